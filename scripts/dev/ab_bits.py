"""A/B bit-identity: run config c3/c2 K steps under two library builds and
compare the downloaded leaf states and leaf sets byte for byte."""
import os
import sys

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, ROOT)
from paper_2107_02750_b200.abi import Backend  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402


def run(path, which, k):
    lib = Backend(path, "fm_")
    lib.call("init", 0)
    sc = S.config3(1) if which == "c3" else S.config2(1)
    s = lib.sim(sc, None)
    s.run(k, gauge_interval=10.0)
    return s.download(), s.num_cells


a_lib, b_lib = sys.argv[1], sys.argv[2]
for which in sys.argv[3:]:
    ua, na = run(a_lib, which, 60)
    ub, nb = run(b_lib, which, 60)
    same = na == nb and all(np.array_equal(np.ascontiguousarray(x).view(np.uint8), np.ascontiguousarray(y).view(np.uint8))
                            for x, y in zip(ua, ub))
    print(which, "leaves", na, nb, "bit-identical" if same else "DIFFERENT")
