import ctypes, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2107_02750_b200 import api
lib = api.lib()
f = ctypes.c_int64(-1)
for which in (2, 0):
    for seed in range(1, 9):
        lib.call("selftest", which, 100_000_000, seed, ctypes.byref(f))
        print("which", which, "seed", seed, "fails", f.value, flush=True)
