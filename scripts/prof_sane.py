"""Throughput on a physically sane DG2 workload (config-0 dam break at
scaled-up size) to separate kernel cost from the config-4 blow-up dynamics."""
import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2107_02750_b200 import api  # noqa: E402
from paper_2107_02750_b200 import scenarios as S  # noqa: E402

lib = api.lib()
# dam break on a 2048^2 grid with dx = 2 m (config-3 terrain, power-of-two cells)
sc = S.config3(1)
sc.solver = "dg2"
h0 = np.where(np.arange(sc.dem.ncols)[None, :] < sc.dem.ncols // 2, 1.5, 0.0) * np.ones((sc.dem.nrows, 1))
sc.initial_depth_raster = S.Raster(h0, cellsize=sc.dem.cellsize)
g = lib.grid(sc.dem, sc.L, sc.eps)
s = lib.sim(sc, g)
s.run(5, gauge_interval=10.0)
prof = s.profile(10)
print("leaves", s.num_cells, "segments", s.num_segments)
for k, (ms, n) in prof.items():
    print(f"{k:18s} {ms / n:.3f} ms/launch x{n}")
u = s.download()[3]
print("max|u|", np.abs(u).max(axis=0)[[0, 3, 6]])
