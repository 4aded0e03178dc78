"""tests/golden/io_small.asc: the reference's write_ascii_grid
(raster.cpp:81-96, through oracle/_ref/libfmref.so) of test_io's small raster.
Run in the build container (needs /root/reference compiled: make -C oracle ref)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2107_02750_b200.abi import Backend  # noqa: E402
import test_io  # noqa: E402

ref = Backend(os.path.join(ROOT, "oracle", "_ref", "libfmref.so"), "ref_")
ref.write_raster(test_io._small_raster(), test_io.GOLDEN)
print(open(test_io.GOLDEN).read())
