"""File formats either side of the path: the ESRI ASCII grid
(raster.cpp:22-96) and the `.nug` text grid (quadgrid.cpp:287-327), plus the
library's binary side formats.

CPU (no device needed — host code of libfm_gpu.so): what fm_raster_write
writes is the reference's file byte for byte; what fm_raster_read reads is
what the reference reads, bit for bit, from the same files (threaded body
parse included); the same files are refused, with the reference's messages.
GPU: fm_grid_write's `.nug` is the reference's write_nug byte for byte for the
same MRA grid, and fm_grid_read rebuilds the grid from it."""
import os

import numpy as np
import pytest

from paper_2107_02750_b200 import scenarios as S
from paper_2107_02750_b200.abi import Backend, FmError
from paper_2107_02750_b200.scenarios import Raster

from conftest import GPU_SO

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "io_small.asc")


@pytest.fixture(scope="module")
def host():
    """libfm_gpu.so without fm_init: the I/O entry points are host code."""
    return Backend(GPU_SO, "fm_")


def _awkward_raster(nr, nc, seed=3):
    rng = np.random.default_rng(seed)
    v = rng.normal(0.0, 50.0, (nr, nc))
    flat = v.reshape(-1)
    flat[::7] = np.round(flat[::7])            # integers print without a point
    flat[1::11] = -9999.0                      # nodata
    flat[2::13] = rng.normal(0, 1, flat[2::13].shape) * 1e-300   # tiny, exponent form
    flat[3::17] = rng.normal(0, 1, flat[3::17].shape) * 1e+200
    special = [-0.0, 5e-324, 1.7976931348623157e308, 0.1]   # -0, smallest denormal, largest
    flat[:len(special)][:flat.size] = special[:flat.size]
    return Raster(v, xll=-123.456789012345678, yll=1e-7, cellsize=1.0 / 3.0, nodata=-9999.0)


def _small_raster():
    v = np.array([[0.0, -0.0, 1.0, 0.1], [1e-7, 123456789.125, -9999.0, 2.5e300],
                  [1.0 / 3.0, -2.0 / 3.0, 5e-324, 17.0]])
    return Raster(v, xll=10.5, yll=-2.25, cellsize=0.1, nodata=-9999.0)


def test_ascii_write_matches_committed_golden(host, tmp_path):
    """tests/golden/io_small.asc was written by the reference's
    write_ascii_grid (scripts/make_golden_io.py)."""
    p = str(tmp_path / "a.asc")
    host.write_raster(_small_raster(), p)
    assert open(p, "rb").read() == open(GOLDEN, "rb").read()
    r = host.read_raster(GOLDEN)
    assert (r.ncols, r.nrows, r.xll, r.yll, r.cellsize, r.nodata) == (4, 3, 10.5, -2.25, 0.1, -9999.0)
    assert r.values.tobytes() == _small_raster().values.tobytes()


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (257, 129), (700, 900)])
def test_ascii_write_byte_identical_to_reference(host, ref, tmp_path, shape):
    r = _awkward_raster(*shape)
    a, b = str(tmp_path / "gpu.asc"), str(tmp_path / "ref.asc")
    host.write_raster(r, a)
    ref.write_raster(r, b)
    assert open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (700, 900)])
def test_ascii_read_bit_identical_to_reference(host, ref, tmp_path, shape):
    """(700, 900): ~12 MB of text, parsed in slices by several threads."""
    r = _awkward_raster(*shape)
    p = str(tmp_path / "r.asc")
    ref.write_raster(r, p)
    x, y = host.read_raster(p), ref.read_raster(p)
    assert (x.ncols, x.nrows, x.xll, x.yll, x.cellsize, x.nodata) == \
        (y.ncols, y.nrows, y.xll, y.yll, y.cellsize, y.nodata)
    assert x.values.tobytes() == y.values.tobytes() == r.values.tobytes()


def test_header_any_order_any_case_and_free_layout(host, ref, tmp_path):
    p = str(tmp_path / "h.asc")
    open(p, "w").write("NROWS 2\nCellSize 2.5\nnodata_VALUE -1\nyllcorner 7\n  ncols   3.0  trailing\n"
                       "XLLCORNER -4e1\n1 2\t3\n\n+4 5e0 .5\n")
    for be in (host, ref):
        r = be.read_raster(p)
        assert (r.ncols, r.nrows, r.xll, r.yll, r.cellsize, r.nodata) == (3, 2, -40.0, 7.0, 2.5, -1.0)
        assert r.values.tolist() == [[1.0, 2.0, 3.0], [4.0, 5.0, 0.5]]


HDR = "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n"
BAD = {
    "truncated_header": "ncols 2\nnrows 2\n",
    "malformed_line": HDR.replace("nrows 2", "nrows two") + "1 2 3 4\n",
    "unknown_keyword": HDR.replace("cellsize", "cellsise") + "1 2 3 4\n",
    "duplicate_keyword": HDR.replace("nrows 2", "ncols 2") + "1 2 3 4\n",
    "bad_dimensions": HDR.replace("cellsize 1", "cellsize 0") + "1 2 3 4\n",
    "too_few": HDR + "1 2 3\n",
    "too_many": HDR + "1 2 3 4 5\n",
    "stops_at_nan": HDR + "1 2 nan 4\n",
    "stops_at_word": HDR + "1 2 3 x 4\n",
    "glued_garbage": HDR + "1 2 3.5abc 4\n",
    "empty_body": HDR,
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_rejected_files_and_messages_match_reference(host, ref, tmp_path, case):
    """Same refusal (ParseError -> FM_ERR_IO) and the same message, including
    the count of values found before the first non-number."""
    p = str(tmp_path / (case + ".asc"))
    open(p, "w").write(BAD[case])
    with pytest.raises(FmError) as eg:
        host.read_raster(p)
    with pytest.raises(FmError) as er:
        ref.read_raster(p)
    assert eg.value.code == er.value.code == 3
    assert str(eg.value) == str(er.value)


def test_missing_and_unwritable_paths(host, tmp_path):
    with pytest.raises(FmError) as e:
        host.read_raster(str(tmp_path / "absent.asc"))
    assert e.value.code == 3 and "cannot open raster file" in str(e.value)
    with pytest.raises(FmError) as e:
        host.write_raster(_small_raster(), str(tmp_path / "no_such_dir" / "x.asc"))
    assert e.value.code == 3 and "cannot write raster file" in str(e.value)


def test_binary_raster_round_trip_exact(host, tmp_path):
    r = _awkward_raster(300, 200)
    r.values[0, 0] = np.nan
    p = str(tmp_path / "r.fmrb")
    host.write_raster(r, p, binary=True)
    assert os.path.getsize(p) == 8 + 8 + 32 + 8 * r.values.size
    x = host.read_raster(p)
    assert (x.ncols, x.nrows, x.xll, x.yll, x.cellsize, x.nodata) == \
        (r.ncols, r.nrows, r.xll, r.yll, r.cellsize, r.nodata)
    assert x.values.tobytes() == r.values.tobytes()
    open(p, "ab").write(b"\0" * 8)
    with pytest.raises(FmError) as e:
        host.read_raster(p)
    assert e.value.code == 3 and "expected 60000 values, found 60001" in str(e.value)


# ---- .nug (GPU: the grid lives on the device) -----------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c0", "c3"])
def test_nug_write_byte_identical_and_read_back(gpu, ref, tmp_path, cfg):
    sc = S.config0(2) if cfg == "c0" else S.config3(1)
    g, r = gpu.grid(sc.dem, sc.L, sc.eps), ref.grid(sc.dem, sc.L, sc.eps)
    a, b = str(tmp_path / "gpu.nug"), str(tmp_path / "ref.nug")
    g.write(a)
    r.write(b)
    assert open(a, "rb").read() == open(b, "rb").read()
    g2, r2 = gpu.read_grid(b), ref.read_grid(b)
    assert g2.info()["L"] == sc.L
    for x, y, z in zip(g.leaves(), g2.leaves(), r2.leaves()):
        assert np.array_equal(x, y) and np.array_equal(x, z)
    # records in any order (make_quadgrid sorts; the payload follows)
    lines = open(b).read().splitlines()
    rng = np.random.default_rng(5)
    body = [lines[1 + k] for k in rng.permutation(len(lines) - 1)]
    c = str(tmp_path / "shuffled.nug")
    open(c, "w").write("\n".join([lines[0]] + body) + "\n")
    for x, y in zip(g.leaves(), gpu.read_grid(c).leaves()):
        assert np.array_equal(x, y)
    # binary side format
    d = str(tmp_path / "g.fmng")
    g.write(d, binary=True)
    assert os.path.getsize(d) == 56 + 36 * g.num_leaves
    for x, y in zip(g.leaves(), gpu.read_grid(d).leaves()):
        assert np.array_equal(x, y)


@pytest.mark.gpu
def test_nug_refusals_match_reference(gpu, ref, tmp_path):
    sc = S.config0(4)
    p = str(tmp_path / "g.nug")
    gpu.grid(sc.dem, sc.L, sc.eps).write(p)
    lines = open(p).read().splitlines()
    cases = {
        "bad_magic": ("gun" + lines[0][3:] + "\n" + "\n".join(lines[1:]) + "\n", 3),
        "short_header": ("nug 3 1\n", 3),
        "hole": ("\n".join(lines[:-1]) + "\n", 5),                       # a leaf missing
        "stops_early": ("\n".join(lines[:5] + ["oops"] + lines[5:]) + "\n", 5),  # read ends at "oops"
        "overlap": ("\n".join(lines + [lines[1]]) + "\n", 5),
    }
    for name, (text, status) in cases.items():
        q = str(tmp_path / (name + ".nug"))
        open(q, "w").write(text)
        with pytest.raises(FmError) as eg:
            gpu.read_grid(q)
        with pytest.raises(FmError) as er:
            ref.read_grid(q)
        assert eg.value.code == er.value.code == status, name
    with pytest.raises(FmError) as e:
        gpu.read_grid(str(tmp_path / "absent.nug"))
    assert e.value.code == 3
