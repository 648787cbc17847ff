"""CSV ingestion and writers (io.hpp:103-188) against the
reference's own io.hpp (oracle/_ref): same values bit for bit, same
exception type and message for every malformed input, same bytes written.
Host-only (no GPU)."""
import os

import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

# reference exception classes (ref_shim.cpp classify) -> ours
KIND = {1: A.InvalidArgument, 4: A.AidwRuntimeError}


def both(path, with_values=True):
    """(ours, reference) outcome: ('ok', arrays) or ('err', type, message)."""
    try:
        s = A.read_data_csv(path) if with_values else A.read_query_csv(path)
        ours = ("ok", s.xs, s.ys, s.zs)
    except (A.InvalidArgument, A.AidwRuntimeError) as e:
        ours = ("err", type(e), str(e))
    try:
        xs, ys, zs = O.ref_read_points_csv(path, with_values)
        ref = ("ok", xs, ys, zs)
    except O.OracleError as e:
        ref = ("err", KIND.get(e.code, A.AidwRuntimeError), e.message)
    return ours, ref


def same(ours, ref):
    assert ours[0] == ref[0], (ours, ref)
    if ours[0] == "err":
        assert ours[1] is ref[1] and ours[2] == ref[2], (ours, ref)
    else:
        for a, b in zip(ours[1:], ref[1:]):
            if b is None:
                assert a is None or len(a) == 0
            else:
                assert np.array_equal(a, b, equal_nan=True)


CASES = {
    "plain": "x,y,z\n1,2,3\n4,5,6\n",
    "no_final_newline": "x,y,z\n1,2,3\n4,5,6",
    "crlf": "x,y,z\r\n1,2,3\r\n4,5,6\r\n",
    "spaces": "x,y,z \n 1 , 2 ,3\t\n",
    "blank_lines": "x,y,z\n1,2,3\n\n  \n\t\n4,5,6\n\n",
    "empty_file": "",
    "header_only": "x,y,z\n",
    "newline_only": "\n",
    "wrong_header": "a,b,c\n1,2,3\n",
    "query_header_in_data": "x,y\n1,2\n",
    "too_few_fields": "x,y,z\n1,2,3\n4,5\n",
    "too_many_fields": "x,y,z\n1,2,3,4\n",
    "non_numeric": "x,y,z\n1,2,zebra\n",
    "empty_field": "x,y,z\n1,,3\n",
    "trailing_comma": "x,y,z\n1,2,3,\n",
    "plus_sign": "x,y,z\n+1,2,3\n",
    "hex": "x,y,z\n0x10,2,3\n",
    "exponent": "x,y,z\n1e-300,-2.5E+300,.5\n",
    "trailing_garbage": "x,y,z\n1,2,3abc\n",
    "nan_value": "x,y,z\n1,2,nan\n",
    "inf_coordinate": "x,y,z\n1,inf,3\n4,5,6\n",
    "nonfinite_later_point": "x,y,z\n1,2,3\n\n4,5,-inf\n",
    "bad_number_then_bad_count": "x,y,z\n1,x,3\n4,5\n",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_data_csv_matches_reference(tmp_path, name):
    path = str(tmp_path / f"{name}.csv")
    with open(path, "w", newline="") as f:
        f.write(CASES[name])
    same(*both(path, True))


@pytest.mark.parametrize("text", ["x,y\n0.25,0.75\n0.5,0.5\n", "x,y\n1,2,3\n", "x,y,z\n1,2,3\n",
                                  "x,y\n\n1,nan\n"])
def test_query_csv_matches_reference(tmp_path, text):
    path = str(tmp_path / "q.csv")
    open(path, "w").write(text)
    same(*both(path, False))


def test_missing_file_matches_reference(tmp_path):
    same(*both(str(tmp_path / "no_such.csv"), True))


def test_large_file_parallel_chunks(tmp_path):
    """~300K rows split across all host threads: values bit-exact, and the
    FIRST malformed line wins when several chunks hold errors."""
    rng = np.random.default_rng(5)
    n = 300_000
    xs, ys, zs = rng.standard_normal(n) * 1e3, rng.random(n), rng.standard_normal(n) * 1e-200
    d = A.PointSet(xs, ys, zs)
    good = str(tmp_path / "big.csv")
    A.write_data_csv(good, d)
    same(*both(good, True))
    lines = open(good).read().split("\n")
    for bad_at in (250_001, 150_001, 5):  # errors late, middle, early (1-based body lines)
        lines[bad_at] = lines[bad_at].replace(",", ";", 1)
    bad = str(tmp_path / "bad.csv")
    open(bad, "w").write("\n".join(lines))
    ours, ref = both(bad, True)
    same(ours, ref)
    assert ":6:" in ours[2]


def test_writers_byte_identical(tmp_path):
    """write_data_csv / write_query_csv / write_result_csv: "%.17g" rows."""
    rng = np.random.default_rng(9)
    v = rng.standard_normal((3, 5000)) * 10.0 ** rng.integers(-300, 300, (3, 5000))
    v[:, :4] = [[0.0, -0.0, 1 / 3, 5e-324]] * 3
    d = A.PointSet(v[0], v[1], v[2])
    p = str(tmp_path / "d.csv")
    A.write_data_csv(p, d)
    want = "x,y,z\n" + "".join(f"{a:.17g},{b:.17g},{c:.17g}\n" for a, b, c in v.T)
    assert open(p).read() == want
    q = str(tmp_path / "q.csv")
    A.write_query_csv(q, A.PointSet(v[0], v[1]))
    assert open(q).read() == "x,y\n" + "".join(f"{a:.17g},{b:.17g}\n" for a, b in v[:2].T)
    r = str(tmp_path / "r.csv")
    A.write_result_csv(r, A.PointSet(v[0], v[1]), A.InterpolationResult(v[2], v[0]))
    assert open(r).read() == "x,y,alpha,z_pred\n" + "".join(
        f"{a:.17g},{b:.17g},{c:.17g},{e:.17g}\n" for a, b, c, e in zip(v[0], v[1], v[0], v[2]))
    # round trip through the reference's reader
    xs, ys, zs = O.ref_read_points_csv(p, True)
    assert np.array_equal(xs, v[0]) and np.array_equal(ys, v[1]) and np.array_equal(zs, v[2])


def test_write_errors(tmp_path):
    with pytest.raises(A.AidwRuntimeError, match="cannot open for writing"):
        A.write_query_csv(str(tmp_path / "no" / "dir.csv"), A.PointSet(np.zeros(1), np.zeros(1)))
    with pytest.raises(A.InvalidArgument, match="result length does not match"):
        A.write_result_csv(str(tmp_path / "r.csv"), A.PointSet(np.zeros(2), np.zeros(2)),
                           A.InterpolationResult(np.zeros(1), np.zeros(1)))


def test_raster_parse_roundtrip_and_errors(tmp_path):  # io.hpp:223-253
    r = A.Raster(4, 3, -1.5, 2.25, 0.125, np.arange(12.0) / 7.0)
    p = str(tmp_path / "r.asc")
    A.write_raster_asc(p, r)
    back = A.parse_raster_asc(p)
    assert (back.ncols, back.nrows) == (4, 3) and np.array_equal(back.values, r.values)
    assert (back.xllcorner, back.yllcorner, back.cellsize) == (-1.5, 2.25, 0.125)
    open(p, "w").write("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2 3\n")
    with pytest.raises(A.AidwRuntimeError, match=r":5: expected 4 values, found 3"):
        A.parse_raster_asc(p)
    open(p, "w").write("ncols 2\nrows 2\n")
    with pytest.raises(A.AidwRuntimeError, match=r":2: expected header line 'nrows <value>'"):
        A.parse_raster_asc(p)
