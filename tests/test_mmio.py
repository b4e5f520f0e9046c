"""Matrix Market I/O (mmio.hpp:50-116) through the host C-ABI vs the
unmodified reference reader (oracle/_ref).  CPU only: no device work."""
import gzip

import numpy as np
import pytest

import oracle

mm = pytest.importorskip("paper_2311_18141_b200.mmio")

FILES = {
    "general.mtx": "%%MatrixMarket matrix coordinate real general\n% a comment\n%another\n"
                   "4 5 6\n1 1 1.5\n4 5 -2\n2 3 0.25\n1 1 2.5\n3 2 1e-3\n2 1 7\n",
    "sym.mtx": "%%MatrixMarket matrix coordinate integer symmetric\n3 3 4\n1 1 3\n2 1 4\n"
               "3 1 5\n3 3 -1\n",
    "pattern.mtx": "%%MatrixMarket matrix coordinate pattern general\n3 4 3\n1 4\n3 1\n2 2\n",
    "crlf.mtx": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 2 3.0\r\n2 1 4\r\n",
    "empty_rows.mtx": "%%MatrixMarket matrix coordinate real general\n6 6 1\n5 2 9\n",
    "zero.mtx": "%%MatrixMarket matrix coordinate real general\n3 3 0\n",
}
BAD = {
    "array.mtx": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex.mtx": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "skew.mtx": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "banner.mtx": "%%MatrixMarkt matrix coordinate real general\n1 1 1\n1 1 1\n",
    "range.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "short.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n",
    "noval.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "size.mtx": "%%MatrixMarket matrix coordinate real general\n2 x 1\n1 1 1\n",
    "empty.mtx": "",
}


def _ref():
    return oracle.ref() if oracle.ref_available() else None


@pytest.mark.parametrize("name", sorted(FILES))
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("gz", [False, True])
def test_read_matches_reference(tmp_path, name, dtype, gz):
    path = tmp_path / (name + (".gz" if gz else ""))
    data = FILES[name].encode()
    path.write_bytes(gzip.compress(data) if gz else data)
    rows, cols, rp, ci, vv = mm.read_matrix_market(path, dtype)
    assert vv.dtype == dtype and rp[-1] == len(ci) == len(vv)
    R = _ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    want = R.read_matrix_market(path, dtype)
    assert (rows, cols) == (want.rows, want.cols)
    assert np.array_equal(rp, want.row_ptr) and np.array_equal(ci, want.col_idx)
    assert np.array_equal(vv, want.values)


@pytest.mark.parametrize("name", sorted(BAD))
def test_rejects_like_reference(tmp_path, name):
    path = tmp_path / name
    path.write_text(BAD[name])
    with pytest.raises(mm.L.MmioError) as ei:
        mm.read_matrix_market(path)
    R = _ref()
    if R is not None:
        with pytest.raises(ValueError) as er:
            R.read_matrix_market(path)
        msg = str(er.value).replace(str(path), "<p>")
        assert msg in str(ei.value).replace(str(path), "<p>")


def test_missing_file(tmp_path):
    with pytest.raises(mm.L.MmioError, match="cannot open"):
        mm.read_matrix_market(tmp_path / "nope.mtx")


def test_write_read_round_trip(tmp_path, golden):
    rp, ci = golden["rmat10_rp"], golden["rmat10_ci"]
    vals = np.random.default_rng(3).standard_normal(len(ci)).astype(np.float32)
    n = len(rp) - 1
    mm.write_matrix_market(tmp_path / "a.mtx", n, n, rp, ci, vals)
    rows, cols, rp2, ci2, v2 = mm.read_matrix_market(tmp_path / "a.mtx", np.float32)
    assert (rows, cols) == (n, n)
    assert np.array_equal(rp2, rp) and np.array_equal(ci2, ci)
    assert np.array_equal(v2, vals)  # %.9g round-trips fp32 exactly
