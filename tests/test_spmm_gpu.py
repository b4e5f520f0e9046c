"""SpMM parity: the sm_100a kernel (through the C-ABI) vs the reference's
spmm_local -- golden fixtures from the reference and the oracle port.

Bar (BASELINE.json north_star): integer-valued inputs bit-exact; real-valued
fp32 within 1e-5 and fp64 within 1e-12 relative to sum |a_ik * b_kj|."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def rd():
    import paper_2311_18141_b200 as rd

    return rd


def dev_csr(rd, h, dtype=None):
    return rd.DeviceCsr.from_host(h.rows, h.cols, h.row_ptr, h.col_idx, h.values,
                                  device=DEV, dtype=dtype)


def run(rd, h, b, c0):
    a = dev_csr(rd, h)
    bt = torch.from_numpy(b).to(DEV)
    ct = torch.from_numpy(c0.copy()).to(DEV)
    m = rd.spmm_local(a, bt, ct)
    torch.cuda.synchronize()
    return ct.cpu().numpy(), m


def tol_check(got, want, h, b, c0, rel):
    absprod = np.abs(h.to_dense()) @ np.abs(b.astype(np.float64)) + np.abs(c0)
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert np.all(err <= rel * absprod + 1e-300), float((err / (absprod + 1e-30)).max())


def test_golden_integer_bit_exact(rd, golden):
    rp = golden["rmat10_rp"]
    h = oracle.Csr(len(rp) - 1, len(rp) - 1, rp, golden["rmat10_ci"], golden["rmat10_v"])
    got, m = run(rd, h, golden["spmm_b"], np.zeros((h.rows, 16), np.float32))
    assert np.array_equal(got, golden["spmm_c"])
    assert m.flops == int(golden["spmm_flops"][0])


@pytest.mark.parametrize("dt,tag,rel", [(np.float32, "f32", 1e-5), (np.float64, "f64", 1e-12)])
def test_golden_real_valued(rd, golden, dt, tag, rel):
    rp = golden["rmat10_rp"]
    nnz = len(golden["rmat10_ci"])
    h = oracle.Csr(len(rp) - 1, len(rp) - 1, rp, golden["rmat10_ci"],
                   oracle.real_twin(nnz, 3, dt))
    b = oracle.real_twin(h.cols * 16, 4, dt).reshape(h.cols, 16)
    c0 = oracle.real_twin(h.rows * 16, 5, dt).reshape(h.rows, 16)
    got, _ = run(rd, h, b, c0)
    want = golden["spmm_real_c_" + tag]
    tol_check(got, want, h, b, c0, rel)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_wide_rows_follow_reference_fma_order(rd, orc, dt):
    """For wide B rows (one 16-B vector per lane and more) the kernels keep the
    reference's k-ascending fma chain from C for every row not cut by a chunk
    boundary, so those rows are bitwise equal to the reference for real data."""
    h = orc.rmat(10, 8, seed=1, dtype=dt)
    h.values = oracle.real_twin(h.nnz, 3, dt)
    n = 128 if dt == np.float32 else 64
    b = oracle.real_twin(h.cols * n, 4, dt).reshape(h.cols, n)
    c0 = oracle.real_twin(h.rows * n, 5, dt).reshape(h.rows, n)
    want = c0.copy()
    orc.spmm_local(h, b, want)
    got, _ = run(rd, h, b, c0)
    tol_check(got, want, h, b, c0, 1e-5 if dt == np.float32 else 1e-12)
    assert np.mean(np.all(got == want, axis=1)) > 0.5


def test_sections_like_reference(rd):
    # test_kernels.cpp:66-105
    diag = oracle.Csr(2, 2, np.array([0, 1, 2], np.uint32), np.array([0, 1], np.uint32),
                      np.array([1, 2], np.float32))
    got, m = run(rd, diag, np.ones((2, 2), np.float32), np.zeros((2, 2), np.float32))
    assert np.array_equal(got, [[1, 1], [2, 2]]) and m.flops == 8
    empty = oracle.Csr(3, 3, np.zeros(4, np.uint32), np.zeros(0, np.uint32),
                       np.zeros(0, np.float32))
    c0 = np.zeros((3, 2), np.float32)
    c0[1, 1] = 5
    got, m = run(rd, empty, np.zeros((3, 2), np.float32), c0)
    assert m.flops == 0 and got[1, 1] == 5
    a = dev_csr(rd, oracle.port().random_csr(4, 5, 0.5, 1))
    with pytest.raises(rd.DimensionError):
        rd.spmm_local(a, torch.zeros((4, 3), device=DEV), torch.zeros((4, 3), device=DEV))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 12, 16, 17, 32, 64, 100, 128, 256, 260, 520, 1030])
def test_widths_match_oracle(rd, orc, n):
    """Every group size / vector width / panel path, integer data, bit-exact."""
    h = orc.rmat(11, 8, seed=7)
    b = orc.random_dense(h.cols, n, 9)
    c0 = orc.random_dense(h.rows, n, 10)
    want = c0.copy()
    orc.spmm_local(h, b, want)
    got, m = run(rd, h, b, c0)
    assert np.array_equal(got, want)
    assert m.flops == 2 * h.nnz * n


@pytest.mark.parametrize("d", [0.05, 0.2, 0.5, 1.0])
@pytest.mark.parametrize("n", [8, 16, 64])
def test_oracle_sweep(rd, orc, n, d):
    # test_kernels.cpp:205-223
    a = orc.random_csr(n, n, d, int(n * 1000 + d * 100))
    bd = orc.random_dense(n, 8, n + 3)
    want = np.zeros((n, 8), np.float32)
    orc.spmm_local(a, bd, want)
    got, _ = run(rd, a, bd, np.zeros((n, 8), np.float32))
    assert np.array_equal(got, want)


def test_strided_and_unaligned(rd, orc):
    h = orc.rmat(10, 8, seed=2)
    b_full = orc.random_dense(h.cols, 70, 4)
    a = dev_csr(rd, h)
    bt = torch.from_numpy(b_full).to(DEV)[:, 1:65]  # ldb=70, 4-byte offset
    ct_full = torch.zeros((h.rows, 66), device=DEV)
    ct = ct_full[:, 2:66]
    rd.spmm_local(a, bt, ct)
    want = np.zeros((h.rows, 64), np.float32)
    orc.spmm_local(h, np.ascontiguousarray(b_full[:, 1:65]), want)
    torch.cuda.synchronize()
    assert np.array_equal(ct.cpu().numpy(), want)
    assert torch.all(ct_full[:, :2] == 0)


def test_fp64_integer(rd, orc):
    h = orc.rmat(12, 8, seed=5, dtype=np.float64)
    b = orc.random_dense(h.cols, 128, 6, dtype=np.float64)
    want = np.zeros((h.rows, 128))
    orc.spmm_local(h, b, want)
    got, _ = run(rd, h, b, np.zeros((h.rows, 128)))
    assert np.array_equal(got, want)


def test_cfg1_minimum_slice_bit_exact(rd, orc):
    """BASELINE cfg1: R-MAT s16 ef8 x random_dense(65536,128,2), bit-exact vs
    the oracle."""
    a = rd.rmat(16, 8, seed=1, device=DEV)
    assert a.nnz == 490_332
    b = rd.random_dense(65536, 128, 2, device=DEV)
    c = torch.zeros((65536, 128), device=DEV)
    m = rd.spmm_local(a, b, c)
    rp, ci, vv = a.to_host()
    h = oracle.Csr(a.rows, a.cols, rp, ci, vv)
    want = np.zeros((65536, 128), np.float32)
    orc.spmm_local(h, b.cpu().numpy(), want)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), want)
    assert m.flops == 125_524_992


def test_cfg3_full_scale_property(rd):
    """BASELINE cfg3 at full size (R-MAT s22 ef16, N=128): integer data, so
    row sums of C equal A @ rowsum(B) exactly (size-independent check), and a
    rerun is bitwise identical (determinism)."""
    a = rd.rmat(22, 16, seed=1, device=DEV)
    b = rd.random_dense(1 << 22, 128, 2, device=DEV)
    c = torch.zeros((1 << 22, 128), device=DEV)
    rd.spmm_local(a, b, c)
    bs = b.double().sum(1)
    rows = torch.repeat_interleave(torch.arange(a.rows, device=DEV),
                                   torch.diff(a.row_ptr.long()))
    want = torch.zeros(a.rows, dtype=torch.float64, device=DEV)
    want.index_add_(0, rows, bs[a.col_idx.long()] * a.values.double())
    assert torch.equal(c.double().sum(1), want)
    c2 = torch.zeros_like(c)
    rd.spmm_local(a, b, c2)
    assert torch.equal(c, c2)


def _hub_csr(rows, cols, seed, dtype):
    """Short random rows, empty rows, and a few hub rows with every column:
    the hub rows span many nnz chunks (head/tail fix-ups), the empty rows
    are skipped by the row window, partial last windows everywhere."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 6, rows)
    lens[rng.random(rows) < 0.4] = 0
    for r in {0, 7, rows // 2, rows - 1}:
        if r < rows:
            lens[r] = cols
    rp = np.zeros(rows + 1, np.uint32)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.arange(cols, dtype=np.uint32) if n == cols else
                         np.sort(rng.choice(cols, n, replace=False)).astype(np.uint32)
                         for n in lens])
    vals = rng.integers(-3, 4, ci.size).astype(dtype)
    return oracle.Csr(rows, cols, rp, ci, vals)


@pytest.mark.parametrize("dt,n", [(np.float32, 128), (np.float64, 64)])
@pytest.mark.parametrize("rows", [5, 3000])
@pytest.mark.parametrize("accumulate", [False, True])
def test_full_row_stream_edges(rd, orc, dt, n, rows, accumulate):
    """spmm_stream_full (rows of 32 16-byte vectors): hub rows cut by chunks,
    empty rows, partial windows, C-zero and accumulate forms, bit-exact."""
    h = _hub_csr(rows, 2048, rows + n, dt)
    b = orc.random_dense(h.cols, n, 3, dtype=dt)
    c0 = orc.random_dense(h.rows, n, 4, dtype=dt) if accumulate else np.zeros((h.rows, n), dt)
    want = c0.copy()
    orc.spmm_local(h, b, want)
    a = dev_csr(rd, h)
    ct = torch.from_numpy(c0.copy()).to(DEV)
    rd.spmm_local(a, torch.from_numpy(b).to(DEV), ct, c_zero=not accumulate)
    torch.cuda.synchronize()
    assert np.array_equal(ct.cpu().numpy(), want)
