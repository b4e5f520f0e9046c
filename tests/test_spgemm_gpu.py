"""SpGEMM / csr_add parity: the sm_100a hash/dense kernels (through the C-ABI)
vs the reference spgemm_local / csr_add (tile.hpp:197-288).

Bar (BASELINE.json north_star): row_ptr and col_idx bit-exact always;
values bit-exact for integer-valued data, and within 1e-5 (fp32) / 1e-12
(fp64) relative to sum |a_ik * b_kj| for real-valued data."""
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


def dev(rd, h, dtype=None):
    return rd.DeviceCsr.from_host(h.rows, h.cols, h.row_ptr, h.col_idx, h.values, device=DEV,
                                  dtype=dtype)


def host(c):
    rp, ci, vv = c.to_host()
    return oracle.Csr(c.rows, c.cols, rp, ci, vv)


def same_structure(got, want):
    assert got.rows == want.rows
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)


def exact(got, want):
    same_structure(got, want)
    assert np.array_equal(got.values, want.values)


def test_golden_rmat9_squared(rd, golden):
    rp = golden["rmat10_rp"]
    a9 = oracle.port().rmat(9, 8, seed=1)
    c, m = rd.spgemm_local(dev(rd, a9), dev(rd, a9))
    g = oracle.Csr(a9.rows, a9.cols, golden["spgemm9_rp"], golden["spgemm9_ci"],
                   golden["spgemm9_v"])
    exact(host(c), g)
    assert m.flops == int(golden["spgemm9_flops"][0])
    assert m.output_nnz == g.nnz
    del rp


@pytest.mark.parametrize("dt,tag,rel", [(np.float32, "f32", 1e-5), (np.float64, "f64", 1e-12)])
def test_golden_real_valued(rd, golden, dt, tag, rel):
    a9 = oracle.port().rmat(9, 8, seed=1)
    ar = oracle.Csr(a9.rows, a9.cols, a9.row_ptr, a9.col_idx, oracle.real_twin(a9.nnz, 3, dt))
    c, _ = rd.spgemm_local(dev(rd, ar), dev(rd, ar))
    got = host(c)
    same_structure(got, oracle.Csr(a9.rows, a9.cols, golden["spgemm9_rp"],
                                   golden["spgemm9_ci"], golden["spgemm9_v"]))
    want = golden["spgemm9_real_v_" + tag]
    # bound: sum over the row's products of |a||b| for each output entry
    absa = oracle.Csr(ar.rows, ar.cols, ar.row_ptr, ar.col_idx, np.abs(ar.values))
    bound, _ = oracle.port().spgemm_local(
        oracle.Csr(absa.rows, absa.cols, absa.row_ptr, absa.col_idx,
                   absa.values.astype(np.float64)),
        oracle.Csr(absa.rows, absa.cols, absa.row_ptr, absa.col_idx,
                   absa.values.astype(np.float64)))
    err = np.abs(got.values.astype(np.float64) - want.astype(np.float64))
    assert np.all(err <= rel * bound.values + 1e-300)


def test_kernel_sections(rd, orc):
    # test_kernels.cpp:111-157
    a = orc.random_csr(4, 4, 0.5, 3)
    eye = oracle.Csr(4, 4, np.arange(5, dtype=np.uint32), np.arange(4, dtype=np.uint32),
                     np.ones(4, np.float32))
    c, m = rd.spgemm_local(dev(rd, eye), dev(rd, a))
    exact(host(c), a)
    assert m.output_nnz == a.nnz and (a.nnz == 0 or m.cf() == 2.0)
    z = oracle.Csr(4, 4, np.zeros(5, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    c, m = rd.spgemm_local(dev(rd, orc.random_csr(4, 4, 0.5, 4)), dev(rd, z))
    assert c.nnz == 0 and m.flops == 0
    a = oracle.Csr(1, 2, np.array([0, 2], np.uint32), np.array([0, 1], np.uint32),
                   np.array([1, -1], np.float32))
    b = oracle.Csr(2, 1, np.array([0, 1, 2], np.uint32), np.array([0, 0], np.uint32),
                   np.array([1, 1], np.float32))
    c, m = rd.spgemm_local(dev(rd, a), dev(rd, b))
    assert c.nnz == 1 and host(c).values[0] == 0 and m.flops == 4  # cancelled zero kept
    with pytest.raises(rd.DimensionError):
        rd.spgemm_local(dev(rd, orc.random_csr(3, 4, 0.5, 1)), dev(rd, orc.random_csr(3, 4, .5, 2)))


@pytest.mark.parametrize("n", [8, 16, 64])
@pytest.mark.parametrize("d", [0.05, 0.2, 0.5, 1.0])
def test_oracle_sweep(rd, orc, n, d):
    # test_kernels.cpp:205-223
    a = orc.random_csr(n, n, d, int(n * 1000 + d * 100))
    b = orc.random_csr(n, n, d, int(n * 2000 + d * 100))
    want, fl = orc.spgemm_local(a, b)
    c, m = rd.spgemm_local(dev(rd, a), dev(rd, b))
    exact(host(c), want)
    assert m.flops == fl


def test_flop_meter_rectangular(rd, orc):
    a = orc.random_csr(12, 10, 0.25, 13)
    b = orc.random_csr(10, 14, 0.25, 17)
    want, fl = orc.spgemm_local(a, b)
    c, m = rd.spgemm_local(dev(rd, a), dev(rd, b))
    exact(host(c), want)
    assert m.flops == fl == orc.spgemm_flops(a, b)


@pytest.mark.parametrize("scale", [12, 14, 16])
def test_rmat_squared_all_tiers(rd, orc, scale):
    a = orc.rmat(scale, 8, seed=scale)
    want, fl = orc.spgemm_local(a, a)
    info = {}
    c, m = rd.spgemm_local(dev(rd, a), dev(rd, a), info=info)
    exact(host(c), want)
    assert m.flops == fl
    if scale == 16:  # hub rows reach the dense-bitmap tier in both passes
        assert info["sym_tiers"][5] > 0 and info["num_tiers"][5] > 0
        assert all(x > 0 for x in info["num_tiers"])


def test_fp64(rd, orc):
    a = orc.rmat(12, 8, seed=4, dtype=np.float64)
    want, _ = orc.spgemm_local(a, a)
    c, _ = rd.spgemm_local(dev(rd, a), dev(rd, a))
    exact(host(c), want)


def test_csr_add_golden_and_identities(rd, orc, golden):
    x = oracle.Csr(9, 7, golden["csradd_x_rp"], golden["csradd_x_ci"], golden["csradd_x_v"])
    y = oracle.Csr(9, 7, golden["csradd_y_rp"], golden["csradd_y_ci"], golden["csradd_y_v"])
    got = host(rd.csr_add(dev(rd, x), dev(rd, y)))
    exact(got, oracle.Csr(9, 7, golden["csradd_rp"], golden["csradd_ci"], golden["csradd_v"]))
    a = orc.random_csr(6, 6, 0.4, 19)
    empty = oracle.Csr(6, 6, np.zeros(7, np.uint32), np.zeros(0, np.uint32),
                       np.zeros(0, np.float32))
    exact(host(rd.csr_add(dev(rd, a), dev(rd, empty))), a)
    d = host(rd.csr_add(dev(rd, a), dev(rd, a)))
    assert np.array_equal(d.values, 2 * a.values)
    with pytest.raises(rd.DimensionError):
        rd.csr_add(dev(rd, a), dev(rd, orc.random_csr(6, 5, 0.4, 1)))


def test_csr_add_keeps_negative_zero(rd):
    a = oracle.Csr(1, 3, np.array([0, 1], np.uint32), np.array([1], np.uint32),
                   np.array([-0.0], np.float32))
    b = oracle.Csr(1, 3, np.array([0, 1], np.uint32), np.array([2], np.uint32),
                   np.array([5.0], np.float32))
    got = host(rd.csr_add(dev(rd, a), dev(rd, b)))
    assert np.signbit(got.values[0]) and got.values[1] == 5.0


def test_multi_term_accumulate(rd, orc):
    """I*C0 + A1*B1 + A2*B2 == csr_add chain of the reference products."""
    c0 = orc.random_csr(40, 30, 0.1, 1)
    a1, b1 = orc.random_csr(40, 25, 0.2, 2), orc.random_csr(25, 30, 0.2, 3)
    a2, b2 = orc.random_csr(40, 35, 0.2, 4), orc.random_csr(35, 30, 0.2, 5)
    p1, _ = orc.spgemm_local(a1, b1)
    p2, _ = orc.spgemm_local(a2, b2)
    want = orc.csr_add(orc.csr_add(c0, p1), p2)
    got, m = rd.spgemm_terms(40, 30, [(None, dev(rd, c0)), (dev(rd, a1), dev(rd, b1)),
                                      (dev(rd, a2), dev(rd, b2))])
    exact(host(got), want)


def test_cfg2_full(rd, orc):
    """BASELINE cfg2: R-MAT s17 ef8 squared; survey goldens + exact vs oracle."""
    a = rd.rmat(17, 8, seed=1, device=DEV)
    c, m = rd.spgemm_local(a, a)
    assert c.nnz == 81_940_178
    assert m.flops == 2 * 144_877_044
    ha = host(a)
    want, fl = orc.spgemm_local(ha, ha)
    exact(host(c), want)


def test_cfg4_full_scale_property(rd):
    """BASELINE cfg4: R-MAT s20 ef8 squared at full size: survey structural
    goldens, and row sums of C == A @ rowsum(A) exactly (integer data)."""
    a = rd.rmat(20, 8, seed=1, device=DEV)
    c, m = rd.spgemm_local(a, a)
    assert c.nnz == 1_390_953_199
    assert m.flops == 2 * 2_348_048_595
    rows_c = torch.repeat_interleave(torch.arange(c.rows, device=DEV),
                                     torch.diff(c.row_ptr.long()))
    got = torch.zeros(c.rows, dtype=torch.float64, device=DEV)
    got.index_add_(0, rows_c, c.values.double())
    del rows_c
    rows_a = torch.repeat_interleave(torch.arange(a.rows, device=DEV),
                                     torch.diff(a.row_ptr.long()))
    rs = torch.zeros(a.rows, dtype=torch.float64, device=DEV)
    rs.index_add_(0, rows_a, a.values.double())
    want = torch.zeros(a.rows, dtype=torch.float64, device=DEV)
    want.index_add_(0, rows_a, rs[a.col_idx.long()] * a.values.double())
    assert torch.equal(got, want)
    # sortedness of every row (bit-exact structure implies strictly increasing)
    ci = c.col_idx.long()
    inc = ci[1:] > ci[:-1]
    starts = torch.zeros(c.nnz, dtype=torch.bool, device=DEV)
    starts[c.row_ptr.long()[1:-1].clamp(max=c.nnz - 1)] = True
    assert bool(torch.all(inc | starts[1:]))


@pytest.mark.parametrize("dt,tag", [(np.float32, "f32"), (np.float64, "f64")])
def test_deterministic_values_equal_reference_bitwise(rd, golden, dt, tag):
    """RDMM_SPGEMM_DETERMINISTIC: real-valued A*A bitwise equal to the
    reference's own result (golden from oracle/_ref, tile.hpp:211-255)."""
    a9 = oracle.port().rmat(9, 8, seed=1)
    ar = oracle.Csr(a9.rows, a9.cols, a9.row_ptr, a9.col_idx, oracle.real_twin(a9.nnz, 3, dt))
    c, _ = rd.spgemm_local(dev(rd, ar), dev(rd, ar), deterministic=True)
    got = host(c)
    same_structure(got, oracle.Csr(a9.rows, a9.cols, golden["spgemm9_rp"],
                                   golden["spgemm9_ci"], golden["spgemm9_v"]))
    assert np.array_equal(got.values, golden["spgemm9_real_v_" + tag])


def test_deterministic_matches_oracle_fma_chain_rmat14(rd, orc):
    """Larger R-MAT (every hash tier and the dense tier's rows): bitwise equal
    to the oracle's fma chain, and identical run to run."""
    h = orc.rmat(14, 8, seed=3)
    h.values = oracle.real_twin(h.nnz, 5, np.float32)
    want, _ = orc.spgemm_local(h, h)
    c1, _ = rd.spgemm_local(dev(rd, h), dev(rd, h), deterministic=True)
    c2, _ = rd.spgemm_local(dev(rd, h), dev(rd, h), deterministic=True)
    g1, g2 = host(c1), host(c2)
    exact(g1, want)
    assert np.array_equal(g1.values.view(np.uint32), g2.values.view(np.uint32))


def test_deterministic_csr_add_keeps_signed_zeros(rd):
    x = oracle.Csr(2, 3, np.array([0, 2, 3], np.uint32), np.array([0, 2, 1], np.uint32),
                   np.array([-0.0, 1.5, 2.0], np.float32))
    y = oracle.Csr(2, 3, np.array([0, 1, 2], np.uint32), np.array([1, 1], np.uint32),
                   np.array([-0.0, -2.0], np.float32))
    out, _ = rd.spgemm_terms(2, 3, [(None, dev(rd, x)), (None, dev(rd, y))],
                             deterministic=True)
    got = host(out)
    assert np.array_equal(got.col_idx, [0, 1, 2, 1])
    assert np.array_equal(got.values, np.array([-0.0, -0.0, 1.5, 0.0], np.float32))
    assert np.signbit(got.values[0]) and np.signbit(got.values[1]) and not np.signbit(got.values[3])
