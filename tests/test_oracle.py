"""The plain-C oracle restatement pinned against the reference's own outputs
(tests/golden/golden.npz, made by tests/golden/make_golden.py from the
unmodified reference) and the reference KATs.  CPU only."""
import numpy as np
import pytest

import oracle

# survey-measured structural goldens for the reference generator at seed 1
#
RMAT_NNZ = {16: 490_332, 17: 991_224}


def csr(g, name):
    rp = g[name + "_rp"]
    return oracle.Csr(len(rp) - 1, 0, rp, g[name + "_ci"], g[name + "_v"])


def same(a, g, name):
    assert np.array_equal(a.row_ptr, g[name + "_rp"])
    assert np.array_equal(a.col_idx, g[name + "_ci"])
    assert np.array_equal(a.values, g[name + "_v"])


def test_splitmix_kat(orc, golden):
    # test_gen_io.cpp:44
    assert orc.splitmix64(0) == 0xE220A8397B1DCDAF
    assert int(golden["kat_splitmix0"][0]) == 0xE220A8397B1DCDAF
    ctr = np.arange(8, dtype=np.uint64)
    assert np.array_equal(oracle.rng_at_np(1, ctr), golden["kat_rng_at_1"])


def test_generators_match_reference(orc, golden):
    same(orc.rmat(10, 8, seed=1), golden, "rmat10")
    same(orc.rmat(10, 8, seed=1, multiplicity=True), golden, "rmat10m")
    same(orc.uniform_tiles(64, 64, 4, 0.25, 3), golden, "unif64")
    same(orc.random_csr(24, 20, 0.25, 6), golden, "rcsr")
    assert np.array_equal(orc.random_dense(20, 28, 7), golden["rdense"])
    same(orc.permute_symmetric(orc.rmat(8, 8, seed=1), 5), golden, "perm8")


@pytest.mark.parametrize("scale", [16, 17])
def test_rmat_structural_goldens(orc, scale):
    a = orc.rmat(scale, 8, seed=1)
    assert a.nnz == RMAT_NNZ[scale]
    assert orc.well_formed(a)


def test_generator_rejects_bad_params(orc):
    with pytest.raises(ValueError):
        orc.rmat(27, 8)  # gen.hpp:49-50 desk-scale guard
    with pytest.raises(ValueError):
        orc.rmat(10, 8, a=0.5)  # probabilities must sum to 1
    with pytest.raises(ValueError):
        orc.uniform_tiles(10, 10, 3, 0.1, 1)  # p not square


def test_spmm_matches_reference(orc, golden):
    a = orc.rmat(10, 8, seed=1)
    b = golden["spmm_b"]
    c = np.zeros((a.rows, 16), np.float32)
    assert orc.spmm_local(a, b, c) == int(golden["spmm_flops"][0])
    assert np.array_equal(c, golden["spmm_c"])
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        ar = oracle.Csr(a.rows, a.cols, a.row_ptr, a.col_idx, oracle.real_twin(a.nnz, 3, dt))
        br = oracle.real_twin(a.cols * 16, 4, dt).reshape(a.cols, 16)
        cr = oracle.real_twin(a.rows * 16, 5, dt).reshape(a.rows, 16)
        orc.spmm_local(ar, br, cr)
        # bit-exact: same k-ascending FMA chain as the reference
        assert np.array_equal(cr, golden["spmm_real_c_" + tag])


def test_spmm_kernel_sections(orc):
    # test_kernels.cpp:66-105
    a = orc.random_csr(2, 2, 1.0, 1)
    a.values[:] = [1, 0, 0, 2] if a.nnz == 4 else a.values
    diag = oracle.Csr(2, 2, np.array([0, 1, 2], np.uint32), np.array([0, 1], np.uint32),
                      np.array([1, 2], np.float32))
    b = np.ones((2, 2), np.float32)
    c = np.zeros((2, 2), np.float32)
    assert orc.spmm_local(diag, b, c) == 8
    assert np.array_equal(c, [[1, 1], [2, 2]])
    empty = oracle.Csr(3, 3, np.zeros(4, np.uint32), np.zeros(0, np.uint32),
                       np.zeros(0, np.float32))
    c = np.zeros((3, 2), np.float32)
    c[1, 1] = 5
    assert orc.spmm_local(empty, np.zeros((3, 2), np.float32), c) == 0
    assert c[1, 1] == 5
    bad = orc.random_csr(4, 5, 0.5, 1)
    with pytest.raises(ValueError):
        orc.spmm_local(bad, np.zeros((4, 3), np.float32), np.zeros((4, 3), np.float32))


def test_spgemm_matches_reference(orc, golden):
    a = orc.rmat(9, 8, seed=1)
    c, fl = orc.spgemm_local(a, a)
    same(c, golden, "spgemm9")
    assert fl == int(golden["spgemm9_flops"][0]) == orc.spgemm_flops(a, a)
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        ar = oracle.Csr(a.rows, a.cols, a.row_ptr, a.col_idx, oracle.real_twin(a.nnz, 3, dt))
        cr, _ = orc.spgemm_local(ar, ar)
        assert np.array_equal(cr.values, golden["spgemm9_real_v_" + tag])


def test_spgemm_cancelled_zero_kept(orc):
    # test_kernels.cpp:149-157
    a = oracle.Csr(1, 2, np.array([0, 2], np.uint32), np.array([0, 1], np.uint32),
                   np.array([1, -1], np.float32))
    b = oracle.Csr(2, 1, np.array([0, 1, 2], np.uint32), np.array([0, 0], np.uint32),
                   np.array([1, 1], np.float32))
    c, fl = orc.spgemm_local(a, b)
    assert c.nnz == 1 and c.values[0] == 0 and fl == 4


def test_csr_add_matches_reference(orc, golden):
    x, y = csr(golden, "csradd_x"), csr(golden, "csradd_y")
    x.cols = y.cols = 7
    same(orc.csr_add(x, y), golden, "csradd")


def test_checksums(orc, golden):
    c = golden["algo_spmm_c"]
    assert orc.checksum_dense(c, 4, 4) == golden["algo_spmm_checksum"][0]
    s = csr(golden, "algo_spgemm")
    s.cols = 10
    assert orc.checksum_sparse(s, 4, 4) == golden["algo_spgemm_checksum"][0]


def test_spmm_all_variants_result_is_serial_product(orc, golden):
    """algos.hpp variants all equal the serial product (test_algos.cpp:98-109)."""
    ga = orc.random_csr(12, 9, 0.35, 5, dtype=np.float64)
    gb = orc.random_dense(9, 10, 6, dtype=np.float64)
    c = orc.random_dense(12, 10, 7, dtype=np.float64)
    orc.spmm_local(ga, gb, c)
    assert np.array_equal(c, golden["algo_spmm_c"])
