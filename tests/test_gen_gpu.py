"""Device generators vs the reference generators (golden fixtures from the
reference itself, and the survey-measured structural goldens)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rd():
    import paper_2311_18141_b200 as rd

    return rd


def same(a, g, name):
    rp, ci, vv = a.to_host()
    assert np.array_equal(rp, g[name + "_rp"])
    assert np.array_equal(ci, g[name + "_ci"])
    assert np.array_equal(vv, g[name + "_v"])


def test_rng_kat(rd, golden):
    from paper_2311_18141_b200.tile import rng_at

    got = rng_at(1, 0, 8).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, golden["kat_rng_at_1"])
    assert int(rng_at(0, 0, 1).cpu().numpy().view(np.uint64)[0]) == int(
        oracle.rng_at_np(0, np.zeros(1, np.uint64))[0])


def test_rmat_matches_reference(rd, golden):
    same(rd.rmat(10, 8, seed=1), golden, "rmat10")
    same(rd.rmat(10, 8, seed=1, multiplicity=True), golden, "rmat10m")


def test_uniform_tiles_matches_reference(rd, golden):
    same(rd.uniform_tiles(64, 64, 4, 0.25, 3), golden, "unif64")


def test_dense_generators(rd, golden):
    assert np.array_equal(rd.random_dense(20, 28, 7).cpu().numpy(), golden["rdense"])
    for dt, npdt in ((torch.float32, np.float32), (torch.float64, np.float64)):
        assert np.array_equal(rd.real_twin(1000, 4, dtype=dt).cpu().numpy(),
                              oracle.real_twin(1000, 4, npdt))


@pytest.mark.parametrize("scale", [13, 15])
def test_rmat_matches_oracle_port(rd, orc, scale):
    g = rd.rmat(scale, 8, seed=3)
    h = orc.rmat(scale, 8, seed=3)
    rp, ci, vv = g.to_host()
    assert np.array_equal(rp, h.row_ptr) and np.array_equal(ci, h.col_idx)


def test_generator_validation(rd):
    with pytest.raises(rd.InvalidArgument):
        rd.rmat(27, 8)
    with pytest.raises(rd.InvalidArgument):
        rd.rmat(10, 8, a=0.5)
    with pytest.raises(rd.InvalidArgument):
        rd.uniform_tiles(10, 10, 3, 0.1, 1)


def test_structural_goldens_at_benchmark_scale(rd):
    """SURVEY §8(c) survey-measured goldens of the reference generator."""
    a = rd.rmat(20, 8, seed=1)
    assert a.nnz == 8_124_707
    del a
    a = rd.rmat(22, 16, seed=1)
    deg = torch.diff(a.row_ptr.long())
    assert a.nnz == 64_827_941
    assert int(deg.max()) == 32_498
    del a, deg
    e = rd.uniform_tiles(1 << 22, 1 << 22, 1, 2.0 ** -18, 1)
    deg = torch.diff(e.row_ptr.long())
    assert e.nnz == 67_108_864
    assert int(deg.max()) == 39
    assert int((deg == 0).sum()) == 1


def test_permute_symmetric_matches_reference(rd, golden, orc):
    """gen.hpp:134-155 on the device: bit-identical to the reference golden
    (perm8 = permute_symmetric(rmat(8, 8, seed=1), 5)) and to the oracle at a
    larger scale, fp32 and fp64."""
    same(rd.permute_symmetric(rd.rmat(8, 8, seed=1), 5), golden, "perm8")
    for dt, ndt in ((torch.float32, np.float32), (torch.float64, np.float64)):
        a = orc.rmat(14, 8, seed=1, dtype=ndt)
        a.values[:] = np.arange(a.nnz) % 7 - 3  # distinct values follow their entries
        want = orc.permute_symmetric(a, 11)
        d = rd.DeviceCsr.from_host(a.rows, a.cols, a.row_ptr, a.col_idx, a.values)
        assert d.dtype == dt
        rp, ci, vv = rd.permute_symmetric(d, 11).to_host()
        assert np.array_equal(rp, want.row_ptr) and np.array_equal(ci, want.col_idx)
        assert np.array_equal(vv, want.values)


def test_permute_symmetric_edges(rd):
    e = rd.DeviceCsr.from_host(4, 4, np.zeros(5, np.uint32), np.zeros(0, np.uint32),
                               np.zeros(0, np.float32))
    rp, ci, vv = rd.permute_symmetric(e, 3).to_host()
    assert np.array_equal(rp, np.zeros(5)) and len(ci) == 0
    r = rd.DeviceCsr.from_host(2, 3, np.array([0, 1, 1], np.uint32), np.array([2], np.uint32),
                               np.array([1.0], np.float32))
    with pytest.raises(rd.DimensionError):
        rd.permute_symmetric(r, 1)
