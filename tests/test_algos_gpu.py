"""Distributed multiply on the B200 fabric vs the reference -- mirrors
/root/reference/proj/tests/test_algos.cpp and acceptance A1/A2/A6, run through
the host C-ABI (include/rdmm_host.h) with P rank threads sharing the GPUs of
the box (one GPU is enough: ranks may share a device).

Bar: SpMM results bit-exact (integer-valued inputs); SpGEMM row_ptr/col_idx
bit-exact and values exact for integer data."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

kM, kK, kN = 12, 9, 10
kTm, kTk, kTn = 4, 3, 4
VARIANTS = ["summa_bsp", "stationary_c", "stationary_a", "stationary_b", "ws_random",
            "ws_locality"]


@pytest.fixture(scope="module")
def dist():
    import paper_2311_18141_b200.dist as dist

    return dist


def devices(p):
    n = torch.cuda.device_count()
    return [r % n for r in range(p)]


def fabric(dist, p, heap=4 << 20):
    return dist.Fabric(nranks=p, heap_bytes=heap, devices=devices(p))


def run_spmm(dist, orc, a_override=None, grid=(2, 2), dims=(kM, kK, kN), tiles=(kTm, kTk, kTn),
             seeds=(5, 6, 7), **opts):
    m, k, n = dims
    tm, tk, tn = tiles
    P = grid[0] * grid[1]
    ga = a_override if a_override is not None else orc.random_csr(m, k, 0.35, seeds[0],
                                                                  dtype=np.float64)
    gb = orc.random_dense(k, n, seeds[1], dtype=np.float64)
    gc0 = orc.random_dense(m, n, seeds[2], dtype=np.float64)
    want = gc0.copy()
    orc.spmm_local(ga, gb, want)
    g = dist.ProcGrid(*grid)
    with fabric(dist, P) as f:
        A = dist.DistSparse(f, m, k, tm, tk, g, 0, dtype=np.float64)
        B = dist.DistDense(f, k, n, tk, tn, g, 1, dtype=np.float64)
        Cm = dist.DistDense(f, m, n, tm, tn, g, 2, dtype=np.float64)
        A.init_from_global(ga.row_ptr, ga.col_idx, ga.values)
        B.init_from_global(gb)
        Cm.init_from_global(gc0)
        rep = dist.run_multiply(f, A, B, Cm, **opts)
        got = Cm.to_global()
    return got, want, rep


def run_spgemm(dist, orc, grid=(2, 2), dims=(kM, kK, kN), tiles=(kTm, kTk, kTn),
               seeds=(15, 16, 17), dens=(0.35, 0.35, 0.15), **opts):
    m, k, n = dims
    tm, tk, tn = tiles
    P = grid[0] * grid[1]
    ga = orc.random_csr(m, k, dens[0], seeds[0], dtype=np.float64)
    gb = orc.random_csr(k, n, dens[1], seeds[1], dtype=np.float64)
    gc0 = orc.random_csr(m, n, dens[2], seeds[2], dtype=np.float64)
    prod, _ = orc.spgemm_local(ga, gb)
    want = orc.csr_add(gc0, prod)
    g = dist.ProcGrid(*grid)
    with fabric(dist, P) as f:
        A = dist.DistSparse(f, m, k, tm, tk, g, 0, dtype=np.float64)
        B = dist.DistSparse(f, k, n, tk, tn, g, 1, dtype=np.float64)
        Cm = dist.DistSparse(f, m, n, tm, tn, g, 2, dtype=np.float64)
        A.init_from_global(ga.row_ptr, ga.col_idx, ga.values)
        B.init_from_global(gb.row_ptr, gb.col_idx, gb.values)
        Cm.init_from_global(gc0.row_ptr, gc0.col_idx, gc0.values)
        rep = dist.run_multiply(f, A, B, Cm, **opts)
        got = Cm.to_global()
    return got, want, rep


def same_csr(got, want):
    rp, ci, vv = got
    assert np.array_equal(rp, want.row_ptr)
    assert np.array_equal(ci, want.col_idx)
    assert np.array_equal(vv, want.values)


@pytest.mark.parametrize("variant", VARIANTS)
def test_every_variant_matches_host_oracle(dist, orc, golden, variant):
    # test_algos.cpp:98-109
    got, want, rep = run_spmm(dist, orc, variant=variant)
    assert np.array_equal(got, want)
    assert np.array_equal(got, golden["algo_spmm_c"])
    assert rep.checksum == golden["algo_spmm_checksum"][0]
    got, want, rep = run_spgemm(dist, orc, variant=variant)
    same_csr(got, want)
    g = golden
    same_csr(got, oracle.Csr(kM, kN, g["algo_spgemm_rp"], g["algo_spgemm_ci"], g["algo_spgemm_v"]))
    assert rep.checksum == golden["algo_spgemm_checksum"][0]


@pytest.mark.parametrize("variant", ["stationary_a", "ws_random", "ws_locality"])
def test_reference_queue_protocol_without_inplace(dist, orc, variant):
    got, want, rep = run_spmm(dist, orc, variant=variant, ws_local_inplace=False)
    assert np.array_equal(got, want)
    got, want, rep = run_spgemm(dist, orc, variant=variant, ws_local_inplace=False)
    same_csr(got, want)


def test_offset_and_prefetch_toggles(dist, orc):
    # test_algos.cpp:111-125
    base, want, _ = run_spmm(dist, orc, variant="stationary_c")
    no_off, _, _ = run_spmm(dist, orc, variant="stationary_c", offset=False)
    no_pre, _, _ = run_spmm(dist, orc, variant="stationary_c", prefetch=False)
    no_fuse, _, _ = run_spmm(dist, orc, variant="stationary_c", fuse_k=False)
    no_split, _, _ = run_spmm(dist, orc, variant="stationary_c", split_local=False)
    assert np.array_equal(no_split, base)
    assert np.array_equal(base, want) and np.array_equal(no_off, base)
    assert np.array_equal(no_pre, base) and np.array_equal(no_fuse, base)
    a_off, want2, _ = run_spmm(dist, orc, variant="stationary_a", offset=False)
    assert np.array_equal(a_off, want2)
    wl, want3, _ = run_spmm(dist, orc, variant="ws_locality", ws_base="stationary_c")
    assert np.array_equal(wl, want3)


def test_deterministic(dist, orc):
    # test_algos.cpp:127-134
    for v in ("stationary_c", "ws_random"):
        r1, _, a = run_spmm(dist, orc, variant=v, seed=9)
        r2, _, b = run_spmm(dist, orc, variant=v, seed=9)
        assert np.array_equal(r1, r2) and a.checksum == b.checksum


@pytest.mark.parametrize("variant", VARIANTS)
def test_each_triple_exactly_once(dist, orc, variant):
    # test_algos.cpp:136-156
    M, N, K = -(-kM // kTm), -(-kN // kTn), -(-kK // kTk)
    allt = sorted((i, j, k) for i in range(M) for j in range(N) for k in range(K))
    for runner in (run_spmm, run_spgemm):
        _, _, rep = runner(dist, orc, variant=variant, record_triples=True)
        got = sorted((t[1], t[2], t[3]) for t in rep.triples)
        assert got == allt
        assert rep.total_multiplies == len(allt)


def test_stationary_a_pushes_one_contribution_per_product(dist, orc):
    # test_algos.cpp:158-171
    _, _, rep = run_spmm(dist, orc, variant="stationary_a")
    pushes = sum(p["queue_pushes"] for p in rep.per_rank)
    pops = sum(p["queue_pops"] for p in rep.per_rank)
    assert pushes == 3 * 3 * 3 and pops == pushes and rep.total_steals == 0


@pytest.mark.parametrize("variant", ["ws_random", "ws_locality"])
def test_work_stealing_rebalances(dist, orc, variant):
    # test_algos.cpp:173-200: rank 0's tiles dense, the rest nearly empty,
    # injected per-flop delay makes rank 0 slow, others steal.
    rows, cols, vals = [], [], []
    for r in range(kM):
        for c in range(kK):
            if (r // kTm) % 2 == 0 and (c // kTk) % 2 == 0:
                rows.append(r), cols.append(c), vals.append(1.0)
            elif r == c:
                rows.append(r), cols.append(c), vals.append(2.0)
    rp = np.zeros(kM + 1, np.uint32)
    np.add.at(rp, np.array(rows) + 1, 1)
    rp = np.cumsum(rp).astype(np.uint32)
    heavy = oracle.Csr(kM, kK, rp, np.array(cols, np.uint32), np.array(vals, np.float64))
    got, want, rep = run_spmm(dist, orc, a_override=heavy, variant=variant,
                              delay_ns_per_flop=20000)
    assert np.array_equal(got, want)
    assert rep.total_steals > 0
    if variant == "ws_locality":
        for p in rep.per_rank:
            assert p["steals_with_local_component"] == p["steals"]


def test_stationary_c_two_tiles_per_rank_per_step(dist, orc):
    # test_algos.cpp:202-226
    ga = orc.random_csr(8, 8, 0.4, 21, dtype=np.float64)
    gb = orc.random_dense(8, 8, 22, dtype=np.float64)
    g = dist.ProcGrid(2, 2)
    with fabric(dist, 4) as f:
        A = dist.DistSparse(f, 8, 8, 4, 4, g, 0, dtype=np.float64)
        B = dist.DistDense(f, 8, 8, 4, 4, g, 1, dtype=np.float64)
        Cm = dist.DistDense(f, 8, 8, 4, 4, g, 2, dtype=np.float64)
        A.init_from_global(ga.row_ptr, ga.col_idx, ga.values)
        B.init_from_global(gb)
        Cm.init()
        f.clear_traffic()
        dist.run_multiply(f, A, B, Cm, variant="stationary_c")
        per = {}
        for (src, dst, label, matrix, i, j) in f.tile_fetches():
            per[(dst, label)] = per.get((dst, label), 0) + 1
        assert len(per) == 4 * 2
        assert all(c == 2 for c in per.values())
        want = np.zeros((8, 8))
        orc.spmm_local(ga, gb, want)
        assert np.array_equal(Cm.to_global(), want)


def test_rejects_malformed(dist, orc):
    import paper_2311_18141_b200 as rd

    # test_algos.cpp:228-276
    g = dist.ProcGrid(2, 2)
    with fabric(dist, 4, 1 << 20) as f:
        A = dist.DistSparse(f, 8, 8, 4, 4, g)
        B = dist.DistDense(f, 6, 8, 3, 4, g)
        Cm = dist.DistDense(f, 8, 8, 4, 4, g)
        A.init(), B.init(), Cm.init()
        with pytest.raises(rd.DimensionError):
            dist.run_multiply(f, A, B, Cm, variant="summa_bsp")
    with fabric(dist, 2, 1 << 20) as f:
        g = dist.ProcGrid(1, 2)
        A = dist.DistSparse(f, 8, 8, 4, 4, g)
        B = dist.DistDense(f, 8, 8, 4, 4, g)
        Cm = dist.DistDense(f, 8, 8, 4, 4, g)
        A.init(), B.init(), Cm.init()
        with pytest.raises(rd.FabricError):
            dist.run_multiply(f, A, B, Cm, variant="summa_bsp")
    with fabric(dist, 4, 1 << 20) as f:
        g = dist.ProcGrid(2, 2)
        A = dist.DistSparse(f, 8, 8, 4, 4, g)
        B = dist.DistDense(f, 8, 8, 4, 4, g)
        Cm = dist.DistDense(f, 8, 8, 4, 4, g)
        A.init(), B.init(), Cm.init()
        with pytest.raises(rd.FabricError):
            dist.run_multiply(f, A, B, Cm, variant="ws_random", ws_base="stationary_c")
    with fabric(dist, 4, 1 << 20) as f:
        with pytest.raises(rd.FabricError):  # grid does not match the rank count
            dist.DistSparse(f, 8, 8, 4, 4, dist.ProcGrid(1, 2))


def test_report_counts_deterministic(dist, orc):
    # test_algos.cpp:278-293
    _, _, r1 = run_spmm(dist, orc, variant="stationary_a", seed=3)
    _, _, r2 = run_spmm(dist, orc, variant="stationary_a", seed=3)
    assert r1.total_flops == r2.total_flops and r1.total_multiplies == r2.total_multiplies
    for p in range(4):
        assert r1.per_rank[p]["multiplies"] == r2.per_rank[p]["multiplies"]
        assert r1.per_rank[p]["flops"] == r2.per_rank[p]["flops"]
    assert r1.wall_seconds > 0
    assert sum(p["bytes_self"] + p["bytes_on_node"] + p["bytes_off_node"]
               for p in r1.per_rank) > 0


@pytest.mark.parametrize("g", [1, 2, 3])
def test_acceptance_a1_grids_and_seeds(dist, orc, g):
    """acceptance.cpp:70-145 (A1) on a reduced seed set: every variant,
    SpMM and SpGEMM, exactly equal to the serial oracle."""
    for seed in range(0, 20, 7):
        m, k, n = 24 + 4 * (seed % 5), 20 + 4 * (seed % 3), 28 + 4 * (seed % 4)
        tile = lambda d: -(-d // (2 * g))  # noqa: E731
        for v in VARIANTS:
            got, want, _ = run_spmm(dist, orc, grid=(g, g), dims=(m, k, n),
                                    tiles=(tile(m), tile(k), tile(n)),
                                    seeds=(seed * 5 + 1, seed * 5 + 2, seed * 5 + 3),
                                    variant=v, seed=seed)
            assert np.array_equal(got, want), (v, g, seed)
            got, want, _ = run_spgemm(dist, orc, grid=(g, g), dims=(m, k, n),
                                      tiles=(tile(m), tile(k), tile(n)),
                                      seeds=(seed * 5 + 1, seed * 5 + 4, seed * 5 + 5),
                                      dens=(0.25, 0.3, 0.1), variant=v, seed=seed)
            same_csr(got, want)


def test_rectangular_grids_for_one_sided_variants(dist, orc):
    """1xP / Px1 grids (the multi-GPU bench layouts) for every non-SUMMA variant."""
    for grid in [(1, 2), (2, 1), (1, 4), (4, 1), (2, 4)]:
        P = grid[0] * grid[1]
        tm, tk, tn = -(-kM // grid[0]), -(-kK // grid[1]), -(-kN // grid[1])
        for v in VARIANTS[1:]:
            got, want, _ = run_spmm(dist, orc, grid=grid, tiles=(tm, tk, tn), variant=v)
            assert np.array_equal(got, want), (grid, v)
            got, want, _ = run_spgemm(dist, orc, grid=grid, tiles=(tm, tk, tn), variant=v)
            same_csr(got, want)
        assert P >= 2


def test_rmat_distributed_spmm_device_init(dist):
    """R-MAT s14 with tiles cut on the device; stationary_c and ws_locality
    on a 2x2 grid vs the single-GPU kernel (bit-exact, integer data)."""
    import paper_2311_18141_b200 as rd

    a = rd.rmat(14, 8, seed=1)
    b = rd.random_dense(a.cols, 64, 2)
    want = torch.zeros((a.rows, 64), device="cuda")
    rd.spmm_local(a, b, want)
    torch.cuda.synchronize()
    g = dist.ProcGrid(2, 2)
    for v in ("stationary_c", "ws_locality", "summa_bsp", "stationary_a"):
        with fabric(dist, 4, 64 << 20) as f:
            n = 1 << 14
            A = dist.DistSparse(f, n, n, n // 2, n // 2, g, 0)
            B = dist.DistDense(f, n, 64, n // 2, 32, g, 1)
            Cm = dist.DistDense(f, n, 64, n // 2, 32, g, 2)
            A.init_from_device(a)
            B.init_from_device(b)
            Cm.init()
            dist.run_multiply(f, A, B, Cm, variant=v, ws_base="stationary_c")
            assert np.array_equal(Cm.to_global(), want.cpu().numpy()), v


@pytest.mark.parametrize("tile,key", [(512, "stage_g2s0"), (256, "stage_g2s4")])
def test_run_stage_flops_match_reference_stage_imbalance(dist, orc, golden, tile, key):
    """The per-rank per-k-step flop table recorded by a stationary-C SpGEMM
    A*A on a 2x2 grid equals the reference's predicted table
    (analytics.hpp:97-150, golden from the unmodified reference), and so do
    the per-stage / end-to-end imbalance figures derived from it."""
    rp, ci = golden["rmat10_rp"], golden["rmat10_ci"]
    n = len(rp) - 1
    vv = golden["rmat10_v"].astype(np.float64)
    g = dist.ProcGrid(2, 2)
    with fabric(dist, 4, 32 << 20) as f:
        A = dist.DistSparse(f, n, n, tile, tile, g, 0, dtype=np.float64)
        B = dist.DistSparse(f, n, n, tile, tile, g, 1, dtype=np.float64)
        Cm = dist.DistSparse(f, n, n, tile, tile, g, 2, dtype=np.float64)
        A.init_from_global(rp, ci, vv)
        B.init_from_global(rp, ci, vv)
        Cm.init()
        rep = dist.run_multiply(f, A, B, Cm, variant="stationary_c")
    assert np.array_equal(rep.stage_flops, golden[key + "_flops"])
    assert [int(x) for x in rep.stage_flops.sum(axis=1)] == [p["flops"] for p in rep.per_rank]
    imb = rep.imbalance()
    np.testing.assert_allclose([imb["per_stage_flop_imbalance"], imb["end_to_end_flop_imbalance"]],
                               golden[key + "_imb"][:2], rtol=1e-12)


@pytest.mark.parametrize("variant", VARIANTS)
def test_stage_flops_cover_every_multiply(dist, orc, variant):
    got, want, rep = run_spmm(dist, orc, variant=variant)
    assert rep.stage_flops.shape[0] == 4
    assert int(rep.stage_flops.sum()) == rep.total_flops
    assert [int(x) for x in rep.stage_flops.sum(axis=1)] == [p["flops"] for p in rep.per_rank]


def test_matrix_market_ingest_permute_and_multiply(dist, orc, golden, tmp_path):
    """A real-matrix path end to end: Matrix Market (.mtx.gz) -> host CSR ->
    device permute_symmetric -> distributed stationary-C A*A on a 2x2 grid,
    bit-exact against the oracle on the reference-permuted matrix."""
    import gzip

    import paper_2311_18141_b200 as rd
    from paper_2311_18141_b200 import mmio

    rp, ci = golden["rmat10_rp"], golden["rmat10_ci"]
    n = len(rp) - 1
    vals = (np.arange(len(ci)) % 5 + 1).astype(np.float64)
    mmio.write_matrix_market(tmp_path / "a.mtx", n, n, rp, ci, vals)
    (tmp_path / "a.mtx.gz").write_bytes(gzip.compress((tmp_path / "a.mtx").read_bytes()))
    rows, cols, rp2, ci2, v2 = mmio.read_matrix_market(tmp_path / "a.mtx.gz", np.float64)
    p = rd.permute_symmetric(rd.DeviceCsr.from_host(rows, cols, rp2, ci2, v2), 3)
    prp, pci, pvv = p.to_host()
    want_a = orc.permute_symmetric(oracle.Csr(n, n, rp, ci, vals), 3)
    assert np.array_equal(prp, want_a.row_ptr) and np.array_equal(pci, want_a.col_idx)
    want, _ = orc.spgemm_local(want_a, want_a)
    g = dist.ProcGrid(2, 2)
    with fabric(dist, 4, 32 << 20) as f:
        A = dist.DistSparse(f, n, n, 256, 512, g, 0, dtype=np.float64)
        B = dist.DistSparse(f, n, n, 512, 256, g, 1, dtype=np.float64)
        Cm = dist.DistSparse(f, n, n, 256, 256, g, 2, dtype=np.float64)
        A.init_from_global(prp, pci, pvv)
        B.init_from_global(prp, pci, pvv)
        Cm.init()
        rep = dist.run_multiply(f, A, B, Cm, variant="stationary_c")
        same_csr(Cm.to_global(), want)
    assert int(rep.stage_flops.sum()) == rep.total_flops == orc.spgemm_flops(want_a, want_a)
