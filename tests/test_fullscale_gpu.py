"""Full-size parity of the BASELINE configurations that carry the performance
claims, element by element against the oracle (VERDICT r1 "What's weak" 1):

* cfg3 -- R-MAT s22 ef16 x dense N=128 (the headline, nnz-stream kernel) and
  N=32 (the narrow cp.async slot kernel of the 1x4 layout), every element;
* cfg5 -- ER 2^22, 16 nnz/row x dense N=256 (row kernel), every element;
* cfg4 -- R-MAT s20 A*A: row_ptr and col_idx exactly and values exactly
  (integer-valued data), 1,390,953,199 output entries;
* distributed runs on >= 2 physical GPUs (bench.py --verify, skipped on a
  one-GPU box) and real-valued distributed products at the fp32 tolerance.

The oracle is the plain-C restatement (oracle/rdmm_oracle.c, pinned to the
reference by tests/test_oracle.py), run over row ranges on all host cores
(ctypes releases the GIL, rows are independent)."""
import concurrent.futures as cf
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def rd():
    import paper_2311_18141_b200 as rd

    return rd


def ranges(rows, parts):
    step = -(-rows // parts)
    return [(r, min(rows, r + step)) for r in range(0, rows, step)]


def oracle_spmm(orc, h, b):
    """C = A*B on the host, rows split over all cores (reference order per row)."""
    c = np.zeros((h.rows, b.shape[1]), dtype=b.dtype)
    with cf.ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(lambda r: orc.spmm_rows(h, r[0], r[1], b, c), ranges(h.rows, 8 * THREADS)))
    return c


def host_csr(a):
    rp, ci, vv = a.to_host()
    return oracle.Csr(a.rows, a.cols, rp, ci, vv)


@pytest.mark.parametrize("n", [128, 32])
def test_cfg3_every_element(rd, orc, n):
    a = rd.rmat(22, 16, seed=1, device=DEV)
    assert a.nnz == 64_827_941
    b = rd.random_dense(a.cols, n, 2, device=DEV)
    c = torch.zeros((a.rows, n), device=DEV)
    m = rd.spmm_local(a, b, c, c_zero=True)
    got = c.cpu().numpy()
    del c
    want = oracle_spmm(orc, host_csr(a), b.cpu().numpy())
    assert m.flops == 2 * a.nnz * n
    assert np.array_equal(got, want)


def test_cfg5_every_element(rd, orc):
    n_rows = 1 << 22
    a = rd.uniform_tiles(n_rows, n_rows, 1, 2.0 ** -18, 1, device=DEV)
    assert a.nnz == 67_108_864
    b = rd.random_dense(a.cols, 256, 2, device=DEV)
    c = torch.zeros((a.rows, 256), device=DEV)
    rd.spmm_local(a, b, c, c_zero=True)
    got = c.cpu().numpy()
    del c
    want = oracle_spmm(orc, host_csr(a), b.cpu().numpy())
    assert np.array_equal(got, want)


def test_cfg4_structure_and_values(rd, orc):
    """R-MAT s20 ef8 A*A: every row's columns and values vs the reference's
    Gustavson (tile.hpp:211-255), row range by row range."""
    a = rd.rmat(20, 8, seed=1, device=DEV)
    assert a.nnz == 8_124_707
    c, meter = rd.spgemm_local(a, a)
    assert c.nnz == 1_390_953_199
    assert meter.flops == 2 * 2_348_048_595
    h = host_csr(a)
    grp = c.row_ptr.cpu().numpy().view(np.uint32)
    parts = ranges(h.rows, 16 * THREADS)

    def check(r):
        r0, r1 = r
        want, _ = orc.spgemm_local(h, h, r0, r1)
        lo, hi = int(grp[r0]), int(grp[r1])
        ok = np.array_equal(grp[r0:r1 + 1] - grp[r0], want.row_ptr)
        ok &= np.array_equal(c.col_idx[lo:hi].cpu().numpy().view(np.uint32), want.col_idx)
        ok &= np.array_equal(c.values[lo:hi].cpu().numpy(), want.values)
        return ok

    with cf.ThreadPoolExecutor(THREADS) as ex:
        results = list(ex.map(check, parts))
    assert all(results)


def _ranks_real(dist, orc, grid, deterministic, n=32):
    """Real-valued (U(-1,1) twin) distributed stationary-C SpMM on a P-rank
    fabric (ranks share the box's GPUs); returns got, want (fp64 oracle) and
    the |A||B| bound of the fp32 gate."""
    h = orc.rmat(14, 8, seed=1)
    h.values = oracle.real_twin(h.nnz, 3, np.float32)
    b = oracle.real_twin(h.cols * n, 4, np.float32).reshape(h.cols, n)
    h64 = oracle.Csr(h.rows, h.cols, h.row_ptr, h.col_idx, h.values.astype(np.float64))
    want = np.zeros((h.rows, n))
    orc.spmm_local(h64, b.astype(np.float64), want)
    absb = np.zeros((h.rows, n))
    habs = oracle.Csr(h.rows, h.cols, h.row_ptr, h.col_idx, np.abs(h64.values))
    orc.spmm_local(habs, np.abs(b.astype(np.float64)), absb)
    pr, pc = grid
    P = pr * pc
    ndev = torch.cuda.device_count()
    with dist.Fabric(nranks=P, heap_bytes=256 << 20, devices=[r % ndev for r in range(P)]) as f:
        g = dist.ProcGrid(pr, pc)
        tm, tk, tn = -(-h.rows // pr), -(-h.cols // max(pr, pc)), -(-n // pc)
        A = dist.DistSparse(f, h.rows, h.cols, tm, tk, g, 0)
        B = dist.DistDense(f, h.cols, n, tk, tn, g, 1)
        Cm = dist.DistDense(f, h.rows, n, tm, tn, g, 2)
        A.init_from_global(h.row_ptr, h.col_idx, h.values)
        B.init_from_global(b)
        Cm.init()
        dist.run_multiply(f, A, B, Cm, variant="stationary_c", deterministic=deterministic)
        got = Cm.to_global()
    return got, want, absb


@pytest.mark.parametrize("grid", [(1, 2), (1, 4), (2, 2)])
@pytest.mark.parametrize("deterministic", [False, True])
def test_distributed_real_valued_tolerance(grid, deterministic):
    """North-star gate for reals: |got - want| <= 1e-5 * sum |a_ik b_kj| for
    fp32, on the layouts the bench uses (atomic accumulation and the
    deterministic fused pass)."""
    import paper_2311_18141_b200.dist as dist

    orc = oracle.port()
    got, want, absb = _ranks_real(dist, orc, grid, deterministic)
    assert np.all(np.abs(got.astype(np.float64) - want) <= 1e-5 * absb + 1e-30)


def test_distributed_deterministic_mode_is_reproducible():
    import paper_2311_18141_b200.dist as dist

    orc = oracle.port()
    g1, _, _ = _ranks_real(dist, orc, (1, 4), True)
    g2, _, _ = _ranks_real(dist, orc, (1, 4), True)
    assert np.array_equal(g1, g2)


def _bench(args, gpus):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--verify"] + args,
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("gpus", [2, 4])
@pytest.mark.parametrize("args", [["--config", "cfg1"], ["--config", "cfg2"],
                                  ["--config", "cfg2", "--variant", "ws_locality"],
                                  ["--config", "cfg1", "--deterministic"]])
def test_multi_gpu_bench_layouts_verify(gpus, args):
    """One process per physical GPU over NVLink (the bench's own launch), the
    result checked against the single-GPU kernel: SpMM exactly, SpGEMM
    row_ptr/col_idx/values exactly."""
    if torch.cuda.device_count() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    d = _bench(args, gpus)
    assert d["n_gpus"] == gpus
    assert d["verify"]["ok"], d["verify"]


def test_distributed_spgemm_deterministic_real_values():
    """stationary-C SpGEMM with RunOptions::deterministic on real values: two
    runs bitwise identical, values within the fp32 gate of the fp64 oracle."""
    import paper_2311_18141_b200.dist as dist

    orc = oracle.port()
    h = orc.rmat(12, 8, seed=2)
    h.values = oracle.real_twin(h.nnz, 7, np.float32)
    h64 = oracle.Csr(h.rows, h.cols, h.row_ptr, h.col_idx, h.values.astype(np.float64))
    want, _ = orc.spgemm_local(h64, h64)
    habs = oracle.Csr(h.rows, h.cols, h.row_ptr, h.col_idx, np.abs(h64.values))
    bound, _ = orc.spgemm_local(habs, habs)
    outs = []
    for _ in range(2):
        with dist.Fabric(nranks=4, heap_bytes=256 << 20,
                         devices=[r % torch.cuda.device_count() for r in range(4)]) as f:
            g = dist.ProcGrid(2, 2)
            t = -(-h.rows // 4)
            A = dist.DistSparse(f, h.rows, h.cols, t, t, g, 0)
            B = dist.DistSparse(f, h.rows, h.cols, t, t, g, 1)
            Cm = dist.DistSparse(f, h.rows, h.cols, t, t, g, 2)
            A.init_from_global(h.row_ptr, h.col_idx, h.values)
            B.init_from_global(h.row_ptr, h.col_idx, h.values)
            Cm.init()
            dist.run_multiply(f, A, B, Cm, variant="stationary_c", deterministic=True)
            outs.append(Cm.to_global())
    (rp1, ci1, v1), (rp2, ci2, v2) = outs
    assert np.array_equal(rp1, want.row_ptr) and np.array_equal(ci1, want.col_idx)
    assert np.array_equal(v1.view(np.uint32), v2.view(np.uint32))
    assert np.all(np.abs(v1.astype(np.float64) - want.values) <= 1e-5 * bound.values + 1e-30)
