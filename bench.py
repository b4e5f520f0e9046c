#!/usr/bin/env python
"""Benchmark driver (measurement contract: DESIGN.md §5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
                    [--variant stationary_c|ws_locality|...|summa_nccl]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)
    python bench.py --impl reference ...                  (reference CPU path)

Prints ONE JSON line (rank 0).  A step is one distributed multiply
C = A*B of BASELINE.json's configuration through the reference entry point
run_multiply (one process per GPU, the one-sided fabric over NVLink), C
reset to zero (SpMM) / empty (SpGEMM) before each step outside the timed
region, inputs resident in HBM.  `value` = total useful GFLOP/s over all
ranks (max-over-ranks device time).  `e2e` repeats the step through the
public API from pinned HOST buffers (upload of A and of the rank's B tiles,
download of the rank's C tiles inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0..4]
    "cfg1": dict(kind="spmm", gen="rmat", scale=16, ef=8, n=128,
                 desc="SpMM R-MAT s16 ef8 x dense 65536x128 fp32"),
    "cfg2": dict(kind="spgemm", gen="rmat", scale=17, ef=8, variant="stationary_c",
                 grid="square", desc="SpGEMM A*A, R-MAT s17 ef8"),
    "cfg3": dict(kind="spmm", gen="rmat", scale=22, ef=16, n=128,
                 desc="SpMM R-MAT s22 ef16 x dense 4194304x128 fp32"),
    "cfg4": dict(kind="spgemm", gen="rmat", scale=20, ef=8, variant="ws_locality",
                 grid="square", desc="SpGEMM A*A, R-MAT s20 ef8"),
    "cfg5": dict(kind="spmm", gen="er", scale=22, n=256, d=2.0 ** -18,
                 desc="SpMM Erdos-Renyi 2^22, 16 nnz/row x dense N=256 fp32"),
}
DEFAULT_CONFIG = "cfg3"
METRIC = "SpMM/SpGEMM useful GFLOP/s at 1/2/4/8 B200; fraction of HBM roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.path = gpu, None, None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for ln in open(self.path):
                f = [x.strip() for x in ln.split(",")]
                if len(f) >= 9 and f[1].replace(".", "").isdigit():
                    rows.append(f)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows)}


def row_sample(rp, ci, vv, stride):
    """Every `stride`-th row of a host CSR (keeps the degree distribution)."""
    import numpy as np

    rows = (len(rp) - 1 + stride - 1) // stride
    deg_all = (rp[1:].astype(np.int64) - rp[:-1])
    row_of = np.repeat(np.arange(len(rp) - 1), deg_all)
    keep = row_of % stride == 0
    deg = deg_all[::stride]
    nrp = np.zeros(rows + 1, np.uint32)
    nrp[1:] = np.cumsum(deg)
    return nrp, ci[keep], vv[keep]


def p2p_peak():
    """Measured peer-copy bandwidth per GPU (tools/p2p_bw.py on this pool's
    B200s, committed under profiles/); nominal NVLink 5 otherwise."""
    for name in ("r2_p2p.json", "r1_diag2/p2p.json"):
        try:
            best = 0.0
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                for ln in fh:
                    ln = ln.strip()
                    if ln.startswith("{"):
                        best = max(best, float(json.loads(ln)["GBps_per_rank"]))
            if best:
                return best, f"measured, profiles/{name} (tools/p2p_bw.py)"
        except Exception:
            pass
    return 900.0, "nominal NVLink 5 per direction"


def cdev():
    """Device of the small tensors of the bench's own collectives: the GPU
    under NCCL, the host under gloo (more ranks than GPUs)."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_backend() == "gloo":
        return torch.device("cpu")
    return torch.device("cuda", torch.cuda.current_device())


def verify(args, cfg, dev, rank, world, A, Cm, grid, tiles, tdist):
    """Compare the distributed result with the single-GPU kernel on the
    global operands (itself pinned to the oracle by tests/): SpMM owned C
    tiles exactly (integer-valued inputs), SpGEMM row_ptr/col_idx/values of
    the gathered C exactly."""
    import numpy as np
    import torch
    import paper_2311_18141_b200 as rd

    a, b = gen_inputs(cfg, dev, args.permute)
    tm, tk, tn = tiles
    ok = True
    if cfg["kind"] == "spmm":
        want = torch.zeros((a.rows, b.shape[1]), device=dev)
        rd.spmm_local(a, b, want, c_zero=True)
        got = torch.zeros((a.rows, b.shape[1]), dtype=torch.float32).pin_memory()
        Cm.owned_to_host(got)
        torch.cuda.synchronize()
        w = want.cpu()
        for i in range(-(-a.rows // tm)):
            for j in range(-(-b.shape[1] // tn)):
                if grid.owner(i, j) == rank:
                    sl = (slice(i * tm, (i + 1) * tm), slice(j * tn, (j + 1) * tn))
                    ok &= bool(torch.equal(got[sl], w[sl]))
        what = "owned C tiles == single-GPU spmm_local(A, B) (exact, integer data)"
    else:
        if rank == 0:
            c, _ = rd.spgemm_local(a, a)
            rp, ci, vv = c.to_host()
            grp, gci, gvv = Cm.to_global()
            ok = bool(np.array_equal(rp, grp) and np.array_equal(ci, gci) and
                      np.array_equal(vv, gvv))
        what = "gathered C row_ptr/col_idx/values == single-GPU spgemm_local(A, A) (exact)"
    if tdist:
        t = torch.tensor([0 if ok else 1], device=cdev())
        tdist.all_reduce(t)
        ok = int(t[0]) == 0
    return {"ok": ok, "checked": what}


def load_traffic(config, kernel, n_gpus):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{config}@{n_gpus}", {}).get(kernel)
    except Exception:
        return None


def layout(cfg, P, args):
    """ProcGrid and tile sizes for P ranks.

    SpMM: a 1 x P grid (B and C split by columns, A by K = P column tiles):
    every rank computes all rows of A against its N/P columns of B, so the
    work is balanced whatever R-MAT's row skew (rank 0 of a P x 1 row split
    holds 0.733^log2(P) of the nonzeros), only A's tiles cross NVLink
    ((P-1)/P of A per rank: 402 MB at P = 4 on cfg3) and B stays
    put.  It needs the narrow-row kernel (spmm_slots_async: N = 32 on cfg3's
    A in 1.12 ms); columns are split while every rank keeps
    >= 16 of them.
    SpGEMM: a square-ish pr x pc grid with 4 pr row tiles of C and K = pr
    (cfg2 stationary-C, cfg4 ws_locality): at 4 GPUs 2x2 beats 4x1 by 1.25x
    (cfg2) and 1.44x (cfg4), profiles/r1_s5, r1_s9.
    """
    n_rows = 1 << cfg["scale"]
    if args.grid:
        pr, pc = (int(x) for x in args.grid.split("x"))
    elif cfg.get("grid") == "square":
        # SpGEMM on a square-ish 2D grid (2x2 at 4 GPUs, 4x2 at 8)
        pc = max(d for d in range(1, int(P ** 0.5) + 1) if P % d == 0)
        pr = P // pc
    else:
        pc = max(d for d in range(1, P + 1) if P % d == 0 and cfg["n"] // d >= 16)
        pr = P // pc
    mt = args.mtiles or (pr if cfg["kind"] == "spmm" else 4 * pr)
    kt = args.ktiles or (max(pr, pc) if cfg["kind"] == "spmm" else pr)
    ncols = cfg["n"] if cfg["kind"] == "spmm" else n_rows
    nt = args.ntiles or pc
    return (pr, pc), (-(-n_rows // mt), -(-n_rows // kt), -(-ncols // nt))


# ----------------------------------------------------------------- our arm


def owned_dense_bytes(grid, rows, cols, tr, tc, rank):
    """fp32 bytes of the dense tiles `rank` owns (ProcGrid owner rule)."""
    tot = 0
    for i in range(-(-rows // tr)):
        for j in range(-(-cols // tc)):
            if grid.owner(i, j) == rank:
                tot += (min(rows, (i + 1) * tr) - i * tr) * (min(cols, (j + 1) * tc) - j * tc) * 4
    return tot


def gen_inputs(cfg, dev, permute=0):
    import paper_2311_18141_b200 as rd
    import torch

    if cfg["gen"] == "rmat":
        a = rd.rmat(cfg["scale"], cfg["ef"], seed=1, device=dev)
    else:
        n = 1 << cfg["scale"]
        a = rd.uniform_tiles(n, n, 1, cfg["d"], 1, device=dev)
    if permute:  # gen.hpp:134-155 symmetric relabelling (not the BASELINE default)
        a = rd.permute_symmetric(a, permute)
    b = rd.random_dense(a.cols, cfg["n"], 2, device=dev) if cfg["kind"] == "spmm" else None
    torch.cuda.synchronize()
    return a, b


def cpu_baseline(a, b, cfg):
    """Reference spmm_local / spgemm_local (oracle/_ref = the unmodified
    reference headers; else the C port) on this host, 1 core, bounded
    sample: every S-th row of A."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle

    impl, kind = (oracle.ref(), "reference") if oracle.ref_available() else (oracle.port(), "port")
    rp, ci, vv = a.to_host()
    if cfg["kind"] == "spmm":
        bh = b.cpu().numpy()
        stride = 1 if a.nnz < 5_000_000 else 4
        nrp, nci, nvv = row_sample(rp, ci, vv, stride)
        h = oracle.Csr(len(nrp) - 1, a.cols, nrp, nci, nvv)
        c = np.zeros((h.rows, bh.shape[1]), np.float32)
        t0 = time.perf_counter()
        fl = impl.spmm_local(h, bh, c)
        dt = time.perf_counter() - t0
        what = "spmm_local"
    else:
        stride = 16 if a.nnz < 2_000_000 else 256
        nrp, nci, nvv = row_sample(rp, ci, vv, stride)
        h = oracle.Csr(len(nrp) - 1, a.cols, nrp, nci, nvv)
        full = oracle.Csr(a.rows, a.cols, rp, ci, vv)
        t0 = time.perf_counter()
        _, fl = impl.spgemm_local(h, full)
        dt = time.perf_counter() - t0
        what = "spgemm_local"
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": kind,
            "sample": f"{what} over every {stride}th row of A ({h.rows} rows, {h.nnz} nnz, "
                      f"{fl} flop), 1 thread, {dt:.2f} s"}


def make_session(world, rank):
    if world == 1:
        return None
    import torch.distributed as dist

    obj = [f"b{os.getpid()}_{time.time_ns() % 10**9}" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def run_ours(args, cfg, dev, rank, world):
    import torch
    import paper_2311_18141_b200 as rd
    import paper_2311_18141_b200.dist as dm
    from paper_2311_18141_b200 import _lib as L
    import numpy as np
    from paper_2311_18141_b200.analytics import imbalance_from_flops, imbalance_from_times

    tdist = torch.distributed if world > 1 else None
    a, b = gen_inputs(cfg, dev, args.permute)
    m, k, nnz_a = a.rows, a.cols, a.nnz
    rp_host = a.row_ptr.cpu().numpy().view("uint32")
    n = cfg["n"] if cfg["kind"] == "spmm" else a.cols
    (pr, pc), (tm, tk, tn) = layout(cfg, world, args)
    grid = dm.ProcGrid(pr, pc)
    session = make_session(world, rank)
    a_bytes = nnz_a * 8 + (m + 1) * 4
    if cfg["kind"] == "spmm":
        heap = int(2 * (a_bytes + 4 * (k * n + m * n)) / world) + (1 << 30)
    else:
        heap = int(4 * a_bytes) + (14 << 30) // world + (2 << 30)
    f = dm.Fabric(nranks=world, heap_bytes=heap, first_local=rank, nlocal=1,
                  devices=[dev.index], session=session)
    A = dm.DistSparse(f, m, k, tm, tk, grid, 0)
    if cfg["kind"] == "spmm":
        B = dm.DistDense(f, k, n, tk, tn, grid, 1)
        Cm = dm.DistDense(f, m, n, tm, tn, grid, 2)
        A.init_from_device(a)
        B.init_from_device(b)
        Cm.init()
        reset = Cm.zero
    else:
        B = dm.DistSparse(f, k, n, tk, tn, grid, 1)
        Cm = dm.DistSparse(f, m, n, tm, tn, grid, 2)
        A.init_from_device(a)
        B.init_from_device(a)
        Cm.init()
        reset = Cm.init
    variant = args.variant
    # ws_random steals stationary-A reservations only (algos.hpp:476-533)
    ws_base = "stationary_a" if variant == "ws_random" else "stationary_c"
    opts = dict(variant=variant, ws_base=ws_base, checksum=False, record_events=False,
                fuse_k=not args.no_fuse, lookahead=args.lookahead,
                split_local=not args.no_split, pipeline=not args.no_pipeline,
                deterministic=args.deterministic,
                row_blocks=args.row_blocks)
    stream = torch.cuda.ExternalStream(f.stream(rank), device=dev)

    def barrier():
        if tdist:
            tdist.barrier()

    for _ in range(args.warmup):
        reset()
        dm.run_multiply(f, A, B, Cm, **opts)
    torch.cuda.synchronize()
    f.clear_traffic()
    L.rdmm_kernel_timing(1)
    launches0 = L.rdmm_kernel_launches()
    per, flops_local, steals = [], 0, 0
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            reset()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = dm.run_multiply(f, A, B, Cm, **opts)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            per.append(e0.elapsed_time(e1))
            flops_local = rep.total_flops
            steals += rep.total_steals
    launches = L.rdmm_kernel_launches() - launches0
    kind_id = 1 if cfg["kind"] == "spmm" else 2
    kms, kcount = L.kernel_time(kind_id)
    L.rdmm_kernel_timing(0)
    ms_local = sum(per) / len(per)
    # NVLink bytes into this rank's GPU per step: the fabric's byte-exact
    # traffic log (gets from peers, contributions read in place)
    nvl_local = f.remote_bytes_in(rank) / args.steps
    # Analytics (analytics.hpp:66-90) on one extra, instrumented run outside
    # the timed loop: the per-rank per-k-step flop table and the per-rank
    # per-k-step device time of the multiply kernels (cudaEvents on the
    # compute stream, RunOptions::time_stages).  Rows of ranks hosted by
    # other processes are zero, so a SUM over processes assembles the tables.
    reset()
    barrier()
    rep_t = dm.run_multiply(f, A, B, Cm, **{**opts, "time_stages": True})
    torch.cuda.synchronize()
    barrier()
    sf = rep_t.stage_flops
    sm_ = rep_t.stage_ms if rep_t.stage_ms is not None else np.zeros(sf.shape)
    width = torch.tensor([sf.shape[1]], device=cdev(), dtype=torch.int64)
    if tdist:
        tdist.all_reduce(width, op=tdist.ReduceOp.MAX)
    tabs = torch.zeros((2, sf.shape[0], int(width[0])), device=cdev(), dtype=torch.float64)
    tabs[0, :, :sf.shape[1]] = torch.as_tensor(sf, dtype=torch.float64)
    tabs[1, :, :sm_.shape[1]] = torch.as_tensor(sm_, dtype=torch.float64)
    if tdist:
        tdist.all_reduce(tabs, op=tdist.ReduceOp.SUM)
    flop_tab, ms_tab = tabs[0].cpu().numpy(), tabs[1].cpu().numpy()
    imbalance = {**imbalance_from_flops(flop_tab), **imbalance_from_times(ms_tab),
                 "per_rank_kernel_ms": [round(float(x), 4) for x in ms_tab.sum(axis=1)],
                 "definition": "analytics.hpp:66-90 (per-stage = sum_s max_r / sum_s avg_r, "
                               "end-to-end = max_r / avg_r) over the run's per-rank per-k-step "
                               "flops and per-rank per-k-step multiply-kernel device time "
                               "(cudaEvents, RankStats::stage_ms)"}
    nvlink = None
    if tdist:  # NVLink bytes per rank per step, against the measured P2P bandwidth
        nv = torch.tensor([nvl_local], device=cdev(), dtype=torch.float64)
        alln = [torch.zeros_like(nv) for _ in range(world)]
        tdist.all_gather(alln, nv)
        nvl = [float(x[0]) for x in alln]
    if tdist:  # max over ranks of the device time; flops summed over ranks
        t = torch.tensor([ms_local, float(flops_local), float(steals)], device=cdev(),
                         dtype=torch.float64)
        tmax = t[:1].clone()
        tdist.all_reduce(tmax, op=tdist.ReduceOp.MAX)
        tsum = t[1:].clone()
        tdist.all_reduce(tsum, op=tdist.ReduceOp.SUM)
        ms, total_flops, steals = float(tmax[0]), int(tsum[0]), int(tsum[1])
        p2p, p2p_src = p2p_peak()
        nvlink = {"bytes_per_step_per_rank": nvl, "bytes_per_step_total": sum(nvl),
                  "achieved_gbs_max_rank": max(nvl) / (ms * 1e-3) / 1e9,
                  "p2p_gbs": p2p, "frac": max(nvl) / (ms * 1e-3) / 1e9 / p2p,
                  "p2p_source": p2p_src,
                  "source": "fabric TrafficLog (fabric.hpp:89-203): bytes each rank fetched "
                            "from peers during the timed steps / step; achieved = busiest "
                            "rank's bytes over the max-over-ranks step time"}
    else:
        ms, total_flops = ms_local, flops_local
    out_nnz = Cm.nnz() if cfg["kind"] == "spgemm" else None

    # ---- roofline of the dominant kernel on this rank
    hbm, peak_src = peaks()
    if cfg["kind"] == "spmm":
        ktiles = -(-k // tk)
        # per-rank compulsory bytes over the owned C tiles (i, j): the A row
        # block's tiles once (row_ptr per k tile + col/val), B(:, j) once, C
        # tile written once
        alg = 0
        for i in range(-(-m // tm)):
            for j in range(-(-n // tn)):
                if grid.owner(i, j) != rank:
                    continue
                r0, r1 = i * tm, min(m, (i + 1) * tm)
                cols = min(n, (j + 1) * tn) - j * tn
                nnz_i = int(rp_host[r1]) - int(rp_host[r0])
                alg += 4 * (r1 - r0 + 1) * ktiles + 8 * nnz_i + 4 * k * cols + 4 * (r1 - r0) * cols
        kernel = "spmm_stream_full|spmm_stream|spmm_slots_async + spmm_fixup (rdmm_spmm_csr), all launches of a step on this rank"
    else:
        alg = (2 * a_bytes + (m + 1) * 4 + 8 * (out_nnz or 0)) // world
        kernel = ("spgemm symbolic + numeric passes (rdmm_spgemm_symbolic/numeric), per step "
                  "on this rank")
    kms_step = kms / max(1, args.steps)
    achieved = alg / (kms_step * 1e-3) / 1e9 if kms_step > 0 else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": (achieved / hbm) if achieved else None,
            "traffic": load_traffic(args.config, "spmm_stream" if kind_id == 1 else "spgemm",
                                    world),
            "algorithmic_bytes": alg, "peak_source": peak_src, "kernel": kernel,
            "kernel_ms_per_step": kms_step, "kernel_launches_timed": kcount}

    # ---- e2e: the same step through the public API from pinned HOST buffers.
    # Every step uploads its inputs (A's CSR arrays and B, pinned host ->
    # device staging on its own stream), builds the distributed operands from
    # them (init_from_device: A's tiles cut, B's tiles scattered on the
    # device), multiplies (run_multiply), and downloads its C tiles
    # (owned_to_host_async on a second stream).  Steps are pipelined the way a
    # serving loop would run them: step s+1's upload (H2D copy engine) and
    # step s's download (D2H copy engine) overlap, with two staging buffers
    # and two C matrices alternating.
    stg_a = [rd.DeviceCsr(a.rows, a.cols, a.nnz, torch.empty_like(a.row_ptr),
                          torch.empty_like(a.col_idx), torch.empty_like(a.values))
             for _ in range(2)]
    rp_h, ci_h, vv_h = (x.cpu().pin_memory() for x in (a.row_ptr, a.col_idx, a.values))
    h2d = sum(x.numel() * x.element_size() for x in (rp_h, ci_h, vv_h))
    if cfg["kind"] == "spmm":
        b_h = b.cpu().pin_memory()
        stg_b = [torch.empty_like(b) for _ in range(2)]
        h2d += b_h.numel() * b_h.element_size()
        c_h = [torch.empty((m, n), dtype=torch.float32).pin_memory() for _ in range(2)]
        C2 = [Cm, dm.DistDense(f, m, n, tm, tn, grid, 3)]
        C2[1].init()
        d2h = owned_dense_bytes(grid, m, n, tm, tn, rank)
    else:
        c_h = torch.empty(int(Cm.owned_bytes() * 1.05) + 4096, dtype=torch.uint8).pin_memory()
    del a, b
    up, down = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    e2e_steps = max(4, min(args.steps, 10))

    def upload(s):
        q = s % 2
        with torch.cuda.stream(up):
            stg_a[q].row_ptr.copy_(rp_h, non_blocking=True)
            stg_a[q].col_idx.copy_(ci_h, non_blocking=True)
            stg_a[q].values.copy_(vv_h, non_blocking=True)
            if cfg["kind"] == "spmm":
                stg_b[q].copy_(b_h, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
        return ev

    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev_in = {0: upload(0)}
    ev_out = {}
    for s_ in range(e2e_steps):
        q = s_ % 2
        if s_ + 1 < e2e_steps:
            ev_in[s_ + 1] = upload(s_ + 1)   # queued behind step s_'s upload
        ev_in[s_].synchronize()
        A.init_from_device(stg_a[q])
        if cfg["kind"] == "spmm":
            B.init_from_device(stg_b[q])
            if s_ - 2 in ev_out:
                ev_out[s_ - 2].synchronize()  # C2[q]'s previous download landed
            C2[q].zero()
            dm.run_multiply(f, A, B, C2[q], **opts)
            C2[q].owned_to_host_async(c_h[q], down)
            ev_out[s_] = torch.cuda.Event()
            ev_out[s_].record(down)
        else:
            B.init_from_device(stg_a[q])
            reset()
            dm.run_multiply(f, A, B, Cm, **opts)
            d2h = Cm.owned_to_host(c_h)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = 1e3 * (time.perf_counter() - t0) / e2e_steps
    if tdist:
        t = torch.tensor([e2e_ms], device=cdev(), dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t[0])

    out = {
        "metric": METRIC,
        "value": total_flops / (ms * 1e-3) / 1e9,
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (reference generators, seeds A=1 B=2, built on device)",
        "config": {"workload": args.config, "desc": cfg["desc"], "permute_seed": args.permute,
                   "rows": m, "cols": k, "n": n,
                   "nnz": nnz_a, "flop_per_step": total_flops,
                   "variant": variant, "fuse_k": not args.no_fuse,
                   "split_local": not args.no_split, "pipeline": not args.no_pipeline, "deterministic": args.deterministic,
                   "row_blocks": args.row_blocks or 8, "lookahead": args.lookahead,
                   "grid": f"{pr}x{pc}", "tiles": [tm, tk, tn],
                   "path": "run_multiply (host C-ABI rdmm_h_run_multiply) over the fabric",
                   "l2": ("inputs > L2 (A %.2f GB, B and C %.2f GB each)"
                          % (nnz_a * 8 / 1e9, m * n * 4 / 1e9)) if cfg["kind"] == "spmm"
                   else "inputs + output > L2", "steals": steals},
        "roofline": roof,
        "e2e": {"value": total_flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "steps": e2e_steps,
                "timer": "host wall clock over the pipelined steps (pinned H2D of A and B, "
                         "init_from_device, run_multiply, D2H of C); step s+1's upload "
                         "overlaps step s's download"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if imbalance:
        out["imbalance"] = imbalance
    if nvlink:
        out["nvlink"] = nvlink
    if args.verify:
        out["verify"] = verify(args, cfg, dev, rank, world, A, Cm, grid, (tm, tk, tn), tdist)
    # the paper's roofline model (model.hpp:139-160) with B200 costs: local
    # HBM bound and NVLink inter-GPU bound for this shape at N GPUs
    from paper_2311_18141_b200 import model as md
    try:
        shp = md.ProblemShape(m, k, n, world, nnz_a / (float(m) * k), 4)
        mod = md.roofline(shp, md.CostModel(mem_bw=hbm * 1e9), cfg["kind"], total_flops,
                          out_nnz or 0)
        out["model"] = {"local_peak_gflops": mod["local_peak"] / 1e9,
                        "internode_bound_gflops": mod["internode_bound"] * world / 1e9,
                        "bound_kind": mod["bound_kind"], "local_ai": mod["local_ai"],
                        "internode_ai": mod["internode_ai"],
                        "value_over_bound": out["value"] / (mod["internode_bound"] * world / 1e9),
                        "source": "model.hpp:139-160, B200 CostModel (NVLink 900 GB/s, "
                                  "measured HBM, fp32 FMA peak); bound x n_gpus"}
    except ValueError as e:
        out["model"] = {"unavailable": str(e)}
    if out_nnz is not None:
        out["config"]["nnz_out"] = out_nnz
    f.close()
    return out


def run_summa_nccl(args, cfg, dev, rank, world):
    """The comparison point: bulk-synchronous SUMMA with NCCL broadcasts of
    A(i,k) along grid rows and B(k,j) along grid columns each phase, the
    same sm_100a SpMM kernel, and a barrier per phase (algos.hpp:348-374
    with the broadcast the reference emulates)."""
    import torch
    import torch.distributed as dist
    import paper_2311_18141_b200 as rd
    from paper_2311_18141_b200.tile import extract_tile

    assert cfg["kind"] == "spmm", "summa_nccl baseline is for SpMM configs"
    a, b = gen_inputs(cfg, dev)
    m, k, n = a.rows, a.cols, cfg["n"]
    (pr, pc), (tm, tk, tn) = layout(cfg, world, args)
    Mt, Kt, Nt = -(-m // tm), -(-k // tk), -(-n // tn)
    gi, gj = rank // pc, rank % pc
    rows_g = [dist.new_group([r * pc + c for c in range(pc)]) for r in range(pr)] \
        if world > 1 else None
    cols_g = [dist.new_group([r * pc + c for r in range(pr)]) for c in range(pc)] \
        if world > 1 else None
    my_row = [i for i in range(Mt) if i % pr == gi]
    my_col = [j for j in range(Nt) if j % pc == gj]
    dims = lambda i, kk: (i * tm, min(tm, m - i * tm), kk * tk, min(tk, k - kk * tk))  # noqa
    A_own = {(i, kk): extract_tile(a, *dims(i, kk)) for i in range(Mt) for kk in range(Kt)
             if i % pr == gi and kk % pc == gj}
    B_own = {(kk, j): b[kk * tk:kk * tk + min(tk, k - kk * tk), j * tn:j * tn + min(tn, n - j * tn)]
             .contiguous() for kk in range(Kt) for j in range(Nt)
             if kk % pr == gi and j % pc == gj}
    nnz_tile = {}
    for i in range(Mt):
        for kk in range(Kt):
            t = extract_tile(a, *dims(i, kk))
            nnz_tile[(i, kk)] = t.nnz
            del t
    C = {(i, j): torch.zeros((min(tm, m - i * tm), min(tn, n - j * tn)), device=dev)
         for i in my_row for j in my_col}
    flops_local = sum(2 * nnz_tile[(i, kk)] * min(tn, n - j * tn)
                      for (i, j) in C for kk in range(Kt))
    del a, b

    def step():
        for kk in range(Kt):
            a_t, b_t = {}, {}
            for i in my_row:
                root = (i % pr) * pc + (kk % pc)
                t = A_own.get((i, kk)) or rd.DeviceCsr.empty(
                    min(tm, m - i * tm), min(tk, k - kk * tk), nnz_tile[(i, kk)], device=dev)
                if world > 1 and pc > 1:
                    dist.broadcast(t.row_ptr, root, group=rows_g[gi])
                    if t.nnz:
                        dist.broadcast(t.col_idx, root, group=rows_g[gi])
                        dist.broadcast(t.values, root, group=rows_g[gi])
                a_t[i] = t
            for j in my_col:
                root = (kk % pr) * pc + (j % pc)
                t = B_own.get((kk, j))
                if t is None:
                    t = torch.empty((min(tk, k - kk * tk), min(tn, n - j * tn)), device=dev)
                if world > 1 and pr > 1:
                    dist.broadcast(t, root, group=cols_g[gj])
                b_t[j] = t
            for (i, j), c in C.items():
                rd.spmm_local(a_t[i], b_t[j], c, c_zero=(kk == 0))
            if world > 1:
                dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    per = []
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
    ms, total = sum(per) / len(per), flops_local
    if world > 1:
        tmax = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = torch.tensor([float(flops_local)], device=dev, dtype=torch.float64)
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms, total = float(tmax[0]), int(tsum[0])
    return {"metric": METRIC, "value": total / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generators, seeds A=1 B=2, built on device)",
            "config": {"workload": args.config, "desc": cfg["desc"], "variant": "summa_nccl",
                       "grid": f"{pr}x{pc}", "tiles": [tm, tk, tn],
                       "path": "NCCL-broadcast SUMMA baseline (torch.distributed + rdmm SpMM)"},
            "clocks": clk.summary()}


# ----------------------------------------------------------- reference arm


def run_reference(args):
    """The reference's own CPU path (oracle/_ref: the unmodified reference
    headers) timed on this host with all its threads: run_multiply
    stationary_c over a ProcGrid as square as possible."""
    import ctypes as C

    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    cfg = CONFIGS[args.config]
    if not oracle.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}
    R, Pn = oracle.ref(), oracle.port()
    threads = int(R._hardware_concurrency()) or os.cpu_count() or 1
    pr = int(np.sqrt(threads))
    while threads % pr:
        pr -= 1
    pc = threads // pr
    a = Pn.rmat(cfg["scale"], cfg["ef"], seed=1) if cfg["gen"] == "rmat" else \
        Pn.uniform_tiles(1 << cfg["scale"], 1 << cfg["scale"], 1, cfg["d"], 1)
    if cfg["kind"] == "spmm":
        n = cfg["n"]
        b = Pn.random_dense(a.cols, n, 2)
        S = 1 if a.nnz < 5_000_000 else 8
        rp, nci, nvv = row_sample(a.row_ptr, a.col_idx, a.values, S)
        hs = oracle.Csr(len(rp) - 1, a.cols, rp, nci, nvv)
        m, k = hs.rows, hs.cols
        tm, tk, tn = -(-m // pr), -(-k // pc), -(-n // pc)
        ao, keep = oracle.as_orc(hs)
        L = R.lib
        L.ref_spmm_session_create.restype = C.c_void_p
        L.ref_spmm_session_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                              C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                              C.POINTER(oracle.OrcCsr), C.c_void_p, C.c_uint64]
        L.ref_spmm_session_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64,
                                           C.POINTER(oracle.RefReport)]
        L.ref_spmm_session_destroy.argtypes = [C.c_void_p]
        sess = L.ref_spmm_session_create(pr, pc, m, k, n, tm, tk, tn, C.byref(ao),
                                         b.ctypes.data, 0)
        if not sess:
            return {"impl": "reference", "unavailable": "reference session setup failed"}
        rep = oracle.RefReport()
        times, flops = [], 0
        for i in range(args.warmup + args.steps):
            rc = L.ref_spmm_session_run(sess, oracle.VARIANTS["stationary_c"],
                                        oracle.VARIANTS["stationary_a"], 0, C.byref(rep))
            if rc:
                return {"impl": "reference", "unavailable": f"run_multiply failed ({rc})"}
            if i >= args.warmup:
                times.append(rep.wall_seconds)
                flops = rep.total_flops
        L.ref_spmm_session_destroy(sess)
        sample = (f"run_multiply stationary_c, {pr}x{pc} ProcGrid, {threads} rank threads, "
                  f"every {S}th row of A ({m} rows, {hs.nnz} nnz) x full B (N={n})")
    else:
        S = 64 if a.nnz < 2_000_000 else 1024
        rp, nci, nvv = row_sample(a.row_ptr, a.col_idx, a.values, S)
        hs = oracle.Csr(len(rp) - 1, a.cols, rp, nci, nvv)
        c0 = oracle.Csr(hs.rows, a.cols, np.zeros(hs.rows + 1, np.uint32),
                        np.zeros(0, np.uint32), np.zeros(0, np.float32))
        times, flops = [], 0
        for i in range(1 + args.steps):
            _, rep = R.run_multiply_spgemm(hs, a, c0, variant="stationary_c", grid=(pr, pc),
                                           tiles=(-(-hs.rows // pr), -(-a.cols // pc),
                                                  -(-a.cols // pc)))
            if i >= 1:
                times.append(rep.max_total_seconds)
                flops = rep.total_flops
        sample = (f"run_multiply stationary_c SpGEMM, {pr}x{pc} ProcGrid, {threads} rank "
                  f"threads, every {S}th row of A ({hs.rows} rows, {hs.nnz} nnz) x full A; "
                  f"max per-rank algorithm time")
    sec = sum(times) / len(times)
    val = flops / sec / 1e9
    return {
        "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators, seeds A=1 B=2)",
        "config": {"workload": args.config, "desc": cfg["desc"], "sample": sample},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def self_spawn(n):
    """`bench.py --gpus N` without torchrun: relaunch as one process per GPU
    (torch.distributed.run on 127.0.0.1) and pass rank 0's line through."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default=None,
                    help="stationary_c | stationary_a | stationary_b | ws_random | "
                         "ws_locality | summa_bsp | summa_nccl (baseline)")
    ap.add_argument("--grid", default=None, help="RxC ProcGrid override")
    ap.add_argument("--mtiles", type=int, default=0)
    ap.add_argument("--ktiles", type=int, default=0)
    ap.add_argument("--ntiles", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--permute", type=int, default=0,
                    help="relabel A with permute_symmetric(seed) first (0 = BASELINE order)")
    ap.add_argument("--no-fuse", action="store_true", help="RunOptions::fuse_k = false")
    ap.add_argument("--no-split", action="store_true", help="RunOptions::split_local = false")
    ap.add_argument("--lookahead", type=int, default=2, help="RunOptions::lookahead")
    ap.add_argument("--deterministic", action="store_true",
                    help="RunOptions::deterministic (fused k-order pass per narrow C tile)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="RunOptions::pipeline = false (whole-tile fetch, then fused pass)")
    ap.add_argument("--row-blocks", type=int, default=0, help="RunOptions::row_blocks")
    ap.add_argument("--verify", action="store_true",
                    help="check the distributed C against the single-GPU kernel")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.variant is None:
        args.variant = cfg.get("variant") or (
            "stationary_c" if cfg["kind"] == "spmm" else "ws_locality")

    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_spawn(args.gpus))

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # one process per GPU; more ranks than GPUs share them round-robin (a
    # functional check of a wider layout on a smaller box, not a bench line)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if world <= torch.cuda.device_count():
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:  # NCCL refuses two ranks on one GPU
            torch.distributed.init_process_group("gloo")
    if args.variant == "summa_nccl":
        out = run_summa_nccl(args, cfg, dev, rank, world)
    else:
        out = run_ours(args, cfg, dev, rank, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        a, b = gen_inputs(cfg, dev)
        out["cpu_baseline"] = cpu_baseline(a, b, cfg)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
