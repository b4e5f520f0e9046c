#!/usr/bin/env python
"""Benchmark driver (see DESIGN.md §5 for the measurement contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
    python bench.py --impl reference ...      # the reference CPU path

One JSON line on stdout (rank 0).  A "step" is one pass of the hot path over
one synthetic input of BASELINE.json's configuration: for SpMM, C += A*B with
A = R-MAT (or Erdos-Renyi) CSR and B dense fp32, everything resident in HBM
when the timed region starts.  `e2e` repeats the step through the public API
from pinned HOST buffers (H2D of A and B, D2H of C inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0..4]
    "cfg1": dict(kind="spmm", gen="rmat", scale=16, ef=8, n=128,
                 desc="SpMM R-MAT s16 ef8 x dense 65536x128 fp32"),
    "cfg2": dict(kind="spgemm", gen="rmat", scale=17, ef=8,
                 desc="SpGEMM A*A, R-MAT s17 ef8"),
    "cfg3": dict(kind="spmm", gen="rmat", scale=22, ef=16, n=128,
                 desc="SpMM R-MAT s22 ef16 x dense 4194304x128 fp32"),
    "cfg4": dict(kind="spgemm", gen="rmat", scale=20, ef=8,
                 desc="SpGEMM A*A, R-MAT s20 ef8"),
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
        self.gpu = gpu
        self.proc = None
        self.path = None

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


def spmm_bytes(m, k, n, nnz, w=4):
    """Compulsory bytes: 4(m+1) + (w+4) nnz + w k n + w m n."""
    return 4 * (m + 1) + (w + 4) * nnz + w * k * n + w * m * n


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


def load_traffic(config, kernel):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(config, {}).get(kernel)
    except Exception:
        return None


# ----------------------------------------------------------------- our arm


def make_spmm_inputs(cfg, dev):
    import paper_2311_18141_b200 as rd
    import torch

    if cfg["gen"] == "rmat":
        a = rd.rmat(cfg["scale"], cfg["ef"], seed=1, device=dev)
    else:
        n = 1 << cfg["scale"]
        a = rd.uniform_tiles(n, n, 1, cfg["d"], 1, device=dev)
    b = rd.random_dense(a.cols, cfg["n"], 2, device=dev)
    c = torch.zeros((a.rows, cfg["n"]), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    return a, b, c


def cpu_baseline_spmm(a, b, cfg_name):
    """Reference spmm_local (oracle/_ref, else the C port) on the host, 1 core."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    impl, kind = (oracle.ref(), "reference") if oracle.ref_available() else (oracle.port(), "port")
    rp, ci, vv = a.to_host()
    bh = b.cpu().numpy()
    # bounded sample: a strided subset of rows (keeps the R-MAT degree mix)
    stride = 1 if cfg_name in ("cfg1",) else 4
    nrp, nci, nvv = row_sample(rp, ci, vv, stride)
    h = oracle.Csr(len(nrp) - 1, a.cols, nrp, nci, nvv)
    rows = np.arange(h.rows)
    c = np.zeros((h.rows, bh.shape[1]), np.float32)
    t0 = time.perf_counter()
    fl = impl.spmm_local(h, bh, c)
    dt = time.perf_counter() - t0
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": kind,
            "sample": f"spmm_local over every {stride}th row of A ({len(rows)} rows, "
                      f"{h.nnz} nnz, {fl} flop) x full B, 1 thread, {dt:.2f} s"}


def run_spmm_local(args, cfg, dev, rank, world):
    """N=1 (or per-rank replica) local path: one spmm_local per step."""
    import paper_2311_18141_b200 as rd
    import torch

    a, b, c = make_spmm_inputs(cfg, dev)
    m, k, n, nnz = a.rows, a.cols, cfg["n"], a.nnz
    flops = 2 * nnz * n
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        rd.spmm_local(a, b, c)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for i in range(args.steps):
            rd.spmm_local(a, b, c)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
        ms = ev[0].elapsed_time(ev[-1]) / args.steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        # ---- e2e through the public API from pinned host buffers
        rp, ci, vv = (x.cpu().pin_memory() for x in (a.row_ptr, a.col_idx, a.values))
        bh = b.cpu().pin_memory()
        ch = torch.empty_like(c, device="cpu").pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in (rp, ci, vv, bh))
        d2h = ch.numel() * ch.element_size()
        e2e_steps = max(1, min(args.steps, 5))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            a.row_ptr.copy_(rp, non_blocking=True)
            a.col_idx.copy_(ci, non_blocking=True)
            a.values.copy_(vv, non_blocking=True)
            b.copy_(bh, non_blocking=True)
            c.zero_()
            rd.spmm_local(a, b, c)
            ch.copy_(c, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
    hbm, peak_src = peaks()
    launch_ms = statistics.mean(per)
    alg = spmm_bytes(m, k, n, nnz)
    achieved = alg / (launch_ms * 1e-3) / 1e9
    total_flops = flops * world
    out = {
        "metric": METRIC,
        "value": total_flops / (ms * 1e-3) / 1e9,
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (reference generators, seeds A=1 B=2, built on device)",
        "config": {"workload": args.config, "desc": cfg["desc"], "rows": m, "cols": k,
                   "n": n, "nnz": nnz, "flop_per_step": flops,
                   "path": "spmm_local (C-ABI rdmm_spmm_csr_f32), 1x1 grid",
                   "l2": "inputs > L2 (B %.2f GB, C %.2f GB)" % (k * n * 4 / 1e9, m * n * 4 / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": load_traffic(args.config, "spmm_chunks"),
                     "algorithmic_bytes": alg, "peak_source": peak_src,
                     "kernel": "spmm_chunks+spmm_fixup (one spmm_local launch pair)",
                     "launch_ms": launch_ms},
        "e2e": {"value": total_flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": 2 * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_spmm(a, b, args.config)
    return out


# ----------------------------------------------------------- reference arm


def run_reference(args):
    """The reference's own CPU path (oracle/_ref: the unmodified reference
    headers) timed on this host with all its threads: run_multiply
    stationary_c over a ProcGrid as square as possible."""
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
    # grid as square as possible with pr*pc = threads
    pr = int(np.sqrt(threads))
    while threads % pr:
        pr -= 1
    pc = threads // pr
    if cfg["kind"] != "spmm":
        return {"impl": "reference", "unavailable": "reference arm implemented for SpMM configs"}
    a = Pn.rmat(cfg["scale"], cfg["ef"], seed=1) if cfg["gen"] == "rmat" else \
        Pn.uniform_tiles(1 << cfg["scale"], 1 << cfg["scale"], 1, cfg["d"], 1)
    n = cfg["n"]
    b = Pn.random_dense(a.cols, n, 2)
    # bounded sample: every S-th row of A so one step is ~1-3 s on this host
    S = 1 if a.nnz < 5_000_000 else 8
    rp, nci, nvv = row_sample(a.row_ptr, a.col_idx, a.values, S)
    hs = oracle.Csr(len(rp) - 1, a.cols, rp, nci, nvv)
    m, k = hs.rows, hs.cols
    tm, tk, tn = -(-m // pr), -(-k // pc), -(-n // pc)
    ao, keep = oracle.as_orc(hs)
    import ctypes as C

    L = R.lib
    L.ref_spmm_session_create.restype = C.c_void_p
    L.ref_spmm_session_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                          C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.POINTER(oracle.OrcCsr), C.c_void_p, C.c_uint64]
    L.ref_spmm_session_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64,
                                       C.POINTER(oracle.RefReport)]
    L.ref_spmm_session_destroy.argtypes = [C.c_void_p]
    sess = L.ref_spmm_session_create(pr, pc, m, k, n, tm, tk, tn, C.byref(ao), b.ctypes.data, 0)
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
    sec = sum(times) / len(times)
    val = flops / sec / 1e9
    sample = (f"run_multiply stationary_c, {pr}x{pc} ProcGrid, {threads} rank threads, "
              f"every {S}th row of A ({m} rows, {hs.nnz} nnz) x full B (N={n})")
    return {
        "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators, seeds A=1 B=2)",
        "config": {"workload": args.config, "desc": cfg["desc"], "sample": sample},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    if cfg["kind"] != "spmm":
        raise SystemExit("SpGEMM configs are not wired into bench.py yet")
    out = run_spmm_local(args, cfg, dev, rank, world)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
