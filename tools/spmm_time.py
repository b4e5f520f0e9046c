"""Time spmm_local on a BASELINE-shaped input (dev tool).  Kernel-family and
chunking switches come from the environment (RDMM_SPMM_KERNEL=rows|stream|vec,
RDMM_SPMM_CPW); the printed `bits` (sum of the fp32 bit patterns of C) lets
runs with different switches be compared for bitwise-identical results."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18141_b200 as rd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--n", type=int, nargs="+", default=[128])
ap.add_argument("--er", action="store_true")
ap.add_argument("--czero", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--tag", default="")
ap.add_argument("--coltiles", type=int, default=0,
                help="time each of K column tiles of A separately (the 1xK passes)")
ap.add_argument("--atomic", type=int, default=0)
args = ap.parse_args()
if args.er:
    a = rd.uniform_tiles(1 << args.scale, 1 << args.scale, 1, 16.0 / (1 << args.scale), 1)
else:
    a = rd.rmat(args.scale, args.ef, seed=1)
if args.coltiles:
    from paper_2311_18141_b200 import _lib as L
    from paper_2311_18141_b200.tile import extract_tile
    import ctypes as C
    K = args.coltiles
    tk = a.cols // K
    for n in args.n:
        b = rd.random_dense(a.cols, n, 2)
        c = torch.zeros((a.rows, n), device="cuda")
        for k in range(K):
            t = extract_tile(a, 0, a.rows, k * tk, tk)
            bk = b[k * tk:(k + 1) * tk]
            flags = (L.SPMM_C_ZERO if args.czero else 0) | (4 if args.atomic else 0)
            fl = C.c_uint64(0)
            def run():
                L.check(L.rdmm_spmm_csr_ex(4, t.rows, t.cols, n, t.nnz, t.row_ptr.data_ptr(),
                                           t.col_idx.data_ptr(), t.values.data_ptr(),
                                           bk.data_ptr(), n, c.data_ptr(), n, flags, None, 0,
                                           None, C.byref(fl)), "spmm")
            for _ in range(2):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.iters):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.iters
            nonempty = int((torch.diff(t.row_ptr.long()) > 0).sum())
            print(json.dumps({"K": K, "k": k, "n": n, "nnz": t.nnz, "nonempty_rows": nonempty,
                              "ms": ms, "atomic": args.atomic, "czero": args.czero}), flush=True)
    sys.exit(0)
for n in args.n:
    b = rd.random_dense(a.cols, n, 2)
    c = torch.zeros((a.rows, n), device="cuda")
    rd.spmm_local(a, b, c, c_zero=True)
    torch.cuda.synchronize()
    bits = int(c.view(torch.int32).long().sum())
    for _ in range(3):
        rd.spmm_local(a, b, c, c_zero=bool(args.czero))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        rd.spmm_local(a, b, c, c_zero=bool(args.czero))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    fl = 2 * a.nnz * n
    print(json.dumps({"tag": args.tag, "ms": ms, "gflops": fl / ms / 1e6, "bits": bits,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("RDMM_")},
                      "czero": args.czero, "scale": args.scale, "n": n, "er": args.er}),
          flush=True)
    del b, c
