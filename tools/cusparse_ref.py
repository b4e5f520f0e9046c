"""Library anchor (BASELINE.md §4 "optionally"): cuSPARSE SpMM / SpGEMM via
torch.sparse on the same inputs as the bench configurations, timed with CUDA
events on one B200.  A reference point for the hand-written kernels, never
on the product path."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18141_b200 as rd  # noqa: E402


def csr(a):
    return torch.sparse_csr_tensor(a.row_ptr.long(), a.col_idx.long(), a.values,
                                   size=(a.rows, a.cols))


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters, out


ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
args = ap.parse_args()
res = {"config": args.config, "library": "cuSPARSE via torch.sparse " + torch.__version__}
if args.config in ("cfg3", "cfg1", "cfg5"):
    if args.config == "cfg5":
        a = rd.uniform_tiles(1 << 22, 1 << 22, 1, 2.0 ** -18, 1)
        n = 256
    else:
        s, ef = (22, 16) if args.config == "cfg3" else (16, 8)
        a = rd.rmat(s, ef, seed=1)
        n = 128
    b = rd.random_dense(a.cols, n, 2)
    A = csr(a)
    ms, c = timed(lambda: torch.sparse.mm(A, b), 10)
    mine = torch.zeros_like(c)
    rd.spmm_local(a, b, mine, c_zero=True)
    res.update(op="SpMM", n=n, ms=ms, gflops=2 * a.nnz * n / ms / 1e6,
               equal_to_rdmm=bool(torch.equal(c, mine)))
else:
    s = 17 if args.config == "cfg2" else 20
    a = rd.rmat(s, 8, seed=1)
    A = csr(a)
    ms, c = timed(lambda: torch.sparse.mm(A, A), 3)
    mine, meter = rd.spgemm_local(a, a)
    res.update(op="SpGEMM", ms=ms, gflops=meter.flops / ms / 1e6, nnz_out=int(c._nnz()),
               same_nnz_as_rdmm=int(c._nnz()) == mine.nnz)
print(json.dumps(res))
