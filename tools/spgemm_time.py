"""Time spgemm_local (A*A, R-MAT) on one GPU (dev tool)."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18141_b200 as rd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=17)
ap.add_argument("--ef", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
a = rd.rmat(args.scale, args.ef, seed=1)
info = {}
c, m = rd.spgemm_local(a, a, info=info)
torch.cuda.synchronize()
del c
ts = []
for _ in range(args.iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c, m = rd.spgemm_local(a, a)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del c
ms = min(ts) * 1e3
print(json.dumps({"scale": args.scale, "ms": ms, "gflops": m.flops / ms / 1e6, "flops": m.flops,
                  "nnz_out": m.output_nnz, "tiers": info}))
