"""Time the fused stationary-C building blocks on one GPU (dev tool): the
column concatenation of K A tiles (rdmm_csr_concat_cols) and the segmented
narrow SpMM over the result, for cfg3's A split into K column tiles."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18141_b200 as rd  # noqa: E402
from paper_2311_18141_b200.tile import concat_cols, extract_tile  # noqa: E402

a = rd.rmat(22, 16, seed=1)
for K, n in ((2, 64), (4, 32), (8, 16)):
    tk = a.cols // K
    tiles = [extract_tile(a, 0, a.rows, k * tk, tk) for k in range(K)]
    b = rd.random_dense(a.cols, n, 2)
    c = torch.zeros((a.rows, n), device="cuda")

    res = {"K": K, "n": n}
    for what in ("concat", "spmm", "both"):
        def run():
            if what == "spmm":
                rd.spmm_local(cat, b, c, c_zero=True)
                return
            x = concat_cols(tiles, tk)
            if what == "both":
                rd.spmm_local(x, b, c, c_zero=True)

        cat = concat_cols(tiles, tk)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[what + "_ms"] = e0.elapsed_time(e1) / 10
    print(json.dumps(res), flush=True)
