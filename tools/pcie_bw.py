"""PCIe copy bandwidth probes for the end-to-end pipeline (dev tool): pinned
H2D / D2H, both at once, and strided 2-D H2D of column panels of a row-major
host matrix (the B panels of a column-split e2e run)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=3):
    s = torch.cuda.Stream()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


n = 1 << 28  # 1 GiB fp32
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
out = {}
out["h2d_gbs"] = 4 * n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e6
out["d2h_gbs"] = 4 * n / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e6
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


out["both_ms"] = timed(both)
out["both_gbs_each"] = 4 * n / out["both_ms"] / 1e6
rows = 1 << 22
hm = h[: rows * 64].view(rows, 64)  # 256-byte rows
for cols in (4, 8, 16, 32):
    dm = d[: rows * cols].view(rows, cols)
    ms = timed(lambda: dm.copy_(hm[:, :cols], non_blocking=True))
    out[f"h2d_2d_{cols * 4}B_gbs"] = rows * cols * 4 / ms / 1e6
print(json.dumps(out))
