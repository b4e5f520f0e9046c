"""Small invocations of every SpMM / SpGEMM kernel family for
compute-sanitizer (racecheck / synccheck are far too slow for the test
suite): narrow cp.async slots (N=16, 32), register slots (N=64), nnz stream
(N=128), rows (N=256), atomic accumulation, device-resident nnz, fused
concat, and SpGEMM hash / dense tiers on an R-MAT s12 A*A."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_18141_b200 as rd  # noqa: E402
from paper_2311_18141_b200 import _lib as L  # noqa: E402
from paper_2311_18141_b200.tile import concat_cols, extract_tile  # noqa: E402

a = rd.rmat(12, 8, seed=1)
for n in (16, 32, 64, 128, 256):
    b = rd.random_dense(a.cols, n, 2)
    c = torch.zeros((a.rows, n), device="cuda")
    rd.spmm_local(a, b, c, c_zero=True)
    rd.spmm_local(a, b, c)
torch.cuda.synchronize()
# fused concat of 4 column tiles + SpMM over it
tk = a.cols // 4
tiles = [extract_tile(a, 0, a.rows, k * tk, tk) for k in range(4)]
cat = concat_cols(tiles, tk)
b = rd.random_dense(a.cols, 32, 2)
c = torch.zeros((a.rows, 32), device="cuda")
rd.spmm_local(cat, b, c, c_zero=True)
# distributed: atomic accumulation (1x4) and the deterministic fused pass
import numpy as np  # noqa: E402
import paper_2311_18141_b200.dist as dm  # noqa: E402

for det in (False, True):
    with dm.Fabric(nranks=4, heap_bytes=64 << 20, devices=[0, 0, 0, 0]) as f:
        g = dm.ProcGrid(1, 4)
        A = dm.DistSparse(f, a.rows, a.cols, a.rows, tk, g, 0)
        B = dm.DistDense(f, a.cols, 32, tk, 8, g, 1)
        Cm = dm.DistDense(f, a.rows, 32, a.rows, 8, g, 2)
        A.init_from_device(a)
        B.init_from_device(b)
        Cm.init()
        dm.run_multiply(f, A, B, Cm, deterministic=det)
        got = Cm.to_global()
        assert np.array_equal(got, c.cpu().numpy())
s = rd.rmat(12, 8, seed=1)
cs, _ = rd.spgemm_local(s, s)
torch.cuda.synchronize()
print("sanitize cases ok", L.loaded_path())
