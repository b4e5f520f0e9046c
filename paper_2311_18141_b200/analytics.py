"""Load-imbalance analytics (reference: analytics.hpp:18-150).

Host-side arithmetic over flop tables; no device work.  `RunReport.imbalance()`
applies `imbalance_from_flops` to the per-rank, per-k-step flops the GPU run
recorded; `stage_imbalance` predicts the same table from A's structure for a
square stationary grid, as the reference does (analytics.hpp:92-150).
"""
from __future__ import annotations

import numpy as np


def _max_over_avg(xs) -> float:
    xs = np.asarray(xs, np.float64)
    s = xs.sum() if xs.size else 0.0
    return 1.0 if s == 0 else float(xs.max() * xs.size / s)


def imbalance_from_flops(stage_flops) -> dict:
    """end-to-end = max_r(sum_s f) / avg_r(sum_s f);
    per-stage = sum_s max_r(f) / sum_s avg_r(f)   (analytics.hpp:66-90).

    `stage_flops` is [ranks, stages]; ragged lists are zero-padded."""
    rows = [np.asarray(r, np.float64) for r in stage_flops]
    if not rows:
        return {"per_stage_flop_imbalance": 1.0, "end_to_end_flop_imbalance": 1.0}
    S = max((r.size for r in rows), default=0)
    f = np.zeros((len(rows), S))
    for i, r in enumerate(rows):
        f[i, :r.size] = r
    avg = f.mean(axis=0).sum() if S else 0.0
    return {"per_stage_flop_imbalance": 1.0 if avg == 0 else float(f.max(axis=0).sum() / avg),
            "end_to_end_flop_imbalance": _max_over_avg(f.sum(axis=1))}


def imbalance_from_times(stage_ms) -> dict:
    """The same two ratios over a [ranks, stages] table of device time (ms)
    per rank per k tile step (RankStats::stage_ms, RunOptions::time_stages):
    the measured counterpart of imbalance_from_flops."""
    r = imbalance_from_flops(stage_ms)
    return {"per_stage_time_imbalance": r["per_stage_flop_imbalance"],
            "end_to_end_time_imbalance": r["end_to_end_flop_imbalance"]}


def nnz_imbalance(row_ptr, col_idx, rows, cols, pr, pc) -> float:
    """max/avg nnz over an even pr x pc block split (analytics.hpp:58-64)."""
    return _max_over_avg(block_nnz(row_ptr, col_idx, rows, cols, pr, pc))


def block_nnz(row_ptr, col_idx, rows, cols, pr, pc) -> np.ndarray:
    if pr < 1 or pc < 1:
        raise ValueError("grid dims must be >= 1")
    rp = np.asarray(row_ptr, np.int64)
    ci = np.asarray(col_idx, np.int64)
    br, bc = -(-rows // pr), -(-cols // pc)
    r = np.repeat(np.arange(rows, dtype=np.int64), np.diff(rp))
    return np.bincount((r // max(br, 1)) * pc + ci // max(bc, 1),
                       minlength=pr * pc).astype(np.int64)


def stage_imbalance(row_ptr, col_idx, n, grid, stages=0) -> dict:
    """Predicted [rank, stage] flops of A*A on a grid x grid mesh with
    stages x stages cyclic tiles (analytics.hpp:92-150): the owner of C(I,J)
    is charged 2 * sum_{t in tile k} colnnz(I, t) * rownnz(J, t) at step k."""
    g = int(grid)
    K = g if stages == 0 else int(stages)
    if g < 1:
        raise ValueError("grid dims must be >= 1")
    if K < g:
        raise ValueError("stages must be >= grid")
    rp = np.asarray(row_ptr, np.int64)
    ci = np.asarray(col_idx, np.int64)
    tm = -(-n // K)
    r = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    colcnt = np.bincount((r // tm) * n + ci, minlength=K * n).reshape(K, n).astype(np.float64)
    rowcnt = np.bincount((ci // tm) * n + r, minlength=K * n).reshape(K, n).astype(np.float64)
    flops = np.zeros((g * g, K), np.int64)
    owner = (np.arange(K)[:, None] % g) * g + (np.arange(K)[None, :] % g)  # [I, J]
    for k in range(K):
        seg = slice(k * tm, min(n, (k + 1) * tm))
        prod = 2 * np.rint(colcnt[:, seg] @ rowcnt[:, seg].T).astype(np.int64)  # [I, J]
        np.add.at(flops[:, k], owner.ravel(), prod.ravel())
    out = imbalance_from_flops(flops)
    tiles = block_nnz(rp, ci, n, n, g, g)
    out.update(stage_flops=flops, per_tile_nnz=tiles, nnz_imbalance=_max_over_avg(tiles))
    return out
