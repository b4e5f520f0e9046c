"""Device CSR utilities on the stationary-C path: column concatenation of the
K A tiles of a C tile (the fused-pass operand, algos.hpp:378-415) and tile
extraction (distmat.hpp:265-282), against numpy restatements."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def rd():
    import paper_2311_18141_b200 as rd

    return rd


def ragged_csr(rng, rows, cols, mean, long_every=0, long_len=0, dtype=np.float32):
    """Sorted, duplicate-free rows: mostly short, some empty, every
    `long_every`-th row long (crosses many 32-entry windows)."""
    lens = rng.poisson(mean, rows).astype(np.int64)
    lens[rng.random(rows) < 0.2] = 0
    if long_every:
        lens[::long_every] = long_len
    lens = np.minimum(lens, cols)
    rp = np.zeros(rows + 1, np.uint32)
    rp[1:] = np.cumsum(lens)
    ci = np.empty(int(rp[-1]), np.uint32)
    for r in range(rows):
        if lens[r]:
            ci[rp[r]:rp[r + 1]] = np.sort(rng.choice(cols, lens[r], replace=False))
    vv = rng.standard_normal(ci.size).astype(dtype)
    return rp, ci, vv


def hstack(tiles, stride):
    rows = len(tiles[0][0]) - 1
    rp = np.zeros(rows + 1, np.uint32)
    ci, vv = [], []
    for r in range(rows):
        for k, (trp, tci, tvv) in enumerate(tiles):
            ci.append(tci[trp[r]:trp[r + 1]] + np.uint32(k * stride))
            vv.append(tvv[trp[r]:trp[r + 1]])
        rp[r + 1] = rp[r] + sum(int(t[0][r + 1] - t[0][r]) for t in tiles)
    return rp, np.concatenate(ci).astype(np.uint32), np.concatenate(vv)


@pytest.mark.parametrize("rows,K,dtype", [(1000, 3, np.float32), (4099, 16, np.float64),
                                          (31, 2, np.float32), (1, 5, np.float32)])
def test_concat_cols_matches_numpy(rd, rows, K, dtype):
    rng = np.random.default_rng(rows * 31 + K)
    stride = 300
    tiles = [ragged_csr(rng, rows, stride if k + 1 < K else 117, 4.0, long_every=97,
                        long_len=90, dtype=dtype) for k in range(K)]
    dev = [rd.DeviceCsr.from_host(rows, stride if k + 1 < K else 117, *t, device=DEV)
           for k, t in enumerate(tiles)]
    out = rd.tile.concat_cols(dev, stride)
    torch.cuda.synchronize()
    rp, ci, vv = out.to_host()
    wrp, wci, wvv = hstack(tiles, stride)
    assert out.cols == stride * (K - 1) + 117
    assert np.array_equal(rp, wrp)
    assert np.array_equal(ci, wci)
    assert np.array_equal(vv, wvv)


def test_concat_cols_with_empty_tiles(rd):
    rng = np.random.default_rng(7)
    rows, stride = 2000, 64
    full = ragged_csr(rng, rows, stride, 6.0)
    empty = (np.zeros(rows + 1, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    tiles = [empty, full, empty]
    dev = [rd.DeviceCsr.from_host(rows, stride, *t, device=DEV) for t in tiles]
    out = rd.tile.concat_cols(dev, stride)
    rp, ci, vv = out.to_host()
    wrp, wci, wvv = hstack(tiles, stride)
    assert np.array_equal(rp, wrp) and np.array_equal(ci, wci) and np.array_equal(vv, wvv)
