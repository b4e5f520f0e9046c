"""Communication-volume and roofline model of the paper (reference:
model.hpp:16-160, PAPER §IV), with B200 cost parameters.

Mirrors include/rdmm/model.hpp: same formulas and argument meaning as the
reference; the CostModel defaults are one B200 box (NVLink 5 peer bandwidth,
measured HBM3e copy bandwidth, fp32 CUDA-core FMA peak) instead of a Summit
node.  bench.py reports `roofline(...)` beside the measured throughput.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class CostModel:  # model.hpp:16-31
    net_bw: float = 900e9        # bytes/s per GPU to any peer (NVLink 5)
    intra_bw: float = 900e9      # bytes/s inside the box
    mem_bw: float = 6446.3e9     # bytes/s HBM3e (MEASURED_PEAKS.json copy bandwidth)
    arith_peak: float = 74.4e12  # flops/s fp32 FMA, 148 SMs x 128 lanes x 2 x 1.965 GHz
    w: float = 4
    latency: float = 0.0

    def validate(self):
        if not (self.net_bw > 0 and self.intra_bw > 0 and self.mem_bw > 0
                and self.arith_peak > 0) or self.latency < 0:
            raise ValueError("cost model parameters must be positive")
        if self.w not in (4, 8):
            raise ValueError("word size must be 4 or 8 bytes")


@dataclass
class ProblemShape:  # model.hpp:33-51
    m: float
    k: float
    n: float
    p: float = 1
    d: float = 1
    w: float = 4

    def validate(self):
        if not (self.m > 0 and self.k > 0 and self.n > 0 and self.p > 0):
            raise ValueError("dims and rank count must be positive")
        if not (0 < self.d <= 1):
            raise ValueError("density must be in (0,1]")

    def p_square(self) -> bool:
        r = round(math.sqrt(self.p))
        return r * r == self.p


def _a_elems(s):
    return s.d * s.m * s.k / s.p


def _iter_elems(s):
    return s.k * s.n / s.p + 2.0 * _a_elems(s) + s.m / math.sqrt(s.p) + 1.0


def _iter_flops(s):
    return 2.0 * _a_elems(s) * (s.n / math.sqrt(s.p))


def comm_elems_per_iter(s: ProblemShape) -> float:  # model.hpp:83-90
    s.validate()
    if not s.p_square():
        raise ValueError("comm_elems_per_iter: p must be a perfect square")
    return _iter_elems(s)


def comm_bytes_per_iter(s: ProblemShape, idx_bytes: float) -> float:  # model.hpp:92-102
    s.validate()
    a = _a_elems(s)
    return (s.k * s.n / s.p + a) * s.w + (a + s.m / math.sqrt(s.p) + 1.0) * idx_bytes


def spmm_internode_ai(s: ProblemShape) -> float:
    s.validate()
    return _iter_flops(s) / (s.w * _iter_elems(s))


def spmm_local_ai(s: ProblemShape) -> float:
    s.validate()
    return _iter_flops(s) / (s.w * (_iter_elems(s) + s.m * s.n / s.p))


def spgemm_local_ai(cf: float, b: float) -> float:  # model.hpp:118-124
    if not (cf > 0 and b > 0):
        raise ValueError("spgemm_local_ai: cf and b must be positive")
    return cf / ((3.0 + 2.0 * cf) * b)


def spgemm_internode_ai(flops: float, s: ProblemShape) -> float:  # model.hpp:126-135
    s.validate()
    if not flops > 0:
        raise ValueError("spgemm_internode_ai: flops must be positive")
    a = 2.0 * s.d * s.m * s.k / s.p + s.m / math.sqrt(s.p) + 1.0
    b = 2.0 * s.d * s.k * s.n / s.p + s.k / math.sqrt(s.p) + 1.0
    return flops / (s.w * (a + b))


def roofline(s: ProblemShape, cost: CostModel | None = None, kind: str = "spmm",
             flops: int = 0, output_nnz: int = 0) -> dict:
    """local peak = min(arith, local AI x mem bw); inter-node bound =
    min(local peak, inter-node AI x net bw) (model.hpp:139-160)."""
    cost = cost or CostModel(w=s.w)
    s.validate()
    cost.validate()
    if kind == "spmm":
        lai, iai = spmm_local_ai(s), spmm_internode_ai(s)
    elif kind == "spgemm":
        if not (flops and output_nnz):
            raise ValueError("roofline: SpGEMM requires measured flops/output nnz")
        lai = spgemm_local_ai(flops / output_nnz, 2.0 * s.w)
        iai = spgemm_internode_ai(flops / s.p, s)
    else:
        raise ValueError(f"unknown multiply kind {kind!r}")
    local_peak = min(cost.arith_peak, lai * cost.mem_bw)
    net = iai * cost.net_bw
    return {"local_ai": lai, "internode_ai": iai, "local_peak": local_peak,
            "internode_bound": min(local_peak, net),
            "bound_kind": "network_bound" if net < local_peak else "compute_bound"}
