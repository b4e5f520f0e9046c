"""Load-imbalance analytics (analytics.hpp:58-150) against goldens made by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""
import os
import subprocess

import numpy as np
import pytest

from paper_2311_18141_b200 import analytics as an

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("grid,stages", [(2, 0), (2, 4), (3, 6)])
def test_stage_imbalance_matches_reference(golden, grid, stages):
    rp, ci = golden["rmat10_rp"], golden["rmat10_ci"]
    r = an.stage_imbalance(rp, ci, len(rp) - 1, grid, stages)
    key = f"stage_g{grid}s{stages}"
    assert np.array_equal(r["stage_flops"], golden[key + "_flops"])
    want = golden[key + "_imb"]
    got = [r["per_stage_flop_imbalance"], r["end_to_end_flop_imbalance"], r["nnz_imbalance"]]
    np.testing.assert_allclose(got, want, rtol=1e-12)


def test_stage_flops_sum_to_spgemm_flops(golden, orc):
    # every (I, J, k) product is charged once: the table sums to 2 * madds(A*A)
    import oracle

    rp, ci = golden["rmat10_rp"], golden["rmat10_ci"]
    a = oracle.Csr(len(rp) - 1, len(rp) - 1, rp, ci, golden["rmat10_v"])
    r = an.stage_imbalance(rp, ci, len(rp) - 1, 2, 4)
    assert int(r["stage_flops"].sum()) == orc.spgemm_flops(a, a)


def test_imbalance_from_flops_matches_reference(golden):
    r = an.imbalance_from_flops(golden["imb_table"])
    np.testing.assert_allclose([r["per_stage_flop_imbalance"], r["end_to_end_flop_imbalance"]],
                               golden["imb_table_out"], rtol=1e-12)


def test_imbalance_edge_cases():
    assert an.imbalance_from_flops([]) == {"per_stage_flop_imbalance": 1.0,
                                           "end_to_end_flop_imbalance": 1.0}
    assert an.imbalance_from_flops(np.zeros((3, 4)))["per_stage_flop_imbalance"] == 1.0
    # ragged rows are zero-padded: rank 1 did nothing in stage 1
    r = an.imbalance_from_flops([[4, 4], [4]])
    assert r["per_stage_flop_imbalance"] == pytest.approx(8 / 6)
    assert r["end_to_end_flop_imbalance"] == pytest.approx(8 / 6)
    with pytest.raises(ValueError):
        an.stage_imbalance([0], [], 0, 2, 1)
    assert an.nnz_imbalance([0, 1, 2], [0, 1], 2, 2, 2, 2) == pytest.approx(2.0)


def test_cpp_analytics_header_compiles(tmp_path, golden):
    # the C++ drop-in header (include/rdmm/analytics.hpp) on a host tile
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "rdmm/analytics.hpp"
#include "rdmm/model.hpp"
#include <cstdio>
int main() {
  rdmm::CsrTile<float> a(4, 4);
  a.row_ptr = {0, 2, 3, 3, 4}; a.col_idx = {0, 3, 1, 2}; a.values = {1, 1, 1, 1};
  auto r = rdmm::stage_imbalance(a, 2);
  rdmm::RunReport run; run.per_rank.resize(2);
  run.per_rank[0].stage_flops = {4, 4}; run.per_rank[1].stage_flops = {4};
  auto q = rdmm::run_imbalance(run);
  rdmm::ProblemShape s; s.m = 4194304; s.k = 4194304; s.n = 128; s.p = 4;
  s.d = 64827941.0 / (4194304.0 * 4194304.0);
  auto rf = rdmm::roofline(s, rdmm::CostModel{}, rdmm::MultiplyKind::spmm);
  std::printf("%.6f %.6f %.6f %.9e\n", r.nnz_imbalance, q.per_stage_flop_imbalance,
              q.end_to_end_flop_imbalance, rf.internode_bound);
}
''')
    exe = tmp_path / "t"
    lib = os.path.join(ROOT, "paper_2311_18141_b200", "lib")
    if not os.path.exists(os.path.join(lib, "librdmm_cuda.so")):
        pytest.skip("librdmm_cuda.so not built")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src),
                    "-o", str(exe), "-L", lib, "-lrdmm_cuda", f"-Wl,-rpath,{lib}", "-pthread"],
                   check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    a_blocks = an.block_nnz([0, 2, 3, 3, 4], [0, 3, 1, 2], 4, 4, 2, 2)
    assert float(out[0]) == pytest.approx(a_blocks.max() / a_blocks.mean(), rel=1e-6)
    assert float(out[1]) == pytest.approx(8 / 6, rel=1e-6)
    assert float(out[2]) == pytest.approx(8 / 6, rel=1e-6)
    assert float(out[3]) == pytest.approx(golden["model_out"][1][3], rel=1e-8)


def test_model_roofline_matches_reference(golden):
    """model.hpp:83-160 (reference) vs paper_2311_18141_b200.model at the
    BASELINE configs' shapes with B200 costs (goldens from the reference)."""
    import sys

    from paper_2311_18141_b200 import model as md

    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import MODEL_CASES, MODEL_COST

    for case, want in zip(MODEL_CASES, golden["model_out"]):
        m, k, n, p, d, w, sg, fl, on = case
        s = md.ProblemShape(m, k, n, p, d, w)
        c = md.CostModel(*MODEL_COST, w=w)
        r = md.roofline(s, c, "spgemm" if sg else "spmm", fl, on)
        got = [r["local_ai"], r["internode_ai"], r["local_peak"], r["internode_bound"],
               0.0 if r["bound_kind"] == "network_bound" else 1.0,
               md.comm_elems_per_iter(s) if s.p_square() else -1.0,
               md.comm_bytes_per_iter(s, 4.0)]
        np.testing.assert_allclose(got, want, rtol=1e-12)
    with pytest.raises(ValueError):
        md.comm_elems_per_iter(md.ProblemShape(8, 8, 8, 2, 0.5))
    with pytest.raises(ValueError):
        md.roofline(md.ProblemShape(8, 8, 8, 4, 0.5), kind="spgemm")
    with pytest.raises(ValueError):
        md.ProblemShape(8, 8, 8, 4, 1.5).validate()
