// rdmm/analytics.hpp -- load-imbalance and virtual-time analytics
// (reference: analytics.hpp, model.hpp:16-31).
//
// Host-side bookkeeping over the flop/traffic records a run produces; nothing
// here touches a device.  The run-derived report (`run_imbalance`) uses the
// per-rank, per-tile-step flop table every variant fills in
// `RankRun::note_multiply` (stage = the k index of the multiplied tiles, as
// in analytics.hpp:93-97), so the north_star's "per-stage and end-to-end
// max/avg" comes from the multiply that actually ran on the GPUs.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "algos.hpp"
#include "model.hpp"  // CostModel

namespace rdmm {

struct ImbalanceReport {  // analytics.hpp:18-25
  std::uint32_t pr = 1, pc = 1;
  std::vector<std::uint64_t> per_tile_nnz;              // pr*pc, row-major
  double nnz_imbalance = 1.0;                           // max/avg
  std::vector<std::vector<std::uint64_t>> stage_flops;  // [rank][stage]
  double per_stage_flop_imbalance = 1.0;
  double end_to_end_flop_imbalance = 1.0;
};

namespace analytics_detail {

// max/avg; an all-zero (or empty) set counts as balanced (analytics.hpp:47-52).
inline double max_over_avg(const std::vector<double>& xs) {
  if (xs.empty()) return 1.0;
  double sum = 0, mx = 0;
  for (double x : xs) {
    sum += x;
    mx = std::max(mx, x);
  }
  return sum == 0 ? 1.0 : mx * double(xs.size()) / sum;
}

// nnz per (row-block, col-block) of an even pr x pc split (analytics.hpp:31-45).
template <typename T>
std::vector<std::uint64_t> block_nnz(const CsrTile<T>& m, std::uint32_t pr, std::uint32_t pc) {
  const std::uint64_t br = (std::uint64_t(m.rows) + pr - 1) / pr;
  const std::uint64_t bc = (std::uint64_t(m.cols) + pc - 1) / pc;
  std::vector<std::uint64_t> n(std::size_t(pr) * pc, 0);
  for (index_t r = 0; r < m.rows; ++r) {
    const std::size_t row_block = br ? r / br : 0;
    for (index_t s = m.row_ptr[r]; s < m.row_ptr[r + 1]; ++s)
      n[row_block * pc + (bc ? m.col_idx[s] / bc : 0)]++;
  }
  return n;
}

}  // namespace analytics_detail

template <typename T>
double nnz_imbalance(const CsrTile<T>& m, std::uint32_t pr, std::uint32_t pc) {
  if (pr < 1 || pc < 1) throw dimension_error("grid dims must be >= 1");
  auto n = analytics_detail::block_nnz(m, pr, pc);
  return analytics_detail::max_over_avg(std::vector<double>(n.begin(), n.end()));
}

// end-to-end = max_r(sum_s f) / avg_r(sum_s f);
// per-stage  = sum_s max_r(f) / sum_s avg_r(f)          (analytics.hpp:66-90)
// Ranks with fewer recorded stages are padded with zeros.
inline void imbalance_from_flops(ImbalanceReport& rep) {
  const auto& f = rep.stage_flops;
  const std::size_t P = f.size();
  if (P == 0) return;
  std::size_t S = 0;
  for (auto& r : f) S = std::max(S, r.size());
  std::vector<double> per_rank(P, 0.0);
  double sum_of_max = 0, sum_of_avg = 0;
  for (std::size_t s = 0; s < S; ++s) {
    double mx = 0, tot = 0;
    for (std::size_t r = 0; r < P; ++r) {
      const double v = s < f[r].size() ? double(f[r][s]) : 0.0;
      per_rank[r] += v;
      tot += v;
      mx = std::max(mx, v);
    }
    sum_of_max += mx;
    sum_of_avg += tot / double(P);
  }
  rep.end_to_end_flop_imbalance = analytics_detail::max_over_avg(per_rank);
  rep.per_stage_flop_imbalance = sum_of_avg == 0 ? 1.0 : sum_of_max / sum_of_avg;
}

// Imbalance of a finished run, from the per-rank per-k-step flops recorded
// by the multiply itself (RankStats::stage_flops).
inline ImbalanceReport run_imbalance(const RunReport& run) {
  ImbalanceReport rep;
  rep.stage_flops.reserve(run.per_rank.size());
  for (const auto& s : run.per_rank) rep.stage_flops.push_back(s.stage_flops);
  imbalance_from_flops(rep);
  return rep;
}

// Predicted stage-resolved imbalance of squaring `a` with a 2D stationary
// algorithm on a grid x grid mesh with `stages` x `stages` tiles mapped
// cyclically (analytics.hpp:92-150).  flops(A_Ik * A_kJ) =
// 2 * sum over t in tile k of (nnz of column t inside row tile I) *
// (nnz of row t inside column tile J), charged to owner(I,J) at step k.
template <typename T>
ImbalanceReport stage_imbalance(const CsrTile<T>& a, std::uint32_t grid,
                                std::uint32_t stages = 0) {
  if (a.rows != a.cols) throw dimension_error("stage_imbalance expects a square matrix");
  if (grid < 1) throw dimension_error("grid dims must be >= 1");
  const std::uint32_t g = grid, K = stages == 0 ? grid : stages;
  if (K < g) throw dimension_error("stages must be >= grid");
  const std::uint64_t n = a.rows, tm = (n + K - 1) / K;
  // colcnt[I][t]: nonzeros of column t in row tile I; rowcnt[J][t]: nonzeros
  // of row t in column tile J (global index t).
  std::vector<std::uint32_t> colcnt(std::size_t(K) * n, 0), rowcnt(std::size_t(K) * n, 0);
  for (index_t r = 0; r < a.rows; ++r)
    for (index_t s = a.row_ptr[r]; s < a.row_ptr[r + 1]; ++s) {
      const index_t c = a.col_idx[s];
      colcnt[std::size_t(r / tm) * n + c]++;
      rowcnt[std::size_t(c / tm) * n + r]++;
    }
  ImbalanceReport rep;
  rep.pr = rep.pc = g;
  rep.per_tile_nnz = analytics_detail::block_nnz(a, g, g);
  rep.nnz_imbalance = analytics_detail::max_over_avg(
      std::vector<double>(rep.per_tile_nnz.begin(), rep.per_tile_nnz.end()));
  rep.stage_flops.assign(std::size_t(g) * g, std::vector<std::uint64_t>(K, 0));
  for (std::uint32_t I = 0; I < K; ++I)
    for (std::uint32_t J = 0; J < K; ++J) {
      auto& owner = rep.stage_flops[std::size_t(I % g) * g + J % g];
      const std::uint32_t* cc = &colcnt[std::size_t(I) * n];
      const std::uint32_t* rc = &rowcnt[std::size_t(J) * n];
      for (std::uint32_t k = 0; k < K; ++k) {
        std::uint64_t dot = 0;
        const std::uint64_t t1 = std::min<std::uint64_t>(n, (k + 1) * tm);
        for (std::uint64_t t = std::uint64_t(k) * tm; t < t1; ++t)
          dot += std::uint64_t(cc[t]) * rc[t];
        owner[k] += 2 * dot;
      }
    }
  imbalance_from_flops(rep);
  return rep;
}

// Per-rank virtual completion time from the run's event log: transfers cost
// bytes/bw + latency (intra bandwidth when src and dst share a node group),
// multiplies cost flops/arith_peak (analytics.hpp:152-174).
inline std::vector<double> virtual_time(const RunReport& report, const CostModel& cost,
                                        rank_t node_group = 6) {
  cost.validate();
  const rank_t grp = node_group == 0 ? 1 : node_group;
  std::vector<double> t(report.events.size(), 0.0);
  for (std::size_t r = 0; r < report.events.size(); ++r)
    for (const Event& e : report.events[r]) {
      if (e.kind == Event::Kind::compute) {
        t[r] += double(e.flops) / cost.arith_peak;
      } else {
        const bool near = e.src / grp == e.dst / grp;
        t[r] += double(e.bytes) / (near ? cost.intra_bw : cost.net_bw) + cost.latency;
      }
    }
  return t;
}

inline double makespan(const std::vector<double>& clocks) {  // analytics.hpp:176-178
  return clocks.empty() ? 0.0 : *std::max_element(clocks.begin(), clocks.end());
}

}  // namespace rdmm
