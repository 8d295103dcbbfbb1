// l4_partition: the §4.2 length-aware stage partition as host code.
//
//   Eq. (1), P:301-315   Q^B = n * sum_k D_k F_k, F = (1, n, sum I, sum I^2, sum L)
//   P:337-339            f_{s,e,l} = min_{e',l'} f_{s-1,e',l'} + (e-e') Q^{n_{l',l}/(e-e')} + c_{l'}
//   P:341                c_{l'}: transfer delay of the fragments straddling the cut
//   P:342 footnote       set division: sort, start at the n/2-th element, every n-th
//   P:345                answer = min over s of f_{s,E,L}
//   P:357-358            exponential buckets as cut candidates, O(1) prefix-sum range statistics
//
// Design for speed (P:642 reports 0.06 s at E=16, 128K): requests are sorted
// once; every range n_{l',l} is a contiguous slice of the sorted array; the
// statistics (count, sum I, sum I^2, sum L) of any strided subset
// S[o::m] of a slice come from int64 prefix sums with stride m (Z16), so each
// stage cost is O(1) (mode 0) or O(m) (mode 1) and the DP is O(E^3 J^2).
//
// Bit-exactness with oracle/partition.py (Z14): identical IEEE-754 binary64
// operation order, no FMA contraction (built with -ffp-contract=off), exact
// int64 feature sums converted to double once, identical tie-breaking.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <vector>

#include "l4_internal.h"

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct Req {
  int64_t I, Lf, idx;
};

struct Stats {  // exact integer features of a request subset
  int64_t n = 0, sI = 0, sI2 = 0, sL = 0;
};

class Partitioner {
 public:
  Partitioner(const l4_partition_params& p, std::vector<Req> reqs, std::vector<int64_t> edges)
      : E_(p.num_instances), mode_(p.stage_cost_mode), chain_(p.chain != 0), kvb_(p.kv_bytes_per_token),
        bw_(p.migrate_bandwidth_Bps), reqs_(std::move(reqs)), edges_(std::move(edges)) {
    for (int k = 0; k < 5; ++k) D_[k] = p.qoe_d[k];
    // Step 4 (Z6): sort by (Lf, I, input index).
    sorted_ = reqs_;
    std::sort(sorted_.begin(), sorted_.end(), [](const Req& a, const Req& b) {
      if (a.Lf != b.Lf) return a.Lf < b.Lf;
      if (a.I != b.I) return a.I < b.I;
      return a.idx < b.idx;
    });
    n_ = (int64_t)sorted_.size();
    J_ = (int)edges_.size() - 1;
    // slice bounds of every edge: first sorted position with Lf >= e_j (Z3 half-open ranges)
    pos_.resize(edges_.size());
    for (size_t j = 0; j < edges_.size(); ++j) {
      pos_[j] = std::lower_bound(sorted_.begin(), sorted_.end(), edges_[j],
                                 [](const Req& r, int64_t e) { return r.Lf < e; }) -
                sorted_.begin();
    }
    // strided prefix sums P_m[i] = x_i + P_m[i - m] for m = 1..E
    pref_.assign((size_t)E_ + 1, {});
    for (int m = 1; m <= E_; ++m) {
      auto& P = pref_[m];
      P.resize((size_t)n_);
      for (int64_t i = 0; i < n_; ++i) {
        Stats s;
        if (i >= m) s = P[(size_t)(i - m)];
        s.n += 1;
        s.sI += sorted_[i].I;
        s.sI2 += sorted_[i].I * sorted_[i].I;
        s.sL += sorted_[i].Lf;
        P[(size_t)i] = s;
      }
    }
    // cut costs c(j') at every edge (j' = 0 pays nothing)
    cut_.assign((size_t)J_ + 1, 0.0);
    for (int j = 1; j <= J_; ++j) {
      const int64_t cut = edges_[j];
      __int128 tokens = 0;
      for (const Req& r : reqs_)  // Z9: straddles iff I < cut < I + O
        if (r.I < cut && cut < r.Lf) tokens += cut;
      cut_[j] = (double)(tokens * (__int128)kvb_) / bw_;
    }
  }

  // Q^B of the subset S[first::m] of the sorted slice [a, b) (Eq. (1)).
  double qoe_strided(int64_t a, int64_t b, int64_t first_off, int m) const {
    const int64_t first = a + first_off;
    if (first >= b) return 0.0;
    const int64_t last = first + ((b - 1 - first) / m) * m;
    const auto& P = pref_[m];
    Stats s = P[(size_t)last];
    if (first >= m) {
      const Stats& t = P[(size_t)(first - m)];
      s.n -= t.n;
      s.sI -= t.sI;
      s.sI2 -= t.sI2;
      s.sL -= t.sL;
    }
    if (s.n == 0) return 0.0;
    // q = (((D0*F0 + D1*F1) + D2*F2) + D3*F3) + D4*F4, Q^B = n * q
    double q = D_[0] * 1.0;
    q = q + D_[1] * (double)s.n;
    q = q + D_[2] * (double)s.sI;
    q = q + D_[3] * (double)s.sI2;
    q = q + D_[4] * (double)s.sL;
    return (double)s.n * q;
  }

  // (e - e') * Q^{n_{l',l}/(e-e')} for the slice of edges [jp, j) and m instances.
  double stage(int jp, int j, int m) const {
    const int64_t a = pos_[jp], b = pos_[j];
    if (mode_ == 0) return (double)m * qoe_strided(a, b, m / 2, m);  // P:342, Z5
    double acc = qoe_strided(a, b, 0, m);                             // mode 1: sum over k in order
    for (int k = 1; k < m; ++k) acc = acc + qoe_strided(a, b, k, m);
    return acc;
  }

  l4_status run(l4_stage* stages_out, int32_t* num_stages_out, double* objective_out) {
    const int E = E_, J = J_;
    const size_t SE = (size_t)(E + 1), SJ = (size_t)(J + 1);
    auto at = [&](int s, int e, int j) { return ((size_t)s * SE + (size_t)e) * SJ + (size_t)j; };
    std::vector<double> f(SE * SE * SJ, kInf);
    std::vector<int32_t> arg_e(SE * SE * SJ, -1), arg_j(SE * SE * SJ, -1);
    // stage cost table [jp][j][m]
    std::vector<double> st((size_t)SJ * SJ * SE, 0.0);
    auto sti = [&](int jp, int j, int m) { return ((size_t)jp * SJ + (size_t)j) * SE + (size_t)m; };
    for (int jp = 0; jp < J; ++jp)
      for (int j = jp + 1; j <= J; ++j)
        for (int m = 1; m <= E; ++m) st[sti(jp, j, m)] = stage(jp, j, m);

    f[at(0, 0, 0)] = 0.0;
    for (int s = 1; s <= E; ++s) {
      for (int e = s; e <= E; ++e) {
        for (int j = 1; j <= J; ++j) {
          double best = kInf;
          int be = -1, bj = -1;
          const int ep_lo = chain_ ? e - 1 : s - 1;
          for (int ep = ep_lo; ep <= e - 1; ++ep) {  // Z1: e' <= e-1
            if (ep < s - 1) continue;
            const int m = e - ep;
            for (int jp = 0; jp < j; ++jp) {
              const double prev = f[at(s - 1, ep, jp)];
              if (prev == kInf) continue;
              const double v = (prev + st[sti(jp, j, m)]) + cut_[jp];
              if (v < best) {  // Z11: first strict minimum
                best = v;
                be = ep;
                bj = jp;
              }
            }
          }
          f[at(s, e, j)] = best;
          arg_e[at(s, e, j)] = be;
          arg_j[at(s, e, j)] = bj;
        }
      }
    }
    int best_s = -1;
    double best = kInf;
    for (int s = 1; s <= E; ++s) {  // Z12: ties -> fewer stages
      if (f[at(s, E, J)] < best) {
        best = f[at(s, E, J)];
        best_s = s;
      }
    }
    if (best_s < 0) return l4::fail(L4_ERR_INFEASIBLE, "l4_partition: no feasible plan");
    std::vector<l4_stage> out;
    int s = best_s, e = E, j = J;
    while (s > 0) {
      const int ep = arg_e[at(s, e, j)], jp = arg_j[at(s, e, j)];
      out.push_back(l4_stage{edges_[jp], edges_[j], (int32_t)(e - ep)});
      s -= 1;
      e = ep;
      j = jp;
    }
    std::reverse(out.begin(), out.end());
    for (size_t k = 0; k < out.size(); ++k) stages_out[k] = out[k];
    *num_stages_out = (int32_t)out.size();
    *objective_out = best;
    return L4_OK;
  }

 private:
  int E_, mode_;
  bool chain_;
  int64_t kvb_;
  double bw_;
  double D_[5];
  std::vector<Req> reqs_, sorted_;
  std::vector<int64_t> edges_;
  std::vector<int64_t> pos_;
  std::vector<std::vector<Stats>> pref_;
  std::vector<double> cut_;
  int64_t n_ = 0;
  int J_ = 0;
};

}  // namespace

extern "C" l4_status l4_partition(const l4_partition_params* p, const int64_t* input_len, const int64_t* output_len,
                                  int64_t n, l4_stage* stages_out, int32_t* num_stages_out, double* objective_out) {
  L4_CHECK_ARG(p != nullptr, "l4_partition: params is NULL");
  L4_CHECK_ARG(stages_out && num_stages_out && objective_out, "l4_partition: output pointer is NULL");
  L4_CHECK_ARG(n >= 0, "l4_partition: n < 0");
  L4_CHECK_ARG(n == 0 || (input_len && output_len), "l4_partition: input_len/output_len is NULL");
  // Step 1 (validation order as in the oracle): E, bandwidth, lengths, mode, edges.
  L4_CHECK_ARG(p->num_instances >= 1, "l4_partition: num_instances must be >= 1");
  if (p->num_instances > 512) return l4::fail(L4_ERR_UNSUPPORTED, "l4_partition: exact DP supports E <= 512");
  L4_CHECK_ARG(p->migrate_bandwidth_Bps > 0.0, "l4_partition: bandwidth must be > 0");
  L4_CHECK_ARG(p->kv_bytes_per_token >= 0, "l4_partition: kv_bytes_per_token must be >= 0");
  std::vector<Req> reqs((size_t)n);
  int64_t max_lf = 0;
  for (int64_t i = 0; i < n; ++i) {
    L4_CHECK_ARG(input_len[i] >= 1 && output_len[i] >= 1, "l4_partition: input/output lengths must be >= 1");
    L4_CHECK_ARG(input_len[i] <= (int64_t)1 << 40 && output_len[i] <= (int64_t)1 << 40,
                 "l4_partition: length too large");
    reqs[(size_t)i] = Req{input_len[i], input_len[i] + output_len[i], i};  // Step 2 (Z4)
    max_lf = std::max(max_lf, reqs[(size_t)i].Lf);
  }
  L4_CHECK_ARG(p->stage_cost_mode == 0 || p->stage_cost_mode == 1, "l4_partition: stage_cost_mode must be 0 or 1");
  // Step 3 (Z10): edges
  std::vector<int64_t> edges;
  if (p->edges == nullptr) {
    int K = 0;
    while (K < 63 && ((int64_t)1 << K) <= max_lf) ++K;  // K = bit_length(max_lf)
    edges.push_back(0);
    for (int j = 1; j <= K + 1; ++j) edges.push_back((int64_t)1 << (j - 1));
  } else {
    L4_CHECK_ARG(p->num_edges >= 2, "l4_partition: need >= 2 edges");
    edges.assign(p->edges, p->edges + p->num_edges);
    L4_CHECK_ARG(edges[0] == 0, "l4_partition: edges[0] must be 0");
    for (size_t k = 1; k < edges.size(); ++k)
      L4_CHECK_ARG(edges[k] > edges[k - 1], "l4_partition: edges must be strictly increasing");
    if (edges.back() <= max_lf) return l4::fail(L4_ERR_INFEASIBLE, "l4_partition: top edge must exceed max(I+O)");
  }
  if (edges.size() > 4096) return l4::fail(L4_ERR_UNSUPPORTED, "l4_partition: too many edges");
  Partitioner part(*p, std::move(reqs), std::move(edges));
  return part.run(stages_out, num_stages_out, objective_out);
}
