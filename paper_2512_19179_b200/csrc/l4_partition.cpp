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
#include <queue>
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
      : E_(p.num_instances), mode_(p.stage_cost_mode), kvb_(p.kv_bytes_per_token),
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

  // Exact DP (or chain DP) over E instances: stages and objective (min over s of f_{s,E,J}).
  bool dp(int E, bool chain, std::vector<l4_stage>* out, double* obj) const {
    const int J = J_;
    const size_t SE = (size_t)(E + 1), SJ = (size_t)(J + 1);
    auto at = [&](int s, int e, int j) { return ((size_t)s * SE + (size_t)e) * SJ + (size_t)j; };
    std::vector<double> f(SE * SE * SJ, kInf);
    std::vector<int32_t> arg_e(SE * SE * SJ, -1), arg_j(SE * SE * SJ, -1);
    f[at(0, 0, 0)] = 0.0;
    for (int s = 1; s <= E; ++s) {
      for (int e = s; e <= E; ++e) {
        for (int j = 1; j <= J; ++j) {
          double best = kInf;
          int be = -1, bj = -1;
          const int ep_lo = chain ? e - 1 : s - 1;
          for (int ep = ep_lo; ep <= e - 1; ++ep) {  // Z1: e' <= e-1
            if (ep < s - 1) continue;
            const int m = e - ep;
            for (int jp = 0; jp < j; ++jp) {
              const double prev = f[at(s - 1, ep, jp)];
              if (prev == kInf) continue;
              const double v = (prev + st_[sti(jp, j, m)]) + cut_[jp];
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
    if (best_s < 0) return false;
    out->clear();
    int s = best_s, e = E, j = J;
    while (s > 0) {
      const int ep = arg_e[at(s, e, j)], jp = arg_j[at(s, e, j)];
      out->push_back(l4_stage{jp, j, (int32_t)(e - ep)});  // edge indices for now
      s -= 1;
      e = ep;
      j = jp;
    }
    std::reverse(out->begin(), out->end());
    *obj = best;
    return true;
  }

  // Objective of a plan given as edge-index stages, in the DP's summation order.
  double objective(const std::vector<l4_stage>& plan) const {
    double acc = 0.0;
    for (const l4_stage& x : plan) acc = (acc + stage_cost((int)x.lo, (int)x.hi, x.instances)) + cut_[x.lo];
    return acc;
  }

  double stage_cost(int jp, int j, int m) const { return m <= E_ ? st_[sti(jp, j, m)] : stage(jp, j, m); }

  // P:360-362 two-phase heuristic (readings Z31-Z33): chain DP over min(E, J) single-instance
  // stages, top-up of the remaining instances, then greedy merging of the adjacent pair with the
  // largest positive gain, tracked in a max-heap with lazy invalidation.
  bool two_phase(std::vector<l4_stage>* out, double* obj) const {
    const int E1 = std::min(E_, J_);
    std::vector<l4_stage> plan;
    double unused;
    if (!dp(E1, true, &plan, &unused)) return false;
    for (int extra = E1; extra < E_; ++extra) {  // Z31
      int best_k = -1;
      double best = 0.0;
      for (size_t k = 0; k < plan.size(); ++k) {
        const double g = stage_cost((int)plan[k].lo, (int)plan[k].hi, plan[k].instances) -
                         stage_cost((int)plan[k].lo, (int)plan[k].hi, plan[k].instances + 1);
        if (best_k < 0 || g > best) {
          best = g;
          best_k = (int)k;
        }
      }
      plan[(size_t)best_k].instances += 1;
    }
    // doubly linked list of stages with versions; heap of (gain, -lo) with lazy invalidation (Z32)
    const int n = (int)plan.size();
    std::vector<int> prev(n), next(n), ver(n, 0);
    std::vector<char> alive(n, 1);
    for (int k = 0; k < n; ++k) {
      prev[k] = k - 1;
      next[k] = k + 1 < n ? k + 1 : -1;
    }
    struct Entry {
      double gain;
      int64_t lo;
      int left, right, vl, vr;
      bool operator<(const Entry& o) const {  // max gain first, then leftmost
        if (gain != o.gain) return gain < o.gain;
        return lo > o.lo;
      }
    };
    std::priority_queue<Entry> heap;
    auto gain_of = [&](int a, int b) {
      const l4_stage& A = plan[(size_t)a];
      const l4_stage& B = plan[(size_t)b];
      const double before = (stage_cost((int)A.lo, (int)A.hi, A.instances) +
                             stage_cost((int)B.lo, (int)B.hi, B.instances)) + cut_[B.lo];
      return before - stage_cost((int)A.lo, (int)B.hi, A.instances + B.instances);
    };
    auto push = [&](int a) {
      const int b = next[a];
      if (a < 0 || b < 0) return;
      const double g = gain_of(a, b);
      if (g > 0.0) heap.push(Entry{g, plan[(size_t)a].lo, a, b, ver[a], ver[b]});
    };
    for (int k = 0; k + 1 < n; ++k) push(k);
    while (!heap.empty()) {
      const Entry t = heap.top();
      heap.pop();
      if (!alive[t.left] || !alive[t.right] || next[t.left] != t.right || ver[t.left] != t.vl || ver[t.right] != t.vr)
        continue;  // stale
      plan[(size_t)t.left].hi = plan[(size_t)t.right].hi;
      plan[(size_t)t.left].instances += plan[(size_t)t.right].instances;
      ver[t.left] += 1;
      alive[t.right] = 0;
      next[t.left] = next[t.right];
      if (next[t.right] >= 0) prev[next[t.right]] = t.left;
      if (prev[t.left] >= 0) push(prev[t.left]);
      push(t.left);
    }
    out->clear();
    for (int k = 0; k >= 0 && k < n; k = next[k]) out->push_back(plan[(size_t)k]);
    *obj = objective(*out);  // Z33
    return true;
  }

  l4_status run(int algorithm, l4_stage* stages_out, int32_t* num_stages_out, double* objective_out) {
    // stage cost table [jp][j][m] for m = 1..E
    st_.assign((size_t)(J_ + 1) * (J_ + 1) * (E_ + 1), 0.0);
    for (int jp = 0; jp < J_; ++jp)
      for (int j = jp + 1; j <= J_; ++j)
        for (int m = 1; m <= E_; ++m) st_[sti(jp, j, m)] = stage(jp, j, m);
    std::vector<l4_stage> plan;
    double obj = 0.0;
    bool ok = algorithm == 2 ? two_phase(&plan, &obj) : dp(E_, algorithm == 1, &plan, &obj);
    if (!ok) return l4::fail(L4_ERR_INFEASIBLE, "l4_partition: no feasible plan");
    for (size_t k = 0; k < plan.size(); ++k)
      stages_out[k] = l4_stage{edges_[(size_t)plan[k].lo], edges_[(size_t)plan[k].hi], plan[k].instances};
    *num_stages_out = (int32_t)plan.size();
    *objective_out = obj;
    return L4_OK;
  }

 private:
  int E_, mode_;
  int64_t kvb_;
  double bw_;
  double D_[5];
  std::vector<Req> reqs_, sorted_;
  std::vector<int64_t> edges_;
  std::vector<int64_t> pos_;
  std::vector<std::vector<Stats>> pref_;
  std::vector<double> cut_;
  std::vector<double> st_;
  int64_t n_ = 0;
  int J_ = 0;
  size_t sti(int jp, int j, int m) const {
    return ((size_t)jp * (size_t)(J_ + 1) + (size_t)j) * (size_t)(E_ + 1) + (size_t)m;
  }
};

}  // namespace

extern "C" l4_status l4_partition(const l4_partition_params* p, const int64_t* input_len, const int64_t* output_len,
                                  int64_t n, l4_stage* stages_out, int32_t* num_stages_out, double* objective_out) {
  l4::NvtxRange nvtx("l4_partition");
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
  L4_CHECK_ARG(p->algorithm >= 0 && p->algorithm <= 2, "l4_partition: algorithm must be 0, 1 or 2");
  Partitioner part(*p, std::move(reqs), std::move(edges));
  return part.run(p->algorithm, stages_out, num_stages_out, objective_out);
}

// ===================================================================== §4.3 refinement
// l4_refine_boundary (include/l4.h): P:369-379, readings Z34-Z37.  The argmin over all
// split points of the merged sorted list uses int64 prefix sums, so each candidate's
// Q^{R[:i]} + Q^{R[i:]} is computed from exact integer features in the oracle's order.
namespace {

struct Seq {
  int64_t I, L;
};

double qoe_of(const double* D, int64_t n, int64_t sI, int64_t sI2, int64_t sL) {
  if (n == 0) return 0.0;
  double q = D[0] * 1.0;
  q = q + D[1] * (double)n;
  q = q + D[2] * (double)sI;
  q = q + D[3] * (double)sI2;
  q = q + D[4] * (double)sL;
  return (double)n * q;
}

bool seq_less(const Seq& a, const Seq& b) { return a.L != b.L ? a.L < b.L : a.I < b.I; }

}  // namespace

extern "C" l4_status l4_refine_boundary(const l4_refine_params* p, const int64_t* local_I, const int64_t* local_L,
                                        int64_t n_local, int32_t n_succ, const int64_t* succ_indptr,
                                        const int64_t* succ_I, const int64_t* succ_L, double boundary_in,
                                        double* boundary_out, int64_t* raw_out, int64_t* split_out) {
  L4_CHECK_ARG(p && boundary_out && raw_out && split_out, "l4_refine_boundary: NULL argument");
  L4_CHECK_ARG(n_local >= 0 && n_succ >= 0, "l4_refine_boundary: negative count");
  L4_CHECK_ARG(n_local == 0 || (local_I && local_L), "l4_refine_boundary: local arrays NULL");
  L4_CHECK_ARG(n_succ == 0 || succ_indptr, "l4_refine_boundary: succ_indptr NULL");
  L4_CHECK_ARG(p->ema_alpha >= 0.0 && p->ema_alpha <= 1.0, "l4_refine_boundary: ema_alpha must be in [0, 1]");
  L4_CHECK_ARG(p->hi - p->lo >= 2, "l4_refine_boundary: need hi - lo >= 2");
  L4_CHECK_ARG(std::isfinite(boundary_in), "l4_refine_boundary: boundary must be finite");
  // successor average: canonical subset of the sorted union (Z35)
  std::vector<Seq> uni;
  if (n_succ > 0) {
    L4_CHECK_ARG(succ_indptr[0] == 0, "l4_refine_boundary: succ_indptr[0] must be 0");
    for (int32_t k = 0; k < n_succ; ++k)
      L4_CHECK_ARG(succ_indptr[k + 1] >= succ_indptr[k], "l4_refine_boundary: succ_indptr not monotone");
    const int64_t tot = succ_indptr[n_succ];
    L4_CHECK_ARG(tot == 0 || (succ_I && succ_L), "l4_refine_boundary: successor arrays NULL");
    uni.reserve((size_t)tot);
    for (int64_t i = 0; i < tot; ++i) uni.push_back(Seq{succ_I[i], succ_L[i]});
    std::sort(uni.begin(), uni.end(), seq_less);
  }
  std::vector<Seq> R;
  R.reserve((size_t)n_local + uni.size());
  for (int64_t i = 0; i < n_local; ++i) R.push_back(Seq{local_I[i], local_L[i]});
  for (size_t i = (size_t)(n_succ / 2); n_succ > 0 && i < uni.size(); i += (size_t)n_succ) R.push_back(uni[i]);
  std::sort(R.begin(), R.end(), seq_less);
  const int64_t N = (int64_t)R.size();
  if (N < p->min_traffic || N == 0) {  // P:379 freeze (Z37)
    *boundary_out = boundary_in;
    *raw_out = -1;
    *split_out = -1;
    return L4_OK;
  }
  std::vector<int64_t> cI(N + 1, 0), cI2(N + 1, 0), cL(N + 1, 0);
  for (int64_t i = 0; i < N; ++i) {
    cI[i + 1] = cI[i] + R[i].I;
    cI2[i + 1] = cI2[i] + R[i].I * R[i].I;
    cL[i + 1] = cL[i] + R[i].L;
  }
  double best = std::numeric_limits<double>::infinity();
  int64_t b = 0;
  for (int64_t i = 0; i < N; ++i) {  // Z36: first strict minimum
    const double v = qoe_of(p->qoe_d, i, cI[i], cI2[i], cL[i]) +
                     qoe_of(p->qoe_d, N - i, cI[N] - cI[i], cI2[N] - cI2[i], cL[N] - cL[i]);
    if (v < best) {
      best = v;
      b = i;
    }
  }
  const int64_t raw = R[(size_t)b].L;
  double nb = p->ema_alpha * (double)raw + (1.0 - p->ema_alpha) * boundary_in;
  nb = std::min(std::max(nb, (double)(p->lo + 1)), (double)(p->hi - 1));
  *boundary_out = nb;
  *raw_out = raw;
  *split_out = b;
  return L4_OK;
}

// ===================================================================== §4.1 QoE fit
// l4_qoe_fit (include/l4.h): least squares Q ~ sum_k D_k F_k by Householder QR
// on max-abs-scaled columns (features span ~12 orders of magnitude); rank < selected
// columns -> L4_ERR_INFEASIBLE.
extern "C" l4_status l4_qoe_fit(const double* F, const double* Q, int64_t n, uint32_t column_mask, double* D_out,
                                double* rms_out) {
  L4_CHECK_ARG(F && Q && D_out, "l4_qoe_fit: NULL argument");
  int cols[5], p = 0;
  for (int k = 0; k < 5; ++k)
    if (column_mask & (1u << k)) cols[p++] = k;
  L4_CHECK_ARG(p >= 1, "l4_qoe_fit: empty column mask");
  if (n < p) return l4::fail(L4_ERR_INVALID_ARG, "l4_qoe_fit: too few samples");
  std::vector<double> A((size_t)n * p), b(Q, Q + n), scale(p);
  for (int c = 0; c < p; ++c) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double v = F[i * 5 + cols[c]];
      A[(size_t)c * n + i] = v;  // column-major
      m = std::max(m, std::fabs(v));
    }
    if (!(m > 0.0) || !std::isfinite(m)) return l4::fail(L4_ERR_INFEASIBLE, "l4_qoe_fit: zero or non-finite column");
    scale[c] = m;
    for (int64_t i = 0; i < n; ++i) A[(size_t)c * n + i] /= m;
  }
  for (int k = 0; k < p; ++k) {  // Householder reflections
    double* ak = &A[(size_t)k * n];
    double norm = 0.0;
    for (int64_t i = k; i < n; ++i) norm += ak[i] * ak[i];
    norm = std::sqrt(norm);
    if (norm == 0.0) return l4::fail(L4_ERR_INFEASIBLE, "l4_qoe_fit: rank deficient feature matrix");
    const double alpha = ak[k] > 0 ? -norm : norm;
    std::vector<double> v((size_t)(n - k));
    for (int64_t i = k; i < n; ++i) v[(size_t)(i - k)] = ak[i];
    v[0] -= alpha;
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn > 0.0) {
      for (int c = k; c < p; ++c) {
        double* ac = &A[(size_t)c * n];
        double dot = 0.0;
        for (int64_t i = k; i < n; ++i) dot += v[(size_t)(i - k)] * ac[i];
        const double f = 2.0 * dot / vn;
        for (int64_t i = k; i < n; ++i) ac[i] -= f * v[(size_t)(i - k)];
      }
      double dot = 0.0;
      for (int64_t i = k; i < n; ++i) dot += v[(size_t)(i - k)] * b[(size_t)i];
      const double f = 2.0 * dot / vn;
      for (int64_t i = k; i < n; ++i) b[(size_t)i] -= f * v[(size_t)(i - k)];
    }
  }
  double rmax = 0.0;
  for (int k = 0; k < p; ++k) rmax = std::max(rmax, std::fabs(A[(size_t)k * n + k]));
  for (int k = 0; k < p; ++k)
    if (std::fabs(A[(size_t)k * n + k]) <= 1e-10 * rmax)
      return l4::fail(L4_ERR_INFEASIBLE, "l4_qoe_fit: rank deficient feature matrix");
  double x[5] = {0, 0, 0, 0, 0};
  for (int k = p - 1; k >= 0; --k) {  // back substitution R x = Q^T b
    double s = b[(size_t)k];
    for (int c = k + 1; c < p; ++c) s -= A[(size_t)c * n + k] * x[c];
    x[k] = s / A[(size_t)k * n + k];
  }
  double D[5] = {0, 0, 0, 0, 0};
  for (int c = 0; c < p; ++c) D[cols[c]] = x[c] / scale[c];
  double ss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double pred = 0.0;
    for (int k = 0; k < 5; ++k) pred += D[k] * F[i * 5 + k];
    ss += (Q[i] - pred) * (Q[i] - pred);
  }
  for (int k = 0; k < 5; ++k) D_out[k] = D[k];
  if (rms_out) *rms_out = std::sqrt(ss / (double)n);
  return L4_OK;
}
