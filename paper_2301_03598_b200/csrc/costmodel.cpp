// costmodel.cpp -- grid-size selection for the device Stream-K schedule.
//
// Restates the reference's Appendix-A model (core/src/costmodel.cpp:13-48,
// PAPER.md:966-1021) for a persistent grid of p CTAs on B200:
//
//   time(g) = e + W(g) * ( a + b*[peers > 1] + c*ipc + d*(peers - 1) + s*segs )
//   ipc      = ceil(total_iters / g)                        costmodel.cpp:13-16
//   peers    = ceil(iters_per_tile / ipc)                   costmodel.cpp:18-20
//   W(g)     = ceil(g / p)                                  waves of the persistent grid
//   segs     = tile segments of one unit: ipc / ipt if ipc % ipt == 0, else ceil(ipc / ipt) + 1
//
// For g <= p this is the reference's predict_time plus two B200 terms: a
// launch constant e and a per-segment epilogue cost s (each segment drains a
// 128-row x 256-col fp32 accumulator, 128 KB per CTA, which is HBM-write-bound
// when k is small).  g = t is data-parallel (W waves of one segment each).
// select_grid_size searches g in {1..p} U {t} like costmodel.cpp:30-48 (ties
// toward larger g) and keeps data-parallel unless a Stream-K grid is predicted
// to be faster by more than `margin`.  calibrate fits {e,a,b,c,d,s} by
// non-negative least squares on relative error (costmodel.cpp:142-225 fits 4
// coefficients on absolute error).
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/skb200.h"

namespace {

constexpr int kF = 6;

int64_t cdiv(int64_t x, int64_t y) { return (x + y - 1) / y; }

void features(const sk_tile_grid_t& g, int64_t gs, int64_t p, double f[kF], double coop_peers = 0.0) {
  const int64_t ipc = cdiv(g.total_iters, gs);
  const int64_t peers = cdiv(g.iters_per_tile, ipc);
  // The kernel's cooperative fixup (one unit per CTA, tiles of >= 8
  // contributors, skb200_api.cu) spreads the fold over all contributors.
  // Its cost in serial-peer-fold units: a publish plus, per folding
  // contributor, ncontrib 32-column chunks (1/8 of a slab each).
  const bool coop = coop_peers > 0.0 && gs <= p && ipc * 4 < g.iters_per_tile && peers + 1 >= 8;
  const double fold_peers =
      coop ? std::min(coop_peers + static_cast<double>(peers + 1) / 8.0, static_cast<double>(peers - 1))
           : static_cast<double>(peers - 1);
  const int64_t segs = ipc % g.iters_per_tile == 0 ? ipc / g.iters_per_tile
                                                   : cdiv(ipc, g.iters_per_tile) + 1;
  const double w = static_cast<double>(cdiv(gs, p));
  f[0] = 1.0;
  f[1] = w;
  f[2] = w * (peers > 1 ? 1.0 : 0.0);
  f[3] = w * static_cast<double>(ipc);
  f[4] = w * fold_peers;
  f[5] = w * static_cast<double>(segs);
}

double dot(const sk_cost_params& c, const double f[kF]) {
  return c.e * f[0] + c.a * f[1] + c.b * f[2] + c.c * f[3] + c.d * f[4] + c.s * f[5];
}

// Lawson-Hanson NNLS for a small dense problem (n x k, k <= 8).
bool nnls(const std::vector<double>& A, const std::vector<double>& b, int n, int k,
          std::vector<double>& x) {
  x.assign(k, 0.0);
  std::vector<bool> passive(k, false);
  std::vector<double> w(k), z(k);
  auto gradient = [&] {
    std::fill(w.begin(), w.end(), 0.0);
    for (int i = 0; i < n; ++i) {
      double r = b[i];
      for (int j = 0; j < k; ++j) r -= A[i * k + j] * x[j];
      for (int j = 0; j < k; ++j) w[j] += A[i * k + j] * r;
    }
  };
  auto solve_passive = [&]() -> bool {  // least squares on the passive set (normal equations)
    std::vector<int> idx;
    for (int j = 0; j < k; ++j)
      if (passive[j]) idx.push_back(j);
    const int m = static_cast<int>(idx.size());
    std::fill(z.begin(), z.end(), 0.0);
    if (m == 0) return true;
    std::vector<double> M(m * m, 0.0), v(m, 0.0);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < m; ++a) {
        v[a] += A[i * k + idx[a]] * b[i];
        for (int c = 0; c < m; ++c) M[a * m + c] += A[i * k + idx[a]] * A[i * k + idx[c]];
      }
    for (int col = 0; col < m; ++col) {
      int piv = col;
      for (int r = col + 1; r < m; ++r)
        if (std::fabs(M[r * m + col]) > std::fabs(M[piv * m + col])) piv = r;
      if (std::fabs(M[piv * m + col]) < 1e-300) return false;
      if (piv != col) {
        for (int c = 0; c < m; ++c) std::swap(M[col * m + c], M[piv * m + c]);
        std::swap(v[col], v[piv]);
      }
      for (int r = col + 1; r < m; ++r) {
        const double f = M[r * m + col] / M[col * m + col];
        for (int c = col; c < m; ++c) M[r * m + c] -= f * M[col * m + c];
        v[r] -= f * v[col];
      }
    }
    for (int r = m - 1; r >= 0; --r) {
      double sum = v[r];
      for (int c = r + 1; c < m; ++c) sum -= M[r * m + c] * z[idx[c]];
      z[idx[r]] = sum / M[r * m + r];
    }
    return true;
  };
  for (int outer = 0; outer < 64; ++outer) {
    gradient();
    int best = -1;
    double bw = 1e-12;
    for (int j = 0; j < k; ++j)
      if (!passive[j] && w[j] > bw) {
        bw = w[j];
        best = j;
      }
    if (best < 0) break;
    passive[best] = true;
    for (int inner = 0; inner < 64; ++inner) {
      if (!solve_passive()) return false;
      bool feasible = true;
      for (int j = 0; j < k; ++j)
        if (passive[j] && z[j] <= 0) feasible = false;
      if (feasible) {
        x = z;
        break;
      }
      double alpha = 1.0;
      for (int j = 0; j < k; ++j)
        if (passive[j] && z[j] <= 0) alpha = std::min(alpha, x[j] / (x[j] - z[j]));
      for (int j = 0; j < k; ++j) {
        x[j] += alpha * (z[j] - x[j]);
        if (passive[j] && x[j] <= 1e-15) {
          passive[j] = false;
          x[j] = 0.0;
        }
      }
    }
  }
  return true;
}

bool valid_grid(const sk_tile_grid_t* g) {
  return g && g->total_tiles >= 1 && g->iters_per_tile >= 1 &&
         g->total_iters == g->total_tiles * g->iters_per_tile;
}

}  // namespace

extern "C" {

sk_status sk_predict_time(const sk_cost_params* c, const sk_tile_grid_t* g, int64_t gs, int64_t p,
                          double* out) {
  if (!c || !valid_grid(g) || gs < 1 || p < 1 || !out) return SK_EINVAL;
  double f[kF];
  features(*g, gs, p, f, c->coop_peers);
  *out = dot(*c, f);
  return SK_OK;
}

sk_status sk_select_grid_size(const sk_cost_params* c, const sk_tile_grid_t* g, int64_t p,
                              int64_t* out) {
  if (!c || !valid_grid(g) || p < 1 || !out) return SK_EINVAL;
  const int64_t dp = std::min(g->total_tiles, g->total_iters);  // == t
  double t_dp = 0.0;
  sk_predict_time(c, g, dp, p, &t_dp);
  int64_t best = dp;
  double bt = t_dp;
  const int64_t cap = std::min(p, g->total_iters);
  for (int64_t x = 1; x <= cap; ++x) {
    double t;
    sk_predict_time(c, g, x, p, &t);
    if (t <= bt) {  // ties break toward larger g (costmodel.cpp:41-45)
      bt = t;
      best = x;
    }
  }
  // Keep the data-parallel schedule unless Stream-K is predicted to win by > margin.
  if (best != dp && !(bt < (1.0 - c->margin) * t_dp)) best = dp;
  *out = best;
  return SK_OK;
}

// Predicted time of a whole schedule: data_parallel, stream_k(g) or the
// two-tile Stream-K + data-parallel hybrid (decompose.cpp:81-121), whose DP
// waves run first and whose SK region is one balanced wave of p units.
sk_status sk_predict_schedule(const sk_cost_params* c, const sk_tile_grid_t* g, int32_t strategy,
                              int64_t param, int64_t p, double* out) {
  if (!c || !valid_grid(g) || p < 1 || !out) return SK_EINVAL;
  switch (strategy) {
    case SK_DATA_PARALLEL:
      return sk_predict_time(c, g, g->total_tiles, p, out);
    case SK_STREAM_K:
      return sk_predict_time(c, g, param, p, out);
    case SK_TWO_TILE_SK_DP: {
      if (param < 1) return SK_EINVAL;
      const int64_t t = g->total_tiles, w = t / param, r = t % param;
      if (r == 0) return sk_predict_time(c, g, t, p, out);
      const int64_t d = w >= 2 ? (w - 1) * param : 0;
      sk_tile_grid_t sk_region = *g;  // the trailing t - d tiles as one Stream-K problem
      sk_region.total_tiles = t - d;
      sk_region.total_iters = (t - d) * g->iters_per_tile;
      double f[kF];
      features(sk_region, param, p, f, c->coop_peers);
      double t_sk = dot(*c, f);
      const double dp_waves = static_cast<double>(cdiv(d, p));
      *out = t_sk + dp_waves * (c->a + c->c * static_cast<double>(g->iters_per_tile) + c->s);
      return SK_OK;
    }
    default:
      return SK_EUNSUPPORTED;
  }
}

// The Stream-K policy: argmin over data_parallel, stream_k(g) for g in 1..p and
// two_tile_sk_dp(p), leaving data-parallel only for a predicted gain > margin.
sk_status sk_select_schedule(const sk_cost_params* c, const sk_tile_grid_t* g, int64_t p,
                             int32_t* strategy, int64_t* param) {
  if (!c || !valid_grid(g) || p < 1 || !strategy || !param) return SK_EINVAL;
  double t_dp;
  sk_predict_schedule(c, g, SK_DATA_PARALLEL, 1, p, &t_dp);
  int32_t best_s = SK_DATA_PARALLEL;
  int64_t best_p = 1;
  double bt = t_dp;
  // Basic Stream-K only while its units stay within ~one tile wave (t < 2p):
  // beyond that every unit spans several tiles at unrelated k offsets, which
  // defeats L2 reuse (not in the model), and the paper's two-tile hybrid takes
  // over; measured: profiles/r01/sweep_corpus_seed0_1000_2sm.csv.
  if (g->total_tiles < 2 * p) {
    int64_t gbest;
    sk_cost_params nomargin = *c;
    nomargin.margin = 0.0;
    sk_select_grid_size(&nomargin, g, p, &gbest);
    if (gbest != std::min(g->total_tiles, g->total_iters)) {
      best_s = SK_STREAM_K;
      best_p = gbest;
      sk_predict_time(c, g, gbest, p, &bt);
    }
  }
  if (g->total_tiles > p && g->total_tiles % p != 0) {
    double t2;
    sk_predict_schedule(c, g, SK_TWO_TILE_SK_DP, p, p, &t2);
    if (t2 < bt) {
      bt = t2;
      best_s = SK_TWO_TILE_SK_DP;
      best_p = p;
    }
  }
  if (best_s != SK_DATA_PARALLEL && !(bt < (1.0 - c->margin) * t_dp)) {
    best_s = SK_DATA_PARALLEL;
    best_p = 1;
  }
  // Cluster fixup: fixed_split(S) whose S k-chunks of a tile reduce through
  // DSMEM, no global partials.  Rule measured on calibration corpora (seed 1)
  // plus configs 3 and skinny (profiles/r02s, r02v): with chunks of >= 8
  // (1-SM) / >= 16 (2-SM pair) iterations it beat the model's pick and
  // data-parallel on ~95 % of such shapes, with no shape > 5 % slower than DP.
  if (c->cluster_min_iters > 0.0) {
    // S = 5, 6, 7 run (the kernel folds whole 32-column boxes, 1-2 per slot)
    // but measured no faster than S = 4 in geomean and up to 10 % slower on
    // the 1-SM kernel; S = 3 beat S = 2 on every sampled shape (1.12-1.14x,
    // profiles/r02z4/).  Candidates: the largest of 8, 4, 3, 2 that fits.
    for (int64_t S : {8, 4, 3, 2}) {
      const int64_t ips = cdiv(g->iters_per_tile, S);
      if ((S - 1) * ips >= g->iters_per_tile) continue;  // an empty chunk: no cluster fixup
      if (static_cast<double>(ips) < c->cluster_min_iters) continue;
      int32_t units = 0;
      const sk_variant v = c->cluster_kernel == 1.0 ? SK_VARIANT_1SM : SK_VARIANT_2SM;
      if (sk_cluster_capacity(v, static_cast<int32_t>(S), -1, &units) != SK_OK) continue;
      if (g->total_tiles * S > units) continue;
      best_s = SK_FIXED_SPLIT;
      best_p = S;
      break;
    }
  }
  *strategy = best_s;
  *param = best_p;
  return SK_OK;
}

sk_status sk_calibrate(const sk_tile_grid_t* grids, const int64_t* gs, const double* times,
                       int64_t n, int64_t p, sk_cost_params* out) {
  if (!grids || !gs || !times || !out || n < kF || p < 1) return SK_EINVAL;
  std::vector<double> A(static_cast<size_t>(n) * kF), b(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    if (!valid_grid(&grids[i]) || gs[i] < 1 || !(times[i] > 0)) return SK_EINVAL;
    double f[kF];
    features(grids[i], gs[i], p, f, out->coop_peers);
    for (int j = 0; j < kF; ++j) A[static_cast<size_t>(i) * kF + j] = f[j] / times[i];
    b[static_cast<size_t>(i)] = 1.0;  // relative error: (pred - t) / t
  }
  std::vector<double> x;
  if (!nnls(A, b, static_cast<int>(n), kF, x)) return SK_EINVAL;
  double res = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double r = 1.0;
    for (int j = 0; j < kF; ++j) r -= A[static_cast<size_t>(i) * kF + j] * x[j];
    res += r * r;
  }
  const double margin = out->margin;
  const double coop_peers = out->coop_peers;
  out->e = x[0];
  out->a = x[1];
  out->b = x[2];
  out->c = x[3];
  out->d = x[4];
  out->s = x[5];
  out->margin = margin;
  out->coop_peers = coop_peers;
  out->fit_residual = std::sqrt(res / static_cast<double>(n));  // RMS relative error
  return SK_OK;
}

// B200 constants (microseconds), fitted with sk_calibrate on samples measured
// by `python -m paper_2301_03598_b200.sweep --calibrate` (corpus seed 1,
// disjoint from the seed-0 evaluation corpus); see profiles/r01/costmodel.json.
// Cooperative fold cost in serial-peer-fold units = coop_peers + contributors / 8
// fits the two measured points (3.7 at 9 contributors, 4.7 at 19) with 2.5, but
// a policy using it (2.5 or a flat 4) picked Stream-K on 1-3-tile deep-k shapes
// where it lost up to 2x and scored config 3 at 1.353 / corpus-1000 at 1.017 vs
// 1.379 / 1.022 without it (profiles/r01/coop_fixup.txt): the default stays the
// reference's owner-fold model, coop_peers = 0.
constexpr double kCoopPeers = 0.0;

sk_status sk_default_cost_params(sk_dtype ab_type, sk_variant variant, sk_cost_params* out) {
  if (!out) return SK_EINVAL;
  if (ab_type != SK_BFLOAT16 && ab_type != SK_FLOAT16 && ab_type != SK_FLOAT64) return SK_EINVAL;
  sk_cost_params c{};
  if (ab_type == SK_FLOAT64) {
    c = {0.0, 5.2158, 0.0, 0.71323, 0.95141, 0.62478, 0.3, 0.0};  // costmodel_fp64.json
  } else if (variant == SK_VARIANT_2SM || variant == SK_VARIANT_2SM_WIDE || variant == SK_VARIANT_AUTO) {
    c = {3.9049, 0.9955, 0.4063, 0.3098, 2.3291, 3.3913, 0.2, 0.0, kCoopPeers, 16.0, 2.0};
    if (variant == SK_VARIANT_2SM_WIDE) c.cluster_min_iters = 0.0;  // no cluster fixup on the wide tile
  } else {
    c = {4.2166, 0.24668, 1.8380, 0.42998, 2.6520, 2.8518, 0.2, 0.0, kCoopPeers, 8.0, 1.0};  // costmodel_1sm.json
  }
  *out = c;
  return SK_OK;
}

}  // extern "C"
