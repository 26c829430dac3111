// costmodel.cpp -- grid-size selection for the device Stream-K schedule.
//
// Restates the reference's Appendix-A model (core/src/costmodel.cpp:13-48,
// PAPER.md:966-1021) and makes it wave-aware for a persistent grid of p CTAs:
//
//   time(g) = e + ceil(g / p) * ( a + b*[peers(g) > 1] + c*ipc(g) + d*(peers(g) - 1) )
//   ipc(g)   = ceil(total_iters / g)                       costmodel.cpp:13-16
//   peers(g) = ceil(iters_per_tile / ipc(g))               costmodel.cpp:18-20
//
// For g <= p (one wave) this is the reference's predict_time plus a constant
// launch term e; for g = t > p (data-parallel with several waves) the per-CTA
// time is multiplied by the wave count, which the reference's desk-scale
// model leaves out.  select_grid_size searches g in {1..p} U {t} like
// costmodel.cpp:30-48 (ties toward larger g); calibrate is a non-negative
// least-squares fit over the 5 features (costmodel.cpp:142-225 fits 4).
// The shipped constants (sk_default_cost_params) were fitted on B200 samples
// measured by paper_2301_03598_b200.sweep (profiles/r01/costmodel_fit.json).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/skb200.h"

namespace {

int64_t cdiv(int64_t x, int64_t y) { return (x + y - 1) / y; }

void features(const sk_tile_grid_t& g, int64_t gs, int64_t p, double f[5]) {
  const int64_t ipc = cdiv(g.total_iters, gs);
  const int64_t peers = cdiv(g.iters_per_tile, ipc);
  const double waves = static_cast<double>(cdiv(gs, p));
  f[0] = 1.0;
  f[1] = waves;
  f[2] = waves * (peers > 1 ? 1.0 : 0.0);
  f[3] = waves * static_cast<double>(ipc);
  f[4] = waves * static_cast<double>(peers - 1);
}

// Lawson-Hanson NNLS on a small dense problem (n x k, k <= 5).
bool nnls(const std::vector<double>& A, const std::vector<double>& b, int n, int k,
          std::vector<double>& x) {
  x.assign(k, 0.0);
  std::vector<bool> passive(k, false);
  auto grad = [&](std::vector<double>& w) {
    w.assign(k, 0.0);
    for (int i = 0; i < n; ++i) {
      double r = b[i];
      for (int j = 0; j < k; ++j) r -= A[i * k + j] * x[j];
      for (int j = 0; j < k; ++j) w[j] += A[i * k + j] * r;
    }
  };
  // unconstrained LS on the passive set via normal equations
  auto solve_passive = [&](std::vector<double>& z) -> bool {
    std::vector<int> idx;
    for (int j = 0; j < k; ++j)
      if (passive[j]) idx.push_back(j);
    const int m = static_cast<int>(idx.size());
    z.assign(k, 0.0);
    if (m == 0) return true;
    std::vector<double> M(m * m, 0.0), v(m, 0.0);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < m; ++a) {
        v[a] += A[i * k + idx[a]] * b[i];
        for (int c = 0; c < m; ++c) M[a * m + c] += A[i * k + idx[a]] * A[i * k + idx[c]];
      }
    for (int col = 0; col < m; ++col) {  // Gaussian elimination with partial pivoting
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
    std::vector<double> y(m, 0.0);
    for (int r = m - 1; r >= 0; --r) {
      double s = v[r];
      for (int c = r + 1; c < m; ++c) s -= M[r * m + c] * y[c];
      y[r] = s / M[r * m + r];
    }
    for (int a = 0; a < m; ++a) z[idx[a]] = y[a];
    return true;
  };
  std::vector<double> w, z;
  for (int outer = 0; outer < 50; ++outer) {
    grad(w);
    int best = -1;
    double bw = 1e-12;
    for (int j = 0; j < k; ++j)
      if (!passive[j] && w[j] > bw) {
        bw = w[j];
        best = j;
      }
    if (best < 0) break;
    passive[best] = true;
    for (int inner = 0; inner < 50; ++inner) {
      if (!solve_passive(z)) return false;
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
        if (passive[j] && std::fabs(x[j]) < 1e-15) {
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
  double f[5];
  features(*g, gs, p, f);
  *out = c->e * f[0] + c->a * f[1] + c->b * f[2] + c->c * f[3] + c->d * f[4];
  return SK_OK;
}

sk_status sk_select_grid_size(const sk_cost_params* c, const sk_tile_grid_t* g, int64_t p,
                              int64_t* out) {
  if (!c || !valid_grid(g) || p < 1 || !out) return SK_EINVAL;
  std::vector<int64_t> cand;
  const int64_t cap = std::min(p, g->total_iters);
  for (int64_t x = 1; x <= cap; ++x) cand.push_back(x);
  cand.push_back(std::min(g->total_tiles, g->total_iters));
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  int64_t best = cand.front();
  double bt = 0.0;
  sk_predict_time(c, g, best, p, &bt);
  for (int64_t x : cand) {
    double t;
    sk_predict_time(c, g, x, p, &t);
    if (t <= bt) {  // ties break toward larger g (costmodel.cpp:41-45)
      bt = t;
      best = x;
    }
  }
  *out = best;
  return SK_OK;
}

sk_status sk_calibrate(const sk_tile_grid_t* grids, const int64_t* gs, const double* times,
                       int64_t n, int64_t p, sk_cost_params* out) {
  if (!grids || !gs || !times || !out || n < 5 || p < 1) return SK_EINVAL;
  std::vector<double> A(static_cast<size_t>(n) * 5), b(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    if (!valid_grid(&grids[i]) || gs[i] < 1) return SK_EINVAL;
    features(grids[i], gs[i], p, &A[static_cast<size_t>(i) * 5]);
    b[static_cast<size_t>(i)] = times[i];
  }
  std::vector<double> x;
  if (!nnls(A, b, static_cast<int>(n), 5, x)) return SK_EINVAL;
  double res = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double r = b[static_cast<size_t>(i)];
    for (int j = 0; j < 5; ++j) r -= A[static_cast<size_t>(i) * 5 + j] * x[j];
    res += r * r;
  }
  out->e = x[0];
  out->a = x[1];
  out->b = x[2];
  out->c = x[3];
  out->d = x[4];
  out->fit_residual = std::sqrt(res);
  return SK_OK;
}

// B200 constants (microseconds), fitted by tests-independent calibration runs
// (paper_2301_03598_b200.sweep --calibrate); see profiles/r01/costmodel_fit.json.
sk_status sk_default_cost_params(sk_dtype ab_type, sk_variant variant, sk_cost_params* out) {
  if (!out) return SK_EINVAL;
  if (ab_type != SK_BFLOAT16 && ab_type != SK_FLOAT16 && ab_type != SK_FLOAT64) return SK_EINVAL;
  sk_cost_params c{};
  if (ab_type == SK_FLOAT64) {
    c = {4.0, 0.5, 2.0, 0.05, 2.0, 0.0};
  } else if (variant == SK_VARIANT_2SM) {
    c = {5.0, 1.0, 4.0, 0.37, 2.0, 0.0};
  } else {
    c = {5.0, 1.0, 3.0, 0.19, 1.5, 0.0};
  }
  *out = c;
  return SK_OK;
}

}  // extern "C"
