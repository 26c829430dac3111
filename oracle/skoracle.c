/*
 * skoracle.c -- CPU restatement of the reference Stream-K path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity *checker*: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2301_03598_b200/, libskb200.so) never
 * links or calls it.
 *
 * Every function restates the reference algorithm at the cited file:line of
 * /root/reference/proj (streamk-lab, C++20).  The restatement is pinned two
 * ways (see tests/test_oracle.py):
 *   - against the reference's own goldens (test_domain.cpp, test_decompose.cpp,
 *     test_executor.cpp, acceptance.cpp), restated as known-answer tests;
 *   - against the reference itself, compiled from its sources into
 *     oracle/_ref/libstreamk_ref.so (oracle/Makefile), via the committed
 *     fixtures in tests/golden/ made by tests/golden/make_golden.py.
 *
 * Floating point: compiled with -ffp-contract=off and no -march, exactly like
 * the reference's default g++ build, so gemm_reference / execute results are
 * bit-identical to the reference for f32/f64 (checked by the golden tests).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t idx_t;

enum { SKOR_OK = 0, SKOR_EINVAL = 1, SKOR_ERANGE = 5, SKOR_ECAP = 6 };
enum {
  SKOR_DATA_PARALLEL = 0,
  SKOR_FIXED_SPLIT = 1,
  SKOR_STREAM_K = 2,
  SKOR_DP_ONE_TILE_SK = 3,
  SKOR_TWO_TILE_SK_DP = 4
};

static idx_t ceil_div(idx_t x, idx_t y) { return (x + y - 1) / y; } /* types.hpp:36 */
static idx_t min_i(idx_t a, idx_t b) { return a < b ? a : b; }

/* types.cpp:33-55 -- validate + tile_grid.  out = {tiles_m, tiles_n, total_tiles,
 * iters_per_tile, total_iters}. */
int skor_tile_grid(idx_t m, idx_t n, idx_t k, idx_t bm, idx_t bn, idx_t bk, idx_t* out) {
  if (m < 1 || n < 1 || k < 1) return SKOR_EINVAL;
  if (bm < 1 || bn < 1 || bk < 1) return SKOR_EINVAL;
  out[0] = ceil_div(m, bm);
  out[1] = ceil_div(n, bn);
  out[2] = out[0] * out[1];
  out[3] = ceil_div(k, bk);
  out[4] = out[2] * out[3];
  return SKOR_OK;
}

/* types.cpp:57-62 -- iter_to_coords (throws out_of_range -> SKOR_ERANGE). */
int skor_iter_to_coords(const idx_t* grid, idx_t i, idx_t* tile, idx_t* local) {
  if (i < 0 || i >= grid[4]) return SKOR_ERANGE;
  *tile = i / grid[3];
  *local = i % grid[3];
  return SKOR_OK;
}

/* decompose.cpp:13-24 -- balanced_ranges: larger shares first. */
static void balanced_ranges(idx_t begin, idx_t end, idx_t count, idx_t first_id, idx_t* out) {
  const idx_t total = end - begin;
  const idx_t base = total / count;
  const idx_t rem = total % count;
  idx_t cursor = begin;
  for (idx_t i = 0; i < count; ++i) {
    const idx_t len = base + (i < rem ? 1 : 0);
    out[2 * (first_id + i)] = cursor;
    out[2 * (first_id + i) + 1] = cursor + len;
    cursor += len;
  }
}

/*
 * Schedule constructors, decompose.cpp:38-121.  `param` is s (fixed_split),
 * g (stream_k) or p (hybrids); ignored for data_parallel.  Writes the grid size
 * to *out_g and, if ranges != NULL and cap >= g, the [g][2] (begin, end) table
 * (cta_id == row index, types.hpp:76-84).
 */
int skor_schedule(int strategy, idx_t m, idx_t n, idx_t k, idx_t bm, idx_t bn, idx_t bk,
                  idx_t param, idx_t* out_g, idx_t* ranges, idx_t cap) {
  idx_t grid[5];
  int st = skor_tile_grid(m, n, k, bm, bn, bk, grid);
  if (st) return st;
  const idx_t t = grid[2], ipt = grid[3], total = grid[4];
  idx_t g = 0;
  switch (strategy) {
    case SKOR_DATA_PARALLEL: /* decompose.cpp:38-48 */
      g = t;
      *out_g = g;
      if (!ranges) return SKOR_OK;
      if (cap < g) return SKOR_ECAP;
      for (idx_t x = 0; x < t; ++x) {
        ranges[2 * x] = x * ipt;
        ranges[2 * x + 1] = (x + 1) * ipt;
      }
      return SKOR_OK;
    case SKOR_FIXED_SPLIT: { /* decompose.cpp:50-69 */
      const idx_t s = param;
      if (s < 1) return SKOR_EINVAL;
      const idx_t ips = ceil_div(ipt, s);
      g = t * s;
      *out_g = g;
      if (!ranges) return SKOR_OK;
      if (cap < g) return SKOR_ECAP;
      for (idx_t x = 0; x < t; ++x) {
        for (idx_t y = 0; y < s; ++y) {
          const idx_t lo = min_i(ipt, y * ips);
          const idx_t hi = min_i(ipt, lo + ips);
          ranges[2 * (x * s + y)] = x * ipt + lo;
          ranges[2 * (x * s + y) + 1] = x * ipt + hi;
        }
      }
      return SKOR_OK;
    }
    case SKOR_STREAM_K: /* decompose.cpp:71-79 */
      if (param < 1) return SKOR_EINVAL;
      g = param;
      *out_g = g;
      if (!ranges) return SKOR_OK;
      if (cap < g) return SKOR_ECAP;
      balanced_ranges(0, total, g, 0, ranges);
      return SKOR_OK;
    case SKOR_DP_ONE_TILE_SK:
    case SKOR_TWO_TILE_SK_DP: { /* decompose.cpp:81-121 */
      const idx_t p = param;
      if (p < 1) return SKOR_EINVAL;
      const idx_t w = t / p, r = t % p;
      if (r == 0) { /* :92-97 degenerate to data-parallel ranges */
        *out_g = t;
        if (!ranges) return SKOR_OK;
        if (cap < t) return SKOR_ECAP;
        for (idx_t x = 0; x < t; ++x) {
          ranges[2 * x] = x * ipt;
          ranges[2 * x + 1] = (x + 1) * ipt;
        }
        return SKOR_OK;
      }
      idx_t dp_tiles;
      if (strategy == SKOR_DP_ONE_TILE_SK) dp_tiles = w * p;
      else dp_tiles = w >= 2 ? (w - 1) * p : 0;
      const idx_t sk_begin = dp_tiles * ipt;
      g = dp_tiles + p;
      *out_g = g;
      if (!ranges) return SKOR_OK;
      if (cap < g) return SKOR_ECAP;
      if (strategy == SKOR_DP_ONE_TILE_SK) { /* :108-112 */
        for (idx_t x = 0; x < dp_tiles; ++x) {
          ranges[2 * x] = x * ipt;
          ranges[2 * x + 1] = (x + 1) * ipt;
        }
        balanced_ranges(sk_begin, total, p, dp_tiles, ranges);
      } else { /* :113-119 SK ids first */
        balanced_ranges(sk_begin, total, p, 0, ranges);
        for (idx_t x = 0; x < dp_tiles; ++x) {
          ranges[2 * (p + x)] = x * ipt;
          ranges[2 * (p + x) + 1] = (x + 1) * ipt;
        }
      }
      return SKOR_OK;
    }
    default:
      return SKOR_EINVAL;
  }
}

/*
 * decompose.cpp:123-136 -- fixup_peers_of, as CSR: offsets[t+1], ids[].
 * ids within a tile are ascending (ranges are visited in ascending cta_id, so
 * the per-tile lists come out sorted without the reference's final sort).
 * *out_nnz receives the total count; ids may be NULL to query it.
 */
int skor_fixup_peers(const idx_t* ranges, idx_t g, idx_t ipt, idx_t t, idx_t* offsets,
                     idx_t* ids, idx_t ids_cap, idx_t* out_nnz) {
  for (idx_t x = 0; x <= t; ++x) offsets[x] = 0;
  for (idx_t c = 0; c < g; ++c) {
    const idx_t b = ranges[2 * c], e = ranges[2 * c + 1];
    if (b == e) continue;
    for (idx_t tile = b / ipt; tile <= (e - 1) / ipt; ++tile) offsets[tile + 1]++;
  }
  for (idx_t x = 0; x < t; ++x) offsets[x + 1] += offsets[x];
  *out_nnz = offsets[t];
  if (!ids) return SKOR_OK;
  if (ids_cap < offsets[t]) return SKOR_ECAP;
  idx_t* fill = (idx_t*)malloc(sizeof(idx_t) * (size_t)(t > 0 ? t : 1));
  if (!fill) return SKOR_EINVAL;
  for (idx_t x = 0; x < t; ++x) fill[x] = offsets[x];
  for (idx_t c = 0; c < g; ++c) {
    const idx_t b = ranges[2 * c], e = ranges[2 * c + 1];
    if (b == e) continue;
    for (idx_t tile = b / ipt; tile <= (e - 1) / ipt; ++tile) ids[fill[tile]++] = c;
  }
  free(fill);
  return SKOR_OK;
}

/* decompose.cpp:138-141 */
int skor_quantization_efficiency(idx_t t, idx_t p, double* out) {
  if (t < 1 || p < 1) return SKOR_EINVAL;
  *out = (double)t / (double)(ceil_div(t, p) * p);
  return SKOR_OK;
}

/* ---- matrix.hpp:39-68: SplitMix64 and random_matrix ------------------------ */
static uint64_t splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double splitmix_double(uint64_t* state) {
  return (double)(splitmix_next(state) >> 11) * 0x1.0p-53;
}

void skor_splitmix_stream(uint64_t seed, idx_t count, uint64_t* out) {
  uint64_t s = seed;
  for (idx_t i = 0; i < count; ++i) out[i] = splitmix_next(&s);
}
void skor_random_matrix_i64(idx_t rows, idx_t cols, uint64_t seed, int64_t* out) {
  uint64_t s = seed;
  for (idx_t i = 0; i < rows * cols; ++i) out[i] = (int64_t)(splitmix_next(&s) & 0x7f) - 64;
}
void skor_random_matrix_f32(idx_t rows, idx_t cols, uint64_t seed, float* out) {
  uint64_t s = seed;
  for (idx_t i = 0; i < rows * cols; ++i) out[i] = (float)(splitmix_double(&s) * 2.0 - 1.0);
}
void skor_random_matrix_f64(idx_t rows, idx_t cols, uint64_t seed, double* out) {
  uint64_t s = seed;
  for (idx_t i = 0; i < rows * cols; ++i) out[i] = splitmix_double(&s) * 2.0 - 1.0;
}

/* ---- sweep.cpp:21-28 log_sample and :79-86 corpus order --------------------- */
static idx_t log_sample(uint64_t* s, idx_t lo, idx_t hi) {
  if (lo == hi) return lo;
  const double u = splitmix_double(s);
  const double v = exp(log((double)lo) + u * (log((double)hi) - log((double)lo)));
  idx_t r = (idx_t)llround(v);
  if (r < lo) r = lo;
  if (r > hi) r = hi;
  return r;
}
/* out[4*i] = {m, n, k, matrix_seed} for sample i. */
void skor_corpus(uint64_t seed, idx_t count, idx_t lo, idx_t hi, uint64_t* out) {
  uint64_t s = seed;
  for (idx_t i = 0; i < count; ++i) {
    out[4 * i + 0] = (uint64_t)log_sample(&s, lo, hi);
    out[4 * i + 1] = (uint64_t)log_sample(&s, lo, hi);
    out[4 * i + 2] = (uint64_t)log_sample(&s, lo, hi);
    out[4 * i + 3] = splitmix_next(&s);
  }
}

/* ---- executor.hpp:22-54 gemm_reference (six-loop blocked) ------------------ */
#define DEFINE_GEMM_REFERENCE(SUF, T)                                                      \
  int skor_gemm_reference_##SUF(idx_t m, idx_t n, idx_t k, idx_t bm, idx_t bn, idx_t bk,   \
                                const T* A, const T* B, T* C) {                            \
    if (m < 1 || n < 1 || k < 1 || bm < 1 || bn < 1 || bk < 1) return SKOR_EINVAL;         \
    for (idx_t mm = 0; mm < m; mm += bm) {                                                 \
      const idx_t m_hi = min_i(mm + bm, m);                                                \
      for (idx_t nn = 0; nn < n; nn += bn) {                                               \
        const idx_t n_hi = min_i(nn + bn, n);                                              \
        for (idx_t i = mm; i < m_hi; ++i)                                                  \
          for (idx_t j = nn; j < n_hi; ++j) C[i * n + j] = (T)0;                           \
        for (idx_t kk = 0; kk < k; kk += bk) {                                             \
          const idx_t k_hi = min_i(kk + bk, k);                                            \
          for (idx_t i = mm; i < m_hi; ++i) {                                              \
            for (idx_t j = nn; j < n_hi; ++j) {                                            \
              T acc = C[i * n + j];                                                        \
              for (idx_t q = kk; q < k_hi; ++q) acc += A[i * k + q] * B[q * n + j];         \
              C[i * n + j] = acc;                                                          \
            }                                                                              \
          }                                                                                \
        }                                                                                  \
      }                                                                                    \
    }                                                                                      \
    return SKOR_OK;                                                                        \
  }
DEFINE_GEMM_REFERENCE(f32, float)
DEFINE_GEMM_REFERENCE(f64, double)
DEFINE_GEMM_REFERENCE(i64, int64_t)

/*
 * executor.hpp:59-88 mac_loop + :130-207 execute, restated sequentially.
 * Per logical CTA and tile segment (:151-184): mac_loop into a zeroed
 * blk_m x blk_n accumulator; local_begin != 0 -> store partial; else fold the
 * peers' partials in ascending cta_id (:165-172) and clamp-store (:175-181).
 * Dispatch order does not change any value (each partial is written once and
 * the fold order is fixed), so a descending sequential sweep reproduces the
 * threaded executor bit-for-bit.
 */
#define DEFINE_EXECUTE(SUF, T)                                                              \
  int skor_execute_##SUF(const idx_t* ranges, idx_t g, idx_t m, idx_t n, idx_t k, idx_t bm, \
                         idx_t bn, idx_t bk, const T* A, const T* B, T* C) {                \
    idx_t grid[5];                                                                          \
    int st = skor_tile_grid(m, n, k, bm, bn, bk, grid);                                     \
    if (st) return st;                                                                      \
    const idx_t tiles_n = grid[1], t = grid[2], ipt = grid[3];                              \
    const size_t slab = (size_t)(bm * bn);                                                  \
    idx_t *offsets = NULL, *ids = NULL, nnz = 0;                                            \
    T* partials = NULL;                                                                     \
    T* accum = NULL;                                                                        \
    offsets = (idx_t*)malloc(sizeof(idx_t) * (size_t)(t + 1));                              \
    if (!offsets) return SKOR_EINVAL;                                                       \
    skor_fixup_peers(ranges, g, ipt, t, offsets, NULL, 0, &nnz);                            \
    ids = (idx_t*)malloc(sizeof(idx_t) * (size_t)(nnz > 0 ? nnz : 1));                      \
    partials = (T*)calloc((size_t)g * slab, sizeof(T));                                     \
    accum = (T*)malloc(sizeof(T) * slab);                                                   \
    if (!ids || !partials || !accum) { st = SKOR_EINVAL; goto done_##SUF; }                 \
    skor_fixup_peers(ranges, g, ipt, t, offsets, ids, nnz, &nnz);                           \
    memset(C, 0, sizeof(T) * (size_t)(m * n));                                              \
    for (idx_t cta = g - 1; cta >= 0; --cta) {                                              \
      idx_t iter = ranges[2 * cta];                                                         \
      const idx_t end = ranges[2 * cta + 1];                                                \
      while (iter < end) {                                                                  \
        const idx_t tile = iter / ipt, tile_iter = tile * ipt;                              \
        const idx_t lb = iter - tile_iter;                                                  \
        const idx_t le = min_i(end, tile_iter + ipt) - tile_iter;                           \
        const idx_t mm = bm * (tile / tiles_n), nn = bn * (tile % tiles_n);                 \
        const idx_t m_ext = min_i(bm, m - mm), n_ext = min_i(bn, n - nn);                   \
        for (size_t e = 0; e < slab; ++e) accum[e] = (T)0;                                  \
        for (idx_t it = lb; it < le; ++it) {                                                \
          const idx_t kk = it * bk, k_hi = min_i(kk + bk, k);                               \
          for (idx_t i = 0; i < m_ext; ++i)                                                 \
            for (idx_t j = 0; j < n_ext; ++j) {                                             \
              T acc = accum[i * bn + j];                                                    \
              for (idx_t q = kk; q < k_hi; ++q) acc += A[(mm + i) * k + q] * B[q * n + nn + j]; \
              accum[i * bn + j] = acc;                                                      \
            }                                                                               \
        }                                                                                   \
        if (lb != 0) {                                                                      \
          memcpy(partials + (size_t)cta * slab, accum, sizeof(T) * slab);                   \
        } else {                                                                            \
          for (idx_t q = offsets[tile]; q < offsets[tile + 1]; ++q) {                       \
            const idx_t peer = ids[q];                                                      \
            if (peer == cta) continue;                                                      \
            const T* p = partials + (size_t)peer * slab;                                    \
            for (size_t e = 0; e < slab; ++e) accum[e] += p[e];                             \
          }                                                                                 \
          for (idx_t i = 0; i < m_ext; ++i)                                                 \
            for (idx_t j = 0; j < n_ext; ++j) C[(mm + i) * n + nn + j] = accum[i * bn + j]; \
        }                                                                                   \
        iter = tile_iter + ipt;                                                             \
      }                                                                                     \
    }                                                                                       \
  done_##SUF:                                                                               \
    free(offsets);                                                                          \
    free(ids);                                                                              \
    free(partials);                                                                         \
    free(accum);                                                                            \
    return st;                                                                              \
  }
DEFINE_EXECUTE(f32, float)
DEFINE_EXECUTE(f64, double)
DEFINE_EXECUTE(i64, int64_t)

/*
 * executor.hpp:217-239 verify.  is_int selects bit-exactness; otherwise
 * |c - ref| <= 8 * eps * k * max(|ref|, 1) with eps the caller's epsilon.
 * Inputs are widened to double by the caller.  Returns 1 on pass.
 * One deliberate tightening: a NaN error fails here, whereas the reference's
 * `abs_err > bound` comparison lets NaN through.
 */
int skor_verify(const double* C, const double* Cref, idx_t count, idx_t k, double eps,
                int is_int, double* max_abs, double* max_rel) {
  int pass = 1;
  double ma = 0.0, mr = 0.0;
  for (idx_t i = 0; i < count; ++i) {
    const double c = C[i], ref = Cref[i];
    const double abs_err = fabs(c - ref);
    const double scale = fabs(ref) > 1.0 ? fabs(ref) : 1.0;
    if (abs_err > ma) ma = abs_err;
    if (abs_err / scale > mr) mr = abs_err / scale;
    if (is_int) {
      if (c != ref) pass = 0;
    } else if (!(abs_err <= 8.0 * eps * (double)k * scale)) {
      pass = 0;
    }
  }
  *max_abs = ma;
  *max_rel = mr;
  return pass;
}
