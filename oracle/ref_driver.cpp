// ref_driver.cpp -- extern "C" driver over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources (/root/reference/proj/core/src/*.cpp, read in place,
// never copied) into oracle/_ref/libstreamk_ref.so.  It lets the Python tests
// and bench.py's reference arm call the reference's public API:
//   streamk::{data_parallel, fixed_split, stream_k, hybrid}   decompose.hpp:12-35
//   streamk::fixup_peers_of / quantization_efficiency         decompose.hpp:37-44
//   streamk::to_text / from_text                              types.hpp:86-90
//   streamk::random_matrix<T>                                 matrix.hpp:56-68
//   streamk::gemm_reference<T> / execute<T>                   executor.hpp:22-207
//   streamk::run_sweep (corpus order, full CSV)                sweep.hpp:29-33
//   streamk::simulate / utilization                           simulate.hpp:34-40
// Exceptions are mapped to status codes (invalid_argument=1, logic_error=4,
// out_of_range=5, other=7).
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>

#include "streamk/decompose.hpp"
#include "streamk/executor.hpp"
#include "streamk/matrix.hpp"
#include "streamk/simulate.hpp"
#include "streamk/sweep.hpp"
#include "streamk/types.hpp"

using namespace streamk;

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::out_of_range&) {
    return 5;
  } catch (const std::logic_error&) {
    return 4;
  } catch (...) {
    return 7;
  }
}

WorkAssignment build(int strategy, int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn,
                     int64_t bk, int64_t param) {
  const GemmProblem p{m, n, k};
  const BlockingFactors b{bm, bn, bk};
  switch (strategy) {
    case 0: return data_parallel(p, b);
    case 1: return fixed_split(p, b, param);
    case 2: return stream_k(p, b, param);
    case 3: return hybrid(p, b, param, HybridVariant::DpOneTileSk);
    case 4: return hybrid(p, b, param, HybridVariant::TwoTileSkDp);
  }
  throw std::invalid_argument("unknown strategy");
}

template <typename T>
Matrix<T> wrap(const T* data, int64_t rows, int64_t cols) {
  Matrix<T> mtx(rows, cols);
  std::memcpy(mtx.data.data(), data, sizeof(T) * static_cast<size_t>(rows * cols));
  return mtx;
}

template <typename T>
int execute_strategy(int strategy, int64_t param, int64_t m, int64_t n, int64_t k, int64_t bm,
                     int64_t bn, int64_t bk, const T* A, const T* B, T* C, int threads) {
  return guarded([&] {
    const WorkAssignment a = build(strategy, m, n, k, bm, bn, bk, param);
    const Matrix<T> Am = wrap(A, m, k), Bm = wrap(B, k, n);
    const Matrix<T> Cm = execute(a, Am, Bm, threads);
    std::memcpy(C, Cm.data.data(), sizeof(T) * static_cast<size_t>(m * n));
  });
}

// An arbitrary range table through the reference's own text parser
// (types.cpp:101-123), then execute<T> (executor.hpp:130-207).
template <typename T>
int execute_table(const int64_t* ranges, int64_t g, int64_t m, int64_t n, int64_t k, int64_t bm,
                  int64_t bn, int64_t bk, const T* A, const T* B, T* C, int threads) {
  return guarded([&] {
    std::ostringstream text;
    text << m << ' ' << n << ' ' << k << '\n' << bm << ' ' << bn << ' ' << bk << '\n'
         << "stream_k " << g << '\n';
    for (int64_t i = 0; i < g; ++i) text << i << ' ' << ranges[2 * i] << ' ' << ranges[2 * i + 1] << '\n';
    const WorkAssignment a = from_text(text.str());
    const Matrix<T> Am = wrap(A, m, k), Bm = wrap(B, k, n);
    const Matrix<T> Cm = execute(a, Am, Bm, threads);
    std::memcpy(C, Cm.data.data(), sizeof(T) * static_cast<size_t>(m * n));
  });
}

template <typename T>
int gemm_ref(int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn, int64_t bk, const T* A,
             const T* B, T* C) {
  return guarded([&] {
    const Matrix<T> Cm = gemm_reference<T>({m, n, k}, {bm, bn, bk}, wrap(A, m, k), wrap(B, k, n));
    std::memcpy(C, Cm.data.data(), sizeof(T) * static_cast<size_t>(m * n));
  });
}

}  // namespace

extern "C" {

int ref_tile_grid(int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn, int64_t bk,
                  int64_t* out) {
  return guarded([&] {
    const TileGrid g = tile_grid({m, n, k}, {bm, bn, bk});
    out[0] = g.tiles_m;
    out[1] = g.tiles_n;
    out[2] = g.total_tiles;
    out[3] = g.iters_per_tile;
    out[4] = g.total_iters;
  });
}

int ref_iter_to_coords(int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn, int64_t bk,
                       int64_t i, int64_t* tile, int64_t* local) {
  return guarded([&] {
    const TileCoords c = iter_to_coords(tile_grid({m, n, k}, {bm, bn, bk}), i);
    *tile = c.tile_idx;
    *local = c.local_iter;
  });
}

// Grid size into *out_g; ranges ([g][2]) written when ranges != NULL and cap >= g.
int ref_schedule(int strategy, int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn,
                 int64_t bk, int64_t param, int64_t* out_g, int64_t* ranges, int64_t cap) {
  return guarded([&] {
    const WorkAssignment a = build(strategy, m, n, k, bm, bn, bk, param);
    *out_g = a.grid_size;
    if (!ranges) return;
    if (cap < a.grid_size) throw std::invalid_argument("cap");
    for (const CtaRange& r : a.ranges) {
      ranges[2 * r.cta_id] = r.iter_begin;
      ranges[2 * r.cta_id + 1] = r.iter_end;
    }
  });
}

// to_text of the strategy's assignment into buf (NUL-terminated); *len = full length.
int ref_to_text(int strategy, int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn,
                int64_t bk, int64_t param, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const std::string s = to_text(build(strategy, m, n, k, bm, bn, bk, param));
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) {
      const size_t c = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), c);
      buf[c] = 0;
    }
  });
}

// from_text round trip: parse text, write back to_text(from_text(text)).
int ref_text_roundtrip(const char* text, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const std::string s = to_text(from_text(std::string(text)));
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) {
      const size_t c = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), c);
      buf[c] = 0;
    }
  });
}

// fixup_peers_of as CSR (offsets[t+1], ids[nnz]); ids may be NULL to size.
int ref_fixup_peers(int strategy, int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn,
                    int64_t bk, int64_t param, int64_t* offsets, int64_t* ids, int64_t cap,
                    int64_t* nnz) {
  return guarded([&] {
    const auto peers = fixup_peers_of(build(strategy, m, n, k, bm, bn, bk, param));
    int64_t total = 0;
    offsets[0] = 0;
    for (size_t t = 0; t < peers.size(); ++t) {
      total += static_cast<int64_t>(peers[t].size());
      offsets[t + 1] = total;
    }
    *nnz = total;
    if (!ids) return;
    if (cap < total) throw std::invalid_argument("cap");
    int64_t q = 0;
    for (const auto& list : peers)
      for (int64_t id : list) ids[q++] = id;
  });
}

int ref_quantization_efficiency(int64_t t, int64_t p, double* out) {
  return guarded([&] { *out = quantization_efficiency(t, p); });
}

void ref_random_matrix_i64(int64_t r, int64_t c, uint64_t seed, int64_t* out) {
  const auto mtx = random_matrix<int64_t>(r, c, seed);
  std::memcpy(out, mtx.data.data(), sizeof(int64_t) * mtx.data.size());
}
void ref_random_matrix_f32(int64_t r, int64_t c, uint64_t seed, float* out) {
  const auto mtx = random_matrix<float>(r, c, seed);
  std::memcpy(out, mtx.data.data(), sizeof(float) * mtx.data.size());
}
void ref_random_matrix_f64(int64_t r, int64_t c, uint64_t seed, double* out) {
  const auto mtx = random_matrix<double>(r, c, seed);
  std::memcpy(out, mtx.data.data(), sizeof(double) * mtx.data.size());
}

int ref_gemm_reference_f32(int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn, int64_t bk,
                           const float* A, const float* B, float* C) {
  return gemm_ref(m, n, k, bm, bn, bk, A, B, C);
}
int ref_gemm_reference_f64(int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn, int64_t bk,
                           const double* A, const double* B, double* C) {
  return gemm_ref(m, n, k, bm, bn, bk, A, B, C);
}
int ref_gemm_reference_i64(int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn, int64_t bk,
                           const int64_t* A, const int64_t* B, int64_t* C) {
  return gemm_ref(m, n, k, bm, bn, bk, A, B, C);
}

int ref_execute_f32(int strategy, int64_t param, int64_t m, int64_t n, int64_t k, int64_t bm,
                    int64_t bn, int64_t bk, const float* A, const float* B, float* C,
                    int threads) {
  return execute_strategy(strategy, param, m, n, k, bm, bn, bk, A, B, C, threads);
}
int ref_execute_f64(int strategy, int64_t param, int64_t m, int64_t n, int64_t k, int64_t bm,
                    int64_t bn, int64_t bk, const double* A, const double* B, double* C,
                    int threads) {
  return execute_strategy(strategy, param, m, n, k, bm, bn, bk, A, B, C, threads);
}
int ref_execute_i64(int strategy, int64_t param, int64_t m, int64_t n, int64_t k, int64_t bm,
                    int64_t bn, int64_t bk, const int64_t* A, const int64_t* B, int64_t* C,
                    int threads) {
  return execute_strategy(strategy, param, m, n, k, bm, bn, bk, A, B, C, threads);
}

// SKMX files through the reference's own save_matrix/load_matrix (matrix.hpp:78-93).
int ref_execute_ranges_f32(const int64_t* ranges, int64_t g, int64_t m, int64_t n, int64_t k,
                           int64_t bm, int64_t bn, int64_t bk, const float* A, const float* B,
                           float* C, int threads) {
  return execute_table(ranges, g, m, n, k, bm, bn, bk, A, B, C, threads);
}
int ref_execute_ranges_f64(const int64_t* ranges, int64_t g, int64_t m, int64_t n, int64_t k,
                           int64_t bm, int64_t bn, int64_t bk, const double* A, const double* B,
                           double* C, int threads) {
  return execute_table(ranges, g, m, n, k, bm, bn, bk, A, B, C, threads);
}
int ref_execute_ranges_i64(const int64_t* ranges, int64_t g, int64_t m, int64_t n, int64_t k,
                           int64_t bm, int64_t bn, int64_t bk, const int64_t* A, const int64_t* B,
                           int64_t* C, int threads) {
  return execute_table(ranges, g, m, n, k, bm, bn, bk, A, B, C, threads);
}

int ref_save_matrix_f32(const char* path, int64_t r, int64_t c, const float* data) {
  return guarded([&] {
    std::ofstream out(path, std::ios::binary);
    save_matrix(wrap(data, r, c), out);
  });
}
int ref_save_matrix_f64(const char* path, int64_t r, int64_t c, const double* data) {
  return guarded([&] {
    std::ofstream out(path, std::ios::binary);
    save_matrix(wrap(data, r, c), out);
  });
}
int ref_save_matrix_i64(const char* path, int64_t r, int64_t c, const int64_t* data) {
  return guarded([&] {
    std::ofstream out(path, std::ios::binary);
    save_matrix(wrap(data, r, c), out);
  });
}
// Loads a float32 SKMX file; returns 7 (runtime_error) on bad magic / dtype.
int ref_load_matrix_f32(const char* path, int64_t* r, int64_t* c, float* data, int64_t cap) {
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    const Matrix<float> m = load_matrix<float>(in);
    *r = m.rows;
    *c = m.cols;
    if (data && cap >= m.rows * m.cols)
      std::memcpy(data, m.data.data(), sizeof(float) * m.data.size());
  });
}

// Corpus dims in run_sweep order (sweep.cpp:79-86), parsed from its CSV with
// the data_parallel strategy only.  out[3*i] = {m, n, k}.
int ref_corpus_dims(uint64_t seed, int64_t count, int64_t lo, int64_t hi, int64_t* out) {
  return guarded([&] {
    SweepSpec spec;
    spec.m_lo = spec.n_lo = spec.k_lo = lo;
    spec.m_hi = spec.n_hi = spec.k_hi = hi;
    spec.sample_count = count;
    spec.seed = seed;
    spec.strategies = {Strategy::DataParallel};
    spec.p = 148;
    std::ostringstream csv;
    run_sweep(spec, {128, 256, 64}, csv);
    std::istringstream in(csv.str());
    std::string line;
    std::getline(in, line);  // # schema=1
    std::getline(in, line);  // header
    int64_t i = 0;
    while (std::getline(in, line) && i < count) {
      std::istringstream row(line);
      std::string f;
      for (int c = 0; c < 3; ++c) {
        std::getline(row, f, ',');
        out[3 * i + c] = std::stoll(f);
      }
      ++i;
    }
  });
}

// run_sweep's whole CSV text (sweep.cpp:75-112) for a corpus with one [lo, hi]
// range on every axis; strategies as codes 0..4 (types.hpp:70 order).
// *len = bytes needed (without the NUL); buf gets them when cap > *len.
int ref_run_sweep(uint64_t seed, int64_t count, int64_t lo, int64_t hi, const int* strategies,
                  int nstrat, int64_t p, int64_t split, int64_t bm, int64_t bn, int64_t bk,
                  char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    SweepSpec spec;
    spec.m_lo = spec.n_lo = spec.k_lo = lo;
    spec.m_hi = spec.n_hi = spec.k_hi = hi;
    spec.sample_count = count;
    spec.seed = seed;
    spec.strategies.clear();
    for (int i = 0; i < nstrat; ++i) spec.strategies.push_back(static_cast<Strategy>(strategies[i]));
    spec.p = p;
    spec.split = split;
    std::ostringstream csv;
    run_sweep(spec, {bm, bn, bk}, csv);
    const std::string out = csv.str();
    *len = static_cast<int64_t>(out.size());
    if (buf && cap > *len) std::memcpy(buf, out.c_str(), out.size() + 1);
  });
}

// simulate (simulate.cpp:23-69) of a closed-form schedule; with_params selects
// CostParams{a, b, c, d}.  Writes makespan and utilization.
int ref_simulate(int strategy, int64_t param, int64_t m, int64_t n, int64_t k, int64_t bm, int64_t bn,
                 int64_t bk, int64_t p, int with_params, double a, double b, double c, double d,
                 double* makespan, double* util) {
  return guarded([&] {
    const WorkAssignment wa = build(strategy, m, n, k, bm, bn, bk, param);
    std::optional<CostParams> prm;
    if (with_params) {
      CostParams cp;
      cp.a = a;
      cp.b = b;
      cp.c = c;
      cp.d = d;
      prm = cp;
    }
    const Timeline tl = simulate(wa, p, prm);
    *makespan = tl.makespan;
    *util = utilization(tl);
  });
}

}  // extern "C"
