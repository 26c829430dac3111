// streamk_b200.hpp -- C++ drop-in for the reference's GEMM entry point.
//
// Include next to the reference's own headers (core/include/streamk/*.hpp) and
// link libskb200.so.  `streamk_b200::execute` takes exactly what
// streamk::execute<T> (executor.hpp:130-132) takes -- a WorkAssignment built by
// streamk::{data_parallel, fixed_split, stream_k, hybrid} and two Matrix<T> --
// and returns a new Matrix<T>, throwing the reference's exception types
// (invalid_argument / out_of_range / logic_error / runtime_error).
//
//   T = int64_t  -> FP64 tensor path, bit-exact (max|A| max|B| k < 2^53)
//   T = double   -> FP64 tensor path (DMMA), tile 64x64x16
//   T = float    -> Precision::Exact: FP64 tensor path on exactly widened inputs;
//                   Precision::BF16 / FP16: tcgen05 tensor cores on rounded inputs,
//                   tile 256x256x64 (2-SM) or 128x256x64 (1-SM)
//
// The assignment's blocking must be the device tile of the chosen precision
// (sk_kernel_blocking); the decomposition knob (s, g or p) is recovered from the
// assignment itself.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "skb200.h"
#include "streamk/executor.hpp"
#include "streamk/matrix.hpp"
#include "streamk/types.hpp"

namespace streamk_b200 {

enum class Precision { Exact, BF16, FP16 };

inline void throw_on(sk_status st) {
  switch (st) {
    case SK_OK: return;
    case SK_EINVAL: throw std::invalid_argument(sk_last_error());
    case SK_ERANGE: throw std::out_of_range(sk_last_error());
    case SK_EPROTOCOL: throw std::logic_error(sk_last_error());  // "fixup flag signaled twice"
    case SK_EIO: throw std::runtime_error(sk_io_error());
    default: throw std::runtime_error(std::string(sk_status_string(st)) + ": " + sk_last_error());
  }
}

inline sk_problem to_sk(const streamk::GemmProblem& p) { return {p.m, p.n, p.k, p.alpha, p.beta}; }
inline sk_blocking to_sk(const streamk::BlockingFactors& b) { return {b.blk_m, b.blk_n, b.blk_k}; }
inline sk_strategy to_sk(streamk::Strategy s) {
  return static_cast<sk_strategy>(static_cast<int>(s));  // same order: types.hpp:70
}

// The closed-form knob (s, g or p) whose schedule reproduces a.ranges exactly;
// 0 for a range table no decomposition produces (run as SK_EXPLICIT).
inline int64_t knob(const streamk::WorkAssignment& a) {
  const sk_problem pr = to_sk(a.problem);
  const sk_blocking bl = to_sk(a.blocking);
  const sk_strategy st = to_sk(a.strategy);
  auto matches = [&](int64_t prm) {
    int64_t g = 0;
    if (sk_schedule(&pr, &bl, st, prm, &g, nullptr, 0) != SK_OK || g != a.grid_size) return false;
    std::vector<int64_t> r(static_cast<size_t>(2 * g));
    if (sk_schedule(&pr, &bl, st, prm, &g, r.data(), g) != SK_OK) return false;
    for (int64_t i = 0; i < g; ++i)
      if (r[2 * i] != a.ranges[i].iter_begin || r[2 * i + 1] != a.ranges[i].iter_end) return false;
    return true;
  };
  switch (a.strategy) {
    case streamk::Strategy::DataParallel:
      if (matches(1)) return 1;
      break;
    case streamk::Strategy::FixedSplit:
      if (matches(a.split)) return a.split;
      break;
    case streamk::Strategy::StreamK:
      if (matches(a.grid_size)) return a.grid_size;
      break;
    default:
      for (int64_t p = 1; p <= a.grid_size; ++p)
        if (matches(p)) return p;
  }
  return 0;
}

template <typename T>
streamk::Matrix<T> execute(const streamk::WorkAssignment& a, const streamk::Matrix<T>& A,
                           const streamk::Matrix<T>& B, Precision prec = Precision::Exact,
                           int device = -1) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double> ||
                    std::is_same_v<T, std::int64_t>,
                "streamk::Matrix<T> element types: int64_t, float, double");
  if (A.rows != a.problem.m || A.cols != a.problem.k || B.rows != a.problem.k ||
      B.cols != a.problem.n)
    throw std::invalid_argument("execute: matrix shapes do not match assignment");
  sk_dtype host = std::is_same_v<T, float> ? SK_FLOAT32
                  : std::is_same_v<T, double> ? SK_FLOAT64 : SK_INT64;
  sk_dtype compute = SK_FLOAT64;
  if constexpr (std::is_same_v<T, float>) {
    if (prec == Precision::BF16) compute = SK_BFLOAT16;
    if (prec == Precision::FP16) compute = SK_FLOAT16;
  }
  const sk_problem pr = to_sk(a.problem);
  const sk_blocking bl = to_sk(a.blocking);
  streamk::Matrix<T> C(a.problem.m, a.problem.n);
  if (const int64_t prm = knob(a)) {
    throw_on(sk_execute(&pr, &bl, to_sk(a.strategy), prm, host, compute, SK_VARIANT_AUTO,
                        A.data.data(), B.data.data(), C.data.data(), device));
    return C;
  }
  // Any other table (e.g. from from_text): ranges by position, as execute<T> reads
  // them (executor.hpp:148); fixup_peers_of keys by cta_id, so they must agree.
  std::vector<int64_t> tbl(2 * a.ranges.size());
  for (size_t i = 0; i < a.ranges.size(); ++i) {
    if (a.ranges[i].cta_id != static_cast<streamk::index_t>(i))
      throw std::invalid_argument("execute: range table cta_ids must be 0..g-1 in order");
    tbl[2 * i] = a.ranges[i].iter_begin;
    tbl[2 * i + 1] = a.ranges[i].iter_end;
  }
  throw_on(sk_execute_ranges(&pr, &bl, tbl.data(), static_cast<int64_t>(a.ranges.size()), host,
                             compute, SK_VARIANT_AUTO, A.data.data(), B.data.data(),
                             C.data.data(), device));
  return C;
}

}  // namespace streamk_b200
