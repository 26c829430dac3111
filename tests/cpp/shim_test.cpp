// shim_test.cpp -- the reference's own C++ API driving libskb200 through
// include/streamk_b200.hpp, checked against the reference's own executor.
// Written in the style of the reference's acceptance suite (one PASS/FAIL line
// per criterion, nonzero exit on failure).  Test infrastructure: built by
// tests/cpp/Makefile against /root/reference/proj headers and sources.
//
//   shim_test --schedule   host only: sk_schedule / sk_fixup_peers == decompose.cpp
//                          on the reference's random-instance generators
//   shim_test --execute    needs a B200: streamk_b200::execute == streamk::execute
//                          (int64 bit-exact, float/double under 8 eps k)
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <sstream>
#include <vector>

#include "streamk/decompose.hpp"
#include "streamk/executor.hpp"
#include "streamk_b200.hpp"
#include "test_util.hpp"

using namespace streamk;
using namespace streamk::testutil;

namespace {

int failures = 0;

void report(const char* what, const std::string& err) {
  std::printf("[%s] %s%s%s\n", err.empty() ? "PASS" : "FAIL", what, err.empty() ? "" : " -- ",
              err.c_str());
  if (!err.empty()) ++failures;
}

std::vector<WorkAssignment> all(const GemmProblem& p, const BlockingFactors& b, Rng& rng) {
  return {data_parallel(p, b), fixed_split(p, b, rng.uniform(1, 5)), stream_k(p, b, rng.uniform(1, 200)),
          hybrid(p, b, rng.uniform(1, 160), HybridVariant::DpOneTileSk),
          hybrid(p, b, rng.uniform(1, 160), HybridVariant::TwoTileSkDp)};
}

std::string schedule_parity() {
  Rng rng(0xb200b200ULL);
  for (int trial = 0; trial < 3000; ++trial) {
    const GemmProblem p = random_problem(rng, 300);
    const BlockingFactors b = random_blocking(rng, 40);
    for (const WorkAssignment& a : all(p, b, rng)) {
      const sk_problem pr = streamk_b200::to_sk(a.problem);
      const sk_blocking bl = streamk_b200::to_sk(a.blocking);
      const int64_t prm = streamk_b200::knob(a);
      int64_t g = 0;
      std::vector<int64_t> r(2 * a.ranges.size());
      if (sk_schedule(&pr, &bl, streamk_b200::to_sk(a.strategy), prm, &g, r.data(),
                      static_cast<int64_t>(a.ranges.size())) != SK_OK ||
          g != a.grid_size)
        return std::string("grid size, ") + strategy_name(a.strategy);
      for (size_t i = 0; i < a.ranges.size(); ++i)
        if (r[2 * i] != a.ranges[i].iter_begin || r[2 * i + 1] != a.ranges[i].iter_end)
          return std::string("ranges, ") + strategy_name(a.strategy);
      const auto peers = fixup_peers_of(a);
      std::vector<int64_t> off(peers.size() + 1);
      int64_t nnz = 0;
      sk_fixup_peers(&pr, &bl, streamk_b200::to_sk(a.strategy), prm, off.data(), nullptr, 0, &nnz);
      std::vector<int64_t> ids(static_cast<size_t>(nnz));
      sk_fixup_peers(&pr, &bl, streamk_b200::to_sk(a.strategy), prm, off.data(), ids.data(), nnz,
                     &nnz);
      for (size_t t = 0; t < peers.size(); ++t) {
        if (static_cast<size_t>(off[t + 1] - off[t]) != peers[t].size())
          return std::string("peer count, ") + strategy_name(a.strategy);
        for (size_t q = 0; q < peers[t].size(); ++q)
          if (ids[static_cast<size_t>(off[t]) + q] != peers[t][q])
            return std::string("peer ids, ") + strategy_name(a.strategy);
      }
    }
  }
  return "";
}

// acceptance.cpp criterion 4 on the device: int64, every strategy, bit-exact.
std::string execute_int64() {
  Rng rng(0xacce9740ULL);
  const BlockingFactors b{64, 64, 16};  // the FP64/int64 device tile
  for (int trial = 0; trial < 60; ++trial) {
    const GemmProblem p = random_problem(rng, 400);
    const auto A = random_matrix<std::int64_t>(p.m, p.k, rng.gen.next());
    const auto B = random_matrix<std::int64_t>(p.k, p.n, rng.gen.next());
    const auto C_ref = naive_multiply(A, B);
    for (const WorkAssignment& a : all(p, b, rng)) {
      const auto C = streamk_b200::execute(a, A, B);
      if (C.data != C_ref.data) return std::string("mismatch, ") + strategy_name(a.strategy);
      if (C.data != execute(a, A, B, 4).data) return "differs from streamk::execute";
    }
  }
  return "";
}

// acceptance.cpp criterion 5 on the device: float and double under 8 eps k.
std::string execute_float_double() {
  Rng rng(0xacce9750ULL);
  const BlockingFactors b{64, 64, 16};
  for (int trial = 0; trial < 30; ++trial) {
    const GemmProblem p = random_problem(rng, 512);
    if (trial % 2 == 0) {
      const auto A = random_matrix<float>(p.m, p.k, rng.gen.next());
      const auto B = random_matrix<float>(p.k, p.n, rng.gen.next());
      for (const WorkAssignment& a : all(p, b, rng)) {
        const auto C = streamk_b200::execute(a, A, B);  // Precision::Exact (FP64 path)
        if (!verify(C, execute(a, A, B, 4), p.k).pass) return "float over the bound";
      }
    } else {
      const auto A = random_matrix<double>(p.m, p.k, rng.gen.next());
      const auto B = random_matrix<double>(p.k, p.n, rng.gen.next());
      for (const WorkAssignment& a : all(p, b, rng)) {
        const auto C = streamk_b200::execute(a, A, B);
        if (!verify(C, gemm_reference(a.problem, a.blocking, A, B), p.k).pass)
          return "double over the bound";
      }
    }
  }
  // BF16 tensor cores on bf16-representable float data (the int64 band): exact.
  const BlockingFactors b16{256, 256, 64};
  const GemmProblem p{700, 900, 1000};
  Matrix<float> A(p.m, p.k), B(p.k, p.n);
  const auto Ai = random_matrix<std::int64_t>(p.m, p.k, 3), Bi = random_matrix<std::int64_t>(p.k, p.n, 4);
  for (size_t i = 0; i < A.data.size(); ++i) A.data[i] = static_cast<float>(Ai.data[i]);
  for (size_t i = 0; i < B.data.size(); ++i) B.data[i] = static_cast<float>(Bi.data[i]);
  const auto want = execute(data_parallel(p, b16), A, B, 8);
  for (const WorkAssignment& a : {stream_k(p, b16, 74), hybrid(p, b16, 74, HybridVariant::TwoTileSkDp)}) {
    if (streamk_b200::execute(a, A, B, streamk_b200::Precision::BF16).data != want.data)
      return "bf16 path not exact on integer-valued data";
  }
  return "";
}

// A table no closed form produces, through the reference's own text parser
// (types.cpp:101-123): random monotone cuts over [0, total), some ranges empty.
WorkAssignment random_table(Rng& rng, const GemmProblem& p, const BlockingFactors& b) {
  const TileGrid g = tile_grid(p, b);
  const int64_t n = rng.uniform(1, 3 * g.total_tiles + 2);
  std::vector<int64_t> cuts(static_cast<size_t>(n - 1));
  for (auto& c : cuts) c = rng.uniform(0, g.total_iters);
  std::sort(cuts.begin(), cuts.end());
  std::ostringstream text;
  text << p.m << ' ' << p.n << ' ' << p.k << '\n' << b.blk_m << ' ' << b.blk_n << ' ' << b.blk_k
       << "\nstream_k " << n << '\n';
  int64_t prev = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t e = i + 1 < n ? cuts[static_cast<size_t>(i)] : g.total_iters;
    const bool drop = rng.uniform(0, 4) == 0;
    text << i << ' ' << prev << ' ' << (drop ? prev : e) << '\n';
    prev = e;
  }
  return from_text(text.str());
}

std::string explicit_peers() {
  Rng rng(0x7ab1e5ULL);
  for (int trial = 0; trial < 500; ++trial) {
    const GemmProblem p = random_problem(rng, 300);
    const BlockingFactors b = random_blocking(rng, 40);
    const WorkAssignment a = random_table(rng, p, b);
    const sk_problem pr = streamk_b200::to_sk(a.problem);
    const sk_blocking bl = streamk_b200::to_sk(a.blocking);
    std::vector<int64_t> tbl;
    for (const CtaRange& r : a.ranges) {
      tbl.push_back(r.iter_begin);
      tbl.push_back(r.iter_end);
    }
    const auto peers = fixup_peers_of(a);
    std::vector<int64_t> off(peers.size() + 1);
    int64_t nnz = 0;
    if (sk_fixup_peers_ranges(&pr, &bl, tbl.data(), a.grid_size, off.data(), nullptr, 0, &nnz) != SK_OK)
      return "sk_fixup_peers_ranges failed";
    std::vector<int64_t> ids(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
    sk_fixup_peers_ranges(&pr, &bl, tbl.data(), a.grid_size, off.data(), ids.data(), nnz, &nnz);
    for (size_t t = 0; t < peers.size(); ++t) {
      if (static_cast<size_t>(off[t + 1] - off[t]) != peers[t].size()) return "peer count";
      for (size_t q = 0; q < peers[t].size(); ++q)
        if (ids[static_cast<size_t>(off[t]) + q] != peers[t][q]) return "peer ids";
    }
  }
  return "";
}

std::string execute_explicit() {
  Rng rng(0xe4b1c17ULL);
  for (int trial = 0; trial < 8; ++trial) {
    const GemmProblem p{rng.uniform(1, 600), rng.uniform(1, 600), rng.uniform(1, 700)};
    const BlockingFactors b = trial % 2 ? BlockingFactors{64, 64, 16} : BlockingFactors{256, 256, 64};
    const WorkAssignment a = random_table(rng, p, b);
    const auto Ai = random_matrix<std::int64_t>(p.m, p.k, 50 + trial);
    const auto Bi = random_matrix<std::int64_t>(p.k, p.n, 51 + trial);
    const auto want = execute(a, Ai, Bi, 1);
    if (trial % 2) {
      if (streamk_b200::execute(a, Ai, Bi).data != want.data) return "int64 explicit table (DMMA)";
    } else {
      Matrix<float> A(p.m, p.k), B(p.k, p.n);
      for (size_t i = 0; i < A.data.size(); ++i) A.data[i] = static_cast<float>(Ai.data[i]);
      for (size_t i = 0; i < B.data.size(); ++i) B.data[i] = static_cast<float>(Bi.data[i]);
      const auto got = streamk_b200::execute(a, A, B, streamk_b200::Precision::BF16);
      for (size_t i = 0; i < got.data.size(); ++i)
        if (got.data[i] != static_cast<float>(want.data[i])) return "bf16 explicit table (tcgen05)";
    }
  }
  return "";
}

std::string errors_map_to_reference_exceptions() {
  const GemmProblem p{64, 64, 64};
  Matrix<double> A(64, 63), B(64, 64);
  try {
    streamk_b200::execute(data_parallel(p, {64, 64, 16}), A, B);
    return "shape mismatch not rejected";
  } catch (const std::invalid_argument&) {
  }
  return "";
}

}  // namespace

int main(int argc, char** argv) {
  const bool sched = argc < 2 || !std::strcmp(argv[1], "--schedule");
  const bool exec = argc >= 2 && !std::strcmp(argv[1], "--execute");
  if (sched) {
    report("sk_schedule / sk_fixup_peers == decompose.cpp (3000 instances x 5 strategies)",
           schedule_parity());
    report("shape errors -> std::invalid_argument", errors_map_to_reference_exceptions());
    report("sk_fixup_peers_ranges == fixup_peers_of on from_text tables (500)", explicit_peers());
  }
  if (exec) {
    report("execute<int64_t>: bit-exact vs naive and streamk::execute (60 instances x 5)",
           execute_int64());
    report("execute<float>/<double> under 8 eps k; bf16 path exact on the int band",
           execute_float_double());
    report("execute on from_text tables (SK_EXPLICIT) == streamk::execute, bit-exact (8)",
           execute_explicit());
  }
  return failures ? 1 : 0;
}
