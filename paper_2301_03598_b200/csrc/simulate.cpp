// simulate.cpp -- the reference's idealised list-scheduling simulator, fed
// with the closed-form schedules (schedule.hpp) and optionally with cost
// constants calibrated from this kernel's device timelines.
//
// Restates simulate (core/src/simulate.cpp:23-69) and utilization (:71-80):
// units are dispatched in cta_id order, each to the earliest-free of p cores
// (lowest index on ties).  Unit cost: a MAC event lasts one time unit per
// iteration and fixups are free.  With params {a, b, c, d} (costmodel.hpp:13-19
// CostParams): a nonempty unit's MAC event lasts a + c * len (+ b when its
// range starts mid-tile, i.e. it emits a partial), and a tile owner appends a
// fixup_reduce event of d per peer it folds (fixup_peers_of, decompose.cpp:
// 123-136).  utilization = sum of MAC durations / (p * makespan), summed in
// event order like the reference, so the sweep CSV's utilization/makespan
// columns are byte-identical to run_sweep's (sweep.cpp:88-108).
#include <algorithm>
#include <vector>

#include "../../include/skb200.h"
#include "schedule.hpp"

using skb200::Schedule;

extern "C" sk_status sk_simulate(const sk_problem* problem, const sk_blocking* blocking,
                                 sk_strategy strategy, int64_t param, const int64_t* ranges,
                                 int64_t num_ranges, int64_t p, const sk_sim_params* params,
                                 double* makespan, double* utilization, double* events,
                                 int64_t capacity, int64_t* num_events) {
  if (!problem || !blocking) return SK_EINVAL;
  if (p < 1) return SK_EINVAL;  // "simulate: p must be >= 1"
  Schedule s;
  std::vector<int64_t> tbl;
  if (strategy == SK_EXPLICIT) {
    if (s.init_explicit(problem->m, problem->n, problem->k, blocking->blk_m, blocking->blk_n,
                        blocking->blk_k, num_ranges) != 0 || num_ranges < 0 || (num_ranges > 0 && !ranges))
      return SK_EINVAL;
    tbl.assign(ranges, ranges + 2 * num_ranges);
    for (int64_t u = 0; u < num_ranges; ++u)
      if (tbl[2 * u] < 0 || tbl[2 * u + 1] < tbl[2 * u] || tbl[2 * u + 1] > s.total_iters) return SK_EINVAL;
  } else {
    if (s.init(problem->m, problem->n, problem->k, blocking->blk_m, blocking->blk_n, blocking->blk_k,
               strategy, param) != 0)
      return SK_EINVAL;
    tbl.resize(static_cast<size_t>(2 * s.grid_size));
    for (int64_t u = 0; u < s.grid_size; ++u) s.range(u, &tbl[2 * u], &tbl[2 * u + 1]);
  }
  const int64_t g = static_cast<int64_t>(tbl.size() / 2), ipt = s.ipt;
  // Partials each tile owner folds in (fixup_peers_of: nonempty ranges
  // intersecting the tile, ascending id; the front is the owner).
  std::vector<int64_t> reduce_count(static_cast<size_t>(g), 0);
  {
    std::vector<int64_t> first(static_cast<size_t>(s.total_tiles), -1), cnt(static_cast<size_t>(s.total_tiles), 0);
    for (int64_t u = 0; u < g; ++u) {
      const int64_t b = tbl[2 * u], e = tbl[2 * u + 1];
      if (b == e) continue;
      for (int64_t t = b / ipt; t <= (e - 1) / ipt; ++t) {
        if (first[static_cast<size_t>(t)] < 0) first[static_cast<size_t>(t)] = u;
        ++cnt[static_cast<size_t>(t)];
      }
    }
    for (int64_t t = 0; t < s.total_tiles; ++t)
      if (cnt[static_cast<size_t>(t)] > 1) reduce_count[static_cast<size_t>(first[static_cast<size_t>(t)])] += cnt[static_cast<size_t>(t)] - 1;
  }
  std::vector<double> free_at(static_cast<size_t>(p), 0.0);
  double span = 0.0, mac_total = 0.0;
  int64_t nev = 0;
  auto emit = [&](int64_t core, int64_t cta, int kind, double st, double en, int64_t tile) {
    if (events && nev < capacity) {
      double* r = events + 6 * nev;
      r[0] = static_cast<double>(core), r[1] = static_cast<double>(cta), r[2] = kind;
      r[3] = st, r[4] = en, r[5] = static_cast<double>(tile);
    }
    ++nev;
  };
  for (int64_t u = 0; u < g; ++u) {
    size_t core = 0;
    for (size_t i = 1; i < free_at.size(); ++i)
      if (free_at[i] < free_at[core]) core = i;
    const int64_t b = tbl[2 * u], e = tbl[2 * u + 1];
    const bool empty = b == e;
    const double len = static_cast<double>(e - b);
    const bool emits_partial = !empty && (b % ipt) != 0;
    double mac_dur = len;
    if (params && !empty) mac_dur = params->a + params->c * len + (emits_partial ? params->b : 0.0);
    const double start = free_at[core];
    const int64_t tile = empty ? 0 : b / ipt;
    emit(static_cast<int64_t>(core), u, 0, start, start + mac_dur, tile);
    mac_total += (start + mac_dur) - start;  // utilization sums end - start per event
    double cursor = start + mac_dur;
    const int64_t reductions = reduce_count[static_cast<size_t>(u)];
    if (params && reductions > 0) {
      const double dur = params->d * static_cast<double>(reductions);
      emit(static_cast<int64_t>(core), u, 2, cursor, cursor + dur, tile);
      cursor += dur;
    }
    free_at[core] = cursor;
    span = std::max(span, cursor);
  }
  if (makespan) *makespan = span;
  if (num_events) *num_events = nev;
  if (utilization) {
    if (nev == 0 || span <= 0.0) {
      *utilization = 0.0;
      return SK_EINVAL;
    }
    *utilization = mac_total / (static_cast<double>(p) * span);
  }
  if (events && nev > capacity) return SK_ECAPACITY;
  return SK_OK;
}
