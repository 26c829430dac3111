// sk_kernel_common.cuh -- shared between the tcgen05 (BF16/FP16) and DMMA (FP64)
// Stream-K kernels: kernel parameter block, the persistent unit iterator, and
// the fixup flag protocol (executor.hpp:95-119 FixupStore, on the GPU).
#pragma once

#include <stdint.h>

#include "ptx.cuh"
#include "schedule.hpp"

namespace skb200 {

// Workspace layout (bytes):
//   [0, 256)                   header: int err word (+ reserved)
//   [256, 256 + flag_bytes)    int32 flags, one per (slab, cta rank), zero between launches
//   [partials_off, ...)        fixup slabs: num_slabs * ranks * slab_elems accumulators
struct WorkspaceLayout {
  size_t flags_off = 256, flag_bytes = 0, partials_off = 0, total = 0;
  static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
  void compute(int64_t num_slabs, int ranks, size_t slab_bytes) {
    flags_off = 256;
    flag_bytes = align256(sizeof(int) * static_cast<size_t>(num_slabs * ranks + 1));
    partials_off = flags_off + flag_bytes;
    total = partials_off + static_cast<size_t>(num_slabs * ranks) * slab_bytes;
  }
};

// Error word bits.
enum : int { kErrDoubleSignal = 1, kErrWatchdog = 1 << 16 };

// Trace layout (ints): per tile {owner, last_peer, storing_unit, segments_folded},
// then per unit {partials_emitted}.
struct KernelParams {
  Schedule s;
  int64_t num_ctas;  // persistent CTAs (pairs for the 2-SM kernel)
  uint32_t idesc;    // tcgen05 instruction descriptor (16-bit kernels)
  int32_t ranks;     // CTAs per logical CTA (1 or 2)
  void* partials;
  int* flags;
  int* err;
  int* trace;
  int64_t watchdog_ns;
};

// The persistent schedule: physical CTA `cta` of `P` runs logical CTAs
// g-1-cta, g-1-cta-P, ... (descending, like executor.hpp:187-193), and inside
// each logical CTA its tile segments in ascending iteration order
// (executor.hpp:149-185).  Every wait targets a strictly higher logical id and
// every CTA's pending ids are lower than its current one, so with all P CTAs
// co-resident the highest in-flight id never waits on unfinished work.
template <class F>
__device__ __forceinline__ void for_each_segment(const Schedule& s, int64_t cta, int64_t P,
                                                 F&& f) {
  for (int64_t u = s.grid_size - 1 - cta; u >= 0; u -= P) {
    int64_t b, e;
    s.range(u, &b, &e);
    int64_t it = b;
    while (it < e) {
      const int64_t tile = it / s.ipt;
      const int64_t tb = tile * s.ipt;
      const int64_t lb = it - tb;
      const int64_t le = imin(e, tb + s.ipt) - tb;
      f(u, tile, lb, le);
      it = tb + s.ipt;
    }
  }
}

// Owner-side wait for one peer flag (FixupStore::wait, executor.hpp:114-118),
// bounded by a watchdog so a protocol bug can never hang the GPU.
__device__ __forceinline__ void wait_flag(const KernelParams& P, const int* flag) {
  if (ptx::ld_acquire(flag) != 0) return;
  const uint64_t t0 = ptx::globaltimer();
  uint32_t backoff = 32;
  while (ptx::ld_acquire(flag) == 0) {
    __nanosleep(backoff);
    if (backoff < 256) backoff <<= 1;
    if (ptx::ld_acquire(P.err) & kErrWatchdog) return;
    if (ptx::globaltimer() - t0 > static_cast<uint64_t>(P.watchdog_ns)) {
      atomicOr(P.err, kErrWatchdog);
      return;
    }
  }
}

// Non-owner signal (FixupStore::signal, executor.hpp:106-112): release after
// the whole slab is written; a nonzero previous value is a double signal.
__device__ __forceinline__ void signal_flag(const KernelParams& P, int* flag) {
  __threadfence();
  const int old = atomicExch(flag, 1);
  if (old != 0) atomicOr(P.err, kErrDoubleSignal);
}

}  // namespace skb200
