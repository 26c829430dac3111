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
//   [table_off, total)         explicit schedules only: ranges, peer offsets, peer ids (int64)
//
// Cooperative fixup (KernelParams::coop, balanced strategies on the 16-bit
// kernels): every balanced unit may publish two slabs, its first segment's
// partial (slab/flag index slab_of(u) * ranks + rank, as in the owner-fold
// protocol) and, as a tile owner, its last segment's accumulator (index
// num_slabs * ranks + the same); then one done counter per (balanced-region
// tile, rank) at flag index 2 * num_slabs * ranks + (tile - first tile) * ranks + rank.
struct WorkspaceLayout {
  size_t flags_off = 256, flag_bytes = 0, partials_off = 0, table_off = 0, total = 0;
  static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
  void compute(int64_t num_slabs, int ranks, size_t slab_bytes, size_t table_bytes = 0,
               int64_t coop_tiles = -1) {
    const int64_t extra = coop_tiles >= 0 ? num_slabs * ranks + coop_tiles * ranks : 0;
    if (coop_tiles >= 0) num_slabs *= 2;
    flags_off = 256;
    flag_bytes = align256(sizeof(int) * static_cast<size_t>(num_slabs * ranks + extra + 1));
    partials_off = flags_off + flag_bytes;
    table_off = align256(partials_off + static_cast<size_t>(num_slabs * ranks) * slab_bytes);
    total = table_bytes ? table_off + table_bytes
                        : partials_off + static_cast<size_t>(num_slabs * ranks) * slab_bytes;
  }
};

// c_done counter of tile (tr, tc) under the pipelining block geometry.
#define SK_CDONE_INDEX(P, tr, tc) ((tr) / (P).pipe_g * (P).pipe_np + (tc) / (P).pipe_w)

// Error word bits.
enum : int { kErrDoubleSignal = 1, kErrWatchdog = 1 << 16, kErrTopology = 1 << 17 };

// Trace layout (ints): per tile {owner, last_peer, storing_unit, segments_folded},
// then per unit {partials_emitted}.
constexpr int kMaxSms = 192;

struct KernelParams {
  Schedule s;
  int64_t num_ctas;  // persistent CTAs (pairs for the 2-SM kernel)
  uint32_t idesc;    // tcgen05 instruction descriptor (16-bit kernels)
  int32_t ranks;     // CTAs per logical CTA (1 or 2)
  void* partials;
  int* flags;
  int* err;
  int* trace;
  long long* cta_clocks;  // optional: per CTA {clock64, globaltimer} at start and end
  long long* events;      // optional timeline: 8 int64 per (unit, segment), see event_slot
  int64_t seg_stride;     // max tile segments of one unit (timeline indexing)
  int64_t watchdog_ns;
  int64_t raster_rows;  // data-parallel tile-row group height (1 = row-major)
  int32_t sk_first;      // TwoTileSkDp phase order: kDpFirst, kSkFirst, kInterleaved
  // Transfer pipelining (sk_execute with pinned host buffers; NULL otherwise):
  // a_ready[tile row] turns nonzero once that row block of A has landed (the
  // producer waits before its first load of the row); c_done[tile row] counts
  // the row's finished C stores (one per storing epilogue warp) so the copy-out
  // stream can start on the row before the kernel ends.
  const int* a_ready;
  int* c_done;
  // Tile-block pipelining (16-bit kernels): B also arrives by panels of pipe_w
  // tile columns (b_ready[panel], NULL = B already complete), and c_done counts
  // per block of pipe_g tile rows x pipe_w tile columns (pipe_np panels per row
  // of blocks); the per-row scheme is pipe_g = 1, pipe_w = tiles_n.
  const int* b_ready;
  int32_t pipe_g, pipe_w, pipe_np;
  const int32_t* dp_perm;  // pipelined: data-parallel slot -> tile order (NULL = raster)
  int32_t k_align;  // balanced units: aligned k order (k_block_of), 0 = ascending
  int32_t l2_policy[4];  // L2 eviction priority for A loads, B loads (data-parallel
                         // units), C stores, B loads (Stream-K / fixed-split units):
                         // 0 normal, 1 evict_first, 2 evict_last
  // Die-aware data-parallel phase (see dp_lane): B200 is two dies, each with
  // half of the SMs and its own L2; die_tab[smid] = die << 8 | rank of the
  // persistent CTA (pair) among those of its die, -1 unknown.  die_n = CTAs
  // (pairs) per die.  Only set for a full persistent grid on a probed device.
  int32_t die_aware;
  // Cooperative fixup: each balanced unit runs alone on its CTA (all of them
  // co-resident), so every contributor of a shared tile publishes its
  // accumulator and then folds 1/ncontrib of the tile's columns from all
  // slabs in the reference's order (owner first, peers ascending), instead of
  // the owner folding every peer slab alone (per-SM bandwidth-bound).
  int32_t coop;
  // Cluster fixup (1-SM kernel, fixed_split(s) with s | ipt, one unit per CTA):
  // the s CTAs of a cluster are the s k-chunks of one tile and reduce through
  // distributed shared memory instead of global slabs; 0 = off.
  int32_t cluster_fix;
  int32_t die_n[2];
  int16_t die_tab[kMaxSms];
};

// The data-parallel slots [first, end) with stride `step` that one persistent
// CTA walks (in the rasterised order).  Default: slot cta, cta + P, ...
struct DpLane {
  int64_t first, step, end;
};
SK_HD DpLane default_lane(const Schedule& s, int64_t cta, int64_t P) {
  return DpLane{cta, P, s.dp_tiles};
}
// Die-aware lane: the rasterised DP order is cut in two contiguous ranges,
// sized by the dies' CTA counts; the CTAs of die d stride through range d only.
// Each die's L2 then holds its own A panels and one compact wave of B panels
// instead of both dies caching (and missing on) the union: measured on 8192^3
// (profiles/r01/die_aware.txt).  `code` = die << 8 | rank from die_tab.
SK_HD DpLane die_lane(const Schedule& s, const int32_t* die_n, int code) {
  const int d = (code >> 8) & 1, r = code & 0xff;
  const int64_t P = die_n[0] + die_n[1];
  const int64_t t0 = (s.dp_tiles * die_n[0] + P / 2) / P;
  return d == 0 ? DpLane{r, die_n[0], t0} : DpLane{t0 + r, die_n[1], s.dp_tiles};
}

// Data-parallel slot i -> tile, a bijection on [0, dp_tiles): whole tile rows
// are visited in groups of `rows` rows, column-major inside a group, so one
// wave of persistent CTAs covers a compact rows x (P / rows) block whose A and
// B panels stay L2-resident; the trailing partial row is visited in order.
// Only the temporal order changes: unit <-> range <-> tile stays the
// reference's (decompose.cpp:42-46), so schedule parity is unaffected.
SK_HD int64_t raster_tile(const Schedule& s, int64_t i, int64_t rows) {
  const int64_t full_rows = s.dp_tiles / s.tiles_n;
  if (rows <= 1 || i >= full_rows * s.tiles_n) return i;
  const int64_t group = rows * s.tiles_n;
  const int64_t gi = i / group, within = i - gi * group;
  const int64_t h = imin(rows, full_rows - gi * rows);
  const int64_t col = within / h, row = gi * rows + (within - col * h);
  return row * s.tiles_n + col;
}

// The persistent schedule (host-callable too: sk_execute predicts the order in
// which tile rows of C complete from it).  Dependencies only run from a tile's owner to
// strictly higher ids inside the balanced (Stream-K) region or inside a
// fixed-split tile; data-parallel units never wait and are never waited on.
//   * data-parallel units: physical CTA `cta` of `P` takes slots cta, cta+P, ...
//     of the rasterised order above;
//   * balanced / fixed-split units: ids hi-1-cta, hi-1-cta-P, ... descending,
//     like the reference's dispatch (executor.hpp:187-193).  Every CTA's pending
//     ids are lower than its current one and every wait targets a higher id, so
//     with all P CTAs co-resident the highest in-flight id never waits on
//     unfinished work (executor.hpp:124-129).
// The phases run in descending-id order of the reference (DP ids above the SK
// ids for TwoTileSkDp, below for DpOneTileSk).  Inside a unit, segments run in
// ascending iteration order (executor.hpp:149-185).  Producer, MMA and epilogue
// roles all walk this same sequence.
// Phase orders for TwoTileSkDp (KernelParams::sk_first):
enum : int { kDpFirst = 0, kSkFirst = 1, kInterleaved = 2 };

// The persistent CTA's segment sequence as an explicit iterator, so each role
// (producer, MMA issuer, epilogue) has ONE copy of its per-segment body:
//   SegmentIter it(s, cta, P, lane, raster_rows, order);
//   int64_t u, tile, lb, le;
//   while (it.next(s, &u, &tile, &lb, &le)) { ... }
// Phases: up to two of {data-parallel slots of `lane` in the rasterised order,
// balanced / fixed-split ids descending from hi - 1 - cta by P}; kInterleaved
// puts the CTA's single balanced unit after `slot` of its data-parallel tiles.
// The schedule is passed to every call rather than stored (a stored pointer to
// the kernel parameter block would force a local-memory copy of it).
struct SegmentIter {
  enum : int { kNone = 0, kDp = 1, kDesc = 2 };
  int64_t cta, P, raster;
  DpLane lane;
  int ph = 0, nph = 0;
  int kind0 = kNone, kind1 = kNone;
  int64_t lo = 0, hi = 0;     // kDesc id range
  int64_t i = 0;              // current DP slot / descending id
  bool fresh = true;          // phase not started yet
  int64_t ins_unit = -1, ins_slot = -1, j = 0;  // kInterleaved: unit, slot, DP tiles so far
  int64_t u = 0, it = 0, e = 0;
  const int32_t* perm = nullptr;  // optional DP slot -> tile permutation (pipelined execute)

  SK_HD SegmentIter(const Schedule& s, int64_t cta_, int64_t P_, const DpLane& lane_,
                    int64_t raster_, int order, const int32_t* perm_ = nullptr)
      : cta(cta_), P(P_), raster(raster_), lane(lane_), perm(perm_) {
    const bool two_tile_dp_first = s.dp_id0 > s.bal.first_id;
    if (s.strategy == kFixedSplit || s.strategy == kExplicit) {
      kind0 = kDesc, nph = 1, lo = 0, hi = s.grid_size;
    } else if (s.bal.count == 0) {
      kind0 = kDp, nph = 1;
    } else {
      lo = s.bal.first_id, hi = s.bal.first_id + s.bal.count;
      if (two_tile_dp_first && order == kInterleaved && s.bal.count <= P_) {
        // TwoTileSkDp with at most one balanced unit per CTA, staggered through
        // the data-parallel waves: unit hi-1-cta runs after `slot` of this CTA's
        // DP tiles, slot rising with cta, so a tile's peers (higher ids = lower
        // cta) never run later than its owner.
        kind0 = kDp, nph = 1;
        const int64_t uu = hi - 1 - cta_;
        const int64_t waves = (s.dp_tiles + P_ - 1) / P_;
        if (uu >= lo) ins_unit = uu, ins_slot = cta_ * (waves + 1) / P_;
      } else if (two_tile_dp_first && order == kDpFirst) {  // DP waves, then the SK region
        kind0 = kDp, kind1 = kDesc, nph = 2;
      } else {  // StreamK, DpOneTileSk, TwoTileSkDp SK-first (Fig. 4c)
        kind0 = kDesc, kind1 = kDp, nph = 2;
      }
    }
  }

  // Next unit of the sequence into (u, it, e); false when exhausted.
  SK_HD bool next_unit(const Schedule& s) {
    while (ph < nph) {
      if ((ph == 0 ? kind0 : kind1) == kDp) {
        if (ins_unit >= 0 && j == ins_slot) {  // interleaved balanced unit, before DP tile j
          const int64_t uu = ins_unit;
          ins_unit = -1;
          return load(s, uu);
        }
        i = fresh ? lane.first : i + lane.step;
        fresh = false;
        if (i < lane.end) {
          ++j;
          return load(s, s.dp_id0 + (perm ? perm[i] : raster_tile(s, i, raster)));
        }
        if (ins_unit >= 0) {  // its slot lies past this CTA's last DP tile
          const int64_t uu = ins_unit;
          ins_unit = -1;
          return load(s, uu);
        }
      } else {
        i = fresh ? hi - 1 - cta : i - P;
        fresh = false;
        if (i >= lo) return load(s, i);
      }
      ++ph;
      fresh = true;
    }
    return false;
  }
  SK_HD bool load(const Schedule& s, int64_t unit) {
    u = unit;
    s.range(unit, &it, &e);
    return true;
  }
  // Next tile segment: unit u, tile, local iterations [lb, le) (executor.hpp:149-185).
  SK_HD bool next(const Schedule& s, int64_t* uo, int64_t* tile, int64_t* lb, int64_t* le) {
    while (it >= e)
      if (!next_unit(s)) return false;
#if defined(__CUDA_ARCH__)  // ids and iterations < 2^31 on the device: 32-bit divide
    const int64_t t = static_cast<uint32_t>(it) / static_cast<uint32_t>(s.ipt);
#else
    const int64_t t = it / s.ipt;
#endif
    const int64_t tb = t * s.ipt;
    *uo = u;
    *tile = t;
    *lb = it - tb;
    *le = imin(e, tb + s.ipt) - tb;
    it = tb + s.ipt;
    return true;
  }
};

#pragma nv_exec_check_disable
template <class F>
SK_HD void for_each_segment(const Schedule& s, int64_t cta, int64_t P, const DpLane& lane,
                            int64_t raster_rows, F&& f, int order = kDpFirst,
                            const int32_t* perm = nullptr) {
  SegmentIter sit(s, cta, P, lane, raster_rows, order, perm);
  int64_t u, tile, lb, le;
  while (sit.next(s, &u, &tile, &lb, &le)) f(u, tile, lb, le);
}

#pragma nv_exec_check_disable
template <class F>
SK_HD void for_each_segment(const Schedule& s, int64_t cta, int64_t P, int64_t raster_rows, F&& f,
                            int order = kDpFirst, const int32_t* perm = nullptr) {
  for_each_segment(s, cta, P, default_lane(s, cta, P), raster_rows, static_cast<F&&>(f), order, perm);
}

// k-block order inside a balanced unit's tile segment (the set of k-blocks is
// the reference's; only the order in which they are multiplied changes, which
// keeps integer-valued results exact and every result deterministic).  All
// balanced units start together and run at the same rate, so a unit-local clock
// tau (iterations since the unit began) is a common clock.  Walking a segment
// that starts mid-tile, [lb, ipt), DOWNWARD reads k-block ipt - 1 - tau at time
// tau in every unit, and walking the unit's last segment, [0, le), downward
// reads (L - 1 - tau) mod ipt (L = unit length); a full middle tile is rotated
// onto that same phase.  Readers of one B column panel then meet on (at most
// two phases of) the same k-block at the same time instead of at unrelated
// offsets, so the panel is fetched from HBM once per phase, not once per tile.
SK_HD int64_t k_rotation(const Schedule& s, int64_t b, int64_t e, int64_t tile, int64_t lb,
                         int64_t le) {
  if (le - lb < s.ipt) return 0;  // partial or last segment: plain descending
  const int64_t t0 = tile * s.ipt - b;  // unit-local time this full segment starts
  const int64_t r = (e - b - 1 - t0) % s.ipt;
  return r < 0 ? r + s.ipt : r;
}
SK_HD int64_t k_block_of(int64_t ipt, int64_t lb, int64_t le, int64_t rot, int64_t i) {
  if (le - lb < ipt) return le - 1 - i;
  const int64_t k = rot - i;
  return k < 0 ? k + ipt : k;
}

// Per-CTA clock stamps (sk_gemm_desc.cta_clocks): the effective SM clock of a
// launch is (clock64 end - start) / (globaltimer end - start).
__device__ __forceinline__ void stamp_clock(const KernelParams& P, int slot) {
  if (P.cta_clocks && threadIdx.x == 0) {
    long long* c = P.cta_clocks + 4 * blockIdx.x + 2 * slot;
    c[0] = static_cast<long long>(clock64());
    c[1] = static_cast<long long>(ptx::globaltimer());
  }
}

// Device timeline (sk_gemm_desc.events): one record per (unit, tile segment)
//   {unit, tile, core, kind, t_mac_start, t_mac_end, t_wait_end, t_done}
// with kind = 1 partial | 2 owner-with-peers | npeer << 8 | smid << 16, times in
// globaltimer ns.
// Rendered as the reference's timeline CSV / Gantt (simulate.cpp:105-168).
enum { kEvUnit = 0, kEvTile, kEvCore, kEvKind, kEvMacStart, kEvMacEnd, kEvWaitEnd, kEvDone };
__device__ __forceinline__ long long* event_slot(const KernelParams& P, int64_t u, int64_t tile) {
  if (!P.events) return nullptr;
  int64_t b, e;
  P.s.range(u, &b, &e);
  return P.events + 8 * (u * P.seg_stride + (tile - b / P.s.ipt));
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
