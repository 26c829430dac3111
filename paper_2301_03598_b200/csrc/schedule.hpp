// schedule.hpp -- closed-form Stream-K schedules, usable on host and device.
//
// Bit-exact restatement of the reference decompositions
// (/root/reference/proj/core/src/decompose.cpp) without materialising the
// range table: every logical CTA ("unit") computes its own [begin, end) and
// every tile its owner and last peer in O(1).
//
//   tile_grid                types.cpp:45-55
//   balanced_ranges          decompose.cpp:13-24     -> Region::range / Region::unit_of
//   data_parallel            decompose.cpp:38-48
//   fixed_split              decompose.cpp:50-69
//   stream_k                 decompose.cpp:71-79
//   hybrid (both variants)   decompose.cpp:81-121
//   fixup_peers_of           decompose.cpp:123-136   -> Schedule::peers (contiguous id interval)
//
// Every strategy is "a data-parallel region + one balanced region" (or fixed
// split):
//   DP            dp ids [0,t)            <-> tiles [0,t)
//   SK(g)         balanced ids [0,g)      over iters [0, T)
//   DpOneTileSk   dp ids [0,D) <-> tiles [0,D);   balanced ids [D, D+p) over [D*ipt, T)
//   TwoTileSkDp   balanced ids [0,p) over [D*ipt, T);  dp ids [p, p+D) <-> tiles [0,D)
//   FS(s)         unit x*s+y  = [x*ipt + min(ipt, y*ips), x*ipt + min(ipt, lo+ips))
// Peers of any tile are a contiguous id interval [owner, last] (checked
// exhaustively against fixup_peers_of by tests/test_schedule.py).
//
// kExplicit carries an arbitrary range table instead (a WorkAssignment that no
// closed form produces, e.g. one read back by from_text, types.cpp:109-123):
// ranges [g][2] and the fixup_peers_of lists in CSR form, validated on the host
// (one starter per tile at most; a starter's peers all have higher ids).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define SK_HD __host__ __device__ __forceinline__
#else
#define SK_HD inline
#endif

namespace skb200 {

enum Strategy : int32_t {
  kDataParallel = 0,
  kFixedSplit = 1,
  kStreamK = 2,
  kDpOneTileSk = 3,
  kTwoTileSkDp = 4,
  kExplicit = 5  // range table (not a reference Strategy value; see above)
};

SK_HD int64_t ceil_div(int64_t x, int64_t y) { return (x + y - 1) / y; }
SK_HD int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

// balanced_ranges(begin, end, count, first_id) in closed form.
struct Region {
  int64_t first_id = 0, count = 0, begin = 0, end = 0, q = 0, r = 0;

  SK_HD void set(int64_t first, int64_t cnt, int64_t b, int64_t e) {
    first_id = first;
    count = cnt;
    begin = b;
    end = e;
    q = cnt > 0 ? (e - b) / cnt : 0;
    r = cnt > 0 ? (e - b) % cnt : 0;
  }
  SK_HD bool contains_id(int64_t u) const { return u >= first_id && u < first_id + count; }
  // decompose.cpp:18-22: len_i = q + (i < r), larger shares first.
  SK_HD void range(int64_t u, int64_t* b, int64_t* e) const {
    const int64_t i = u - first_id;
    *b = begin + i * q + imin(i, r);
    *e = *b + q + (i < r ? 1 : 0);
  }
  // Inverse: id of the (nonempty) range holding iteration j in [begin, end).
  SK_HD int64_t unit_of(int64_t j) const {
    const int64_t d = j - begin;
    const int64_t big = r * (q + 1);
#if defined(__CUDA_ARCH__)  // < 2^31 on the device (see Schedule::tile_rc)
    const uint32_t d32 = static_cast<uint32_t>(d), big32 = static_cast<uint32_t>(big);
    const uint32_t q32 = static_cast<uint32_t>(q);
    return first_id + (d32 < big32 ? d32 / (q32 + 1) : static_cast<uint32_t>(r) + (d32 - big32) / q32);
#else
    return first_id + (d < big ? d / (q + 1) : r + (d - big) / q);
#endif
  }
};

struct Schedule {
  // tile grid (types.cpp:45-55)
  int64_t m = 0, n = 0, k = 0;
  int64_t blk_m = 1, blk_n = 1, blk_k = 1;
  int64_t tiles_m = 0, tiles_n = 0, total_tiles = 0, ipt = 0, total_iters = 0;
  // decomposition
  int32_t strategy = kDataParallel;
  int64_t param = 1;
  int64_t grid_size = 0;  // g: number of logical CTAs
  // data-parallel region: ids [dp_id0, dp_id0 + dp_tiles) <-> tiles [0, dp_tiles)
  int64_t dp_id0 = 0, dp_tiles = 0;
  // balanced region (stream_k / hybrid SK part)
  Region bal;
  // fixed split
  int64_t split = 1, ips = 1;
  // fixup slabs: which units emit a partial, compact slab index
  int64_t num_slabs = 0;
  // Tile id -> C block (tile_rc).  1: row-major, the reference's
  // executor.hpp:69-70.  G > 1: ids run through groups of G tile rows,
  // column-major inside a group (the last group may be shorter), so every
  // contiguous id range -- a wave of data-parallel tiles, a hybrid's trailing
  // Stream-K region -- covers a compact block of C.  Ids, ranges, owners and
  // peers are untouched; only which block of C an id denotes changes.
  int64_t tile_group = 1;
  // kExplicit: [g][2] ranges and per-tile ascending peer ids (CSR); the first
  // peer of a tile is its starter when that range covers local k = 0.
  const int64_t* xr = nullptr;
  const int64_t* xoff = nullptr;
  const int64_t* xids = nullptr;

  SK_HD int init_explicit(int64_t m_, int64_t n_, int64_t k_, int64_t bm, int64_t bn, int64_t bk,
                          int64_t g) {
    if (init(m_, n_, k_, bm, bn, bk, kDataParallel, 1) != 0) return 1;
    strategy = kExplicit;
    param = g;
    grid_size = g;
    dp_tiles = 0;
    num_slabs = g;  // slab = unit id (a unit emits at most its first segment)
    return 0;
  }

  // Returns 0 on success, 1 (EINVAL) on a non-positive extent or parameter.
  SK_HD int init(int64_t m_, int64_t n_, int64_t k_, int64_t bm, int64_t bn, int64_t bk,
                 int32_t strat, int64_t prm) {
    if (m_ < 1 || n_ < 1 || k_ < 1 || bm < 1 || bn < 1 || bk < 1) return 1;  // types.cpp:33-43
    m = m_;
    n = n_;
    k = k_;
    blk_m = bm;
    blk_n = bn;
    blk_k = bk;
    tiles_m = ceil_div(m, bm);
    tiles_n = ceil_div(n, bn);
    total_tiles = tiles_m * tiles_n;
    ipt = ceil_div(k, bk);
    total_iters = total_tiles * ipt;
    strategy = strat;
    param = prm;
    dp_id0 = 0;
    dp_tiles = 0;
    bal.set(0, 0, 0, 0);
    split = 1;
    ips = ipt;
    num_slabs = 0;
    switch (strat) {
      case kDataParallel:  // decompose.cpp:38-48
        grid_size = total_tiles;
        dp_tiles = total_tiles;
        return 0;
      case kFixedSplit:  // decompose.cpp:50-69
        if (prm < 1) return 1;
        split = prm;
        ips = ceil_div(ipt, split);
        grid_size = total_tiles * split;
        // chunks y >= 1 start mid-tile; nonempty iff y * ips < ipt
        num_slabs = total_tiles * (split - 1);
        return 0;
      case kStreamK:  // decompose.cpp:71-79
        if (prm < 1) return 1;
        grid_size = prm;
        bal.set(0, prm, 0, total_iters);
        num_slabs = prm;
        return 0;
      case kDpOneTileSk:
      case kTwoTileSkDp: {  // decompose.cpp:81-121
        if (prm < 1) return 1;
        const int64_t p = prm, w = total_tiles / p, rem = total_tiles % p;
        if (rem == 0) {  // :92-97
          grid_size = total_tiles;
          dp_tiles = total_tiles;
          return 0;
        }
        const int64_t d = (strat == kDpOneTileSk) ? w * p : (w >= 2 ? (w - 1) * p : 0);
        grid_size = d + p;
        dp_tiles = d;
        if (strat == kDpOneTileSk) {
          dp_id0 = 0;
          bal.set(d, p, d * ipt, total_iters);
        } else {
          bal.set(0, p, d * ipt, total_iters);
          dp_id0 = p;
        }
        num_slabs = p;
        return 0;
      }
      default:
        return 1;
    }
  }

  // On the device every id and iteration is < 2^31 (sk_gemm rejects larger
  // problems), so the divisions run in 32 bits: a 64-bit division is a
  // ~100-instruction routine on the per-segment critical path.
  SK_HD void tile_rc(int64_t tile, int64_t* r, int64_t* c) const {
#if defined(__CUDA_ARCH__)
    const uint32_t t = static_cast<uint32_t>(tile), tn = static_cast<uint32_t>(tiles_n);
    if (tile_group <= 1) {
      const uint32_t q = t / tn;
      *r = q;
      *c = t - q * tn;
      return;
    }
    const uint32_t G = static_cast<uint32_t>(tile_group), span = G * tn;
    const uint32_t g = t / span, w = t - g * span;
    const uint32_t h = min(G, static_cast<uint32_t>(tiles_m) - g * G);
    const uint32_t cc = w / h;
    *c = cc;
    *r = g * G + (w - cc * h);
#else
    if (tile_group <= 1) {
      *r = tile / tiles_n;
      *c = tile % tiles_n;
      return;
    }
    const int64_t span = tile_group * tiles_n;
    const int64_t g = tile / span, w = tile - g * span;
    const int64_t h = imin(tile_group, tiles_m - g * tile_group);
    *c = w / h;
    *r = g * tile_group + (w - *c * h);
#endif
  }

  // Range of logical CTA u in [0, grid_size).
  SK_HD void range(int64_t u, int64_t* b, int64_t* e) const {
    if (strategy == kExplicit) {
      *b = xr[2 * u];
      *e = xr[2 * u + 1];
      return;
    }
    if (strategy == kFixedSplit) {
      const int64_t x = u / split, y = u % split;
      const int64_t lo = imin(ipt, y * ips);
      *b = x * ipt + lo;
      *e = x * ipt + imin(ipt, lo + ips);
      return;
    }
    if (bal.contains_id(u)) {
      bal.range(u, b, e);
      return;
    }
    const int64_t x = u - dp_id0;  // data-parallel unit
    *b = x * ipt;
    *e = (x + 1) * ipt;
  }

  // Peers of `tile` (fixup_peers_of, decompose.cpp:123-136): the contiguous id
  // interval [owner, last].  owner covers local k = 0.
  SK_HD void peers(int64_t tile, int64_t* owner, int64_t* last) const {
    if (strategy == kFixedSplit) {
      *owner = tile * split;
      *last = tile * split + ceil_div(ipt, ips) - 1;
      return;
    }
    if (tile < dp_tiles) {
      *owner = *last = dp_id0 + tile;
      return;
    }
    *owner = bal.unit_of(tile * ipt);
    *last = bal.unit_of((tile + 1) * ipt - 1);
  }

  // Number of peers an owner u of `tile` folds (its covering ranges other than
  // itself) and the i-th of them, i in [1, npeer], ascending id.
  SK_HD int npeers(int64_t tile, int64_t u) const {
    if (strategy == kExplicit) return static_cast<int>(xoff[tile + 1] - xoff[tile] - 1);
    int64_t owner, last;
    peers(tile, &owner, &last);
    return static_cast<int>(last - u);
  }
  SK_HD int64_t peer(int64_t tile, int64_t u, int i) const {
    return strategy == kExplicit ? xids[xoff[tile] + i] : u + i;
  }
  // A partial whose tile no range starts is never folded (the reference's
  // executor leaves that tile of C at zero): explicit tables only.
  SK_HD bool orphan(int64_t tile) const {
    if (strategy != kExplicit) return false;
    return xr[2 * xids[xoff[tile]]] > tile * ipt;
  }

  // Compact slab index of a partial-emitting unit (only units whose first
  // segment starts mid-tile emit; at most one partial per unit).
  SK_HD int64_t slab_of(int64_t u) const {
    if (strategy == kExplicit) return u;
    if (strategy == kFixedSplit) return (u / split) * (split - 1) + (u % split) - 1;
    return u - bal.first_id;
  }
};

}  // namespace skb200
