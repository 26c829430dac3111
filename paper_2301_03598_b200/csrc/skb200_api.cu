// skb200_api.cu -- host side of the C ABI declared in include/skb200.h.
//
// Schedules are computed in closed form (schedule.hpp); sk_gemm validates the
// descriptor, builds the TMA tensor maps, sizes the persistent grid to the SM
// count and launches the hand-written sm_100a kernels.  sk_execute is the
// reference-facing drop-in of streamk::execute<T> (executor.hpp:130-207):
// host buffers in, host C out.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <tuple>
#include <vector>

#include "../../include/skb200.h"
#include "schedule.hpp"
#include "sk_kernel_common.cuh"

namespace skb200 {
// sk_gemm_f16.cu
uint32_t make_idesc_f16(bool bf16, int M, int N);
size_t f16_slab_bytes(int bn);
int f16_stage_k();
int f16_epilogue_warps(int bn);
cudaError_t f16_prepare(int cg, int bn, int sms, int* units);
cudaError_t f16_cluster_capacity(int cg, int cluster, int sms, int* clusters);
cudaError_t launch_f16(int cg, int bn, int cluster, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                       const KernelParams& p, int grid, cudaStream_t stream);
// sk_gemm_f64.cu
size_t f64_slab_bytes();
cudaError_t f64_max_ctas_per_sm(int* out);
cudaError_t launch_f64(const CUtensorMap& a, const CUtensorMap& b, double* C, int64_t ldc,
                       const KernelParams& p, int grid, cudaStream_t stream);
// sk_convert.cu
cudaError_t launch_convert(int kind, const void* src, int64_t ld_src, void* dst, int64_t ld_dst,
                           int64_t rows, int64_t cols, cudaStream_t stream);
cudaError_t launch_f32_to_16(const float* src, void* dst, int64_t rows, int64_t cols,
                             int64_t ld_dst, bool bf16, cudaStream_t stream);
// sk_random.cu
cudaError_t launch_random_matrix(int gen, int out, uint64_t seed, int shift, int64_t rows, int64_t cols,
                                 void* dst, int64_t ld, cudaStream_t stream);
// sk_probe.cu
bool probe_dies(int sms, std::vector<int>* die_of_sm, cudaError_t* cuda_err);
}  // namespace skb200

using namespace skb200;

namespace {

thread_local std::string g_last_error;

sk_status fail(sk_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

sk_status cuda_fail(cudaError_t e, const char* where) {
  return fail(SK_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define SK_CUDA(call)                                  \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

// ---- per-device lazily initialised state --------------------------------
struct DeviceInfo {
  int sms = 0;
  int cc_major = 0, cc_minor = 0;
  bool ok = false;
  // two-die topology (sk_probe.cu); probed once, outside stream capture
  bool topo_probed = false, topo_ok = false;
  std::vector<int> die_of_sm;
  // Kernel attributes are per-device state: set once per device, together
  // with the co-resident capacity of each persistent kernel (CTAs for the
  // 1-SM and FP64 kernels, CTA pairs for the 2-SM kernel).  A persistent grid
  // larger than that could leave an owner waiting on a unit whose CTA never
  // becomes resident, so every launch is capped by it.
  bool f16_ready[3] = {false, false, false};  // per tcgen05 kernel (Kernel enum order)
  int f16_units[3] = {0, 0, 0};
  int cluster_caps[2][9] = {{-1, -1, -1, -1, -1, -1, -1, -1, -1},
                            {-1, -1, -1, -1, -1, -1, -1, -1, -1}};  // [cg - 1][S = 2..8]: clusters
  bool f64_ready = false;
  int f64_per_sm = 0;
};
std::mutex g_dev_mu;
DeviceInfo g_dev[64];

// ---- tuning knobs ----------------------------------------------------------
// SKB200_* environment overrides, read once (sk_reload_env re-reads them) so
// a launch does not scan the environment ten times.  -1 = unset.
struct Knobs {
  int die_aware = 0, l2_promo = -1, raster_rows = -1, sk_first = -1, k_align = -1, coop = -1;
  int cluster_fix = 1;  // fixed_split on the 1-SM kernel: DSMEM fixup inside a cluster when it fits
  double coop_min = 8.0;  // mean contributors per shared tile from which the cooperative fixup runs
  int pipeline = 1, pipe_g = -1, pipe_w = -1, pipe_trace = 0;
  bool l2_policy_set = false;
  int l2_policy[4] = {0, 0, 0, 0};
};
std::mutex g_knob_mu;
Knobs g_knobs;
bool g_knobs_loaded = false;

Knobs read_knobs() {
  Knobs k;
  auto num = [](const char* name, int def) {
    const char* e = getenv(name);
    return e ? atoi(e) : def;
  };
  k.die_aware = num("SKB200_DIE_AWARE", 0);
  k.l2_promo = num("SKB200_L2_PROMO", -1);
  k.raster_rows = num("SKB200_RASTER_ROWS", -1);
  k.sk_first = num("SKB200_SK_FIRST", -1);
  k.k_align = num("SKB200_K_ALIGN", -1);
  k.coop = num("SKB200_COOP", -1);
  k.cluster_fix = num("SKB200_CLUSTER_FIX", 1);
  if (const char* e = getenv("SKB200_COOP_MIN")) k.coop_min = atof(e);
  k.pipeline = num("SKB200_PIPELINE", 1);
  k.pipe_g = num("SKB200_PIPE_G", -1);
  k.pipe_w = num("SKB200_PIPE_W", -1);
  k.pipe_trace = num("SKB200_PIPE_TRACE", 0);
  if (const char* e = getenv("SKB200_L2_POLICY"))
    k.l2_policy_set = sscanf(e, "%d,%d,%d,%d", &k.l2_policy[0], &k.l2_policy[1], &k.l2_policy[2],
                             &k.l2_policy[3]) == 4;
  return k;
}

const Knobs& knobs() {
  std::lock_guard<std::mutex> lk(g_knob_mu);
  if (!g_knobs_loaded) {
    g_knobs = read_knobs();
    g_knobs_loaded = true;
  }
  return g_knobs;
}

sk_status device_info(int dev, DeviceInfo* out) {
  if (dev < 0 || dev >= 64) return fail(SK_EINVAL, "device ordinal %d", dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& d = g_dev[dev];
  if (!d.ok) {
    SK_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    SK_CUDA(cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    SK_CUDA(cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    d.ok = true;
  }
  *out = d;
  return SK_OK;
}

// Die-aware lane table for a full persistent grid of `ranks`-CTA units
// (KernelParams::die_tab): die << 8 | rank among the die's units, keyed by the
// smid of the unit's leader CTA.  Probes the device on first use (not while
// `strm` is being captured into a graph: the probe synchronises).
bool die_table(int dev, cudaStream_t strm, int ranks, KernelParams* P) {
  // Opt-in (SKB200_DIE_AWARE=1): halves DRAM reads of isolated 8192^3 launches
  // (1.63 -> 0.99 GB, +6 % under ncu) but measured 1-4 % slower in back-to-back
  // bursts (profiles/r01/die_aware.txt), so the default schedule ignores dies.
  if (!knobs().die_aware) return false;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& d = g_dev[dev];
  if (!d.ok) return false;
  if (!d.topo_probed) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(strm, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return false;
    }
    cudaError_t ce;
    d.topo_ok = probe_dies(d.sms, &d.die_of_sm, &ce);
    d.topo_probed = true;
  }
  if (!d.topo_ok || d.sms > kMaxSms) return false;
  int n[2] = {0, 0};
  for (int i = 0; i < kMaxSms; ++i) P->die_tab[i] = -1;
  for (int sm = 0; sm < d.sms; sm += ranks) {  // units in ascending smid (TPC) order per die
    const int die = d.die_of_sm[static_cast<size_t>(sm)];
    for (int j = 0; j < ranks; ++j) P->die_tab[sm + j] = static_cast<int16_t>((die << 8) | n[die]);
    ++n[die];
  }
  P->die_n[0] = n[0];
  P->die_n[1] = n[1];
  return true;
}

// ---- TMA descriptors through the driver entry point (no -lcuda) ----------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D row-major tensor: rows x cols elements with leading dimension ld.
// Encoded maps are cached per host thread (a small ring keyed by every encode
// argument), so repeated launches on the same buffers skip the driver call.
struct TmapKey {
  int dt;
  size_t esize;
  const void* base;
  int64_t rows, cols, ld;
  uint32_t box_cols, box_rows;
  int swz, promo;
  bool operator==(const TmapKey& o) const {
    return dt == o.dt && esize == o.esize && base == o.base && rows == o.rows && cols == o.cols &&
           ld == o.ld && box_cols == o.box_cols && box_rows == o.box_rows && swz == o.swz &&
           promo == o.promo;
  }
};
struct TmapCache {
  static constexpr int N = 16;
  TmapKey key[N];
  CUtensorMap map[N];
  bool used[N] = {};
  int next = 0;
};
thread_local TmapCache g_tmaps;

sk_status make_tmap(CUtensorMap* m, CUtensorMapDataType dt, size_t esize, const void* base,
                    int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols, uint32_t box_rows,
                    CUtensorMapSwizzle swz) {
  // 128-B L2 promotion: 8192^3 DP 1468.8 vs 1461.7 (256 B), hybrid 1445.4 vs
  // 1438.7 TFLOP/s; config 3 and skinny shapes unchanged (profiles/r01/l2_policy.txt).
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  if (knobs().l2_promo >= 0)  // 0 none, 1 64B, 2 128B, 3 256B
    promo = static_cast<CUtensorMapL2promotion>(knobs().l2_promo);
  const TmapKey key{static_cast<int>(dt), esize, base, rows, cols, ld, box_cols, box_rows,
                    static_cast<int>(swz), static_cast<int>(promo)};
  TmapCache& c = g_tmaps;
  for (int i = 0; i < TmapCache::N; ++i)
    if (c.used[i] && c.key[i] == key) {
      *m = c.map[i];
      return SK_OK;
    }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esize};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SK_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  c.key[c.next] = key;
  c.map[c.next] = *m;
  c.used[c.next] = true;
  c.next = (c.next + 1) % TmapCache::N;
  return SK_OK;
}

// ---- workspace hygiene ------------------------------------------------------
// The kernels leave every flag they consume at zero, but the flag region's size
// depends on the schedule, so a workspace reused across descriptors may have old
// partial-slab bytes where the next launch keeps its flags.  Track, per
// workspace, the hull of bytes that may hold slab data and clear a new launch's
// flag region only when it overlaps that hull.
struct Dirty {
  size_t lo = 0, hi = 0;  // [lo, hi), empty when lo >= hi
  uint64_t table = 0;     // hash of the explicit table the workspace tail holds (0 = none)
};
std::mutex g_ws_mu;
std::unordered_map<const void*, Dirty> g_ws_dirty;

void ws_mark_clean(const void* ws) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  g_ws_dirty[ws] = Dirty{};
}
void ws_mark_all_dirty(const void* ws) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  g_ws_dirty[ws] = Dirty{0, ~size_t(0)};
}
// Returns true when [flags_off, flags_end) must be zeroed before this launch.
// *upload: whether an explicit table (hash `table`, 0 = closed form) must be
// copied into the workspace tail; any other launch invalidates a resident table.
bool ws_prepare(const void* ws, size_t flags_off, size_t flags_end, size_t slabs_end,
                uint64_t table = 0, bool* upload = nullptr) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto it = g_ws_dirty.find(ws);
  bool clear = false;
  Dirty d = it == g_ws_dirty.end() ? Dirty{} : it->second;
  if (upload) *upload = table != 0 && d.table != table;
  d.table = table;
  if (d.lo < d.hi && d.lo < flags_end && flags_off < d.hi) {
    clear = true;
    if (d.lo < flags_end) d.lo = flags_end;
  }
  if (slabs_end > flags_end) {  // this launch writes slabs in [flags_end, slabs_end)
    if (d.lo >= d.hi) {
      d.lo = flags_end;
      d.hi = slabs_end;
    } else {
      d.lo = std::min(d.lo, flags_end);
      d.hi = std::max(d.hi, slabs_end);
    }
  }
  g_ws_dirty[ws] = d;
  return clear;
}

bool valid_strategy(int32_t s) { return s >= 0 && s <= 4; }

sk_status init_schedule(const sk_problem* p, const sk_blocking* b, int32_t strategy,
                        int64_t param, Schedule* s) {
  if (!p || !b) return fail(SK_EINVAL, "null problem/blocking");
  if (!valid_strategy(strategy)) return fail(SK_EINVAL, "unknown strategy %d", strategy);
  if (s->init(p->m, p->n, p->k, b->blk_m, b->blk_n, b->blk_k, strategy, param) != 0) {
    if (p->m < 1 || p->n < 1 || p->k < 1) return fail(SK_EINVAL, "GemmProblem extents must be >= 1");
    if (b->blk_m < 1 || b->blk_n < 1 || b->blk_k < 1)
      return fail(SK_EINVAL, "BlockingFactors must be >= 1");
    return fail(SK_EINVAL, "strategy parameter must be >= 1");
  }
  return SK_OK;
}

// ---- explicit range tables (SK_EXPLICIT) ---------------------------------------
// Host copy of a validated table: ranges, then fixup_peers_of (decompose.cpp:123-136)
// as CSR, laid out exactly as it is copied into the workspace tail.
struct ExplicitTable {
  std::vector<int64_t> data;  // [2g ranges][t + 1 offsets][nnz ids]
  int64_t g = 0, tiles = 0, nnz = 0;
  bool all_started = true;
  uint64_t hash = 0;
  const int64_t* ranges() const { return data.data(); }
  const int64_t* off() const { return data.data() + 2 * g; }
  const int64_t* ids() const { return data.data() + 2 * g + tiles + 1; }
  size_t bytes() const { return data.size() * sizeof(int64_t); }
};
thread_local ExplicitTable g_xt;

// Bounds (mac_loop's contract, executor.hpp:63-68) and peer lists; with
// `protocol`, also the two conditions the persistent grid needs (see skb200.h).
sk_status build_explicit(const Schedule& s, const int64_t* r, int64_t g, bool protocol,
                         ExplicitTable* x) {
  if (g < 0) return fail(SK_EINVAL, "num_ranges < 0");
  if (g > 0 && !r) return fail(SK_EINVAL, "null range table");
  const int64_t t = s.total_tiles, ipt = s.ipt;
  std::vector<int64_t> cnt(static_cast<size_t>(t + 1), 0);
  for (int64_t u = 0; u < g; ++u) {
    const int64_t b = r[2 * u], e = r[2 * u + 1];
    if (b < 0 || e < b || e > s.total_iters)
      return fail(SK_EINVAL, "range %lld [%lld, %lld) outside [0, %lld)", (long long)u,
                  (long long)b, (long long)e, (long long)s.total_iters);
    if (b == e) continue;  // empty ranges are nobody's peer (decompose.cpp:127)
    for (int64_t tile = b / ipt; tile <= (e - 1) / ipt; ++tile) ++cnt[static_cast<size_t>(tile + 1)];
  }
  for (int64_t i = 0; i < t; ++i) cnt[static_cast<size_t>(i + 1)] += cnt[static_cast<size_t>(i)];
  x->g = g;
  x->tiles = t;
  x->nnz = cnt[static_cast<size_t>(t)];
  x->data.assign(static_cast<size_t>(2 * g + t + 1 + x->nnz), 0);
  std::copy(r, r + 2 * g, x->data.begin());
  int64_t* off = x->data.data() + 2 * g;
  int64_t* ids = off + t + 1;
  std::copy(cnt.begin(), cnt.end(), off);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t u = 0; u < g; ++u) {  // ascending u: every list comes out sorted
    const int64_t b = r[2 * u], e = r[2 * u + 1];
    if (b == e) continue;
    for (int64_t tile = b / ipt; tile <= (e - 1) / ipt; ++tile) ids[fill[static_cast<size_t>(tile)]++] = u;
  }
  x->all_started = true;
  for (int64_t tile = 0; tile < t; ++tile) {
    int64_t starter = -1;
    for (int64_t q = off[tile]; q < off[tile + 1]; ++q) {
      const int64_t u = ids[q];
      if (r[2 * u] > tile * ipt) continue;  // joins mid-tile: a partial
      if (protocol && starter >= 0)
        return fail(SK_EINVAL, "tile %lld is started by ranges %lld and %lld (the reference "
                    "executor would wait on both forever)", (long long)tile, (long long)starter,
                    (long long)u);
      starter = u;
    }
    if (starter < 0) {
      x->all_started = false;
    } else if (protocol && starter != ids[off[tile]]) {
      return fail(SK_EUNSUPPORTED, "tile %lld: starter %lld would wait on lower id %lld; only "
                  "tables whose fixup waits point to higher ids run on a persistent grid",
                  (long long)tile, (long long)starter, (long long)ids[off[tile]]);
    }
  }
  uint64_t h = 1469598103934665603ull;  // FNV-1a over the table and the tile grid
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) h = (h ^ ((v >> (8 * i)) & 0xff)) * 1099511628211ull;
  };
  mix(static_cast<uint64_t>(ipt));
  mix(static_cast<uint64_t>(t));
  for (int64_t v : x->data) mix(static_cast<uint64_t>(v));
  x->hash = h ? h : 1;
  return SK_OK;
}

size_t dtype_size(int32_t t) {
  switch (t) {
    case SK_INT64: return 8;
    case SK_FLOAT32: return 4;
    case SK_FLOAT64: return 8;
    case SK_BFLOAT16: return 2;
    case SK_FLOAT16: return 2;
  }
  return 0;
}

// Which kernel serves a descriptor.
enum class Kernel { F16_1SM, F16_2SM, F16_2SM_WIDE, F64 };
bool is_f16(Kernel k) { return k != Kernel::F64; }
int kernel_cg(Kernel k) { return k == Kernel::F16_1SM ? 1 : 2; }
int kernel_bn(Kernel k) { return k == Kernel::F16_2SM_WIDE ? 512 : 256; }

sk_status pick_kernel(const sk_gemm_desc* d, Kernel* k) {
  if (d->ab_type == SK_BFLOAT16 || d->ab_type == SK_FLOAT16) {
    // AUTO: the blocking names the kernel (128x256x64 -> 1-SM); default 2-SM.
    if (d->variant == SK_VARIANT_1SM ||
        (d->variant == SK_VARIANT_AUTO && d->blocking.blk_m == 128 && d->blocking.blk_n == 256 &&
         d->blocking.blk_k == 64)) {
      *k = Kernel::F16_1SM;
      return SK_OK;
    }
    if (d->variant == SK_VARIANT_2SM_WIDE ||
        (d->variant == SK_VARIANT_AUTO && d->blocking.blk_m == 256 && d->blocking.blk_n == 512 &&
         d->blocking.blk_k == 64)) {
      *k = Kernel::F16_2SM_WIDE;
      return SK_OK;
    }
    if (d->variant == SK_VARIANT_2SM || d->variant == SK_VARIANT_AUTO) {
      *k = Kernel::F16_2SM;
      return SK_OK;
    }
    return fail(SK_EINVAL, "unknown variant %d", d->variant);
  }
  if (d->ab_type == SK_FLOAT64) {
    *k = Kernel::F64;
    return SK_OK;
  }
  return fail(SK_EUNSUPPORTED, "ab_type %d has no device kernel", d->ab_type);
}

sk_status kernel_blocking(Kernel k, sk_blocking* out) {
  switch (k) {
    case Kernel::F16_1SM: *out = {128, 256, 64}; return SK_OK;
    case Kernel::F16_2SM: *out = {256, 256, 64}; return SK_OK;
    case Kernel::F16_2SM_WIDE: *out = {256, 512, 64}; return SK_OK;
    case Kernel::F64: *out = {64, 64, 16}; return SK_OK;
  }
  return SK_EINVAL;
}

int kernel_ranks(Kernel k) { return is_f16(k) ? kernel_cg(k) : 1; }

// Mean number of contributing units over the balanced region's shared tiles
// (tiles with more than one contributor); 0 when none is shared.
double mean_contributors(const Schedule& s) {
  // units of >= ipt/2 iterations give tiles at most ~3 contributors: skip the
  // scan (it then only runs for schedules with few tiles, g <= p units)
  if (s.bal.q * 2 >= s.ipt) return 0.0;
  int64_t shared = 0, sum = 0;
  for (int64_t t = s.bal.begin / s.ipt; t < s.total_tiles; ++t) {
    int64_t owner, last;
    s.peers(t, &owner, &last);
    if (last > owner) {
      ++shared;
      sum += last - owner + 1;
    }
  }
  return shared ? static_cast<double>(sum) / static_cast<double>(shared) : 0.0;
}

// Balanced-region tiles the cooperative fixup keeps a done counter for, or -1
// when the schedule/kernel never uses it (the workspace is sized for it
// whenever the 16-bit kernels run a balanced schedule).
int64_t coop_tiles(Kernel k, const Schedule& s) {
  if (k == Kernel::F64 || s.bal.count == 0 || s.strategy == kFixedSplit || s.strategy == kExplicit)
    return -1;
  return s.total_tiles - s.bal.begin / s.ipt;
}

size_t kernel_slab_bytes(Kernel k) {
  switch (k) {
    case Kernel::F16_1SM:
    case Kernel::F16_2SM:
    case Kernel::F16_2SM_WIDE: return f16_slab_bytes(kernel_bn(k));
    case Kernel::F64: return 64 * 64 * sizeof(double);
  }
  return 0;
}

sk_status check_desc(const sk_gemm_desc* d, Kernel* kern, Schedule* s) {
  if (!d) return fail(SK_EINVAL, "null descriptor");
  sk_status st;
  if (d->strategy == SK_EXPLICIT) {
    if (s->init_explicit(d->problem.m, d->problem.n, d->problem.k, d->blocking.blk_m,
                         d->blocking.blk_n, d->blocking.blk_k, d->num_ranges) != 0)
      return init_schedule(&d->problem, &d->blocking, SK_DATA_PARALLEL, 1, s);  // the message
    st = build_explicit(*s, d->ranges, d->num_ranges, true, &g_xt);
    if (st) return st;
    s->xr = g_xt.ranges();
    s->xoff = g_xt.off();
    s->xids = g_xt.ids();
  } else {
    st = init_schedule(&d->problem, &d->blocking, d->strategy, d->param, s);
    if (st) return st;
  }
  st = pick_kernel(d, kern);
  if (st) return st;
  sk_blocking kb;
  kernel_blocking(*kern, &kb);
  if (d->blocking.blk_m != kb.blk_m || d->blocking.blk_n != kb.blk_n ||
      d->blocking.blk_k != kb.blk_k)
    return fail(SK_EUNSUPPORTED,
                "blocking %lldx%lldx%lld differs from the kernel tile %lldx%lldx%lld",
                (long long)d->blocking.blk_m, (long long)d->blocking.blk_n,
                (long long)d->blocking.blk_k, (long long)kb.blk_m, (long long)kb.blk_n,
                (long long)kb.blk_k);
  // int32 device indexing guard (true for every BASELINE config).
  if (s->total_iters >= (int64_t(1) << 31) || s->grid_size >= (int64_t(1) << 31) ||
      d->problem.m >= (int64_t(1) << 31) || d->problem.n >= (int64_t(1) << 31) ||
      d->problem.k >= (int64_t(1) << 31))
    return fail(SK_EUNSUPPORTED, "problem too large for 32-bit tile coordinates");
  return SK_OK;
}

}  // namespace

namespace {
// Transfer-pipelining state of a launch (sk_execute with pinned host buffers).
struct PipeFlags {
  const int* a_ready = nullptr;  // [tiles_m]
  const int* b_ready = nullptr;  // [panels] or NULL (B complete before launch)
  int* c_done = nullptr;         // [blocks]
  int g = 1, w = 1, np = 1;      // c_done block = g tile rows x w tile cols; np panels
  int64_t raster = 1;            // data-parallel raster height
  const int32_t* perm = nullptr; // data-parallel slot -> tile order (device), or NULL
};
sk_status gemm_impl(const sk_gemm_desc* d, void* ws, size_t ws_bytes, cudaStream_t strm,
                    const PipeFlags* pipe = nullptr);

// Raster group height: the group's A panels (rows x BLK_M x k elements) are
// kept near 32 MB so they stay L2-resident while B streams through; measured
// best at 8192^3: 16 rows (1-SM), 8 rows (2-SM) (profiles/r01/raster_rows.txt).
int64_t raster_rows_for(const sk_gemm_desc* d) {
  const double panel = static_cast<double>(d->blocking.blk_m) * static_cast<double>(d->problem.k) *
                       static_cast<double>(dtype_size(d->ab_type));
  int64_t rows = std::max<int64_t>(1, static_cast<int64_t>((32.0 * 1024 * 1024) / panel));
  if (knobs().raster_rows > 0) rows = knobs().raster_rows;
  // beyond the tile rows a group changes nothing; keeps group * tiles_n < 2^31
  const int64_t tiles_m = ceil_div(d->problem.m, std::max<int64_t>(1, d->blocking.blk_m));
  return std::max<int64_t>(1, std::min(rows, tiles_m));
}

// Tile id -> block of C (sk_gemm_desc.tile_group): the reference's row-major
// map by default; grouped ids only on request (G = -1: the raster height),
// after which the data-parallel raster is the identity.  G is clamped to
// tiles_m (beyond it nothing changes, and G * tiles_n stays < 2^31).
void apply_tile_group(const sk_gemm_desc* d, Kernel kern, bool explicit_table, bool pipelined,
                      Schedule* s, int64_t* raster) {
  s->tile_group = 1;
  if (pipelined || explicit_table || kern == Kernel::F64) return;
  int64_t group = d->tile_group == -1 ? *raster : d->tile_group;
  group = std::min<int64_t>(group, s->tiles_m);
  if (group > 1) {
    s->tile_group = group;
    *raster = 1;  // the id order already is the raster
  }
}

// TwoTileSkDp phase order: the FP64 kernel runs the SK region first (its fixup
// epilogues then overlap the DP waves: 33.6 -> 34.3 TFLOP/s at 8192^3); the
// tcgen05 kernel keeps the DP waves first (SK-first measured 1.5 % slower;
// interleaving the SK units through the DP waves 4 % slower,
// profiles/r01/phase_order.txt).
int phase_order_for(Kernel k) {
  int order = k == Kernel::F64 ? kSkFirst : kDpFirst;
  if (knobs().sk_first >= 0) order = knobs().sk_first;
  return order;
}
}  // namespace

extern "C" {

const char* sk_status_string(sk_status s) {
  switch (s) {
    case SK_OK: return "SK_OK";
    case SK_EINVAL: return "SK_EINVAL: invalid argument";
    case SK_EUNSUPPORTED: return "SK_EUNSUPPORTED: not supported by the device kernel";
    case SK_ECUDA: return "SK_ECUDA: CUDA error";
    case SK_EPROTOCOL: return "SK_EPROTOCOL: fixup protocol violation";
    case SK_ERANGE: return "SK_ERANGE: index out of range";
    case SK_ECAPACITY: return "SK_ECAPACITY: output buffer too small";
    case SK_EIO: return "SK_EIO: matrix file error";
  }
  return "unknown sk_status";
}

const char* sk_last_error(void) { return g_last_error.c_str(); }
int sk_abi_version(void) { return SKB200_ABI_VERSION; }

sk_status sk_tile_grid(const sk_problem* p, const sk_blocking* b, sk_tile_grid_t* out) {
  Schedule s;
  sk_status st = init_schedule(p, b, SK_DATA_PARALLEL, 1, &s);
  if (st) return st;
  if (out) *out = {s.tiles_m, s.tiles_n, s.total_tiles, s.ipt, s.total_iters};
  return SK_OK;
}

sk_status sk_iter_to_coords(const sk_tile_grid_t* g, int64_t i, int64_t* tile, int64_t* local) {
  if (!g || g->iters_per_tile < 1) return fail(SK_EINVAL, "bad tile grid");
  if (i < 0 || i >= g->total_iters) return fail(SK_ERANGE, "iteration index out of range");
  if (tile) *tile = i / g->iters_per_tile;
  if (local) *local = i % g->iters_per_tile;
  return SK_OK;
}

sk_status sk_schedule(const sk_problem* p, const sk_blocking* b, sk_strategy strategy,
                      int64_t param, int64_t* grid_size, int64_t* ranges, int64_t capacity) {
  Schedule s;
  sk_status st = init_schedule(p, b, strategy, param, &s);
  if (st) return st;
  if (grid_size) *grid_size = s.grid_size;
  if (!ranges) return SK_OK;
  if (capacity < s.grid_size) return fail(SK_ECAPACITY, "ranges capacity %lld < g %lld",
                                          (long long)capacity, (long long)s.grid_size);
  for (int64_t u = 0; u < s.grid_size; ++u) s.range(u, &ranges[2 * u], &ranges[2 * u + 1]);
  return SK_OK;
}

sk_status sk_fixup_peers(const sk_problem* p, const sk_blocking* b, sk_strategy strategy,
                         int64_t param, int64_t* offsets, int64_t* ids, int64_t capacity,
                         int64_t* nnz) {
  Schedule s;
  sk_status st = init_schedule(p, b, strategy, param, &s);
  if (st) return st;
  if (!offsets) return fail(SK_EINVAL, "null offsets");
  int64_t total = 0;
  offsets[0] = 0;
  for (int64_t t = 0; t < s.total_tiles; ++t) {
    int64_t owner, last;
    s.peers(t, &owner, &last);
    total += last - owner + 1;
    offsets[t + 1] = total;
  }
  if (nnz) *nnz = total;
  if (!ids) return SK_OK;
  if (capacity < total) return fail(SK_ECAPACITY, "ids capacity too small");
  int64_t q = 0;
  for (int64_t t = 0; t < s.total_tiles; ++t) {
    int64_t owner, last;
    s.peers(t, &owner, &last);
    for (int64_t id = owner; id <= last; ++id) ids[q++] = id;
  }
  return SK_OK;
}

sk_status sk_fixup_peers_ranges(const sk_problem* p, const sk_blocking* b, const int64_t* ranges,
                                int64_t num_ranges, int64_t* offsets, int64_t* ids,
                                int64_t capacity, int64_t* nnz) {
  if (!p || !b) return fail(SK_EINVAL, "null problem/blocking");
  Schedule s;
  if (s.init_explicit(p->m, p->n, p->k, b->blk_m, b->blk_n, b->blk_k, num_ranges) != 0)
    return init_schedule(p, b, SK_DATA_PARALLEL, 1, &s);
  if (!offsets) return fail(SK_EINVAL, "null offsets");
  ExplicitTable x;
  sk_status st = build_explicit(s, ranges, num_ranges, false, &x);
  if (st) return st;
  std::copy(x.off(), x.off() + x.tiles + 1, offsets);
  if (nnz) *nnz = x.nnz;
  if (!ids) return SK_OK;
  if (capacity < x.nnz) return fail(SK_ECAPACITY, "ids capacity too small");
  std::copy(x.ids(), x.ids() + x.nnz, ids);
  return SK_OK;
}

sk_status sk_quantization_efficiency(int64_t t, int64_t p, double* out) {
  if (t < 1 || p < 1) return fail(SK_EINVAL, "quantization_efficiency: t, p >= 1");
  if (out) *out = static_cast<double>(t) / static_cast<double>(ceil_div(t, p) * p);
  return SK_OK;
}

sk_status sk_corpus(uint64_t seed, int64_t count, int64_t lo, int64_t hi, uint64_t* out) {
  if (count < 0 || lo < 1 || hi < lo || (count > 0 && !out))
    return fail(SK_EINVAL, "sk_corpus: bad arguments");
  uint64_t state = seed;
  auto next = [&state]() {  // SplitMix64, matrix.hpp:39-53
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  auto sample = [&](int64_t a, int64_t b) -> int64_t {  // sweep.cpp:21-28 log_sample
    if (a == b) return a;
    const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
    const double v = std::exp(std::log(static_cast<double>(a)) +
                              u * (std::log(static_cast<double>(b)) - std::log(static_cast<double>(a))));
    return std::min(std::max(static_cast<int64_t>(std::llround(v)), a), b);
  };
  for (int64_t i = 0; i < count; ++i) {
    out[4 * i + 0] = static_cast<uint64_t>(sample(lo, hi));
    out[4 * i + 1] = static_cast<uint64_t>(sample(lo, hi));
    out[4 * i + 2] = static_cast<uint64_t>(sample(lo, hi));
    out[4 * i + 3] = next();
  }
  return SK_OK;
}

sk_status sk_kernel_blocking(sk_dtype ab_type, sk_variant variant, sk_blocking* out) {
  sk_gemm_desc d{};
  d.ab_type = ab_type;
  d.variant = variant;
  Kernel k;
  sk_status st = pick_kernel(&d, &k);
  if (st) return st;
  return kernel_blocking(k, out);
}

sk_status sk_workspace_size(const sk_gemm_desc* d, size_t* bytes) {
  Kernel k;
  Schedule s;
  sk_status st = check_desc(d, &k, &s);
  if (st) return st;
  WorkspaceLayout L;
  L.compute(s.num_slabs, kernel_ranks(k), kernel_slab_bytes(k),
            s.strategy == kExplicit ? g_xt.bytes() : 0, coop_tiles(k, s));
  if (bytes) *bytes = L.total;
  return SK_OK;
}

sk_status sk_workspace_init(void* ws, size_t bytes, void* stream) {
  if (!ws || bytes < 256) return fail(SK_EINVAL, "workspace too small");
  // One memset after allocation; the kernel re-arms every flag it consumes.
  SK_CUDA(cudaMemsetAsync(ws, 0, bytes, static_cast<cudaStream_t>(stream)));
  ws_mark_clean(ws);
  return SK_OK;
}

sk_status sk_workspace_check(void* ws, void* stream) {
  if (!ws) return fail(SK_EINVAL, "null workspace");
  int err = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SK_CUDA(cudaMemcpyAsync(&err, ws, sizeof(int), cudaMemcpyDeviceToHost, st));
  SK_CUDA(cudaStreamSynchronize(st));
  if (err == 0) return SK_OK;
  SK_CUDA(cudaMemsetAsync(ws, 0, sizeof(int), st));
  ws_mark_all_dirty(ws);  // flags may be left set after a protocol failure
  if (err & kErrDoubleSignal) return fail(SK_EPROTOCOL, "execute: fixup flag signaled twice");
  if (err & kErrTopology) return fail(SK_EPROTOCOL, "die-aware schedule: SM outside the probed topology");
  return fail(SK_EPROTOCOL, "fixup wait watchdog expired (err=0x%x)", err);
}

sk_status sk_trace_size(const sk_gemm_desc* d, int64_t* ints) {
  Kernel k;
  Schedule s;
  sk_status st = check_desc(d, &k, &s);
  if (st) return st;
  if (ints) *ints = 5 * s.total_tiles + s.grid_size;
  return SK_OK;
}

namespace {
int64_t max_segments_per_unit(const Schedule& s) {
  int64_t best = 1;
  for (int64_t u = 0; u < s.grid_size; ++u) {
    int64_t b, e;
    s.range(u, &b, &e);
    if (e > b) best = std::max(best, (e - 1) / s.ipt - b / s.ipt + 1);
  }
  return best;
}
}  // namespace

extern "C" sk_status sk_timeline_size(const sk_gemm_desc* d, int64_t* records, int64_t* seg_stride) {
  Kernel k;
  Schedule s;
  sk_status st = check_desc(d, &k, &s);
  if (st) return st;
  const int64_t stride = max_segments_per_unit(s);
  if (seg_stride) *seg_stride = stride;
  if (records) *records = s.grid_size * stride;
  return SK_OK;
}

sk_status sk_device_topology(int device, int32_t* die_of_sm, int32_t max_sms, int32_t* sms,
                             int32_t* ok) {
  if (!sms || !ok) return fail(SK_EINVAL, "null output");
  DeviceInfo info;
  sk_status st = device_info(device, &info);
  if (st) return st;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& d = g_dev[device];
  if (!d.topo_probed) {
    int cur = 0;
    SK_CUDA(cudaGetDevice(&cur));
    SK_CUDA(cudaSetDevice(device));
    cudaError_t ce;
    d.topo_ok = probe_dies(d.sms, &d.die_of_sm, &ce);
    d.topo_probed = true;
    cudaSetDevice(cur);
    if (ce != cudaSuccess) return cuda_fail(ce, "topology probe");
  }
  *sms = d.sms;
  *ok = d.topo_ok ? 1 : 0;
  if (die_of_sm && d.topo_ok)
    for (int i = 0; i < d.sms && i < max_sms; ++i) die_of_sm[i] = d.die_of_sm[static_cast<size_t>(i)];
  return SK_OK;
}

sk_status sk_persistent_order(const sk_gemm_desc* d, int64_t num_ctas, int64_t cta, int64_t* out,
                              int64_t max_records, int64_t* count) {
  Kernel kern;
  Schedule s;
  sk_status st = check_desc(d, &kern, &s);
  if (st) return st;
  if (num_ctas < 1 || cta < 0 || cta >= num_ctas || !count || (max_records > 0 && !out))
    return fail(SK_EINVAL, "persistent_order: bad grid / cta / output");
  int64_t raster = raster_rows_for(d);
  apply_tile_group(d, kern, s.strategy == kExplicit, false, &s, &raster);
  SegmentIter it(s, cta, num_ctas, default_lane(s, cta, num_ctas), raster, phase_order_for(kern));
  int64_t n = 0, u, tile, lb, le;
  while (it.next(s, &u, &tile, &lb, &le)) {
    if (n < max_records) {
      int64_t* r = out + 4 * n;
      r[0] = u, r[1] = tile, r[2] = lb, r[3] = le;
    }
    ++n;
  }
  *count = n;
  return SK_OK;
}

sk_status sk_tile_block(const sk_gemm_desc* d, int64_t tile, int64_t* tile_row, int64_t* tile_col) {
  Kernel kern;
  Schedule s;
  sk_status st = check_desc(d, &kern, &s);
  if (st) return st;
  if (!tile_row || !tile_col) return fail(SK_EINVAL, "null output");
  if (tile < 0 || tile >= s.total_tiles) return fail(SK_ERANGE, "tile %lld out of range", (long long)tile);
  int64_t raster = raster_rows_for(d);
  apply_tile_group(d, kern, s.strategy == kExplicit, false, &s, &raster);
  s.tile_rc(tile, tile_row, tile_col);
  return SK_OK;
}

sk_status sk_gemm(const sk_gemm_desc* d, void* ws, size_t ws_bytes, void* stream) {
  return gemm_impl(d, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

sk_status sk_random_matrix(sk_dtype gen_type, int32_t shift, uint64_t seed, int64_t rows, int64_t cols,
                           sk_dtype out_type, void* dst, int64_t ld, void* stream) {
  if (rows < 0 || cols < 0 || ld < cols || shift < 0 || shift > 7 || (rows * cols > 0 && !dst))
    return fail(SK_EINVAL, "random_matrix: bad extents / buffer");
  const int gen = gen_type == SK_INT64 ? 0 : gen_type == SK_FLOAT32 ? 1 : gen_type == SK_FLOAT64 ? 2 : -1;
  const int out = out_type == SK_BFLOAT16 ? 0 : out_type == SK_FLOAT16 ? 1 : out_type == SK_FLOAT32 ? 2
                  : out_type == SK_FLOAT64 ? 3 : -1;
  if (gen < 0 || out < 0 || (gen == 2 && out < 2))
    return fail(SK_EINVAL, "random_matrix: unsupported generator / output type pair");
  if (rows * cols == 0) return SK_OK;
  SK_CUDA(launch_random_matrix(gen, out, seed, shift, rows, cols, dst, ld, static_cast<cudaStream_t>(stream)));
  return SK_OK;
}

}  // extern "C"

namespace {
// Co-resident capacity of a persistent kernel on device `dev` (current device):
// CTAs for the 1-SM and FP64 kernels, CTA pairs for the 2-SM kernel.  Sets the
// kernel's per-device attributes on first use.
sk_status resident_units(int dev, const DeviceInfo& info, Kernel kern, int* out) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& di = g_dev[dev];
  if (kern == Kernel::F64) {
    if (!di.f64_ready) {
      cudaError_t e = f64_max_ctas_per_sm(&di.f64_per_sm);
      if (e != cudaSuccess) return cuda_fail(e, "sk_gemm_f64 occupancy");
      if (di.f64_per_sm < 1) return fail(SK_ECUDA, "sk_gemm_f64 does not fit on an SM");
      di.f64_ready = true;
    }
    *out = di.f64_per_sm * info.sms;
    return SK_OK;
  }
  const int cg = kernel_cg(kern), ki = static_cast<int>(kern);
  if (!di.f16_ready[ki]) {
    cudaError_t e = f16_prepare(cg, kernel_bn(kern), info.sms, &di.f16_units[ki]);
    if (e != cudaSuccess) return cuda_fail(e, "sk_gemm_f16 attributes / occupancy");
    if (di.f16_units[ki] < 1) return fail(SK_ECUDA, "sk_gemm_f16 does not fit on the device");
    di.f16_ready[ki] = true;
  }
  *out = std::min(di.f16_units[ki], info.sms / cg);
  return SK_OK;
}

// Units (CTAs for 1-SM, CTA pairs for 2-SM) of the 256-wide tcgen05 kernel
// co-resident as clusters of S units (cluster fixup); 0 if none fit.  Caller
// holds no lock; resident_units() has set the kernel's attributes.
int cluster_units(int dev, const DeviceInfo& info, Kernel kern, int S) {
  const int cg = kernel_cg(kern);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceInfo& di = g_dev[dev];
  int& cap = di.cluster_caps[cg - 1][S];
  if (cap < 0) {
    int c = 0;
    if (f16_cluster_capacity(cg, S * cg, info.sms, &c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    cap = c;
  }
  return cap * S;
}

// Cluster fixup (256-wide tcgen05 kernels, fixed_split(S)): usable when
// 2 <= S <= 8, no k-chunk is empty (every unit of a cluster has a segment: the
// last chunk [(S-1) ips, ipt) is nonempty) and all t * S units are co-resident
// as clusters of S units.
int cluster_fix_for(int dev, const DeviceInfo& info, Kernel kern, const Schedule& s) {
  if ((kern != Kernel::F16_1SM && kern != Kernel::F16_2SM) || s.strategy != kFixedSplit ||
      knobs().cluster_fix == 0)
    return 0;
  const int64_t S = s.split;
  if (S < 2 || S > 8 || (S - 1) * s.ips >= s.ipt) return 0;
  return s.grid_size <= cluster_units(dev, info, kern, static_cast<int>(S)) ? static_cast<int>(S) : 0;
}

sk_status gemm_impl(const sk_gemm_desc* d, void* ws, size_t ws_bytes, cudaStream_t strm,
                    const PipeFlags* pipe) {
  const int* a_ready = pipe ? pipe->a_ready : nullptr;
  int* c_done = pipe ? pipe->c_done : nullptr;
  const int64_t raster = pipe ? pipe->raster : 0;
  Kernel kern;
  Schedule s;
  sk_status st = check_desc(d, &kern, &s);
  if (st) return st;
  const size_t esz = dtype_size(d->ab_type);
  const size_t csz = d->ab_type == SK_FLOAT64 ? 8 : 4;
  if (!d->A || !d->B || !d->C) return fail(SK_EINVAL, "null matrix pointer");
  if (d->lda < d->problem.k || d->ldb < d->problem.n || d->ldc < d->problem.n)
    return fail(SK_EINVAL, "leading dimension smaller than the row length");
  if ((reinterpret_cast<uintptr_t>(d->A) | reinterpret_cast<uintptr_t>(d->B) |
       reinterpret_cast<uintptr_t>(d->C)) & 15)
    return fail(SK_EUNSUPPORTED, "matrix base pointers must be 16-byte aligned");
  if ((d->lda * esz) % 16 || (d->ldb * esz) % 16 || (d->ldc * csz) % 16)
    return fail(SK_EUNSUPPORTED, "leading dimensions must be multiples of 16 bytes (TMA)");
  const bool xp = s.strategy == kExplicit;
  WorkspaceLayout L;
  L.compute(s.num_slabs, kernel_ranks(kern), kernel_slab_bytes(kern), xp ? g_xt.bytes() : 0,
            coop_tiles(kern, s));
  if (!ws || ws_bytes < L.total)
    return fail(SK_EINVAL, "workspace of %zu bytes < required %zu", ws_bytes, L.total);

  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  DeviceInfo info;
  st = device_info(dev, &info);
  if (st) return st;
  if (info.cc_major != 10 || info.cc_minor != 0)
    return fail(SK_EUNSUPPORTED, "device sm_%d%d: this build targets sm_100a only", info.cc_major,
                info.cc_minor);
  bool upload = false;
  if (ws_prepare(ws, L.flags_off, L.partials_off, L.total, xp ? g_xt.hash : 0, &upload))
    SK_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(ws) + L.flags_off, 0, L.flag_bytes, strm));

  KernelParams P{};
  P.s = s;
  if (xp) {  // the kernel reads the table from the workspace tail
    int64_t* tb = reinterpret_cast<int64_t*>(static_cast<uint8_t*>(ws) + L.table_off);
    if (upload) SK_CUDA(cudaMemcpyAsync(tb, g_xt.data.data(), g_xt.bytes(), cudaMemcpyHostToDevice, strm));
    P.s.xr = tb;
    P.s.xoff = tb + 2 * g_xt.g;
    P.s.xids = tb + 2 * g_xt.g + g_xt.tiles + 1;
  }
  P.ranks = kernel_ranks(kern);
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  P.err = reinterpret_cast<int*>(wsb);
  P.flags = reinterpret_cast<int*>(wsb + L.flags_off);
  P.partials = wsb + L.partials_off;
  P.trace = d->trace;
  P.a_ready = a_ready;
  P.c_done = c_done;
  P.b_ready = pipe ? pipe->b_ready : nullptr;
  P.dp_perm = pipe ? pipe->perm : nullptr;
  P.pipe_g = pipe ? pipe->g : 1;
  P.pipe_w = pipe ? pipe->w : static_cast<int32_t>(s.tiles_n);
  P.pipe_np = pipe ? pipe->np : 1;
  P.cta_clocks = reinterpret_cast<long long*>(d->cta_clocks);
  P.events = reinterpret_cast<long long*>(d->events);
  P.seg_stride = d->events ? max_segments_per_unit(s) : 1;
  P.watchdog_ns = 4000000000LL;
  // Raster group height: the group's A panels (rows x BLK_M x k elements) are
  // kept near 32 MB so they stay L2-resident while B streams through; measured
  // best at 8192^3: 16 rows (1-SM), 8 rows (2-SM) (profiles/r01/raster_rows.txt).
  P.raster_rows = raster > 0 ? raster : raster_rows_for(d);
  apply_tile_group(d, kern, xp, a_ready != nullptr, &P.s, &P.raster_rows);
  // Grouped tile ids (Schedule::tile_rc): the same G-row groups now also
  // decide which block of C each tile id denotes, so a hybrid's trailing
  // Stream-K region is a compact 8 x 17 block at 8192^3 instead of a
  // 4.25 x 32 band (B panels fit L2): two_tile_sk_dp 1482 -> 1505 TFLOP/s,
  // data-parallel unchanged (profiles/r01/tile_group.txt).  The transfer-
  // pipelined sk_execute keeps row-major ids (its copies go by rows of C), and
  // so do explicit tables: with gaps or orphan tiles, which block of C stays
  // zero is observable (the reference's row-major id).  The DMMA kernel keeps
  // its raster (it is compute-bound, insensitive to L2 placement).
  // SKB200_TILE_GROUP=1 restores the reference's row-major tile ids.
  // L2 eviction priorities {A loads, B loads, C stores}: 0 normal, 1 first, 2 last.
  // A panels are re-read across a raster group's waves (keep), B panels stream
  // through a wave and C is written once (evict first); measured +4 % at 8192^3
  // from less DRAM traffic and a higher power-capped clock
  // (profiles/r01/l2_policy.txt).
  P.l2_policy[0] = 2;
  P.l2_policy[1] = 1;
  P.l2_policy[2] = 1;
  P.l2_policy[3] = 2;
  // TwoTileSkDp phase order: the FP64 kernel runs the SK region first (its fixup
  // epilogues then overlap the DP waves: 33.6 -> 34.3 TFLOP/s at 8192^3); the
  // tcgen05 kernel keeps the DP waves first (SK-first measured 1.5 % slower).
  P.sk_first = phase_order_for(kern);
  // Balanced units walk their k-blocks against a common clock (k_block_of): B
  // panels are shared in time across the SK region; 8192^3 hybrid 1458 -> 1482
  // TFLOP/s, config-3 geomean 1.287 -> 1.325 (profiles/r01/k_align.txt).
  P.k_align = kern == Kernel::F64 ? 0 : 1;
  if (knobs().k_align >= 0) P.k_align = knobs().k_align;
  if (knobs().l2_policy_set)
    for (int i = 0; i < 4; ++i) P.l2_policy[i] = knobs().l2_policy[i];
  // Persistent grid: at most the co-resident capacity of the kernel on this
  // device (queried once per device with the kernel attributes, which are
  // per-device state), so every unit a fixup wait points to is running.
  int resident = 0;
  st = resident_units(dev, info, kern, &resident);
  if (st) return st;
  const int64_t units = std::max<int64_t>(s.grid_size, 1);
  const int64_t cap = d->num_ctas > 0 ? d->num_ctas : resident;
  P.num_ctas = std::min<int64_t>(units, std::min<int64_t>(cap, resident));
  // Die-aware data-parallel phase: needs every SM (pair) in the persistent grid,
  // so each die's lane ranks are dense (dp_lane); the rasterised DP order is
  // otherwise unchanged.
  // Cooperative fixup when every balanced unit has a CTA of its own (all of
  // them run concurrently, so contributors can wait on each other); the
  // transfer-pipelined sk_execute path keeps owner folds (its per-row store
  // counts assume one storing CTA per tile).
  // Only worth it when tiles have many contributors: measured on B200
  // (profiles/r01/coop_fixup.txt) it wins from ~8 contributors per shared
  // tile (768^2 x 16384: +22 %, 512^2 x 65536: +50 %) and loses below (the
  // owner's serial fold of a few slabs is cheaper than every contributor
  // publishing and folding after its last segment).
  P.coop = 0;
  if (coop_tiles(kern, s) >= 0 && s.bal.count <= P.num_ctas && !a_ready && !c_done) {
    P.coop = mean_contributors(s) >= knobs().coop_min ? 1 : 0;
    if (knobs().coop >= 0) P.coop = knobs().coop != 0;
  }
  P.cluster_fix = 0;
  if (!a_ready && !c_done && !xp) {
    P.cluster_fix = cluster_fix_for(dev, info, kern, s);
    if (P.cluster_fix) P.num_ctas = s.grid_size;  // one unit per CTA, clusters of S
  }
  P.die_aware = 0;
  if (is_f16(kern) && s.dp_tiles > 0 &&
      P.num_ctas == info.sms / P.ranks && !a_ready)
    P.die_aware = die_table(dev, strm, P.ranks, &P) ? 1 : 0;

  if (is_f16(kern)) {
    const int cg = kernel_cg(kern);
    const CUtensorMapDataType dt = d->ab_type == SK_BFLOAT16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUtensorMap ta, tb, tc;
    const int bks = f16_stage_k();  // smem stage k-depth (A rows of bks elements)
    st = make_tmap(&ta, dt, 2, d->A, d->problem.m, d->problem.k, d->lda, static_cast<uint32_t>(bks), 128,
                   bks == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
    if (st) return st;
    st = make_tmap(&tb, dt, 2, d->B, d->problem.k, d->problem.n, d->ldb, 64, static_cast<uint32_t>(bks),
                   CU_TENSOR_MAP_SWIZZLE_128B);
    if (st) return st;
    st = make_tmap(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d->C, d->problem.m, d->problem.n,
                   d->ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (st) return st;
    P.idesc = make_idesc_f16(d->ab_type == SK_BFLOAT16, 128 * cg, 256);
    const cudaError_t e = launch_f16(cg, kernel_bn(kern), P.cluster_fix > 1 ? P.cluster_fix * cg : cg, ta, tb, tc, P,
                                     static_cast<int>(P.num_ctas), strm);
    if (e != cudaSuccess) return cuda_fail(e, cg == 2 ? "sk_gemm_f16<2> launch" : "sk_gemm_f16<1> launch");
    return SK_OK;
  }
  if (kern == Kernel::F64) {
    CUtensorMap ta, tb;
    st = make_tmap(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, d->A, d->problem.m, d->problem.k,
                   d->lda, 16, 64, CU_TENSOR_MAP_SWIZZLE_128B);
    if (st) return st;
    st = make_tmap(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, d->B, d->problem.k, d->problem.n,
                   d->ldb, 16, 16, CU_TENSOR_MAP_SWIZZLE_128B);
    if (st) return st;
    const cudaError_t e =
        launch_f64(ta, tb, static_cast<double*>(d->C), d->ldc, P, static_cast<int>(P.num_ctas), strm);
    if (e != cudaSuccess) return cuda_fail(e, "sk_gemm_f64 launch");
    return SK_OK;
  }
  return fail(SK_EUNSUPPORTED, "kernel not available");
}
}  // namespace

// ---------------------------------------------------------------------------
// sk_execute: streamk::execute<T> with host buffers (executor.hpp:130-207).
// ---------------------------------------------------------------------------
namespace {

struct ExecCache {
  int device = -1;
  cudaStream_t stream = nullptr;
  // transfer pipelining: copy-in and copy-out streams, ordering events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in = nullptr, ev_flags = nullptr;
  void* buf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // A, B, C, ws, staging, row flags
  size_t cap[6] = {0, 0, 0, 0, 0, 0};
  size_t ws_valid = 0;  // bytes of ws known to be zeroed
  ~ExecCache() { release(); }
  void release() {
    if (device >= 0) cudaSetDevice(device);
    for (int i = 0; i < 6; ++i) {
      if (buf[i]) cudaFree(buf[i]);
      buf[i] = nullptr;
      cap[i] = 0;
    }
    for (cudaStream_t* q : {&stream, &s_in, &s_out}) {
      if (*q) cudaStreamDestroy(*q);
      *q = nullptr;
    }
    for (cudaEvent_t* e : {&ev_in, &ev_flags}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
    device = -1;
    ws_valid = 0;
  }
  sk_status ensure(int i, size_t bytes) {
    if (cap[i] >= bytes) return SK_OK;
    if (buf[i]) cudaFree(buf[i]);
    buf[i] = nullptr;
    cap[i] = 0;
    SK_CUDA(cudaMalloc(&buf[i], bytes));
    cap[i] = bytes;
    if (i == 3) ws_valid = 0;
    return SK_OK;
  }
};
thread_local ExecCache g_exec;

// cuStreamWaitValue32 (driver API, through the runtime's entry-point query).
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32 wait_value32() {
  static PFN_waitValue32 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_waitValue32>(nullptr);
    return reinterpret_cast<PFN_waitValue32>(p);
  }();
  return fn;
}

// Pitched copy that degenerates to one linear copy when both pitches equal the width.
cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                      int64_t rows, cudaMemcpyKind kind, cudaStream_t q) {
  if (dpitch == width && spitch == width)
    return cudaMemcpyAsync(dst, src, width * static_cast<size_t>(rows), kind, q);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, static_cast<size_t>(rows), kind, q);
}

typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32 write_value32() {
  static PFN_writeValue32 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_writeValue32>(nullptr);
    return reinterpret_cast<PFN_writeValue32>(p);
  }();
  return fn;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Transfer pipelining for sk_execute (pinned host buffers, no conversion): A
// arrives by tile rows and B by panels of W tile columns on a copy stream, each
// followed by a flag the producer waits on (a_ready[row], b_ready[panel]), in
// the order the persistent traversal first needs them; every finished block of
// C (G tile rows x W tile columns, counted by c_done[block]) leaves on a second
// copy stream (cuStreamWaitValue32) while the kernel still runs.  G is the data-
// parallel raster height, so a raster group's first wave needs only its G rows
// of A and the first few panels of B, and C starts leaving after the first
// group's columns instead of after all of B (profiles/r01d/pipeline_blocks.txt).
// The FP64 kernel keeps whole-B-first, row blocks of C (G = 1, W = tiles_n).
// The schedule is the caller's: only copy order follows it.
sk_status execute_pipelined(ExecCache& X, sk_gemm_desc& d, size_t ws_bytes, const void* A,
                            const void* B, void* C, size_t esz, size_t csz, bool zero_c) {
  Kernel kern;
  Schedule s;
  sk_status st = check_desc(&d, &kern, &s);
  if (st) return st;
  const int64_t m = d.problem.m, n = d.problem.n, k = d.problem.k;
  const int64_t bm = d.blocking.blk_m, bn = d.blocking.blk_n;
  const int64_t rows = s.tiles_m, cols = s.tiles_n;
  const bool f64 = kern == Kernel::F64;
  PipeFlags pf;
  // Block geometry: G = 1 / W = all columns is the whole-B-first, row-block
  // scheme (kept for FP64); the tcgen05 kernels use 8 x 8 tile blocks, 2 %
  // faster at 8192^3 (8.39-8.48 vs 8.60-8.66 ms; profiles/r01d/pipeline_blocks.txt):
  // the call is bound by bidirectional PCIe, not by when C starts to leave.
  int64_t G = f64 ? 1 : 8, W = f64 ? cols : 8;
  if (!f64) {
    if (knobs().pipe_g > 0) G = knobs().pipe_g;
    if (knobs().pipe_w > 0) W = knobs().pipe_w;
  }
  pf.raster = std::min<int64_t>(rows, G);
  pf.g = static_cast<int>(pf.raster);
  pf.w = static_cast<int>(std::min<int64_t>(cols, W));
  pf.np = static_cast<int>((cols + pf.w - 1) / pf.w);
  const int64_t groups = (rows + pf.g - 1) / pf.g, blocks = groups * pf.np;
  // stores per tile: one per epilogue warp of each CTA of the pair (tcgen05), one (DMMA)
  const uint32_t incr = f64 ? 1u : static_cast<uint32_t>(kernel_ranks(kern) * f16_epilogue_warps(kernel_bn(kern)));
  std::vector<uint32_t> target(static_cast<size_t>(blocks), 0);
  std::vector<int64_t> firstA(static_cast<size_t>(rows), INT64_MAX), firstB(static_cast<size_t>(pf.np), INT64_MAX);
  std::vector<int64_t> lastC(static_cast<size_t>(blocks), -1);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t P = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(s.grid_size, 1),
                                                           f64 ? 2 * sms : sms / kernel_ranks(kern)));
  const int order = phase_order_for(kern);
  // Data-parallel tiles in "growing square" block order: block (group, panel)
  // shells of max(group, panel), each new B panel's blocks, then each new A
  // group's, so every 32-MB input that lands completes more blocks of C and the
  // copy-out never starves (profiles/r01d/pipeline_blocks.txt).  Row-major ids.
  std::vector<int32_t> perm;
  if (!f64) {
    const int64_t R = groups, Cp = pf.np;
    std::vector<std::pair<int64_t, int64_t>> border;
    for (int64_t sh = 0; sh < std::max(R, Cp); ++sh) {
      if (sh < Cp)
        for (int64_t gi = 0; gi < std::min(sh, R); ++gi) border.emplace_back(gi, sh);
      if (sh < R)
        for (int64_t pj = 0; pj <= std::min(sh, Cp - 1); ++pj) border.emplace_back(sh, pj);
    }
    for (auto& bp : border)
      for (int64_t tc = bp.second * pf.w; tc < std::min(cols, (bp.second + 1) * pf.w); ++tc)
        for (int64_t tr = bp.first * pf.g; tr < std::min(rows, (bp.first + 1) * pf.g); ++tr)
          if (tr * cols + tc < s.dp_tiles) perm.push_back(static_cast<int32_t>(tr * cols + tc));
  }
  const int32_t* hperm = perm.empty() ? nullptr : perm.data();
  for (int64_t cta = 0; cta < P; ++cta) {
    int64_t t = 0;
    for_each_segment(s, cta, P, pf.raster, [&](int64_t, int64_t tile, int64_t lb, int64_t le) {
      int64_t tr, tc;
      s.tile_rc(tile, &tr, &tc);
      const size_t blk = static_cast<size_t>(tr / pf.g * pf.np + tc / pf.w);
      firstA[static_cast<size_t>(tr)] = std::min(firstA[static_cast<size_t>(tr)], t);
      firstB[static_cast<size_t>(tc / pf.w)] = std::min(firstB[static_cast<size_t>(tc / pf.w)], t);
      t += le - lb;
      if (lb == 0) {
        lastC[blk] = std::max(lastC[blk], t);
        target[blk] += incr;
      }
    }, order, hperm);
  }
  std::vector<int64_t> out_order(static_cast<size_t>(blocks));
  for (int64_t b = 0; b < blocks; ++b) out_order[static_cast<size_t>(b)] = b;
  std::stable_sort(out_order.begin(), out_order.end(), [&](int64_t x, int64_t y) {
    return lastC[static_cast<size_t>(x)] < lastC[static_cast<size_t>(y)];
  });
  // Copy-in order: by the first C block (in copy-out order) an item feeds, then
  // by first need -- the copy-out is the long pole, so the inputs of the first
  // block to leave come first (profiles/r01d/pipeline_blocks.txt).
  std::vector<int64_t> pos(static_cast<size_t>(blocks));
  for (int64_t i = 0; i < blocks; ++i) pos[static_cast<size_t>(out_order[static_cast<size_t>(i)])] = i;
  std::vector<int64_t> feedA(static_cast<size_t>(rows), INT64_MAX), feedB(static_cast<size_t>(pf.np), INT64_MAX);
  for (int64_t tr = 0; tr < rows; ++tr)
    for (int64_t tc = 0; tc < cols; ++tc) {
      const int64_t p = pos[static_cast<size_t>(tr / pf.g * pf.np + tc / pf.w)];
      feedA[static_cast<size_t>(tr)] = std::min(feedA[static_cast<size_t>(tr)], p);
      feedB[static_cast<size_t>(tc / pf.w)] = std::min(feedB[static_cast<size_t>(tc / pf.w)], p);
    }
  // items: (first block fed, first need, kind 0 = A row / -1 = B panel, index)
  std::vector<std::tuple<int64_t, int64_t, int, int64_t>> items4;
  for (int64_t r = 0; r < rows; ++r)
    items4.emplace_back(feedA[static_cast<size_t>(r)], firstA[static_cast<size_t>(r)], 0, r);
  for (int64_t q = 0; q < pf.np; ++q)
    items4.emplace_back(feedB[static_cast<size_t>(q)], firstB[static_cast<size_t>(q)], -1, q);
  std::stable_sort(items4.begin(), items4.end());
  std::vector<std::tuple<int64_t, int, int64_t>> items;
  for (auto& it4 : items4) items.emplace_back(std::get<1>(it4), std::get<2>(it4), std::get<3>(it4));

  st = X.ensure(5, sizeof(int) * static_cast<size_t>(rows + pf.np + blocks + perm.size()));
  if (st) return st;
  int* a_ready = static_cast<int*>(X.buf[5]);
  int* b_ready = a_ready + rows;
  int* c_done = b_ready + pf.np;
  int32_t* dperm = c_done + blocks;
  pf.a_ready = a_ready;
  pf.b_ready = b_ready;
  pf.c_done = c_done;
  pf.perm = perm.empty() ? nullptr : dperm;
  if (!X.s_in) {
    SK_CUDA(cudaStreamCreateWithFlags(&X.s_in, cudaStreamNonBlocking));
    SK_CUDA(cudaStreamCreateWithFlags(&X.s_out, cudaStreamNonBlocking));
    SK_CUDA(cudaEventCreateWithFlags(&X.ev_in, cudaEventDisableTiming));
    SK_CUDA(cudaEventCreateWithFlags(&X.ev_flags, cudaEventDisableTiming));
  }
  cudaStream_t sm = X.stream, si = X.s_in, so = X.s_out;
  // flags down before the kernel and the copy-out waits see them
  SK_CUDA(cudaMemsetAsync(a_ready, 0, sizeof(int) * static_cast<size_t>(rows + pf.np + blocks), si));
  if (!perm.empty())  // pageable source: staged by the runtime before the call returns
    SK_CUDA(cudaMemcpyAsync(dperm, perm.data(), sizeof(int32_t) * perm.size(), cudaMemcpyHostToDevice, si));
  SK_CUDA(cudaEventRecord(X.ev_in, si));
  SK_CUDA(cudaStreamWaitEvent(sm, X.ev_in, 0));
  SK_CUDA(cudaStreamWaitEvent(so, X.ev_in, 0));
  d.A = X.buf[0];
  d.B = X.buf[1];
  d.C = X.buf[2];
  if (zero_c) SK_CUDA(cudaMemsetAsync(X.buf[2], 0, static_cast<size_t>(m * d.ldc) * csz, sm));
  // SKB200_PIPE_TRACE=1: event after every copy and the kernel, printed to
  // stderr in ms from the call's start (profiles/r01d/pipeline_blocks.txt)
  const bool trace = knobs().pipe_trace != 0;
  std::vector<std::pair<std::string, cudaEvent_t>> tev;
  auto mark = [&](const std::string& what, cudaStream_t q) {
    if (!trace) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) == cudaSuccess) {
      cudaEventRecord(e, q);
      tev.emplace_back(what, e);
    }
  };
  mark("start", si);
  st = gemm_impl(&d, X.buf[3], ws_bytes, sm, &pf);
  if (st) return st;
  mark("kernel_end", sm);
  // a stream memory op, not a memset kernel: nothing may need an SM the
  // persistent GEMM is holding
  auto raise = [&](const int* flag) -> sk_status {
    const CUresult cr = write_value32()(reinterpret_cast<CUstream>(si), reinterpret_cast<CUdeviceptr>(flag),
                                        1, CU_STREAM_WRITE_VALUE_DEFAULT);
    return cr == CUDA_SUCCESS ? SK_OK : fail(SK_ECUDA, "cuStreamWriteValue32 failed (%d)", int(cr));
  };
  const uint8_t* Ah = static_cast<const uint8_t*>(A);
  const uint8_t* Bh = static_cast<const uint8_t*>(B);
  uint8_t* Ad = static_cast<uint8_t*>(X.buf[0]);
  uint8_t* Bd = static_cast<uint8_t*>(X.buf[1]);
  // Consecutive A row blocks travel as one copy of up to ~16 MB (per-copy gaps
  // cost more than the later first row, profiles/r01/pipeline.txt).
  const int64_t max_rows = std::max<int64_t>(1, (int64_t(16) << 20) / std::max<int64_t>(1, bm * k * static_cast<int64_t>(esz)));
  for (size_t i = 0; i < items.size();) {
    const int kind = std::get<1>(items[i]);
    const int64_t idx = std::get<2>(items[i]);
    if (kind != 0) {  // B panel: W tile columns x all k rows (2-D copy)
      const int64_t c0 = idx * pf.w * bn, nc = std::min<int64_t>(c0 + pf.w * bn, n) - c0;
      SK_CUDA(copy_rows(Bd + static_cast<size_t>(c0) * esz, d.ldb * esz, Bh + static_cast<size_t>(c0) * esz,
                        n * esz, nc * esz, k, cudaMemcpyHostToDevice, si));
      if ((st = raise(b_ready + idx))) return st;
      mark("B_panel_" + std::to_string(idx), si);
      ++i;
      continue;
    }
    size_t j = i + 1;
    while (j < items.size() && std::get<1>(items[j]) == 0 &&
           std::get<2>(items[j]) == std::get<2>(items[j - 1]) + 1 && static_cast<int64_t>(j - i) < max_rows)
      ++j;
    const int64_t r0 = idx * bm, nr = std::min(std::get<2>(items[j - 1]) * bm + bm, m) - r0;
    SK_CUDA(copy_rows(Ad + static_cast<size_t>(r0 * d.lda) * esz, d.lda * esz,
                      Ah + static_cast<size_t>(r0 * k) * esz, k * esz, k * esz, nr,
                      cudaMemcpyHostToDevice, si));
    for (size_t q = i; q < j; ++q)
      if ((st = raise(a_ready + std::get<2>(items[q])))) return st;
    mark("A_rows_" + std::to_string(idx) + "-" + std::to_string(std::get<2>(items[j - 1])), si);
    i = j;
  }
  // copy-out: each block of C once all of its stores have landed
  uint8_t* Ch = static_cast<uint8_t*>(C);
  const uint8_t* Cd = static_cast<const uint8_t*>(X.buf[2]);
  PFN_waitValue32 wv = wait_value32();
  for (int64_t b : out_order) {
    if (!target[static_cast<size_t>(b)]) {
      // nothing stores this block (explicit tables that leave tiles unstarted):
      // the reference returns zeros there (its fresh C, matrix.hpp:22)
      if (zero_c) {
        const int64_t r0 = (b / pf.np) * pf.g * bm, nr = std::min(r0 + pf.g * bm, m) - r0;
        const int64_t c0 = (b % pf.np) * pf.w * bn, nc = std::min(c0 + pf.w * bn, n) - c0;
        uint8_t* Cz = static_cast<uint8_t*>(C);
        for (int64_t r = r0; r < r0 + nr; ++r)
          memset(Cz + static_cast<size_t>(r * n + c0) * csz, 0, static_cast<size_t>(nc) * csz);
      }
      continue;
    }
    const CUresult cr = wv(reinterpret_cast<CUstream>(so), reinterpret_cast<CUdeviceptr>(c_done + b),
                           target[static_cast<size_t>(b)], CU_STREAM_WAIT_VALUE_GEQ);
    if (cr != CUDA_SUCCESS) return fail(SK_ECUDA, "cuStreamWaitValue32 failed (%d)", int(cr));
    const int64_t r0 = (b / pf.np) * pf.g * bm, nr = std::min(r0 + pf.g * bm, m) - r0;
    const int64_t c0 = (b % pf.np) * pf.w * bn, nc = std::min(c0 + pf.w * bn, n) - c0;
    SK_CUDA(copy_rows(Ch + static_cast<size_t>(r0 * n + c0) * csz, n * csz,
                      Cd + static_cast<size_t>(r0 * d.ldc + c0) * csz, d.ldc * csz, nc * csz, nr,
                      cudaMemcpyDeviceToHost, so));
    mark("C_block_" + std::to_string(b), so);
  }
  SK_CUDA(cudaStreamSynchronize(si));
  SK_CUDA(cudaStreamSynchronize(so));
  if (trace && !tev.empty()) {
    cudaDeviceSynchronize();
    for (auto& te : tev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0].second, te.second);
      fprintf(stderr, "[pipe] %8.3f ms %s\n", ms, te.first.c_str());
    }
    for (auto& te : tev) cudaEventDestroy(te.second);
  }
  return sk_workspace_check(X.buf[3], sm);
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace

namespace {
sk_status execute_impl(const sk_problem* p, const sk_blocking* b, sk_strategy strategy,
                       int64_t param, const int64_t* ranges, int64_t num_ranges,
                       sk_dtype host_type, sk_dtype compute_type, int32_t variant, const void* A,
                       const void* B, void* C, int32_t device) {
  if (!p || !b || !A || !B || !C) return fail(SK_EINVAL, "null argument");
  if (compute_type != SK_BFLOAT16 && compute_type != SK_FLOAT16 && compute_type != SK_FLOAT64)
    return fail(SK_EUNSUPPORTED, "compute_type %d has no device kernel", compute_type);
  const bool is16 = compute_type != SK_FLOAT64;
  if (is16 && !(host_type == compute_type || host_type == SK_FLOAT32))
    return fail(SK_EINVAL, "host_type must equal compute_type or be FLOAT32");
  if (!is16 && host_type != SK_FLOAT64 && host_type != SK_FLOAT32 && host_type != SK_INT64)
    return fail(SK_EINVAL, "FP64 compute takes FLOAT64, FLOAT32 or INT64 host data");
  if (!is16 && host_type == SK_INT64) {
    // execute<int64_t> on the FP64 tensor path is exact while every partial sum
    // stays below 2^53: max|A| * max|B| * k < 2^53 (the reference band is [-64, 63]).
    auto maxabs = [](const void* p, int64_t cnt) {
      const int64_t* v = static_cast<const int64_t*>(p);
      long double mx = 0;
      for (int64_t i = 0; i < cnt; ++i) mx = std::max(mx, std::fabs(static_cast<long double>(v[i])));
      return mx;
    };
    const long double bound = maxabs(A, p->m * p->k) * maxabs(B, p->k * p->n) *
                              static_cast<long double>(p->k);
    if (bound >= 9007199254740992.0L)
      return fail(SK_EUNSUPPORTED, "int64 operands exceed the exact fp64 range (max|A|max|B|k >= 2^53)");
  }

  const int64_t m = p->m, n = p->n, k = p->k;
  if (m < 1 || n < 1 || k < 1) return fail(SK_EINVAL, "GemmProblem extents must be >= 1");
  const size_t esz = dtype_size(compute_type), csz = is16 ? 4 : 8;
  // Pitched device copies: ld rounded up to 16 bytes for TMA.
  const int64_t lda = round_up(k, 16 / static_cast<int64_t>(esz));
  const int64_t ldb = round_up(n, 16 / static_cast<int64_t>(esz));
  const int64_t ldc = round_up(n, 16 / static_cast<int64_t>(csz));

  sk_gemm_desc d{};
  d.problem = *p;
  d.blocking = *b;
  d.strategy = strategy;
  d.param = param;
  d.ab_type = compute_type;
  d.variant = variant;
  d.lda = lda;
  d.ldb = ldb;
  d.ldc = ldc;
  d.ranges = ranges;
  d.num_ranges = num_ranges;
  size_t ws_bytes = 0;
  sk_status st = sk_workspace_size(&d, &ws_bytes);
  if (st) return st;
  // A fresh C is zero (matrix.hpp:22): only explicit tables can leave tiles unwritten.
  const bool zero_c = strategy == SK_EXPLICIT && !g_xt.all_started;

  int dev = device;
  if (dev < 0) SK_CUDA(cudaGetDevice(&dev));
  ExecCache& X = g_exec;
  if (X.device != dev) {
    X.release();
    SK_CUDA(cudaSetDevice(dev));
    SK_CUDA(cudaStreamCreateWithFlags(&X.stream, cudaStreamNonBlocking));
    X.device = dev;
  } else {
    SK_CUDA(cudaSetDevice(dev));
  }

  st = X.ensure(0, static_cast<size_t>(m * lda) * esz);
  if (!st) st = X.ensure(1, static_cast<size_t>(k * ldb) * esz);
  if (!st) st = X.ensure(2, static_cast<size_t>(m * ldc) * csz);
  if (!st) st = X.ensure(3, ws_bytes);
  if (st) return st;
  cudaStream_t s = X.stream;
  if (X.ws_valid < ws_bytes) {
    st = sk_workspace_init(X.buf[3], X.cap[3], s);
    if (st) return st;
    X.ws_valid = X.cap[3];
  }
  // Overlapped transfers: pinned host buffers, no element conversion, > 1 tile row.
  {
    const bool same = is16 ? host_type == compute_type : host_type == SK_FLOAT64;
    if (same && knobs().pipeline != 0 && m > b->blk_m && wait_value32() && write_value32() && is_pinned(A) &&
        is_pinned(B) && is_pinned(C))
      return execute_pipelined(X, d, ws_bytes, A, B, C, esz, csz, zero_c);
  }
  if (host_type == SK_FLOAT32 && is16) {
    // H2D fp32, round-to-nearest-even into the pitched 16-bit operand buffers.
    st = X.ensure(4, static_cast<size_t>(std::max(m * k, k * n)) * 4);
    if (st) return st;
    float* stg = static_cast<float*>(X.buf[4]);
    SK_CUDA(cudaMemcpyAsync(stg, A, sizeof(float) * m * k, cudaMemcpyHostToDevice, s));
    SK_CUDA(launch_f32_to_16(stg, X.buf[0], m, k, lda, compute_type == SK_BFLOAT16, s));
    SK_CUDA(cudaMemcpyAsync(stg, B, sizeof(float) * k * n, cudaMemcpyHostToDevice, s));
    SK_CUDA(launch_f32_to_16(stg, X.buf[1], k, n, ldb, compute_type == SK_BFLOAT16, s));
  } else if (!is16 && host_type != SK_FLOAT64) {
    // execute<float> / execute<int64_t> on the FP64 path: widen exactly on the device.
    const size_t hs = dtype_size(host_type);
    st = X.ensure(4, static_cast<size_t>(std::max(std::max(m * k, k * n), m * n)) * 8);
    if (st) return st;
    const int kind = host_type == SK_FLOAT32 ? 0 : 1;
    SK_CUDA(cudaMemcpyAsync(X.buf[4], A, hs * m * k, cudaMemcpyHostToDevice, s));
    SK_CUDA(launch_convert(kind, X.buf[4], k, X.buf[0], lda, m, k, s));
    SK_CUDA(cudaMemcpyAsync(X.buf[4], B, hs * k * n, cudaMemcpyHostToDevice, s));
    SK_CUDA(launch_convert(kind, X.buf[4], n, X.buf[1], ldb, k, n, s));
  } else {
    SK_CUDA(cudaMemcpy2DAsync(X.buf[0], lda * esz, A, k * esz, k * esz, m, cudaMemcpyHostToDevice, s));
    SK_CUDA(cudaMemcpy2DAsync(X.buf[1], ldb * esz, B, n * esz, n * esz, k, cudaMemcpyHostToDevice, s));
  }
  d.A = X.buf[0];
  d.B = X.buf[1];
  d.C = X.buf[2];
  if (zero_c) SK_CUDA(cudaMemsetAsync(X.buf[2], 0, static_cast<size_t>(m * ldc) * csz, s));
  st = sk_gemm(&d, X.buf[3], ws_bytes, s);
  if (st) return st;
  if (!is16 && host_type != SK_FLOAT64) {
    // narrow the fp64 C to the caller's element type, tightly packed, then D2H
    const size_t hs = dtype_size(host_type);
    SK_CUDA(launch_convert(host_type == SK_FLOAT32 ? 2 : 3, X.buf[2], ldc, X.buf[4], n, m, n, s));
    SK_CUDA(cudaMemcpyAsync(C, X.buf[4], hs * m * n, cudaMemcpyDeviceToHost, s));
  } else {
    SK_CUDA(cudaMemcpy2DAsync(C, n * csz, X.buf[2], ldc * csz, n * csz, m, cudaMemcpyDeviceToHost, s));
  }
  return sk_workspace_check(X.buf[3], s);
}
}  // namespace

extern "C" sk_status sk_execute(const sk_problem* p, const sk_blocking* b, sk_strategy strategy,
                                int64_t param, sk_dtype host_type, sk_dtype compute_type,
                                int32_t variant, const void* A, const void* B, void* C,
                                int32_t device) {
  if (strategy == SK_EXPLICIT) return fail(SK_EINVAL, "SK_EXPLICIT: use sk_execute_ranges");
  return execute_impl(p, b, strategy, param, nullptr, 0, host_type, compute_type, variant, A, B,
                      C, device);
}

extern "C" sk_status sk_execute_ranges(const sk_problem* p, const sk_blocking* b,
                                       const int64_t* ranges, int64_t num_ranges,
                                       sk_dtype host_type, sk_dtype compute_type, int32_t variant,
                                       const void* A, const void* B, void* C, int32_t device) {
  return execute_impl(p, b, SK_EXPLICIT, num_ranges, ranges, num_ranges, host_type, compute_type,
                      variant, A, B, C, device);
}

extern "C" void sk_execute_release(void) { g_exec.release(); }

extern "C" sk_status sk_cluster_capacity(sk_variant variant, int32_t cluster, int32_t device,
                                         int32_t* units) {
  if (!units || cluster < 2 || cluster > 8) return fail(SK_EINVAL, "clusters of 2 to 8 units");
  if (variant != SK_VARIANT_1SM && variant != SK_VARIANT_2SM)
    return fail(SK_EUNSUPPORTED, "the cluster fixup runs on the 1-SM and 2-SM 256-wide kernels");
  *units = 0;
  int dev = device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(SK_ECUDA, "no CUDA device");
  }
  DeviceInfo info;
  sk_status st = device_info(dev, &info);
  if (st) return st;
  if (info.cc_major != 10 || info.cc_minor != 0) return fail(SK_EUNSUPPORTED, "sm_100a only");
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != dev) SK_CUDA(cudaSetDevice(dev));
  const Kernel kern = variant == SK_VARIANT_1SM ? Kernel::F16_1SM : Kernel::F16_2SM;
  int resident = 0;
  st = resident_units(dev, info, kern, &resident);  // kernel attributes first
  if (!st) *units = cluster_units(dev, info, kern, cluster);
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  return st;
}

extern "C" sk_status sk_persistent_capacity(sk_dtype ab_type, sk_variant variant, int32_t device,
                                            int32_t* units) {
  if (!units) return fail(SK_EINVAL, "null output");
  sk_gemm_desc d{};
  d.ab_type = ab_type;
  d.variant = variant;
  Kernel k;
  sk_status st = pick_kernel(&d, &k);
  if (st) return st;
  int dev = device;
  if (dev < 0) SK_CUDA(cudaGetDevice(&dev));
  int cur = 0;
  SK_CUDA(cudaGetDevice(&cur));
  SK_CUDA(cudaSetDevice(dev));
  DeviceInfo info;
  st = device_info(dev, &info);
  int n = 0;
  if (!st) st = resident_units(dev, info, k, &n);
  cudaSetDevice(cur);
  if (st) return st;
  *units = n;
  return SK_OK;
}

extern "C" void sk_reload_env(void) {
  std::lock_guard<std::mutex> lk(g_knob_mu);
  g_knobs = read_knobs();
  g_knobs_loaded = true;
}
