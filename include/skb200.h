/*
 * skb200.h -- C ABI of the B200-native Stream-K GEMM (libskb200.so).
 *
 * This is the drop-in boundary for the reference's GEMM hot path
 * (/root/reference/proj, "streamk-lab"):
 *
 *   reference (C++ templates, header-only)         this ABI (extern "C", POD only)
 *   -----------------------------------------------------------------------------
 *   tile_grid            types.cpp:45-55            sk_tile_grid
 *   iter_to_coords       types.cpp:57-62            sk_iter_to_coords
 *   data_parallel / fixed_split / stream_k / hybrid
 *                        decompose.cpp:38-121       sk_schedule
 *   fixup_peers_of       decompose.cpp:123-136      sk_fixup_peers
 *   quantization_efficiency decompose.cpp:138-141   sk_quantization_efficiency
 *   execute<T>(assignment, A, B, threads)
 *                        executor.hpp:130-207       sk_execute   (host buffers, synchronous)
 *                                                   sk_gemm      (device buffers, stream-ordered)
 *   detail::FixupStore   executor.hpp:95-119        sk_workspace_size / sk_workspace_init /
 *                                                   sk_workspace_check (device fixup slabs + flags)
 *
 * Conventions mirror the reference: row-major A (m x k), B (k x n), C (m x n);
 * tiles linearised row-major over (tiles_m, tiles_n); C = A * B with alpha/beta
 * ignored exactly as executor.hpp:142,179 ignores them.  Exceptions become status
 * codes: std::invalid_argument -> SK_EINVAL, std::out_of_range -> SK_ERANGE,
 * std::logic_error (double signal) -> SK_EPROTOCOL.  No C++ types cross the ABI.
 *
 * Threading: every entry point is reentrant.  Per-device state (SM count, kernel
 * attributes) is initialised lazily under a mutex; sk_execute keeps one
 * device-buffer cache per host thread.  Workspaces belong to the caller.
 */
#ifndef SKB200_H_
#define SKB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKB200_ABI_VERSION 5

typedef enum sk_status {
  SK_OK = 0,
  SK_EINVAL = 1,        /* std::invalid_argument in the reference */
  SK_EUNSUPPORTED = 2,  /* valid for the reference, not for this kernel (blocking, alignment) */
  SK_ECUDA = 3,         /* CUDA runtime / driver error; see sk_last_error() */
  SK_EPROTOCOL = 4,     /* fixup protocol violation: double signal or wait watchdog */
  SK_ERANGE = 5,        /* std::out_of_range (iter_to_coords) */
  SK_ECAPACITY = 6,     /* caller buffer too small; the required size is still reported */
  SK_EIO = 7            /* std::runtime_error of the SKMX reader/writer; see sk_io_error() */
} sk_status;

/* Strategy tags: types.hpp:70 Strategy / decompose.hpp:9 HybridVariant. */
typedef enum sk_strategy {
  SK_DATA_PARALLEL = 0,
  SK_FIXED_SPLIT = 1,   /* param = s */
  SK_STREAM_K = 2,      /* param = g */
  SK_DP_ONE_TILE_SK = 3, /* param = p */
  SK_TWO_TILE_SK_DP = 4, /* param = p */
  SK_EXPLICIT = 5        /* an arbitrary range table (sk_gemm_desc.ranges / sk_execute_ranges):
                            a WorkAssignment no closed form produces, e.g. from from_text
                            (types.cpp:109-123).  Not accepted by sk_schedule/sk_fixup_peers. */
} sk_strategy;

typedef enum sk_dtype {
  SK_INT64 = 0,    /* reference DType::Int64 (CPU-only in the reference; no device kernel) */
  SK_FLOAT32 = 1,  /* reference DType::Float32 */
  SK_FLOAT64 = 2,  /* reference DType::Float64 */
  SK_BFLOAT16 = 3, /* tensor-core input types (accumulate and store in FLOAT32) */
  SK_FLOAT16 = 4
} sk_dtype;

/* Kernel family: one tile configuration per precision. */
typedef enum sk_variant {
  SK_VARIANT_AUTO = 0, /* the kernel whose tile equals the blocking; 2-SM by default */
  SK_VARIANT_1SM = 1, /* BF16/FP16: 128x256x64, tcgen05 cta_group::1, persistent grid = #SMs */
  SK_VARIANT_2SM = 2, /* BF16/FP16: 256x256x64, tcgen05 cta_group::2, persistent grid = #SMs/2 pairs */
  SK_VARIANT_2SM_WIDE = 3 /* BF16/FP16: 256x512x64, two N=256 cta_group::2 MMAs share each A stage
                             (48 instead of 64 B of operands per SM per MAC step); one TMEM
                             accumulator, so the epilogue does not overlap the mainloop */
} sk_variant;

/* types.hpp:20-27.  alpha/beta carried but ignored (executor.hpp:142,179). */
typedef struct sk_problem {
  int64_t m, n, k;
  double alpha, beta;
} sk_problem;

/* types.hpp:30-34 */
typedef struct sk_blocking {
  int64_t blk_m, blk_n, blk_k;
} sk_blocking;

/* types.hpp:41-47 */
typedef struct sk_tile_grid_t {
  int64_t tiles_m, tiles_n, total_tiles, iters_per_tile, total_iters;
} sk_tile_grid_t;

/* Device GEMM descriptor for sk_gemm.  All pointers are device pointers owned
 * by the caller; leading dimensions are in elements. */
typedef struct sk_gemm_desc {
  sk_problem problem;
  sk_blocking blocking; /* must equal sk_kernel_blocking(ab_type, variant) */
  int32_t strategy;     /* sk_strategy */
  int32_t ab_type;      /* SK_BFLOAT16 | SK_FLOAT16 | SK_FLOAT64 */
  int64_t param;        /* s, g or p (ignored for data_parallel) */
  int32_t variant;      /* sk_variant */
  int32_t num_ctas;     /* persistent CTAs (pairs for 2-SM); 0 = all SMs */
  const void* A;
  int64_t lda;          /* >= k, lda * sizeof(ab) % 16 == 0 */
  const void* B;
  int64_t ldb;          /* >= n, ldb * sizeof(ab) % 16 == 0 */
  void* C;              /* FLOAT32 for BF16/FP16 inputs, FLOAT64 for FP64 */
  int64_t ldc;          /* >= n, ldc * sizeof(c) % 16 == 0 */
  int32_t* trace;       /* optional device buffer, see sk_trace_size(); NULL = off */
  int64_t* cta_clocks;  /* optional device buffer of 4 * grid int64: per launched CTA
                           {clock64 start, globaltimer ns start, clock64 end, globaltimer end} */
  int64_t* events;      /* optional device timeline, 8 int64 per record, see sk_timeline_size:
                           {unit, tile, core, kind, t_mac_start, t_mac_end, t_wait_end, t_done},
                           kind = 1 partial | 2 owner with peers | npeer << 8 |
                           smid << 16 (SM that ran the epilogue); ns */
  /* ABI v2: strategy == SK_EXPLICIT only.  HOST table [num_ranges][2] of
   * (iter_begin, iter_end), row index == cta_id, executed like execute<T> executes
   * assignment.ranges (executor.hpp:147-185).  Validated on every call:
   *   0 <= iter_begin <= iter_end <= total_iters, else SK_EINVAL (mac_loop's
   *   invalid_argument, executor.hpp:63-68);
   *   a tile started (local k = 0) by two ranges -> SK_EINVAL (the reference
   *   would wait forever: each starter waits on the other);
   *   a starter with a lower-id peer -> SK_EUNSUPPORTED (its wait would point
   *   to a lower id, which a persistent grid cannot order; every closed-form
   *   schedule has all waits pointing up, executor.hpp:124-129).
   * Tiles no range starts are not written (the reference leaves them zero in its
   * fresh C; sk_execute_ranges zero-fills).  The table (ranges + peer lists) is
   * copied into the workspace tail (sk_workspace_size counts it) and re-copied
   * only when the workspace last ran a different table. */
  const int64_t* ranges;
  int64_t num_ranges;
  /* ABI v3: which block of C a tile id denotes.
   *   0 (default) or 1: the reference's row-major map, tile -> (tile / tiles_n,
   *     tile % tiles_n) (executor.hpp:69-70,173-174).  Data-parallel units are
   *     still visited in a grouped raster order (temporal order only).
   *   G > 1: ids run through groups of G tile rows, column-major inside a group
   *     (an opt-in locality layout: ids, ranges, owners and peers stay the
   *     reference's, but the block of C an id denotes does not).  Clamped to
   *     tiles_m.  Ignored by explicit tables, the pipelined sk_execute and FP64.
   *   -1: G = the data-parallel raster height (the round-1 default). */
  int32_t tile_group;
  int32_t reserved0; /* must be 0 */
} sk_gemm_desc;

const char* sk_status_string(sk_status status);
/* Thread-local detail string for the last non-OK status on this thread. */
const char* sk_last_error(void);
int sk_abi_version(void);

/* ---- integer schedule (host, closed form; bit-exact with decompose.cpp) ---- */
sk_status sk_tile_grid(const sk_problem* problem, const sk_blocking* blocking,
                       sk_tile_grid_t* out);
sk_status sk_iter_to_coords(const sk_tile_grid_t* grid, int64_t i, int64_t* tile_idx,
                            int64_t* local_iter);
/* Writes the grid size to *grid_size and, when ranges != NULL and capacity >= g,
 * the [g][2] (iter_begin, iter_end) table; row index == cta_id. */
sk_status sk_schedule(const sk_problem* problem, const sk_blocking* blocking,
                      sk_strategy strategy, int64_t param, int64_t* grid_size, int64_t* ranges,
                      int64_t capacity);
/* fixup_peers_of as CSR: offsets[total_tiles + 1], ids[nnz] ascending per tile.
 * ids may be NULL to query *nnz. */
sk_status sk_fixup_peers(const sk_problem* problem, const sk_blocking* blocking,
                         sk_strategy strategy, int64_t param, int64_t* offsets, int64_t* ids,
                         int64_t capacity, int64_t* nnz);
sk_status sk_quantization_efficiency(int64_t t, int64_t p, double* out);

/* ---- geometry corpus (sweep.cpp:21-28, 79-86) ---------------------------- */
/* The paper's log-sampled shape corpus in run_sweep order: out[4*i] =
 * {m, n, k, matrix_seed} of sample i, dims = clamp(llround(exp(ln lo + u (ln hi -
 * ln lo))), lo, hi) with u from SplitMix64(seed); matrix_seed = next(). */
sk_status sk_corpus(uint64_t seed, int64_t count, int64_t lo, int64_t hi, uint64_t* out);

/* ---- SKMX matrix files (matrix.hpp:70-93, matrix.cpp:13-61) --------------- */
/* 16-byte LE header "SKMX", u32 dtype tag, u32 rows, u32 cols; row-major payload. */
sk_status sk_save_matrix(const char* path, sk_dtype dtype, int64_t rows, int64_t cols,
                         const void* data);
sk_status sk_load_matrix_header(const char* path, sk_dtype* dtype, int64_t* rows, int64_t* cols);
/* dtype tag must equal `expect` (else SK_EIO, the reference's runtime_error). */
sk_status sk_load_matrix(const char* path, sk_dtype expect, int64_t rows, int64_t cols, void* data);
const char* sk_io_error(void);

/* ---- grid-size model (costmodel.hpp:13-60, wave-aware) -------------------- */
/* time(g) = e + ceil(g/p) * (a + b*[peers>1] + c*ipc + d*(peers-1) + s*segs), microseconds;
 * segs = tile segments per unit.  margin: minimum predicted Stream-K gain over
 * data-parallel before select_grid_size leaves g = t.  sk_calibrate keeps the
 * caller's margin and writes the RMS relative fit error to fit_residual. */
typedef struct sk_cost_params {
  double e, a, b, c, d, s;
  double margin;
  double fit_residual;
  /* > 0: the kernel's cooperative fixup (g <= p, tiles of >= 8 contributors)
   * costs like coop_peers + contributors / 8 serial peer folds, not peers - 1
   * (0 = the reference's model: the owner folds every peer). */
  double coop_peers;
  /* > 0: the kernel's cluster fixup (fixed_split(S), S in {8, 4, 3, 2}; the
   * kernel runs any 2 <= S <= 8), the S
   * k-chunks of a tile reduced through DSMEM) is a candidate of
   * sk_select_schedule when every chunk is nonempty, the largest chunk has at
   * least this many iterations and t * S units are co-resident as clusters of S
   * on the current device (sk_cluster_capacity); 0 = not a candidate. */
  double cluster_min_iters;
  double cluster_kernel; /* the sk_variant those constants describe (1 or 2) */
} sk_cost_params;
/* B200-calibrated constants for a kernel family. */
sk_status sk_default_cost_params(sk_dtype ab_type, sk_variant variant, sk_cost_params* out);
sk_status sk_predict_time(const sk_cost_params* params, const sk_tile_grid_t* grid, int64_t g,
                          int64_t p, double* out);
/* argmin over g in {1..p} U {t} (costmodel.cpp:30-48); g == t is data-parallel. */
sk_status sk_select_grid_size(const sk_cost_params* params, const sk_tile_grid_t* grid, int64_t p,
                              int64_t* g);
/* Predicted time of data_parallel, stream_k(param) or two_tile_sk_dp(param). */
sk_status sk_predict_schedule(const sk_cost_params* params, const sk_tile_grid_t* grid,
                              int32_t strategy, int64_t param, int64_t p, double* out);
/* The Stream-K policy: argmin over data_parallel, stream_k(1..p) and
 * two_tile_sk_dp(p); data-parallel unless another wins by > margin.  With
 * cluster_min_iters > 0, fixed_split(S) on the cluster fixup is taken first
 * when it applies (largest S), measured faster on 95 % of such shapes. */
sk_status sk_select_schedule(const sk_cost_params* params, const sk_tile_grid_t* grid, int64_t p,
                             int32_t* strategy, int64_t* param);
/* Non-negative least squares over n >= 6 measured (grid, g, time) samples. */
sk_status sk_calibrate(const sk_tile_grid_t* grids, const int64_t* g, const double* times,
                       int64_t n, int64_t p, sk_cost_params* out);

/* ---- device GEMM -------------------------------------------------------- */
/* The tile configuration the device kernel uses for an input type/variant. */
sk_status sk_kernel_blocking(sk_dtype ab_type, sk_variant variant, sk_blocking* out);
/* Bytes of device workspace (fixup flags + fp32/fp64 partial slabs). */
sk_status sk_workspace_size(const sk_gemm_desc* desc, size_t* bytes);
/* Zero a workspace once after allocation (stream-ordered).  The kernel leaves
 * it zeroed again after every successful launch (self-cleaning flags). */
sk_status sk_workspace_init(void* workspace, size_t bytes, void* stream);
/* Synchronises the stream, reads and clears the workspace error word. */
sk_status sk_workspace_check(void* workspace, void* stream);
/* Ints needed for the optional ownership trace: per tile id {owner, last_peer,
 * storing_unit, segments}, then per unit {partials_emitted}, then per block of C
 * in row-major block order (tile_row * tiles_n + tile_col) {unit that stored it}
 * -- 5 * total_tiles + grid_size ints.  The block section shows the tile -> C
 * map actually used (executor.hpp:69-70 under the default tile_group). */
sk_status sk_trace_size(const sk_gemm_desc* desc, int64_t* ints);
/* Records of the optional device timeline: grid_size * seg_stride (record of
 * unit u's i-th tile segment at u * seg_stride + i; unused records stay zero). */
sk_status sk_timeline_size(const sk_gemm_desc* desc, int64_t* records, int64_t* seg_stride);
/* Two-die topology of a device as the die-aware schedule sees it (probed once
 * per device, synchronising): *ok = 1 and die_of_sm[0..*sms) in {0, 1} when
 * the device shows a clean two-die split with TPC-aligned 2-CTA clusters, else
 * *ok = 0.  die_of_sm may be NULL; at most max_sms entries are written. */
sk_status sk_device_topology(int device, int32_t* die_of_sm, int32_t max_sms, int32_t* sms,
                             int32_t* ok);
/* The persistent sequence CTA (pair) `cta` of a `num_ctas`-CTA launch of
 * `desc` walks -- producer, MMA issuer and epilogue all follow it: records of
 * {unit, tile, local_begin, local_end} (executor.hpp:149-185 segments), at
 * most max_records written, *count = the sequence length.  Host-side. */
sk_status sk_persistent_order(const sk_gemm_desc* desc, int64_t num_ctas, int64_t cta,
                              int64_t* out, int64_t max_records, int64_t* count);
/* The block of C (tile row, tile column) that tile id `tile` denotes in a
 * launch of `desc`: row-major like executor.hpp:69-70 unless desc->tile_group
 * selects the grouped layout (tcgen05 kernels, closed-form schedules). */
sk_status sk_tile_block(const sk_gemm_desc* desc, int64_t tile, int64_t* tile_row, int64_t* tile_col);
/* Co-resident capacity of the persistent kernel for (ab_type, variant) on
 * `device` (< 0: current): CTAs for the 1-SM and FP64 kernels, CTA pairs for
 * the 2-SM kernel.  sk_gemm never launches a larger persistent grid, so every
 * unit a fixup wait points to is resident.  Sets the kernel's per-device
 * attributes on first use. */
sk_status sk_persistent_capacity(sk_dtype ab_type, sk_variant variant, int32_t device, int32_t* units);
/* Units (CTAs of the 1-SM kernel, CTA pairs of the 2-SM kernel) co-resident
 * as clusters of `cluster` units (2 to 8) on `device` (-1 = current): the
 * capacity of the cluster fixup, fixed_split(S) with t * S <= units. */
sk_status sk_cluster_capacity(sk_variant variant, int32_t cluster, int32_t device, int32_t* units);
/* Stream-ordered, asynchronous.  Does not synchronise. */
sk_status sk_gemm(const sk_gemm_desc* desc, void* workspace, size_t workspace_bytes,
                  void* stream);

/* ---- reference-facing drop-in of streamk::execute<T> ------------------- */
/* Host buffers in, host C out (tight row-major, ld = cols), synchronous.
 * compute_type BFLOAT16/FLOAT16: host_type is the same 16-bit type (raw bits)
 *   or FLOAT32 (rounded to nearest on the device); C is float32.
 * compute_type FLOAT64 (tensor-core DMMA): host_type FLOAT64 (C double),
 *   FLOAT32 (widened exactly, C float -- execute<float> without input rounding)
 *   or INT64 (C int64, exact; SK_EUNSUPPORTED unless max|A| max|B| k < 2^53 --
 *   execute<int64_t>).
 * Device buffers, workspace and the stream are cached per host thread.
 * device < 0 = current device. */
sk_status sk_execute(const sk_problem* problem, const sk_blocking* blocking,
                     sk_strategy strategy, int64_t param, sk_dtype host_type,
                     sk_dtype compute_type, int32_t variant, const void* A, const void* B,
                     void* C, int32_t device);
/* sk_execute over an explicit range table ([num_ranges][2], see sk_gemm_desc.ranges):
 * the drop-in for execute<T> on an arbitrary WorkAssignment.  C is zero-filled
 * first when some tile has no starting range, like the reference's fresh C. */
sk_status sk_execute_ranges(const sk_problem* problem, const sk_blocking* blocking,
                            const int64_t* ranges, int64_t num_ranges, sk_dtype host_type,
                            sk_dtype compute_type, int32_t variant, const void* A,
                            const void* B, void* C, int32_t device);
/* fixup_peers_of (decompose.cpp:123-136) of an explicit range table, CSR as in
 * sk_fixup_peers; validates the ranges like sk_gemm (bounds only). */
sk_status sk_fixup_peers_ranges(const sk_problem* problem, const sk_blocking* blocking,
                                const int64_t* ranges, int64_t num_ranges, int64_t* offsets,
                                int64_t* ids, int64_t capacity, int64_t* nnz);
/* Releases the calling thread's sk_execute cache. */
void sk_execute_release(void);

/* ---- reference input generator (matrix.hpp:39-68), on the device ---------- */
/* Fills the pitched device buffer dst (rows x cols, ld elements) with
 * random_matrix<gen_type>(rows, cols, seed): element i (row-major) is the i-th
 * SplitMix64 draw, as (next() & 0x7f) - 64 for SK_INT64 (then >> shift,
 * arithmetic), (float)(u * 2 - 1) for SK_FLOAT32 and u * 2 - 1 for SK_FLOAT64
 * (u = (next() >> 11) * 2^-53), rounded to nearest-even into out_type
 * (SK_BFLOAT16 | SK_FLOAT16 | SK_FLOAT32 | SK_FLOAT64; FLOAT64 generation only
 * into FLOAT32/FLOAT64).  Stream-ordered. */
sk_status sk_random_matrix(sk_dtype gen_type, int32_t shift, uint64_t seed, int64_t rows,
                           int64_t cols, sk_dtype out_type, void* dst, int64_t ld, void* stream);

/* ---- simulator (simulate.cpp:23-80) --------------------------------------- */
/* Reference CostParams (costmodel.hpp:13-19): a fixed per-unit cost, b partial
 * output cost, c per-iteration cost, d per-peer reduction cost. */
typedef struct sk_sim_params {
  double a, b, c, d;
} sk_sim_params;
/* Greedy list scheduling of the schedule's units in cta_id order onto p cores
 * (earliest free, lowest index on ties).  params NULL: unit cost (1 per MAC
 * iteration, zero-length fixups).  Writes the makespan, the utilization (sum of
 * MAC durations / (p * makespan); SK_EINVAL for an empty timeline, as the
 * reference throws) and, when events != NULL, up to `capacity` records of 6
 * doubles {core, cta, kind (0 mac, 2 fixup_reduce), start, end, tile}.
 * strategy SK_EXPLICIT takes the [num_ranges][2] table. */
sk_status sk_simulate(const sk_problem* problem, const sk_blocking* blocking, sk_strategy strategy,
                      int64_t param, const int64_t* ranges, int64_t num_ranges, int64_t p,
                      const sk_sim_params* params, double* makespan, double* utilization,
                      double* events, int64_t capacity, int64_t* num_events);

/* Re-reads the SKB200_* tuning overrides from the environment (they are read
 * once, at the first launch; DESIGN.md lists them). */
void sk_reload_env(void);

#ifdef __cplusplus
}
#endif
#endif /* SKB200_H_ */
