// sk_gemm_f16.cu -- persistent, warp-specialised Stream-K GEMM for sm_100a.
//
// C (fp32, m x n) = A (bf16|fp16, m x k, row-major) * B (bf16|fp16, k x n, row-major)
// under any of the reference's five decompositions (decompose.cpp:38-121).
//
// Replaces the reference executor (executor.hpp:130-207):
//   mac_loop (executor.hpp:59-88)     -> TMA producer warp -> smem ring -> tcgen05.mma
//                                        issuer, fp32 accumulator in TMEM
//   FixupStore (executor.hpp:95-119)  -> fp32 slabs in global memory + int flags with
//                                        release/acquire (sk_kernel_common.cuh)
//   owner fold + StoreTile (:164-181) -> epilogue warps: TMEM -> regs (+ peer slabs in
//                                        ascending id) -> swizzled smem -> TMA store
//   worker loop (:187-193)            -> persistent grid (sk_kernel_common.cuh)
//
// Kernels (sk_gemm_f16<CG, BN, CF>), one tile config each:
//   CG = 1, BN = 256: 1-SM, tile 128x256x64, tcgen05.mma.cta_group::1 M=128 N=256,
//           grid = #SMs
//   CG = 2, BN = 256: 2-SM, tile 256x256x64, tcgen05.mma.cta_group::2 M=256 N=256 on
//           a CTA pair (cluster ranks 2i, 2i+1), grid = #SMs/2 pairs.  Each CTA of
//           the pair loads its own 128 rows of A and its own 128 columns of B; the
//           leader issues the MMA for both and every CTA drains its own 128 lanes.
//   CG = 2, BN = 512: the wide 2-SM tile 256x512x64: two N=256 MMAs per k step
//           share each A stage (48 instead of 64 B of operands per SM per MAC
//           step); one 512-column TMEM accumulator, handed back by halves.
//   CF = true (BN = 256): the cluster-fixup instantiation for fixed_split(S),
//           2 <= S <= 8, launches whose t*S units fit as clusters of S units: a
//           tile's S k-chunks reduce through DSMEM inside their cluster.
//
// Warp roles (192 threads, 1 CTA per SM):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + tcgen05.mma issuer (one lane; leader CTA only for CG=2)
//   warps 2..5  epilogue; warp w drains TMEM lanes 32*(w%4) .. +31
// Smem ring: STAGES k-blocks of A (rows x 64, K-major, 128B swizzle) and B
// (64 x cols as 64x64 boxes, MN-major, 128B swizzle).  TMEM (BN = 256): two
// 256-column fp32 accumulators, so one segment's epilogue overlaps the next
// mainloop.  All roles walk the same SegmentIter sequence (sk_kernel_common.cuh);
// tile ids denote C blocks through Schedule::tile_rc (the reference's row-major
// map unless grouped ids are requested).  Fixup: the owner folds its peers
// (executor.hpp order); schedules of >= 8 contributors per tile, one unit per
// CTA: every contributor publishes and folds a column share (coop_fold); the
// cluster fixup above.  Pieces of a tile outside C are skipped throughout.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ptx.cuh"
#include "schedule.hpp"
#include "sk_kernel_common.cuh"

namespace skb200 {
namespace f16 {

constexpr int ROWS = 128;  // rows per CTA (= TMEM lanes)
constexpr int MMA_N = 256; // N of one tcgen05.mma; a tile is BN / MMA_N of them side by side
constexpr int BK = 64;  // k-depth of one Stream-K iteration (the blocking factor)
// k-depth of one smem stage: 64 (one iteration) or 32 (half-depth stages: twice
// as many, released after 2 MMAs instead of 4, A in 64-B swizzle).
#ifndef SKB200_STAGE_K
#define SKB200_STAGE_K 64
#endif
constexpr int BKS = SKB200_STAGE_K;
constexpr int SUB = BK / BKS;
static_assert(BKS == 64 || BKS == 32, "stage k-depth 64 or 32");
constexpr int UMMA_K = 16;
// Epilogue warps: 4 (one per TMEM lane quarter) or 8 (two per quarter, each
// draining half of the 256 accumulator columns -- twice the loads/stores in
// flight for the fixup fold and the partial/C stores).  Measured on B200
// (profiles/r01/epilogue_warps.txt): 8 warps speed the Stream-K fold ~15 % but
// cost data-parallel ~1 %, because end-of-kernel fixups are L2-bandwidth-bound
// rather than latency-bound; 4 is the default.
#ifndef SKB200_EPI_WARPS
#define SKB200_EPI_WARPS 4
#endif
#ifndef SKB200_EPI_BUFS
#define SKB200_EPI_BUFS (SKB200_EPI_WARPS == 8 ? 1 : 2)
#endif
constexpr int EPI_WARPS = SKB200_EPI_WARPS;
// -DSKB200_DISCARD: drop consumed fixup-slab lines from L2 (discard.global.L2)
// instead of letting them age out.  Off: the discards sit on the owner's fold
// path and cost more than the write-backs they save -- Stream-K picks on the
// 225 near-regression corpus shapes 1.006x -> 1.024x of DP, 9 -> 0 shapes more
// than 5 % slower, config 3 1.40 -> 1.42, 8192^3 unchanged
// (profiles/r02/epilogue_ab.txt).

// Epilogue warps of the wide tile (A/B knob): 8 = two per TMEM lane quarter,
// interleaved by 64-column steps so both drain half 0 first.  Measured slower
// than 4 (8192^3 hybrid 1561 vs 1574 TFLOP/s, the inter-tile gap unchanged:
// profiles/r03b/), so 4.
#ifndef SKB200_EPI_WARPS_WIDE
#define SKB200_EPI_WARPS_WIDE 4
#endif
static_assert(EPI_WARPS == 4 || EPI_WARPS == 8, "4 or 8 epilogue warps");
// SPLIT_RELEASE (wide tile): hand each accumulator half back to the MMA warp as
// soon as it is read (A/B knob; measured in profiles/r02k/README.txt).
#ifndef SKB200_SPLIT_RELEASE
#define SKB200_SPLIT_RELEASE 1
#endif
#ifndef SKB200_EPI_BUFS_WIDE
#define SKB200_EPI_BUFS_WIDE SKB200_EPI_BUFS
#endif
constexpr int EPI_BUF_BYTES = 32 * 32 * 4;  // 32 rows x 32 fp32 = 4 KB
constexpr int TMEM_COLS = 512;                    // all of TMEM: 512 fp32 columns x 128 lanes
constexpr int B_BOX_BYTES = 64 * BKS * 2;         // BKS k-rows x 64 cols

// Tile width BN: 256 (one MMA, two TMEM accumulators so a tile's epilogue
// overlaps the next mainloop) or, 2-SM only, 512 ("wide": two N = 256 MMAs
// share every A stage, so a CTA loads 48 B of operands per 128x512x64 MAC step
// instead of 64; one accumulator fills TMEM, so the epilogue no longer overlaps).
template <int CG, int BN>
struct Cfg {
  static_assert(BN == 256 || (BN == 512 && CG == 2), "tile widths: 256, 512 (2-SM)");
  static constexpr int NMMA = BN / MMA_N;                   // MMAs per 16-deep k step
  static constexpr int BPM = MMA_N / CG / 64;               // 64-col B boxes per MMA per CTA
  static constexpr int NACC = TMEM_COLS / BN;               // TMEM accumulators
  static constexpr int EPI_WARPS = BN == 512 ? SKB200_EPI_WARPS_WIDE : SKB200_EPI_WARPS;
  static constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;   // 192 (4 epilogue warps) or 320
  static constexpr int EPI_COLS = BN / (EPI_WARPS / 4);     // accumulator columns per epilogue warp
  static constexpr int SLAB_ELEMS = ROWS * BN;              // fp32 partial per CTA rank
  static constexpr int B_COLS = BN / CG;                    // B columns held per CTA
  // 4-KB TMA-store staging boxes per epilogue warp
  static constexpr int EPI_BUFS = EPI_WARPS == 8 ? 1 : (BN == 512 ? SKB200_EPI_BUFS_WIDE : SKB200_EPI_BUFS);
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_BUFS * EPI_BUF_BYTES;
  static constexpr int A_STAGE = ROWS * BKS * 2;            // 16 KB (BKS = 64)
  static constexpr int B_STAGE = B_COLS * BKS * 2;          // 32 KB (1-SM) / 16 KB (2-SM)
  static constexpr int STAGE = A_STAGE + B_STAGE;
#ifndef SKB200_STAGES_1SM
#define SKB200_STAGES_1SM 4
#endif
#ifndef SKB200_STAGES_2SM
#define SKB200_STAGES_2SM 6
#endif
#ifndef SKB200_STAGES_WIDE
#define SKB200_STAGES_WIDE 4
#endif
  static constexpr int STAGES =
      (CG == 1 ? SKB200_STAGES_1SM : (BN == 512 ? SKB200_STAGES_WIDE : SKB200_STAGES_2SM)) * SUB;
  static constexpr int a_off = 0;
  static constexpr int b_off = a_off + STAGES * A_STAGE;
  static constexpr int epi_off = b_off + STAGES * B_STAGE;
  static constexpr int bar_off = epi_off + EPI_BYTES;
  static constexpr int bar_bytes = (2 * STAGES + 5) * 8 + 16;
  static constexpr int alloc = bar_off + bar_bytes + 1024;  // + runtime 1 KB alignment
  static_assert(alloc <= 232448, "smem budget");
};

// Slab layout: for chunk c (32 cols) and float4 column-group j (0..7), the 128
// rows are contiguous, so a warp's 32 lanes move 512 contiguous bytes per access.
__device__ __forceinline__ float4* slab_ptr(float* slab, int c, int j, int row) {
  return reinterpret_cast<float4*>(slab) + ((c * 8 + j) * ROWS + row);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctas() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// shared::cluster address of `p`'s twin in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(ptx::smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_to_leader(void* dst, const CUtensorMap* m,
                                                      uint32_t bar_cluster_addr, int32_t c0,
                                                      int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster_addr), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void st_shared_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr)
               : "memory");
}

// Epilogue probe (experiments only, -DSKB200_EPI_PROBE): per (CTA, epilogue
// warp) globaltimer stamps of the warp's last segment in cta_clocks[16 * slot].
#ifdef SKB200_EPI_PROBE
#define EPI_STAMP(slot)                                                                              \
  do {                                                                                               \
    if (P.cta_clocks && lane == 0)                                                                   \
      P.cta_clocks[(static_cast<int64_t>(blockIdx.x) * EPI_WARPS + (warp - 2)) * 16 + (slot)] =      \
          static_cast<long long>(ptx::globaltimer());                                                \
  } while (0)
#else
#define EPI_STAMP(slot) \
  do {                  \
  } while (0)
#endif

// Column (relative to the tile) of this CTA's B box i: MMA i / BPM, this CTA's
// 256 / CG columns of it, 64-column box i % BPM.
template <int CG, int BN>
__device__ __forceinline__ int32_t b_col_of(int i, uint32_t rank) {
  using K = Cfg<CG, BN>;
  return (i / K::BPM) * MMA_N + static_cast<int32_t>(rank) * (MMA_N / CG) + 64 * (i % K::BPM);
}

template <int CG, int BN, bool CF>  // CF: the cluster-fixup instantiation (fixed_split over DSMEM)
__global__ void __launch_bounds__(Cfg<CG, BN>::NUM_THREADS, 1)
    sk_gemm_f16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const KernelParams P) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using K = Cfg<CG, BN>;
  constexpr int EPI_COLS = K::EPI_COLS;
  constexpr int EPI_WARPS = K::EPI_WARPS;
  constexpr int SLAB_ELEMS = K::SLAB_ELEMS;
  constexpr int EPI_BUFS = K::EPI_BUFS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem + K::a_off;
  uint8_t* sB = smem + K::b_off;
  float* sEpi = reinterpret_cast<float*>(smem + K::epi_off);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + K::bar_off);
  uint64_t* empty_bar = full_bar + K::STAGES;
  uint64_t* tfull_bar = empty_bar + K::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* xfix_bar = tempty_bar + 2;  // cluster fixup: peers' accumulators are in their smem
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(xfix_bar + 1);
  int* lane_code_smem = reinterpret_cast<int*>(tmem_base_smem + 1);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const Schedule& s = P.s;
  // 2-SM: a CTA pair is cluster ranks (2i, 2i + 1) -- the tcgen05 peer CTAs; a
  // cluster holds one pair, or S pairs under the cluster fixup.
  const uint32_t crank = CG == 2 ? cluster_rank() : 0;
  const uint32_t rank = crank & 1u;        // rank inside the pair
  const uint32_t pair_base = crank & ~1u;  // cluster rank of the pair's leader
  const bool leader_cta = rank == 0;
  const int64_t cta = CG == 2 ? static_cast<int64_t>(cluster_id_x()) * (cluster_nctas() / 2) + crank / 2
                              : static_cast<int64_t>(blockIdx.x);
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << pair_base);
  auto b_col = [rank](int i) { return b_col_of<CG, BN>(i, rank); };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmC);
    for (int i = 0; i < K::STAGES; ++i) {
      ptx::mbar_init(&full_bar[i], 1);
      ptx::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull_bar[i], 1);
      ptx::mbar_init(&tempty_bar[i], EPI_WARPS * CG);
    }
    if (CF) ptx::mbar_init(xfix_bar, EPI_WARPS * (P.cluster_fix - 1));
    ptx::fence_barrier_init();
    // Die-aware DP lane (die_lane): keyed by the leader CTA's SM, shared with the peer.
    if (P.die_aware && leader_cta) {
      const int code = P.die_tab[ptx::smid()];
      *lane_code_smem = code;
      if constexpr (CG == 2) st_shared_cluster(mapa(lane_code_smem, pair_base + 1), code);
    }
  }
  if (warp == 1) ptx::tmem_alloc<CG>(tmem_base_smem, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  // peer barriers initialised before any remote use
  if (CG == 2 || CF) cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  DpLane dp_lane = default_lane(s, cta, P.num_ctas);
  if (P.die_aware) {
    const int code = *lane_code_smem;
    if (code >= 0) dp_lane = die_lane(s, P.die_n, code);
    else if (threadIdx.x == 0) atomicOr(P.err, kErrTopology);  // host validated: unreachable
  }
  // Programmatic dependent launch: the prologue above overlaps the previous
  // kernel's tail; nothing below touches global memory before it completes.
  ptx::grid_dependency_wait();
  ptx::launch_dependents();
#ifndef SKB200_EPI_PROBE
  stamp_clock(P, 0);
#endif

  if (warp == 0) {
    // ===================== TMA producer (every CTA of the pair) =====================
    if (lane == 0) {
      const uint64_t pol_a = ptx::make_policy(P.l2_policy[0]);
      const uint64_t pol_b_dp = ptx::make_policy(P.l2_policy[1]);
      const uint64_t pol_b_sk = ptx::make_policy(P.l2_policy[3]);
      uint32_t stage = 0, phase = 0;
      for_each_segment(s, cta, P.num_ctas, dp_lane, P.raster_rows,
                       [&](int64_t u, int64_t tile, int64_t lb, int64_t le) {
        int64_t tr, tc;
        s.tile_rc(tile, &tr, &tc);
        const int32_t m0 = static_cast<int32_t>(tr * (ROWS * CG) + rank * ROWS);
        const int32_t n0 = static_cast<int32_t>(tc * BN);
        // B panels stream through a data-parallel wave but are revisited at
        // unrelated k offsets by Stream-K units: separate L2 priorities.
        const bool sk_unit = s.strategy == kFixedSplit || s.bal.contains_id(u);
        const uint64_t pol_b = sk_unit ? pol_b_sk : pol_b_dp;
        if (P.a_ready) {  // row block of A (and column panel of B) in HBM
          wait_flag(P, P.a_ready + tr);
          if (P.b_ready) wait_flag(P, P.b_ready + tc / P.pipe_w);
        }
        // k order of a balanced unit's segments (P.k_align): see k_block_of.
        int64_t rot = -1;
        if (P.k_align && sk_unit && s.strategy != kFixedSplit) {
          int64_t b, e;
          s.range(u, &b, &e);
          rot = k_rotation(s, b, e, tile, lb, le);
        }
        for (int64_t i = lb; i < le; ++i) {
          const int64_t kb = rot < 0 ? i : k_block_of(s.ipt, lb, le, rot, i - lb);
          for (int h = 0; h < SUB; ++h) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          const int32_t k0 = static_cast<int32_t>(kb * BK + h * BKS);
          uint8_t* a_dst = sA + stage * K::A_STAGE;
          uint8_t* b_dst = sB + stage * K::B_STAGE;
          if constexpr (CG == 1) {
            ptx::mbar_expect_tx(&full_bar[stage], K::STAGE);
            ptx::tma_load_2d(a_dst, &tmA, &full_bar[stage], k0, m0, pol_a);
#pragma unroll
            for (int i = 0; i < K::B_COLS / 64; ++i)
              ptx::tma_load_2d(b_dst + i * B_BOX_BYTES, &tmB, &full_bar[stage], n0 + b_col(i), k0, pol_b);
          } else {
            // Both CTAs' bytes land on the leader's full barrier; only the leader arrives.
            if (leader_cta) ptx::mbar_expect_tx(&full_bar[stage], 2 * K::STAGE);
            const uint32_t fb = mapa(&full_bar[stage], pair_base);
            tma_load_2d_to_leader(a_dst, &tmA, fb, k0, m0, pol_a);
#pragma unroll
            for (int i = 0; i < K::B_COLS / 64; ++i)
              tma_load_2d_to_leader(b_dst + i * B_BOX_BYTES, &tmB, fb, n0 + b_col(i), k0, pol_b);
          }
          if (++stage == K::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          }
        }
      }, P.sk_first, P.dp_perm);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    if (lane == 0 && leader_cta) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      // One k step (BKS deep) of MMAs j0 .. j1-1 on smem stage `stg`; step index
      // `si` within the segment (0 = first: overwrite the accumulator).
      auto issue = [&](uint32_t d_tmem, uint32_t stg, int64_t si, int j0, int j1) {
        const uint32_t a0 = ptx::smem_u32(sA + stg * K::A_STAGE);
        const uint32_t b0 = ptx::smem_u32(sB + stg * K::B_STAGE);
#pragma unroll
        for (int kk = 0; kk < BKS / UMMA_K; ++kk) {
          // A: K-major, swizzle = row bytes (128 B at BKS 64, 64 B at 32), +32 B per
          // 16-element k step; SBO = 8 rows x row bytes.
          const uint64_t ad = BKS == 64 ? ptx::make_sdesc_sw128(a0 + kk * 32, 16, 1024)
                                        : ptx::make_sdesc_sw64(a0 + kk * 32, 16, 512);
          // B: MN-major SW128, +16 k-rows x 128 B per k step; LBO = next 64-col box,
          // SBO = 8 k-rows x 128 B.  MMA j reads this CTA's boxes j * BPM ..; its
          // accumulator is TMEM columns j * 256 ..
#pragma unroll
          for (int j = 0; j < K::NMMA; ++j) {
            if (j < j0 || j >= j1) continue;
            const uint64_t bd =
                ptx::make_sdesc_sw128(b0 + j * K::BPM * B_BOX_BYTES + kk * 2048, B_BOX_BYTES, 1024);
            ptx::umma_f16<CG>(d_tmem + j * MMA_N, ad, bd, P.idesc, (si > 0 || kk > 0) ? 1u : 0u);
          }
        }
      };
      auto release = [&](uint32_t stg) {  // free the smem slot once these MMAs have read it
        if constexpr (CG == 1) ptx::umma_commit(&empty_bar[stg]);
        else ptx::umma_commit_mc(&empty_bar[stg], pair_mask);
      };
      auto advance = [&]() {
        if (++stage == K::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      };
      for_each_segment(s, cta, P.num_ctas, dp_lane, P.raster_rows,
                       [&](int64_t u, int64_t tile, int64_t lb, int64_t le) {
        const int64_t nsteps = (le - lb) * SUB;
        const uint32_t d_tmem = tmem_base + acc * BN;
        int64_t si = 0;
        if constexpr (K::NACC == 1) {
          // One accumulator (wide tile): the epilogue frees its two 256-column
          // halves one after the other.  Start the segment on half 0 alone for up
          // to STAGES steps (the ring holds them), then run those steps' half-1
          // MMAs once half 1 is drained.  Each half still sees k in order.
          ptx::mbar_wait(&tempty_bar[0], acc_phase ^ 1);
          ptx::tc_fence_after();
          if (long long* ev = event_slot(P, u, tile)) ev[kEvMacStart] = ptx::globaltimer();
          const int64_t d = nsteps < K::STAGES ? nsteps : K::STAGES;
          uint32_t st = stage, ph = phase;
          for (int64_t i = 0; i < d; ++i) {
            ptx::mbar_wait(&full_bar[st], ph);
            ptx::tc_fence_after();
            issue(d_tmem, st, i, 0, 1);
            if (++st == K::STAGES) {
              st = 0;
              ph ^= 1;
            }
          }
          ptx::mbar_wait(&tempty_bar[1], acc_phase ^ 1);
          ptx::tc_fence_after();
          for (; si < d; ++si) {
            issue(d_tmem, stage, si, 1, K::NMMA);
            release(stage);
            advance();
          }
        } else {
          ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          ptx::tc_fence_after();
          if (long long* ev = event_slot(P, u, tile)) ev[kEvMacStart] = ptx::globaltimer();
        }
        for (; si < nsteps; ++si) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          issue(d_tmem, stage, si, 0, K::NMMA);
          release(stage);
          advance();
        }
        // Accumulator ready for the epilogue warps (of both CTAs for CG = 2).
        if constexpr (CG == 1) ptx::umma_commit(&tfull_bar[acc]);
        else ptx::umma_commit_mc(&tfull_bar[acc], pair_mask);
        if (++acc == K::NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }, P.sk_first, P.dp_perm);
    }
    __syncwarp();
  } else {
    // ===================== epilogue =====================
    const uint32_t q = warp % 4;  // TMEM lane quarter this warp may access
    const int row = static_cast<int>(q * 32 + lane);
    const bool leader = (threadIdx.x == 64);
    float* stage_buf = sEpi + (warp - 2) * EPI_BUFS * (EPI_BUF_BYTES / 4);
    float* partials = static_cast<float*>(P.partials);
    const uint64_t pol_c = ptx::make_policy(P.l2_policy[2]);
    uint32_t acc = 0, acc_phase = 0, nstores = 0;
    // flag / slab index of a (unit, rank): each CTA of a pair runs its own protocol
    auto fidx = [&](int64_t u) { return s.slab_of(u) * CG + rank; };
    const int64_t own_base = s.num_slabs * CG;  // cooperative: owners' published accumulators
    const int64_t done_base = 2 * s.num_slabs * CG;
    const int64_t bal_tile0 = s.bal.begin / s.ipt;
    auto slab = [&](int64_t idx) { return partials + idx * static_cast<int64_t>(SLAB_ELEMS); };
    // epilogue warp group (two groups share each TMEM lane quarter with 8 warps)
    const int grp = static_cast<int>((warp - 2) / 4);
    constexpr int NG = EPI_WARPS / 4;
    const int c_lo = grp * (EPI_COLS / 32);  // cooperative fold: this group's contiguous columns
    // One 32x32 fp32 box of C (this warp's rows, 32 columns at n0 + 32 * c): stage
    // through a ring of EPI_BUFS swizzled smem boxes (16-B chunk j of row r at
    // j ^ (r % 8)); EPI_BUFS - 1 TMA stores stay in flight while the next is written.
    auto store_box = [&](const float* v32, int32_t n0, int32_t m0, int c) {
      float* buf = stage_buf + (nstores % EPI_BUFS) * (EPI_BUF_BYTES / 4);
      if (nstores >= EPI_BUFS) {
        if (lane == 0) ptx::tma_store_wait_read<EPI_BUFS - 1>();
        __syncwarp();
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int jj = j ^ static_cast<int>(lane & 7);
        *reinterpret_cast<float4*>(buf + lane * 32 + jj * 4) =
            make_float4(v32[4 * j], v32[4 * j + 1], v32[4 * j + 2], v32[4 * j + 3]);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_2d_hint(&tmC, buf, n0 + c * 32, m0 + static_cast<int32_t>(q * 32), pol_c);
        ptx::tma_store_commit();
      }
      ++nstores;
    };
    // Cooperative fold of one shared tile by contributor u: wait for every
    // contributor's slab, fold the 32-column chunks c = idx, idx + ncon, ...
    // (owner's accumulator, then peers ascending: executor.hpp:165-172), store
    // them, and let the last contributor to finish re-arm the tile's flags.
    auto coop_fold = [&](int64_t u, int64_t tile) {
      int64_t owner, last;
      s.peers(tile, &owner, &last);
      const int ncon = static_cast<int>(last - owner + 1);
      const int idx = static_cast<int>(u - owner);
      int64_t tr, tc;
      s.tile_rc(tile, &tr, &tc);
      const int32_t m0 = static_cast<int32_t>(tr * (ROWS * CG) + rank * ROWS);
      const int32_t n0 = static_cast<int32_t>(tc * BN);
      if (idx < EPI_COLS / 32) {  // else: no chunk to fold (more contributors than chunks)
        if (lane == 0) {
          wait_flag(P, P.flags + own_base + fidx(owner));
          for (int64_t pu = owner + 1; pu <= last; ++pu) wait_flag(P, P.flags + fidx(pu));
        }
        __syncwarp();
        const float* os = slab(own_base + fidx(owner));
        const int c_end = m0 + static_cast<int32_t>(q * 32) >= s.m
                              ? c_lo
                              : imin(c_lo + EPI_COLS / 32, 2 * ceil_div(s.n - n0, 64));
#pragma unroll 1
        for (int c = c_lo + idx; c < c_end; c += ncon) {
          float4 a[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) a[j] = ptx::ld_cg_f4(slab_ptr(const_cast<float*>(os), c, j, row));
          int64_t pu = owner + 1;
#pragma unroll 1
          for (; pu + 1 <= last; pu += 2) {  // two peer slabs in flight, folded in id order
            float* p0 = slab(fidx(pu));
            float* p1 = slab(fidx(pu + 1));
            float4 w0[8], w1[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              w0[j] = ptx::ld_cg_f4(slab_ptr(p0, c, j, row));
              w1[j] = ptx::ld_cg_f4(slab_ptr(p1, c, j, row));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              a[j].x += w0[j].x; a[j].y += w0[j].y; a[j].z += w0[j].z; a[j].w += w0[j].w;
              a[j].x += w1[j].x; a[j].y += w1[j].y; a[j].z += w1[j].z; a[j].w += w1[j].w;
            }
          }
          if (pu <= last) {
            float* p0 = slab(fidx(pu));
            float4 w0[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) w0[j] = ptx::ld_cg_f4(slab_ptr(p0, c, j, row));
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              a[j].x += w0[j].x; a[j].y += w0[j].y; a[j].z += w0[j].z; a[j].w += w0[j].w;
            }
          }
#ifdef SKB200_DISCARD
          // Every lane has consumed the chunk: its slab lines are dead, drop them
          // from L2 without a write-back (lane l: line l of the warp's 4 KB).
          __syncwarp();
          ptx::discard_l2(reinterpret_cast<const char*>(slab_ptr(const_cast<float*>(os), c, lane / 4, q * 32)) +
                          (lane % 4) * 128);
          for (int64_t pd = owner + 1; pd <= last; ++pd)
            ptx::discard_l2(reinterpret_cast<const char*>(slab_ptr(slab(fidx(pd)), c, lane / 4, q * 32)) +
                            (lane % 4) * 128);
#endif
          store_box(reinterpret_cast<const float*>(a), n0, m0, c);
        }
      }
      // every epilogue warp of this CTA has read its slabs: count the contributor
      ptx::named_bar_sync(1, 32 * EPI_WARPS);
      if (leader) {
        int* done = P.flags + done_base + (tile - bal_tile0) * CG + rank;
        __threadfence();
        if (atomicAdd(done, 1) == ncon - 1) {  // the last reader re-arms the tile
          ptx::st_relaxed(P.flags + own_base + fidx(owner), 0);
          for (int64_t pu = owner + 1; pu <= last; ++pu) ptx::st_relaxed(P.flags + fidx(pu), 0);
          ptx::st_relaxed(done, 0);
        }
      }
    };
    int64_t pend0 = 0, pend1 = 0;  // this unit's published shared tiles (at most two)
    int npend = 0;
    for_each_segment(s, cta, P.num_ctas, dp_lane, P.raster_rows,
                     [&](int64_t u, int64_t tile, int64_t lb, int64_t le) {
      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      EPI_STAMP(0);
      long long* ev = (leader && rank == 0) ? event_slot(P, u, tile) : nullptr;
      if (ev) ev[kEvMacEnd] = ptx::globaltimer();
      const uint32_t tsrc = tmem_base + acc * BN + ((q * 32) << 16);
      int64_t tr, tc;
      s.tile_rc(tile, &tr, &tc);
      const int32_t m0 = static_cast<int32_t>(tr * (ROWS * CG) + rank * ROWS);
      const int32_t n0 = static_cast<int32_t>(tc * BN);
      const bool partial = lb != 0;  // not the tile starter (executor.hpp:160)
      if constexpr (CF) {
        {
          // Cluster fixup (fixed_split(S), one unit per CTA / CTA pair): the S
          // units of this cluster are the S k-chunks of this tile, chunk y on
          // unit slot i = S - 1 - y of the cluster (SegmentIter's descending
          // ids), so the owner (y = 0) is slot S - 1; slot i is cluster rank
          // i * CG + (rank in the pair).  1) every CTA parks its 128 accumulator
          // rows in its own (now idle) operand ring as [64 float4 column
          // groups][128 rows]; 2) release-arrive on the barrier of every other
          // slot's CTA holding the same rows; 3) slot i folds column groups
          // [i * 64/S, (i + 1) * 64/S) of all S accumulators through DSMEM,
          // owner first, then y = 1, 2, ... (executor.hpp:165-172: the owner
          // fold's order, so C is bit-identical to it), and TMA-stores them.
          const int S = P.cluster_fix;
          const uint32_t cr = cluster_rank();
          const uint32_t slot = cr / CG, hr = cr % CG;
          float4* park = reinterpret_cast<float4*>(smem);
          const int jn = (BN / 4) / S, j0 = static_cast<int>(slot) * jn;  // S = 2, 4, 8
#pragma unroll 1
          for (int c = 0; c < BN / 32; c += 2) {
            float v[64];
            ptx::tmem_ld64(tsrc + c * 32, v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
              park[(c * 8 + j) * ROWS + row] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          ptx::tc_fence_before();
          ptx::fence_acq_rel_cluster();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) ptx::mbar_arrive(&tempty_bar[acc]);
            else mbar_arrive_remote(mapa(&tempty_bar[acc], pair_base));
            for (int qq = 0; qq < S; ++qq)
              if (qq != static_cast<int>(slot))
                ptx::mbar_arrive_cluster(xfix_bar, static_cast<uint32_t>(qq * CG) + hr);
          }
          ptx::mbar_wait_cluster(xfix_bar, 0);
          const long long t_ready = ev ? static_cast<long long>(ptx::globaltimer()) : 0;
          const bool rows_in = m0 + static_cast<int32_t>(q * 32) < s.m;
          // The fold is DSMEM-latency-bound: each thread's share (64/S column
          // groups x S contributors = 64 float4) is read in two batches of 32
          // loads in flight, folded in y order (owner first), then stored.
          auto fold = [&](auto s_const) {
            constexpr int SS = decltype(s_const)::value;
            constexpr int GPB = 32 / SS;  // column groups per batch
            uint32_t base[SS];
#pragma unroll
            for (int y = 0; y < SS; ++y) base[y] = mapa(park, static_cast<uint32_t>((SS - 1 - y) * CG) + hr);
            float4 a[GPB < 8 ? 8 : GPB];
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int gb = j0 + b * GPB;  // first column group of this batch
              float4 w[SS][GPB];
#pragma unroll
              for (int y = 0; y < SS; ++y)
#pragma unroll
                for (int g = 0; g < GPB; ++g) w[y][g] = ptx::ld_dsmem_f4(base[y] + ((gb + g) * ROWS + row) * 16);
              float4* dst = GPB < 8 ? a + b * GPB : a;
#pragma unroll
              for (int g = 0; g < GPB; ++g) {
                float4 x = w[0][g];
#pragma unroll
                for (int y = 1; y < SS; ++y) {
                  x.x += w[y][g].x; x.y += w[y][g].y; x.z += w[y][g].z; x.w += w[y][g].w;
                }
                dst[g] = x;
              }
              if (GPB >= 8) {  // whole 32-column chunks: store them now
#pragma unroll
                for (int cc = 0; cc < GPB / 8; ++cc)
                  if (n0 + (gb + 8 * cc) * 4 < s.n) store_box(reinterpret_cast<const float*>(a + 8 * cc), n0, m0, (gb + 8 * cc) / 8);
              }
            }
            if (GPB < 8 && n0 + j0 * 4 < s.n) store_box(reinterpret_cast<const float*>(a), n0, m0, j0 / 8);
          };
          // S = 3, 5, 6, 7: slot i folds the whole 32-column boxes
          // [i * 8 / S, (i + 1) * 8 / S) (1-3 boxes; the same boxes the
          // power-of-two split gives for S = 2, 4, 8), one box (S <= 4) or half
          // a box (S > 4) of all S contributors in flight per batch.
          auto fold_boxes = [&](auto s_const) {
            constexpr int SS = decltype(s_const)::value;
            constexpr int GPB = SS <= 4 ? 8 : 4;  // column groups per batch: <= 32 loads in flight
            uint32_t base[SS];
#pragma unroll
            for (int y = 0; y < SS; ++y) base[y] = mapa(park, static_cast<uint32_t>((SS - 1 - y) * CG) + hr);
            const int bx0 = static_cast<int>(slot) * (BN / 32) / SS;
            const int bx1 = (static_cast<int>(slot) + 1) * (BN / 32) / SS;
#pragma unroll 1
            for (int bx = bx0; bx < bx1 && n0 + bx * 32 < s.n; ++bx) {
              float4 a[8];
#pragma unroll
              for (int h = 0; h < 8 / GPB; ++h) {
                const int gb = bx * 8 + h * GPB;
                float4 w[SS][GPB];
#pragma unroll
                for (int y = 0; y < SS; ++y)
#pragma unroll
                  for (int g = 0; g < GPB; ++g) w[y][g] = ptx::ld_dsmem_f4(base[y] + ((gb + g) * ROWS + row) * 16);
#pragma unroll
                for (int g = 0; g < GPB; ++g) {
                  float4 x = w[0][g];
#pragma unroll
                  for (int y = 1; y < SS; ++y) {
                    x.x += w[y][g].x; x.y += w[y][g].y; x.z += w[y][g].z; x.w += w[y][g].w;
                  }
                  a[h * GPB + g] = x;
                }
              }
              store_box(reinterpret_cast<const float*>(a), n0, m0, bx);
            }
          };
          if (rows_in) {
            switch (S) {
              case 2: fold(std::integral_constant<int, 2>{}); break;
              case 3: fold_boxes(std::integral_constant<int, 3>{}); break;
              case 4: fold(std::integral_constant<int, 4>{}); break;
              case 5: fold_boxes(std::integral_constant<int, 5>{}); break;
              case 6: fold_boxes(std::integral_constant<int, 6>{}); break;
              case 7: fold_boxes(std::integral_constant<int, 7>{}); break;
              default: fold(std::integral_constant<int, 8>{}); break;
            }
          }
          if (leader && rank == 0 && P.trace) {  // ownership / partial counts as the reference's protocol
            if (partial) {
              atomicAdd(P.trace + 4 * s.total_tiles + u, 1);
            } else {
              const int npeer = s.npeers(tile, u);
              int* t = P.trace + 4 * tile;
              t[0] = static_cast<int>(u);
              t[1] = static_cast<int>(s.peer(tile, u, npeer));
              t[2] = static_cast<int>(u);
              t[3] = npeer;
              P.trace[4 * s.total_tiles + s.grid_size + tr * s.tiles_n + tc] = static_cast<int>(u);
            }
          }
          if (ev) {  // MacEnd -> parked, every chunk here (WaitEnd) -> folded, stores issued (Done)
            ev[kEvWaitEnd] = t_ready;
            ev[kEvUnit] = u;
            ev[kEvTile] = tile;
            ev[kEvCore] = cta;
            ev[kEvKind] = (partial ? 1 : 2) | (static_cast<long long>(S - 1) << 8) |
                          (static_cast<long long>(ptx::smid()) << 16);
            ev[kEvDone] = ptx::globaltimer();
          }
          if (++acc == K::NACC) {
            acc = 0;
            acc_phase ^= 1;
          }
          return;
        }
      }
      const bool orphan = partial && s.orphan(tile);  // explicit table: nobody folds it
      const int npeer = (!partial && (le < s.ipt || s.strategy == kExplicit)) ? s.npeers(tile, u) : 0;
      // Cooperative schedule: the owner of a shared tile publishes its
      // accumulator like a partial and every contributor folds a share later.
      const bool coop_t = P.coop && (partial || npeer > 0);
      const bool publish = partial || coop_t;
      const int fold_n = coop_t ? 0 : npeer;  // peers this owner folds itself
      if (fold_n > 0) {
        if (lane == 0)
          for (int p = 1; p <= fold_n; ++p) wait_flag(P, P.flags + fidx(s.peer(tile, u, p)));
        __syncwarp();
      }
      if (ev) ev[kEvWaitEnd] = ptx::globaltimer();
      EPI_STAMP(15);
      const int64_t my_idx = partial ? fidx(u) : own_base + fidx(u);
      float* my_slab = publish ? slab(my_idx) : nullptr;
      // 64 columns (two 32-column chunks) per step: one tcgen05.ld.x64, 16 float4
      // of peer slab in flight per thread, two 32x32 TMA-store boxes.
      // Only chunks that hold part of C: this warp's 32 rows and the 64-column
      // steps left of n (ragged edges, skinny m or n); every contributor of the
      // tile skips the same (rows, chunk) pairs, so publish and fold stay matched.
      // 64-column steps c = 2 grp, 2 grp + 2 NG, ... below c_end (32-column chunks).
      const int c_end = (orphan || m0 + static_cast<int32_t>(q * 32) >= s.m)
                            ? 0
                            : imin(BN / 32, 2 * ceil_div(s.n - n0, 64));
      const int c_first = 2 * grp;
      // TMEM hand-back: NACC = 2, the whole accumulator once its last columns are
      // in registers; NACC = 1 (wide), each 256-column half as soon as this warp
      // has read its part of it (the MMA warp restarts on half 0 first).
      auto hand_back = [&](int which) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) ptx::mbar_arrive(&tempty_bar[which]);
          else mbar_arrive_remote(mapa(&tempty_bar[which], pair_base));
        }
      };
      constexpr int H0_END = MMA_N / 32;  // chunks of accumulator half 0
      bool h0_back = K::NACC == 2;  // NACC = 2: no half to hand back separately
      auto hand_back_last = [&]() {  // the whole accumulator is in registers
        if (!h0_back) {
          hand_back(0);
          h0_back = true;
        }
        hand_back(K::NACC == 1 ? 1 : acc);
      };
      constexpr std::true_type kFold{};
      constexpr std::false_type kNoFold{};
      auto after_read = [&](int next) {  // this warp's chunks below `next` are in registers
        if (SKB200_SPLIT_RELEASE && !h0_back && (next >= H0_END || next >= c_end)) {
          hand_back(0);
          h0_back = true;
        }
      };
      // One 64-column step on registers r (chunks c, c + 1): publish, or fold the
      // peers (own accumulator, then peers in ascending id, executor.hpp:165-172)
      // and store.
      auto step = [&](uint32_t (&r)[64], int c, auto fold) {
        float* v = reinterpret_cast<float*>(r);
        EPI_STAMP(1 + 3 * (c / 2 % 4));
        if (!decltype(fold)::value && publish) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            ptx::st_cg_f4(slab_ptr(my_slab, c + j / 8, j % 8, row),
                          make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
          EPI_STAMP(2 + 3 * (c / 2 % 4));
        } else {
#pragma unroll 1
          for (int p = 1; decltype(fold)::value && p <= fold_n; ++p) {
            float* ps = slab(fidx(s.peer(tile, u, p)));
            float4 w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) w[j] = ptx::ld_cg_f4(slab_ptr(ps, c + j / 8, j % 8, row));
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              v[4 * j] += w[j].x;
              v[4 * j + 1] += w[j].y;
              v[4 * j + 2] += w[j].z;
              v[4 * j + 3] += w[j].w;
            }
#ifdef SKB200_DISCARD
            // The slab lines this warp just consumed are dead: drop them from L2
            // without a DRAM write-back (one lane per 128-B line).
            __syncwarp();
            if ((lane & 7) == 0) {
#pragma unroll
              for (int j = 0; j < 16; ++j) ptx::discard_l2(slab_ptr(ps, c + j / 8, j % 8, row));
            }
#endif
          }
          EPI_STAMP(2 + 3 * (c / 2 % 4));
          store_box(v, n0, m0, c);
          store_box(v + 32, n0, m0, c + 1);
        }
        EPI_STAMP(3 + 3 * (c / 2 % 4));
      };
      // Publish / plain store: software pipeline, the TMEM load of the next 64
      // columns is in flight while this step's registers are stored.  Owner fold:
      // one step at a time (its peer loads need the registers).
      // One 64-column step at a time (a software-pipelined TMEM load measured
      // slower: profiles/r02k/README.txt).
#pragma unroll 1
      for (int c = c_first; c < c_end; c += 2 * NG) {
        uint32_t r[64];
        ptx::tmem_ld64(tsrc + c * 32, reinterpret_cast<float(&)[64]>(r));
        after_read(c + 2 * NG);
        if (c + 2 * NG >= c_end) hand_back_last();
        if (fold_n > 0) step(r, c, kFold);
        else step(r, c, kNoFold);
      }
      if (c_first >= c_end) hand_back_last();  // nothing of C in this warp's rows / columns
      if (publish && !orphan) {
        __threadfence();
        ptx::named_bar_sync(1, 32 * EPI_WARPS);
        if (leader) {
          signal_flag(P, P.flags + my_idx);
          if (P.trace && rank == 0 && partial) atomicAdd(P.trace + 4 * s.total_tiles + u, 1);
        }
      }
      EPI_STAMP(13);
      if (!partial) {
        if (P.c_done) {  // this warp's rows of the tile are in HBM: count them for copy-out
          if (lane == 0) {
            ptx::tma_store_wait_all<0>();
            ptx::fence_proxy_async_global();
            __threadfence_system();
            atomicAdd(P.c_done + SK_CDONE_INDEX(P, tr, tc), 1);
          }
          __syncwarp();
        }
        if (fold_n > 0) {
          ptx::named_bar_sync(1, 32 * EPI_WARPS);
          if (leader)  // every epilogue warp has read the slabs: re-arm the flags
            for (int p = 1; p <= fold_n; ++p) ptx::st_relaxed(P.flags + fidx(s.peer(tile, u, p)), 0);
        }
        if (leader && P.trace && rank == 0) {
          int* t = P.trace + 4 * tile;
          t[0] = static_cast<int>(u);
          t[1] = static_cast<int>(s.peer(tile, u, npeer));
          t[2] = static_cast<int>(u);
          t[3] = npeer;
          // the block of C this unit stored (trace section 3, row-major blocks)
          P.trace[4 * s.total_tiles + s.grid_size + tr * s.tiles_n + tc] = static_cast<int>(u);
        }
      }
      if (ev) {
        ev[kEvUnit] = u;
        ev[kEvTile] = tile;
        ev[kEvCore] = cta;
        ev[kEvKind] = (partial ? 1 : 0) | (npeer > 0 ? 2 : 0) | (static_cast<long long>(npeer) << 8) |
                      (static_cast<long long>(ptx::smid()) << 16);
        ev[kEvDone] = ptx::globaltimer();
      }
      if (++acc == K::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
      // Cooperative: shared tiles are folded once the unit has published all of
      // its segments (at most its first and its last), so no fold ever waits
      // behind this unit's own later mainloop work.
      if (coop_t && !orphan) (npend++ == 0 ? pend0 : pend1) = tile;
      if (npend > 0) {
        int64_t b, e;
        s.range(u, &b, &e);
        if (tile * s.ipt + le == e) {
          if (npend > 0) coop_fold(u, pend0);
          if (npend > 1) coop_fold(u, pend1);
          if (ev && npend) ev[kEvDone] = ptx::globaltimer();
          npend = 0;
        }
      }
    }, P.sk_first, P.dp_perm);
    if (lane == 0) ptx::tma_store_wait_all<0>();
    __syncwarp();
    EPI_STAMP(14);
  }

  ptx::tc_fence_before();
  __syncthreads();
  // 2-SM: the leader's MMAs touch the peer's smem/TMEM; cluster fixup: peers read this smem
  if (CG == 2 || CF) cluster_sync();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<CG>(tmem_base, TMEM_COLS);
#ifndef SKB200_EPI_PROBE
  stamp_clock(P, 1);
#endif
#endif
}

}  // namespace f16

// tcgen05 instruction descriptor, kind::f16:
//   [4,6) D format (1 = F32)  [7,10) A format  [10,13) B format (0 = F16, 1 = BF16)
//   [15] A major (0 = K)  [16] B major (1 = MN)  [17,23) N >> 3  [24,29) M >> 4
uint32_t make_idesc_f16(bool bf16, int M, int N) {
  const uint32_t ab = bf16 ? 1u : 0u;
  return (1u << 4) | (ab << 7) | (ab << 10) | (0u << 15) | (1u << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

size_t f16_slab_bytes(int bn) { return sizeof(float) * f16::ROWS * bn; }
int f16_stage_k() { return f16::BKS; }
int f16_epilogue_warps(int bn) {
  return bn == 512 ? f16::Cfg<2, 512>::EPI_WARPS : f16::Cfg<2, 256>::EPI_WARPS;
}

// Per-device setup of kernel (CG, BN) on the CURRENT device (the caller holds the
// device-state mutex and records that it ran): the dynamic-smem / cluster-size
// opt-ins, then how many CTAs (1-SM) or CTA pairs (2-SM) can be co-resident --
// the persistent grid is capped by it (a non-resident unit could be waited on).
template <int CG, int BN>
static cudaError_t prepare_cg(int sms, int* units) {
  auto kern = f16::sk_gemm_f16<CG, BN, false>;
  using K = f16::Cfg<CG, BN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::alloc);
  if (e != cudaSuccess) return e;
  if (CG == 2) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(sms - sms % 2));
    cfg.blockDim = dim3(K::NUM_THREADS);
    cfg.dynamicSmemBytes = K::alloc;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(units, kern, &cfg);
  }
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K::NUM_THREADS, K::alloc);
  *units = per_sm * sms;
  return e;
}

cudaError_t f16_prepare(int cg, int bn, int sms, int* units) {
  if (cg == 1) return prepare_cg<1, 256>(sms, units);
  return bn == 512 ? prepare_cg<2, 512>(sms, units) : prepare_cg<2, 256>(sms, units);
}

template <int CG, int BN, bool CF>
static cudaError_t launch_cg(int cluster, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                             const KernelParams& p, int pairs_or_ctas, cudaStream_t stream) {
  auto kern = f16::sk_gemm_f16<CG, BN, CF>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(pairs_or_ctas * CG));
  cfg.blockDim = dim3(f16::Cfg<CG, BN>::NUM_THREADS);
  cfg.dynamicSmemBytes = f16::Cfg<CG, BN>::alloc;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);  // CG, or S for the cluster fixup
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, a, b, c, p);
}

cudaError_t launch_f16(int cg, int bn, int cluster, const CUtensorMap& a, const CUtensorMap& b,
                       const CUtensorMap& c, const KernelParams& p, int grid, cudaStream_t stream) {
  const bool cf = cluster > cg;  // the cluster fixup: S units per cluster
  if (cg == 1) return cf ? launch_cg<1, 256, true>(cluster, a, b, c, p, grid, stream)
                         : launch_cg<1, 256, false>(cluster, a, b, c, p, grid, stream);
  if (bn == 512) return launch_cg<2, 512, false>(cluster, a, b, c, p, grid, stream);
  return cf ? launch_cg<2, 256, true>(cluster, a, b, c, p, grid, stream)
            : launch_cg<2, 256, false>(cluster, a, b, c, p, grid, stream);
}

// Co-resident clusters of `cluster` CTAs of the 256-wide kernel with CG CTAs per
// unit (cluster fixup); prepare_cg<CG, 256> has set the smem / cluster opt-ins.
template <int CG>
static cudaError_t cluster_capacity_cg(int cluster, int sms, int* clusters) {
  auto kern = f16::sk_gemm_f16<CG, 256, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       f16::Cfg<CG, 256>::alloc);
  if (e != cudaSuccess) return e;
  if (cluster > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(sms - sms % cluster));
  cfg.blockDim = dim3(f16::Cfg<CG, 256>::NUM_THREADS);
  cfg.dynamicSmemBytes = f16::Cfg<CG, 256>::alloc;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(clusters, kern, &cfg);
}

cudaError_t f16_cluster_capacity(int cg, int cluster, int sms, int* clusters) {
  return cg == 2 ? cluster_capacity_cg<2>(cluster, sms, clusters) : cluster_capacity_cg<1>(cluster, sms, clusters);
}

}  // namespace skb200
