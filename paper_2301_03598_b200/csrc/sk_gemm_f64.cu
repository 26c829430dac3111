// sk_gemm_f64.cu -- persistent Stream-K DGEMM for sm_100a (BASELINE config 4).
//
// C (fp64) = A (fp64, m x k, row-major) * B (fp64, k x n, row-major) under any
// of the reference's decompositions, with the paper's single FP64 tile config
// 64x64x16.  sm_100 has no f64 tcgen05 kind, so the MAC loop
// runs on the FP64 tensor pipe through warp-level DMMA
// (mma.sync.aligned.m16n8k16.row.col.f64), fed by TMA:
//
//   warp 4        TMA producer: A 64x16 box + four 16x16 B boxes per k-iteration,
//                 128-B swizzled, STAGES-deep mbarrier ring
//   warps 0..3    consumers: warp w owns the 32x32 sub-tile (w/2, w%2), 2 x 4
//                 m16n8 fragments = 32 fp64 accumulators per thread; after a
//                 segment they run the fixup protocol and store C
//
// Fixup (executor.hpp:95-119,160-181): a non-owner writes its 32 KB fp64 slab
// (thread-strided, coalesced), fences and signals; the owner waits on the
// flags of its peers and adds their slabs in ascending id after its own
// accumulator, then stores the clamped tile.  Same persistent order and
// deadlock argument as the 16-bit kernel (sk_kernel_common.cuh).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"
#include "schedule.hpp"
#include "sk_kernel_common.cuh"

namespace skb200 {
namespace f64 {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 8;        // 8 KB
constexpr int B_BOX_BYTES = BK * 16 * 8;    // 16 k-rows x 16 n = 2 KB
constexpr int B_BYTES = 4 * B_BOX_BYTES;    // 8 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int CONSUMERS = 4;
constexpr int NUM_THREADS = 32 * (CONSUMERS + 1);
constexpr int SLAB_ELEMS = BM * BN;
constexpr int SMEM = STAGES * STAGE_BYTES + (2 * STAGES) * 8 + 1024;

// Byte offset of element (r, c) inside a box with 128-B rows and 128-B swizzle.
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * 128 + ((((c >> 1) ^ (r & 7))) << 4) + ((c & 1) << 3));
}

__device__ __forceinline__ void dmma_16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0, %1, %2, %3}, {%4, %5, %6, %7, %8, %9, %10, %11}, {%12, %13, %14, %15}, "
      "{%0, %1, %2, %3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__device__ __forceinline__ double ld_smem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__global__ void __launch_bounds__(NUM_THREADS, 2)
    sk_gemm_f64(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                double* __restrict__ Cg, int64_t ldc, const KernelParams P) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const Schedule& s = P.s;
  const int64_t cta = blockIdx.x;

  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full_bar[i], 1);
      ptx::mbar_init(&empty_bar[i], CONSUMERS);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  ptx::grid_dependency_wait();
  ptx::launch_dependents();
  stamp_clock(P, 0);

  if (warp == CONSUMERS) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_a = ptx::make_policy(P.l2_policy[0]);
      const uint64_t pol_b = ptx::make_policy(P.l2_policy[1]);
      uint32_t stage = 0, phase = 0;
      for_each_segment(s, cta, P.num_ctas, P.raster_rows,
                       [&](int64_t, int64_t tile, int64_t lb, int64_t le) {
        int64_t tr, tc;
        s.tile_rc(tile, &tr, &tc);
        const int32_t m0 = static_cast<int32_t>(tr * BM);
        const int32_t n0 = static_cast<int32_t>(tc * BN);
        if (P.a_ready) {  // row block of A (and column panel of B) in HBM
          wait_flag(P, P.a_ready + tr);
          if (P.b_ready) wait_flag(P, P.b_ready + tc / P.pipe_w);
        }
        for (int64_t kb = lb; kb < le; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          uint8_t* st = smem + stage * STAGE_BYTES;
          const int32_t k0 = static_cast<int32_t>(kb * BK);
          ptx::tma_load_2d(st, &tmA, &full_bar[stage], k0, m0, pol_a);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            ptx::tma_load_2d(st + A_BYTES + j * B_BOX_BYTES, &tmB, &full_bar[stage], n0 + 16 * j, k0,
                             pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }, P.sk_first, P.dp_perm);
    }
    return;
  }

  // ===================== DMMA consumers =====================
  const int wm = static_cast<int>(warp / 2) * 32, wn = static_cast<int>(warp % 2) * 32;
  const int g = static_cast<int>(lane >> 2), tq = static_cast<int>(lane & 3);
  const int tid = static_cast<int>(threadIdx.x);  // 0..127
  double* partials = static_cast<double*>(P.partials);
  uint32_t stage = 0, phase = 0;
  for_each_segment(s, cta, P.num_ctas, P.raster_rows,
                   [&](int64_t u, int64_t tile, int64_t lb, int64_t le) {
    long long* ev = tid == 0 ? event_slot(P, u, tile) : nullptr;
    if (ev) ev[kEvMacStart] = ptx::globaltimer();
    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

    for (int64_t kb = lb; kb < le; ++kb) {
      ptx::mbar_wait(&full_bar[stage], phase);
      const uint32_t sa = ptx::smem_u32(smem + stage * STAGE_BYTES);
      const uint32_t sb = sa + A_BYTES;
      double af[2][8], bf[4][4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r)  // a[r]: m = g + 8*(r%2), k = tq + 4*(r/2)
          af[i][r] = ld_smem_f64(sa + swz(wm + 16 * i + g + 8 * (r & 1), tq + 4 * (r >> 1)));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn + 8 * j + g;  // b[v]: k = tq + 4v, n = g
#pragma unroll
        for (int v = 0; v < 4; ++v)
          bf[j][v] = ld_smem_f64(sb + (n >> 4) * B_BOX_BYTES + swz(tq + 4 * v, n & 15));
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_16816(acc[i][j], af[i], bf[j]);
      // The MMAs consumed every fragment register, so this warp is done with the stage.
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty_bar[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    const bool partial = lb != 0;
    const int npeer = (!partial && (le < s.ipt || s.strategy == kExplicit)) ? s.npeers(tile, u) : 0;
    if (ev) {
      ev[kEvMacEnd] = ptx::globaltimer();
      ev[kEvUnit] = u;
      ev[kEvTile] = tile;
      ev[kEvCore] = cta;
      ev[kEvKind] = (partial ? 1 : 0) | (npeer > 0 ? 2 : 0) | (static_cast<long long>(npeer) << 8) |
                      (static_cast<long long>(ptx::smid()) << 16);
    }
    if (partial && s.orphan(tile)) {  // explicit table: no range starts this tile
      if (ev) ev[kEvWaitEnd] = ev[kEvDone] = ptx::globaltimer();
      return;
    }
    if (partial) {
      double* slab = partials + s.slab_of(u) * static_cast<int64_t>(SLAB_ELEMS);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) __stcg(slab + ((i * 4 + j) * 4 + e) * 128 + tid, acc[i][j][e]);
      __threadfence();
      ptx::named_bar_sync(1, 128);
      if (tid == 0) {
        signal_flag(P, P.flags + s.slab_of(u));
        if (P.trace) atomicAdd(P.trace + 4 * s.total_tiles + u, 1);
      }
      if (ev) ev[kEvWaitEnd] = ev[kEvDone] = ptx::globaltimer();
      return;
    }
    if (npeer > 0) {
      if (tid == 0)
        for (int p = 1; p <= npeer; ++p) wait_flag(P, P.flags + s.slab_of(s.peer(tile, u, p)));
      ptx::named_bar_sync(1, 128);
      if (ev) ev[kEvWaitEnd] = ptx::globaltimer();
      // Owner fold: own accumulator, then peers in ascending id (executor.hpp:165-172).
      for (int p = 1; p <= npeer; ++p) {
        const double* slab = partials + s.slab_of(s.peer(tile, u, p)) * static_cast<int64_t>(SLAB_ELEMS);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] += __ldcg(slab + ((i * 4 + j) * 4 + e) * 128 + tid);
      }
      ptx::named_bar_sync(1, 128);
      if (tid == 0)
        for (int p = 1; p <= npeer; ++p) ptx::st_relaxed(P.flags + s.slab_of(s.peer(tile, u, p)), 0);
    }
    // Clamped store of the owner's tile (executor.hpp:175-181).
    int64_t tr, tc;
    s.tile_rc(tile, &tr, &tc);
    if (tid == 0 && P.trace) {
      int* t = P.trace + 4 * tile;
      t[0] = static_cast<int>(u);
      t[1] = static_cast<int>(s.peer(tile, u, npeer));
      t[2] = static_cast<int>(u);
      t[3] = npeer;
      P.trace[4 * s.total_tiles + s.grid_size + tr * s.tiles_n + tc] = static_cast<int>(u);
    }
    const int64_t m0 = tr * BM, n0 = tc * BN;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t r = m0 + wm + 16 * i + g + 8 * h;
          const int64_t c = n0 + wn + 8 * j + 2 * tq;
          if (r >= s.m) continue;
          double* dst = Cg + r * ldc + c;
          if (c + 1 < s.n) {
            __stcs(reinterpret_cast<double2*>(dst), make_double2(acc[i][j][2 * h], acc[i][j][2 * h + 1]));
          } else if (c < s.n) {
            __stcs(dst, acc[i][j][2 * h]);
          }
        }
    if (P.c_done) {  // the tile is in HBM: count it for copy-out
      __threadfence_system();
      ptx::named_bar_sync(1, 128);
      if (tid == 0) atomicAdd(P.c_done + SK_CDONE_INDEX(P, tr, tc), 1);
    }
    if (ev) {
      if (npeer == 0) ev[kEvWaitEnd] = ev[kEvMacEnd];
      ev[kEvDone] = ptx::globaltimer();
    }
  }, P.sk_first, P.dp_perm);
  stamp_clock(P, 1);
#endif
}

}  // namespace f64

size_t f64_slab_bytes() { return sizeof(double) * f64::SLAB_ELEMS; }

// Per-device setup on the CURRENT device (the caller records that it ran).
cudaError_t f64_max_ctas_per_sm(int* out) {
  cudaError_t e = cudaFuncSetAttribute(f64::sk_gemm_f64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       f64::SMEM);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, f64::sk_gemm_f64, f64::NUM_THREADS,
                                                    f64::SMEM);
  if (e == cudaSuccess && *out > 2) *out = 2;
  return e;
}

cudaError_t launch_f64(const CUtensorMap& a, const CUtensorMap& b, double* C, int64_t ldc,
                       const KernelParams& p, int grid, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(f64::NUM_THREADS);
  cfg.dynamicSmemBytes = f64::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, f64::sk_gemm_f64, a, b, C, ldc, p);
}

}  // namespace skb200
