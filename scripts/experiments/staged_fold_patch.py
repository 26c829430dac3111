import sys
root = sys.argv[1]
p = root + '/paper_2301_03598_b200/csrc/ptx.cuh'
s = open(p).read()
s = s.replace('''// Invalidate one 128-B L2 line''', '''__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Invalidate one 128-B L2 line''')
open(p, 'w').write(s)
p = root + '/paper_2301_03598_b200/csrc/sk_gemm_f16.cu'
s = open(p).read()
s = s.replace('''  return reinterpret_cast<float4*>(slab) + ((c * 8 + j) * ROWS + row);''',
              '''  return reinterpret_cast<float4*>(slab) + (((row >> 5) * 8 + c) * 8 + j) * 32 + (row & 31);''')
s = s.replace('''  static constexpr int bar_off = epi_off + EPI_BYTES;
  static constexpr int bar_bytes = (2 * STAGES + 4) * 8 + 16;''', '''  static constexpr int RING = STAGES * STAGE;
  static constexpr int FOLD_BUF = 8192;
  static constexpr int FOLD_NB = RING / EPI_WARPS / FOLD_BUF;
  static constexpr int bar_off = epi_off + EPI_BYTES;
  static constexpr int bar_bytes = (2 * STAGES + 4 + EPI_WARPS * FOLD_NB) * 8 + 16;''')
s = s.replace('''  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty_bar + 2);''', '''  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* fold_bar = tempty_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(fold_bar + EPI_WARPS * K::FOLD_NB);''')
s = s.replace('''      ptx::mbar_init(&tempty_bar[i], EPI_WARPS * CG);
    }''', '''      ptx::mbar_init(&tempty_bar[i], EPI_WARPS * CG);
    }
    for (int i = 0; i < EPI_WARPS * K::FOLD_NB; ++i) ptx::mbar_init(&fold_bar[i], 1);''')
s = s.replace('''    int64_t pend0 = 0, pend1 = 0;  // this unit's published shared tiles (at most two)
    int npend = 0;''', '''    int64_t pend0 = 0, pend1 = 0;
    int npend = 0;
    int64_t nseg = 0, seg_i = 0;
    {
      SegmentIter cnt(s, cta, P.num_ctas, dp_lane, P.raster_rows, P.sk_first);
      int64_t a0, a1, a2, a3;
      while (cnt.next(s, &a0, &a1, &a2, &a3)) ++nseg;
    }
    uint8_t* fold_ring = smem + K::a_off + (warp - 2) * (K::RING / EPI_WARPS);
    uint64_t* fbar = fold_bar + (warp - 2) * K::FOLD_NB;''')
s = s.replace('''      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      long long* ev = (leader && rank == 0) ? event_slot(P, u, tile) : nullptr;''', '''      ptx::mbar_wait(&tfull_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const bool last_seg = ++seg_i == nseg;
      long long* ev = (leader && rank == 0) ? event_slot(P, u, tile) : nullptr;''')
s = s.replace('''      // 64 columns (two 32-column chunks) per step: one tcgen05.ld.x64, 16 float4
      // of peer slab in flight per thread, two 32x32 TMA-store boxes.
#pragma unroll 1
      for (int c = c_lo; c < (orphan ? c_lo : c_lo + EPI_COLS / 32); c += 2) {
        float v[64];
        ptx::tmem_ld64(tsrc + c * 32, v);
        if (publish) {''', '''      const bool staged = !publish && fold_n > 0 && last_seg;
      const int fold_total = staged ? (EPI_COLS / 64) * fold_n : 0;
      auto fold_src = [&](int i) -> const float4* {
        return slab_ptr(slab(fidx(s.peer(tile, u, 1 + i % fold_n))), c_lo + 2 * (i / fold_n), 0,
                        static_cast<int>(q * 32));
      };
      if (staged && lane == 0) {
        ptx::fence_proxy_async_global();
        for (int i = 0; i < fold_total && i < K::FOLD_NB; ++i) {
          ptx::mbar_expect_tx(&fbar[i], K::FOLD_BUF);
          ptx::bulk_load(fold_ring + i * K::FOLD_BUF, fold_src(i), K::FOLD_BUF, &fbar[i]);
        }
      }
      int fi = 0;
#ifdef SKB200_DEBUG_FOLD
      const bool dbg = fold_n > 0 && lane == 0 && rank == 0 && (cta % 16) == 0 && warp == 2;
      unsigned long long dt[24];
      int ndt = 0;
      if (dbg) dt[ndt++] = ptx::globaltimer();
#endif
#pragma unroll 1
      for (int c = c_lo; c < (orphan ? c_lo : c_lo + EPI_COLS / 32); c += 2) {
        float v[64];
        ptx::tmem_ld64(tsrc + c * 32, v);
        if (staged) {
#pragma unroll 1
          for (int p = 1; p <= fold_n; ++p, ++fi) {
            const int b = fi % K::FOLD_NB;
            ptx::mbar_wait(&fbar[b], static_cast<uint32_t>(fi / K::FOLD_NB) & 1u);
            const float4* buf = reinterpret_cast<const float4*>(fold_ring + b * K::FOLD_BUF);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float4 w = buf[j * 32 + lane];
              v[4 * j] += w.x;
              v[4 * j + 1] += w.y;
              v[4 * j + 2] += w.z;
              v[4 * j + 3] += w.w;
            }
            __syncwarp();
            if (lane == 0 && fi + K::FOLD_NB < fold_total) {
              ptx::fence_proxy_async_smem();
              ptx::mbar_expect_tx(&fbar[b], K::FOLD_BUF);
              ptx::bulk_load(fold_ring + b * K::FOLD_BUF, fold_src(fi + K::FOLD_NB), K::FOLD_BUF, &fbar[b]);
            }
          }
#ifdef SKB200_DEBUG_FOLD
          if (dbg) dt[ndt++] = ptx::globaltimer();
#endif
          store_box(v, n0, m0, c);
          store_box(v + 32, n0, m0, c + 1);
#ifdef SKB200_DEBUG_FOLD
          if (dbg) dt[ndt++] = ptx::globaltimer();
#endif
        } else if (publish) {''')
s = s.replace('''          store_box(v, n0, m0, c);
          store_box(v + 32, n0, m0, c + 1);
        }
      }
      // Accumulator drained''', '''#ifdef SKB200_DEBUG_FOLD
          if (dbg) dt[ndt++] = ptx::globaltimer();
#endif
          store_box(v, n0, m0, c);
          store_box(v + 32, n0, m0, c + 1);
#ifdef SKB200_DEBUG_FOLD
          if (dbg) dt[ndt++] = ptx::globaltimer();
#endif
        }
      }
#ifdef SKB200_DEBUG_FOLD
      if (dbg) {
        ptx::tma_store_wait_all<0>();
        dt[ndt++] = ptx::globaltimer();
        printf("FOLD staged=%d cta %d tile %d npeer %d ns:", (int)staged, (int)cta, (int)tile, fold_n);
        for (int i = 1; i < ndt; ++i) printf(" %d", (int)(dt[i] - dt[i - 1]));
        printf("\\n");
      }
#endif
      // Accumulator drained''')
open(p, 'w').write(s)
