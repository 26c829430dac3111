// sk_probe.cu -- one-time per-device topology probe: which die is each SM on,
// and do 2-CTA clusters land on one TPC (SM pair)?
//
// B200 is two dies; each has half of the SMs and its own L2, and an L2 line has
// one home die.  Atomics resolve at the line's home L2 slice, so a chain of
// dependent atomics on one word is ~2x slower from the far die (measured ~75 vs
// ~170 cycles).  One CTA per SM (200 KB of smem forces that), launched as
// clusters of 2, runs the chain on a few words one CTA at a time (ticket
// order, so chains never contend) and records {smid, cluster rank, latency}.
// The host classifies the SMs into two dies and checks that each cluster's
// two CTAs share a TPC (smid / 2), which the die-aware persistent schedule
// needs (sk_kernel_common.cuh dp_lane).  Every wait is bounded by %globaltimer,
// so a busy or unusual device yields "no topology", never a hang.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ptx.cuh"

namespace skb200 {

constexpr int kProbeWords = 4;
constexpr int kProbeIters = 48;
constexpr int kProbeSmem = 200 * 1024;

// out[cta] = {smid, cluster rank, lat word 0..kProbeWords-1}; words 4 KB apart
__global__ void __cluster_dims__(2, 1, 1) die_probe(unsigned* words, int* ticket, int* out, int* err) {
  extern __shared__ uint8_t probe_smem[];
  if (threadIdx.x != 0) return;
  probe_smem[0] = 0;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint64_t t_start = ptx::globaltimer();
  const int my = atomicAdd(ticket, 1);
  volatile int* turn = ticket + 1;
  while (*turn != my) {
    if (ptx::globaltimer() - t_start > 200000000ull) {  // 200 ms
      atomicOr(err, 1);
      return;
    }
  }
  int* o = out + blockIdx.x * (2 + kProbeWords);
  o[0] = static_cast<int>(ptx::smid());
  o[1] = static_cast<int>(rank);
  for (int w = 0; w < kProbeWords; ++w) {
    unsigned* p = words + w * 1024;
    unsigned v = 0;
    const long long t0 = clock64();
    for (int i = 0; i < kProbeIters; ++i) v = atomicAdd(p + (v >> 30), 1u);  // dependent chain (v < 2^30)
    const long long t1 = clock64();
    o[2 + w] = static_cast<int>((t1 - t0) / kProbeIters) + static_cast<int>(v >> 30);
  }
  __threadfence();
  atomicAdd(ticket + 1, 1);
}

// Fills die_of_sm[0..sms) with 0/1 and returns true when the device shows a
// clean two-die split with TPC-aligned clusters; false otherwise (no error:
// the caller just keeps the topology-oblivious schedule).
bool probe_dies(int sms, std::vector<int>* die_of_sm, cudaError_t* cuda_err) {
  *cuda_err = cudaSuccess;
  if (sms <= 0 || sms % 2 || sms > 192) return false;
  const size_t words_bytes = kProbeWords * 4096;
  const size_t out_ints = static_cast<size_t>(sms) * (2 + kProbeWords);
  uint8_t* buf = nullptr;
  const size_t bytes = words_bytes + 64 + out_ints * 4;
  cudaError_t e = cudaMalloc(&buf, bytes);
  if (e != cudaSuccess) {
    *cuda_err = e;
    return false;
  }
  bool ok = false;
  std::vector<int> h(out_ints + 1, -1);
  do {
    if ((e = cudaMemset(buf, 0, bytes)) != cudaSuccess) break;
    unsigned* words = reinterpret_cast<unsigned*>(buf);
    int* ticket = reinterpret_cast<int*>(buf + words_bytes);
    int* err = ticket + 2;
    int* out = reinterpret_cast<int*>(buf + words_bytes + 64);
    if ((e = cudaMemset(out, 0xff, out_ints * 4)) != cudaSuccess) break;
    if ((e = cudaFuncSetAttribute(die_probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kProbeSmem)) != cudaSuccess)
      break;
    die_probe<<<sms, 32, kProbeSmem>>>(words, ticket, out, err);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) break;
    if ((e = cudaMemcpy(h.data(), out, out_ints * 4, cudaMemcpyDeviceToHost)) != cudaSuccess) break;
    if ((e = cudaMemcpy(&h[out_ints], err, 4, cudaMemcpyDeviceToHost)) != cudaSuccess) break;
    if (h[out_ints] != 0) break;
    // every SM exactly once, clusters TPC-aligned
    std::vector<int> seen(sms, 0);
    std::vector<std::vector<int>> lat(kProbeWords, std::vector<int>(sms, 0));
    bool good = true;
    for (int c = 0; c < sms && good; ++c) {
      const int* o = &h[static_cast<size_t>(c) * (2 + kProbeWords)];
      if (o[0] < 0 || o[0] >= sms || seen[o[0]]++) good = false;
      else
        for (int w = 0; w < kProbeWords; ++w) lat[w][o[0]] = o[2 + w];
      if (good && (c & 1)) {
        const int* l = o - (2 + kProbeWords);  // the cluster's other CTA
        if (l[0] / 2 != o[0] / 2 || l[1] == o[1]) good = false;
      }
    }
    if (!good) break;
    // classify on word 0: near (< midpoint) = die 0; require a clear gap, and
    // every other word must give the same or the complementary partition
    std::vector<int> die(sms);
    for (int w = 0; w < kProbeWords && good; ++w) {
      const auto mm = std::minmax_element(lat[w].begin(), lat[w].end());
      const int lo = *mm.first, hi = *mm.second, mid = (lo + hi) / 2;
      int max_near = 0, min_far = 1 << 30;
      for (int i = 0; i < sms; ++i) {
        if (lat[w][i] < mid) max_near = std::max(max_near, lat[w][i]);
        else min_far = std::min(min_far, lat[w][i]);
      }
      if (max_near * 4 > min_far * 3) {  // no clean bimodal split
        good = false;
        break;
      }
      int same = 0;
      for (int i = 0; i < sms; ++i) {
        const int d = lat[w][i] < mid ? 0 : 1;
        if (w == 0) die[i] = d;
        else same += d == die[i];
      }
      if (w > 0 && same != sms && same != 0) good = false;
    }
    if (!good) break;
    for (int t = 0; t < sms / 2; ++t)  // a TPC never straddles dies
      if (die[2 * t] != die[2 * t + 1]) good = false;
    const int n0 = static_cast<int>(std::count(die.begin(), die.end(), 0));
    if (!good || n0 == 0 || n0 == sms) break;
    *die_of_sm = die;
    ok = true;
  } while (false);
  cudaFree(buf);
  if (e != cudaSuccess) {
    *cuda_err = e;
    cudaGetLastError();  // clear
    return false;
  }
  return ok;
}

}  // namespace skb200
