// die_map.cu -- which die is each SM on?  (B200 = two dies, each with half the
// SMs and half the L2; an L2 line has one home partition.)
//
// One CTA per SM runs a chain of dependent atomics on a single word.  Atomics
// resolve at the line's home L2 slice, so the chain's latency is bimodal:
// near-die SMs vs far-die SMs.  Repeating with several words (different homes)
// and taking the per-SM latency vector separates the two dies.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o die_map scripts/die_map.cu && ./die_map
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void chase(unsigned* words, int nwords, int iters, long long* out, volatile int* turn) {
  if (threadIdx.x != 0) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  // serialise the CTAs (one per SM, all co-resident) so the chains never contend
  while (*turn != static_cast<int>(smid)) {
  }
  for (int w = 0; w < nwords; ++w) {
    unsigned* p = words + w * 1024;  // 4 KB apart: different L2 slices / homes
    unsigned v = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) v = atomicAdd(p + (v & 0), 1u) & 0;
    long long t1 = clock64();
    out[smid * nwords + w] = (t1 - t0) / iters + v;
  }
  __threadfence();
  atomicAdd(const_cast<int*>(turn), 1);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nwords = 16, iters = 256;
  unsigned* words;
  long long* out;
  cudaMalloc(&words, nwords * 4096);
  cudaMemset(words, 0, nwords * 4096);
  cudaMalloc(&out, sizeof(long long) * 256 * nwords);
  int* turn;
  cudaMalloc(&turn, sizeof(int));
  cudaMemset(turn, 0, sizeof(int));
  cudaMemset(out, 0, sizeof(long long) * 256 * nwords);
  // one CTA per SM: large smem request forces spreading
  cudaFuncSetAttribute(chase, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  chase<<<sms, 32, 200 * 1024>>>(words, nwords, iters, out, turn);
  cudaDeviceSynchronize();
  std::vector<long long> h(256 * nwords);
  cudaMemcpy(h.data(), out, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("smid");
  for (int w = 0; w < nwords; ++w) printf(",w%d", w);
  printf("\n");
  for (int s = 0; s < sms; ++s) {
    printf("%d", s);
    for (int w = 0; w < nwords; ++w) printf(",%lld", h[s * nwords + w]);
    printf("\n");
  }
  return 0;
}
