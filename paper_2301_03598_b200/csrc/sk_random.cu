// sk_random.cu -- the reference's seeded matrix fill, generated on the device.
//
// random_matrix<T>(rows, cols, seed) (matrix.hpp:39-68) draws one SplitMix64
// value per element in row-major order.  SplitMix64 is a counter-based
// generator in disguise: the i-th draw (0-based) mixes state = seed + (i + 1) *
// 0x9e3779b97f4a7c15, so every element is computed independently, with no
// sequential state, by its own thread:
//   int64:  (next() & 0x7f) - 64                      (matrix.hpp:62)
//   float:  (float)((next() >> 11) * 2^-53 * 2 - 1)   (matrix.hpp:52,64)
//   double: (next() >> 11) * 2^-53 * 2 - 1
// then (int64 only) an arithmetic right shift, then RNE into the operand type
// (bf16 / fp16 / fp32 / fp64) in a pitched buffer.  Sweeps and benches feed
// the kernels the reference's own inputs at any size without a host-side fill
// or a PCIe copy.  HBM-bound (one store per element); grid = 8 x SMs.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace skb200 {

__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ULL;  // matrix.hpp:45
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// gen: 0 int64, 1 float, 2 double.  out: 0 bf16, 1 fp16, 2 fp32, 3 fp64.
template <int GEN, int OUT>
__global__ void __launch_bounds__(256) random_matrix_kernel(uint64_t seed, int shift, int64_t rows,
                                                            int64_t cols, void* dst, int64_t ld) {
  const int64_t total = rows * cols;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += stride) {
    const uint64_t z = splitmix_draw(seed, static_cast<uint64_t>(i));
    double v;
    float vf;
    if constexpr (GEN == 0) {
      const int64_t x = (static_cast<int64_t>(z & 0x7f) - 64) >> shift;
      v = static_cast<double>(x);
      vf = static_cast<float>(x);
    } else {
      v = static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
      vf = static_cast<float>(v);  // random_matrix<float>: (T)(u * 2 - 1)
      if constexpr (GEN == 1) v = static_cast<double>(vf);
    }
    const int64_t r = i / cols, c = i - r * cols;
    const int64_t o = r * ld + c;
    if constexpr (OUT == 0) {
      static_cast<__nv_bfloat16*>(dst)[o] = __float2bfloat16_rn(vf);
    } else if constexpr (OUT == 1) {
      static_cast<__half*>(dst)[o] = __float2half_rn(vf);
    } else if constexpr (OUT == 2) {
      static_cast<float*>(dst)[o] = vf;
    } else {
      static_cast<double*>(dst)[o] = v;
    }
  }
}

template <int GEN, int OUT>
static cudaError_t launch_rm(uint64_t seed, int shift, int64_t rows, int64_t cols, void* dst,
                             int64_t ld, cudaStream_t stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (rows * cols + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
  random_matrix_kernel<GEN, OUT><<<static_cast<int>(blocks), 256, 0, stream>>>(seed, shift, rows, cols,
                                                                             dst, ld);
  return cudaGetLastError();
}

cudaError_t launch_random_matrix(int gen, int out, uint64_t seed, int shift, int64_t rows, int64_t cols,
                                 void* dst, int64_t ld, cudaStream_t stream) {
#define SK_RM_CASE(G, O) \
  if (gen == G && out == O) return launch_rm<G, O>(seed, shift, rows, cols, dst, ld, stream);
  SK_RM_CASE(0, 0) SK_RM_CASE(0, 1) SK_RM_CASE(0, 2) SK_RM_CASE(0, 3)
  SK_RM_CASE(1, 0) SK_RM_CASE(1, 1) SK_RM_CASE(1, 2) SK_RM_CASE(1, 3)
  SK_RM_CASE(2, 2) SK_RM_CASE(2, 3)
#undef SK_RM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace skb200
