// sk_convert.cu -- fp32 -> bf16/fp16 (round-to-nearest-even) into a pitched
// operand buffer.  Used only by sk_execute when the caller hands the drop-in
// fp32 matrices (the reference's Matrix<float>, matrix.hpp:15-28) to a 16-bit
// tensor-core kernel.  HBM-bound: 4 B read + 2 B written per element, grid
// sized to a multiple of the SM count, 8 elements (32 B in, 16 B out) per step.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace skb200 {

template <bool BF16>
__global__ void __launch_bounds__(256) f32_to_16_kernel(const float* __restrict__ src,
                                                        uint16_t* __restrict__ dst, int64_t rows,
                                                        int64_t cols, int64_t ld_dst) {
  const int64_t total = rows * cols;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    const float v = src[i];
    uint16_t bits;
    if constexpr (BF16) {
      __nv_bfloat16 h = __float2bfloat16_rn(v);
      bits = *reinterpret_cast<uint16_t*>(&h);
    } else {
      __half h = __float2half_rn(v);
      bits = *reinterpret_cast<uint16_t*>(&h);
    }
    dst[r * ld_dst + c] = bits;
  }
}

cudaError_t launch_f32_to_16(const float* src, void* dst, int64_t rows, int64_t cols,
                             int64_t ld_dst, bool bf16, cudaStream_t stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = rows * cols;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (bf16)
    f32_to_16_kernel<true><<<static_cast<int>(blocks), 256, 0, stream>>>(
        src, static_cast<uint16_t*>(dst), rows, cols, ld_dst);
  else
    f32_to_16_kernel<false><<<static_cast<int>(blocks), 256, 0, stream>>>(
        src, static_cast<uint16_t*>(dst), rows, cols, ld_dst);
  return cudaGetLastError();
}

}  // namespace skb200

namespace skb200 {

// Pitched elementwise conversions for the fp64-compute drop-ins of
// execute<float> and execute<int64_t> (sk_execute): f32/i64 operands are
// widened exactly to f64, the f64 result is narrowed back (f32: round to
// nearest; i64: the value is an exact integer when the caller's range check
// passed).  HBM-bound; grid-stride over rows x cols.
template <typename S, typename D>
__global__ void __launch_bounds__(256) convert_2d_kernel(const S* __restrict__ src, int64_t ld_src,
                                                         D* __restrict__ dst, int64_t ld_dst,
                                                         int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    const S v = src[r * ld_src + c];
    if constexpr (sizeof(D) == 8 && static_cast<D>(0.5) == 0) {
      dst[r * ld_dst + c] = static_cast<D>(llrint(static_cast<double>(v)));  // f64 -> i64
    } else {
      dst[r * ld_dst + c] = static_cast<D>(v);
    }
  }
}

template <typename S, typename D>
static cudaError_t launch_conv(const void* src, int64_t ld_src, void* dst, int64_t ld_dst,
                               int64_t rows, int64_t cols, cudaStream_t stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (rows * cols + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > static_cast<int64_t>(sms) * 8 ? static_cast<int64_t>(sms) * 8 : blocks);
  convert_2d_kernel<S, D><<<static_cast<int>(blocks), 256, 0, stream>>>(
      static_cast<const S*>(src), ld_src, static_cast<D*>(dst), ld_dst, rows, cols);
  return cudaGetLastError();
}

// kind: 0 f32->f64, 1 i64->f64, 2 f64->f32, 3 f64->i64
cudaError_t launch_convert(int kind, const void* src, int64_t ld_src, void* dst, int64_t ld_dst,
                           int64_t rows, int64_t cols, cudaStream_t stream) {
  switch (kind) {
    case 0: return launch_conv<float, double>(src, ld_src, dst, ld_dst, rows, cols, stream);
    case 1: return launch_conv<long long, double>(src, ld_src, dst, ld_dst, rows, cols, stream);
    case 2: return launch_conv<double, float>(src, ld_src, dst, ld_dst, rows, cols, stream);
    case 3: return launch_conv<double, long long>(src, ld_src, dst, ld_dst, rows, cols, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace skb200
