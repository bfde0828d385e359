// Exact squared-error sum for MSE / PSNR (pkg/src/irdenoise/metrics.py:22-40).
//
// The reference accumulates sum((a - b)^2) in Python integers and divides once, so
// the result is independent of summation order; the GPU sum is an exact u64: one call
// takes at most 2^32 - 1 u16 elements ((2^32 - 1) * 65535^2 < 2^64; any u8 size
// below 2^47 fits), larger inputs are split by the caller.
// HBM-bound streaming reduction: 16-byte loads, per-thread u64 partials, one
// atomic per warp.
#pragma once
#include <cstdint>

namespace irdn {
namespace metrics {

constexpr int THREADS = 256;

template <typename T>
__device__ __forceinline__ uint64_t sq_vec(const uint4& a, const uint4& b) {
  const uint32_t* pa = reinterpret_cast<const uint32_t*>(&a);
  const uint32_t* pb = reinterpret_cast<const uint32_t*>(&b);
  uint64_t acc = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (sizeof(T) == 1) {
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int d = (int)((pa[j] >> (8 * q)) & 0xFFu) - (int)((pb[j] >> (8 * q)) & 0xFFu);
        s += (uint32_t)(d * d);
      }
      acc += s;
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t x = (pa[j] >> (16 * q)) & 0xFFFFu, y = (pb[j] >> (16 * q)) & 0xFFFFu;
        const uint32_t d = x > y ? x - y : y - x;
        acc += (uint64_t)(d * d);  // < 2^32: no signed overflow
      }
    }
  }
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(THREADS) sq_err_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                         int64_t n, bool vec, unsigned long long* out) {
  constexpr int V = 16 / sizeof(T);
  uint64_t acc = 0;
  const int64_t nvec = vec ? n / V : 0;  // vec: both pointers 16-byte aligned
  const int64_t stride = (int64_t)gridDim.x * THREADS;
  const uint4* va = reinterpret_cast<const uint4*>(a);
  const uint4* vb = reinterpret_cast<const uint4*>(b);
  for (int64_t v = (int64_t)blockIdx.x * THREADS + threadIdx.x; v < nvec; v += stride)
    acc += sq_vec<T>(__ldcs(va + v), __ldcs(vb + v));
  for (int64_t i = nvec * V + (int64_t)blockIdx.x * THREADS + threadIdx.x; i < n; i += stride) {
    const int64_t d = (int64_t)a[i] - (int64_t)b[i];
    acc += (uint64_t)(d * d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

}  // namespace metrics
}  // namespace irdn
