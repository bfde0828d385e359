// Generic FNR / MF kernel: any odd k >= 3, any frame size, any row pitch,
// u8 or u16 pixels. One thread per output pixel; window values are read
// through L1 with replicate-edge clamping and the median is found by an
// exact bitwise radix selection (no sort). This is the correctness anchor
// for shapes the specialised tile kernels do not cover (unaligned pitches
// such as the reference's 364-pixel rows, tiny images, k >= 13).
//
// Reference semantics followed (pkg/src/irdenoise/...):
//   filters.py:148-167  clamp-gather of the k*k window (raster order irrelevant
//                       for min/max/median, all duplicates included)
//   filters.py:169-178  FNR: noisy iff centre == min or == max; noisy -> median
//   filters.py:179-180  MF: every pixel -> median
//   sorting.py:51-56    median = element (n-1)/2 of the sorted window
#pragma once
#include "fnr_common.cuh"

namespace irdn {

// Exact rank selection by bitwise construction: the largest t with
// #{v < t} <= rank is the rank-th smallest value. Bits above the highest
// bit where min and max differ are shared by every window value, so the
// search starts below them.
template <typename T>
__device__ __forceinline__ uint32_t generic_window_select(const T* __restrict__ frame,
                                                          const PassGeom& g, int x, int y,
                                                          int r, uint32_t vmin, uint32_t vmax,
                                                          int rank) {
  uint32_t diff = vmin ^ vmax;
  if (diff == 0u) return vmin;
  int hb = 31 - __clz(diff);
  uint32_t m = vmin & ~((2u << hb) - 1u);
  for (int b = hb; b >= 0; --b) {
    const uint32_t t = m | (1u << b);
    int below = 0;
    for (int dy = -r; dy <= r; ++dy) {
      const T* row = frame + (int64_t)(clampi(y + dy, 0, g.height - 1) - g.in_row0) * g.in_pitch;
      for (int dx = -r; dx <= r; ++dx) below += (uint32_t)row[clampi(x + dx, 0, g.width - 1)] < t;
    }
    if (below <= rank) m = t;
  }
  return m;
}

template <typename T>
__global__ void __launch_bounds__(256) fnr_generic_kernel(const T* __restrict__ in,
                                                          T* __restrict__ out, PassGeom g, int k,
                                                          int method,
                                                          unsigned long long* counts) {
  const int r = k >> 1;
  const int rank = (k * k - 1) >> 1;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = g.row_begin + blockIdx.y * 8 + (threadIdx.x >> 5);
  uint32_t detected = 0, replaced = 0;
  for (int b = blockIdx.z; b < g.batch; b += gridDim.z) {
    if (x < g.width && y < g.row_end) {
      const T* frame = in + (int64_t)b * g.in_frame_stride;
      const uint32_t c = frame[(int64_t)(y - g.in_row0) * g.in_pitch + x];
      uint32_t vmin = 0xffffffffu, vmax = 0u;
      for (int dy = -r; dy <= r; ++dy) {
        const T* row = frame + (int64_t)(clampi(y + dy, 0, g.height - 1) - g.in_row0) * g.in_pitch;
        for (int dx = -r; dx <= r; ++dx) {
          const uint32_t v = row[clampi(x + dx, 0, g.width - 1)];
          vmin = min(vmin, v);
          vmax = max(vmax, v);
        }
      }
      uint32_t o = c;
      if (method != 0) {
        o = generic_window_select<T>(frame, g, x, y, r, vmin, vmax, rank);
      } else if (c == vmin || c == vmax) {
        o = generic_window_select<T>(frame, g, x, y, r, vmin, vmax, rank);
        detected += 1;
        replaced += (o != c);
      }
      out[(int64_t)b * g.out_frame_stride + (int64_t)(y - g.row_begin) * g.out_pitch + x] = (T)o;
    }
  }
  if (method == 0) block_add_counts<256>(detected, replaced, counts);
}

}  // namespace irdn
