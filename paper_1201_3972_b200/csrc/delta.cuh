// Sparse result return for the host-buffer run_filter (irdn_run_filter_*).
//
// FNR rewrites only the flagged pixels whose median differs from the centre
// (filters.py:172-176: 2-50 % of the pixels on the BASELINE scenes); every other output
// pixel is the input pixel the caller already holds in host memory. So instead of a
// full device->host copy of the filtered image, the device sends the difference
// between output and input, and the host rebuilds the output from its own input.
//
// Region of a chunk of n pixels, nb = ceil(n / BLK) blocks of BLK = 4096 pixels:
//   [ u32 total, 3 x u32 pad                      ]  16 bytes
//   [ u32 count[nb]   (16-byte padded)            ]  changed pixels of block b
//   [ u32 offset[nb]  (16-byte padded)            ]  index of block b's first value in values[]
//   [ u32 mask[nb][BLK / 32]                      ]  bit j of word w <=> pixel b*BLK + 32w + j changed
//   [ T values[total] (capacity n)                ]  the changed output pixels, block by block
// Blocks claim their value range with one atomicAdd on `total`, so the values are
// packed densely (block order is arbitrary, `offset` says where each block's run is);
// a block without a change writes only its count (its mask slot is stale, the decoder
// skips it). The fixed part (header, counts, offsets, masks) has a known size, so the
// host copies it plus a budget of values with one DMA (delta_budget in irdn_api.cu) and
// fetches the rest only when `total` exceeds the budget.
//
// One CTA per block compares in / out (16-byte loads; both are L2-resident right after
// the filter), compacts the changed values in shared memory and writes the block's
// run with 16-byte-aligned stores where it can. The host side (delta_host.cpp) expands
// the values into a copy of its own input (AVX-512 VBMI2 expand-load where available).
#pragma once
#include <cstdint>

namespace irdn {
namespace delta {

constexpr int BLK = 4096;            // pixels per block
constexpr int THREADS = 256;         // 16 pixels per thread
constexpr int PPT = BLK / THREADS;   // pixels per thread
constexpr int MASK_WORDS = BLK / 32;

__host__ __device__ inline int64_t nblocks(int64_t n) { return (n + BLK - 1) / BLK; }
__host__ __device__ inline int64_t table_bytes(int64_t n) { return ((nblocks(n) * 4) + 15) & ~int64_t(15); }
__host__ __device__ inline int64_t counts_offset(int64_t) { return 16; }
__host__ __device__ inline int64_t offsets_offset(int64_t n) { return 16 + table_bytes(n); }
__host__ __device__ inline int64_t mask_offset(int64_t n) { return 16 + 2 * table_bytes(n); }
__host__ __device__ inline int64_t values_offset(int64_t n) { return mask_offset(n) + nblocks(n) * (BLK / 8); }
template <typename T>
__host__ __device__ inline int64_t region_bytes(int64_t n) {
  return ((values_offset(n) + n * (int64_t)sizeof(T)) + 15) & ~int64_t(15);
}

// dst must be 16-byte aligned and its first 16 bytes zero (total = 0) at launch.
template <typename T>
__global__ void __launch_bounds__(THREADS) encode_kernel(const T* __restrict__ in, const T* __restrict__ out,
                                                          int64_t n, uint8_t* __restrict__ dst, int vec_ok) {
  __shared__ __align__(16) T s_val[BLK];
  __shared__ __align__(16) uint32_t s_mask[MASK_WORDS];
  __shared__ int s_warp[THREADS / 32];
  __shared__ uint32_t s_base;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t b = blockIdx.x;
  const int64_t p0 = b * BLK + (int64_t)t * PPT;
  T a[PPT], o[PPT];
  if (vec_ok && p0 + PPT <= n) {
    constexpr int V = PPT * (int)sizeof(T) / 16;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      *reinterpret_cast<uint4*>(a + v * 16 / sizeof(T)) = __ldcs(reinterpret_cast<const uint4*>(in + p0) + v);
      *reinterpret_cast<uint4*>(o + v * 16 / sizeof(T)) = __ldcs(reinterpret_cast<const uint4*>(out + p0) + v);
    }
  } else {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const bool ok = p0 + j < n;
      a[j] = ok ? in[p0 + j] : T(0);
      o[j] = ok ? out[p0 + j] : T(0);
    }
  }
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) m |= (a[j] != o[j] ? 1u : 0u) << j;
  const int c = __popc(m);
  int incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += u;
  }
  if (lane == 31) s_warp[warp] = incl;
  // two threads form one 32-pixel mask word (thread 2w: low half, 2w + 1: high half)
  const uint32_t hi = __shfl_down_sync(0xffffffffu, m, 1);
  if ((t & 1) == 0) s_mask[t >> 1] = m | (hi << 16);
  __syncthreads();
  int base = 0, total = 0;
#pragma unroll
  for (int w = 0; w < THREADS / 32; ++w) {
    const int x = s_warp[w];
    base += w < warp ? x : 0;
    total += x;
  }
  int pos = base + incl - c;
  uint32_t mm = m;
  while (mm) {
    const int j = __ffs(mm) - 1;
    mm &= mm - 1u;
#pragma unroll
    for (int q = 0; q < PPT; ++q)
      if (q == j) s_val[pos] = o[q];
    ++pos;
  }
  if (t == 0) s_base = total ? atomicAdd(reinterpret_cast<unsigned int*>(dst), (unsigned)total) : 0u;
  __syncthreads();
  const uint32_t off = s_base;
  if (t == 0) {
    reinterpret_cast<uint32_t*>(dst + counts_offset(n))[b] = (uint32_t)total;
    reinterpret_cast<uint32_t*>(dst + offsets_offset(n))[b] = off;
  }
  if (total == 0) return;
  uint4* dmask = reinterpret_cast<uint4*>(dst + mask_offset(n) + b * (BLK / 8));
  if (t < MASK_WORDS / 4) dmask[t] = reinterpret_cast<const uint4*>(s_mask)[t];
  T* dval = reinterpret_cast<T*>(dst + values_offset(n)) + off;
  // the run starts at an arbitrary element: a scalar head up to 16-byte alignment, then uint4s
  constexpr int E = 16 / (int)sizeof(T);
  const int head = (int)(((16 - ((uintptr_t)dval & 15)) & 15) / sizeof(T));
  const int h = head < total ? head : total;
  if (t < h) dval[t] = s_val[t];
  const int rest = total - h;
  const int nvec = rest / E;
  for (int i = t; i < nvec; i += THREADS) {
    uint4 v;
    T* pv = reinterpret_cast<T*>(&v);
#pragma unroll
    for (int e = 0; e < E; ++e) pv[e] = s_val[h + i * E + e];
    reinterpret_cast<uint4*>(dval + h)[i] = v;
  }
  for (int i = h + nvec * E + t; i < total; i += THREADS) dval[i] = s_val[i];
}

}  // namespace delta
}  // namespace irdn
