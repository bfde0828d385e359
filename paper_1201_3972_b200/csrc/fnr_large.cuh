// Tiled FNR / MF kernel for large windows (k >= 13, r <= LMAX_R) and for layouts the TMA
// kernels cannot take (row pitch or frame stride not a multiple of 16 bytes, e.g. the
// reference's 364-pixel rows). Any frame size, u8 or u16, row strips (global clamp).
//
// One 256-thread CTA per 64 x 16 output tile:
//   1. the tile plus an r-pixel halo is loaded into shared memory once, with the
//      replicate-edge clamp applied at load time (image.py:117-130);
//   2. detector (filters.py:169-171): separable window min / max — a k-wide horizontal
//      min / max per halo row, then a k-tall vertical one per output pixel — instead of
//      k^2 compares per pixel; signal pixels are written straight out, flagged ones are
//      queued in shared memory (MF queues every pixel);
//   3. median (filters.py:172-176, sorting.py:51-56): one WARP per queued pixel — the k^2
//      window values are spread over the 32 lanes and the (k^2-1)/2-th smallest is built
//      bit by bit (the largest t with #{v < t} <= rank), one warp-wide sum per bit,
//      starting below the highest bit where the window's min and max differ.
// Exact integer selection, so the result equals the introsort median bit for bit.
#pragma once
#include "fnr_common.cuh"

namespace irdn {
namespace large {

constexpr int TW = 64, TH = 16, THREADS = 256;  // TW = 64: index math uses >> 6
constexpr int LMAX_R = 31;  // k <= 63 (shared memory: (16 + 62) x (64 + 62) pixels)

template <typename T>
struct Smem {
  static constexpr int MAXW = TW + 2 * LMAX_R, MAXH = TH + 2 * LMAX_R;
  T tile[MAXH * MAXW];
  T hmin[MAXH * TW];
  T hmax[MAXH * TW];
  uint16_t q[TW * TH];
  int nq;
};

// Medians of the queued pixels, one warp per pixel. V > 0: lane l holds window elements
// l, l + 32, ... (at most V of them, offsets precomputed in `off`) in registers for the whole
// bit-by-bit search; V = 0 (k > 31): the elements are re-read from shared memory per bit.
template <typename T, int V>
__device__ __forceinline__ uint32_t select_queue(const Smem<T>& S, int nq, int SW, int r, const int (&off)[V > 0 ? V : 1],
                                                 int rank, T* oframe, int y0, int x0, const PassGeom& g, bool fnr,
                                                 int k = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t replaced = 0;
  for (int e = warp; e < nq; e += THREADS / 32) {
    const int oy = S.q[e] >> 8, ox = S.q[e] & 0xFF;
    const T* win = S.tile + oy * SW + ox;
    uint32_t mn = 0xFFFFFFFFu, mx = 0u, m;
    if constexpr (V > 0) {
      uint32_t v[V];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const bool ok = off[j] >= 0;
        v[j] = ok ? (uint32_t)win[off[j]] : 0xFFFFFFFFu;  // never below a threshold t < 2^16
        mn = min(mn, v[j]);
        mx = max(mx, ok ? v[j] : 0u);
      }
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      m = mn;
      const uint32_t diff = mn ^ mx;
      if (diff) {
        const int hb = 31 - __clz(diff);
        m = mn & ~((2u << hb) - 1u);
        for (int bit = hb; bit >= 0; --bit) {
          const uint32_t t = m | (1u << bit);
          uint32_t below = 0;
#pragma unroll
          for (int j = 0; j < V; ++j) below += v[j] < t;
          below = __reduce_add_sync(0xffffffffu, below);
          if ((int)below <= rank) m = t;
        }
      }
    } else {
      const int kk = k * k, dy0 = lane / k, dx0 = lane - dy0 * k;
      for (int i = lane, dy = dy0, dx = dx0; i < kk; i += 32) {
        const uint32_t x = win[dy * SW + dx];
        mn = min(mn, x);
        mx = max(mx, x);
        dx += 32;
        while (dx >= k) dx -= k, ++dy;
      }
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      m = mn;
      const uint32_t diff = mn ^ mx;
      if (diff) {
        const int hb = 31 - __clz(diff);
        m = mn & ~((2u << hb) - 1u);
        for (int bit = hb; bit >= 0; --bit) {
          const uint32_t t = m | (1u << bit);
          uint32_t below = 0;
          for (int i = lane, dy = dy0, dx = dx0; i < kk; i += 32) {
            below += (uint32_t)win[dy * SW + dx] < t;
            dx += 32;
            while (dx >= k) dx -= k, ++dy;
          }
          below = __reduce_add_sync(0xffffffffu, below);
          if ((int)below <= rank) m = t;
        }
      }
    }
    if (lane == 0) {
      oframe[(int64_t)(y0 + oy - g.row_begin) * g.out_pitch + x0 + ox] = (T)m;
      if (fnr) replaced += m != (uint32_t)win[r * SW + r];
    }
  }
  return replaced;
}

// V: window elements per lane held in registers by the median search (kk <= 32 V), 0 = none
template <typename T, int V>
__global__ void __launch_bounds__(THREADS) fnr_large_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                            PassGeom g, int k, int method,
                                                            unsigned long long* counts) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem<T>& S = *reinterpret_cast<Smem<T>*>(smem_raw);
  const int r = k >> 1, rank = (k * k - 1) >> 1;
  const int SW = TW + 2 * r, SH = TH + 2 * r;  // halo tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles_x = (g.width + TW - 1) / TW;
  const int x0 = (blockIdx.x % tiles_x) * TW;
  const int y0 = g.row_begin + (blockIdx.x / tiles_x) * TH;
  const bool fnr = method == 0;
  uint32_t detected = 0, replaced = 0;
  // this lane's window elements l, l + 32, ... as offsets into the halo tile (-1: none)
  const int kk = k * k;
  int off[V > 0 ? V : 1];
#pragma unroll
  for (int j = 0; j < (V > 0 ? V : 1); ++j) {
    const int i = lane + 32 * j;
    off[j] = i < kk ? (i / k) * SW + (i % k) : -1;
  }
  pdl_wait_and_trigger();

  for (int b = blockIdx.y; b < g.batch; b += gridDim.y) {
    const T* frame = in + (int64_t)b * g.in_frame_stride;
    T* oframe = out + (int64_t)b * g.out_frame_stride;
    if (tid == 0) S.nq = 0;
    // 1. halo tile, clamped against the global frame (replicate edge) and then to the rows
    //    the input strip holds: rows past the strip only feed output rows past row_end of a
    //    partial last tile, which are never stored, and must not be read (strip contract).
    const int ylo = max(0, g.in_row0), yhi = min(g.height, g.in_row0 + g.in_rows) - 1;
    for (int iy = warp; iy < SH; iy += THREADS / 32) {
      const int gy = clampi(clampi(y0 - r + iy, 0, g.height - 1), ylo, yhi);
      const T* src = frame + (int64_t)(gy - g.in_row0) * g.in_pitch;
      for (int ix = lane; ix < SW; ix += 32) S.tile[iy * SW + ix] = src[clampi(x0 - r + ix, 0, g.width - 1)];
    }
    __syncthreads();
    // 2a. horizontal k-wide min / max of every halo row (only the TW output columns)
    for (int i = tid; i < SH * TW; i += THREADS) {
      const int iy = i >> 6, ix = i & (TW - 1);  // TW = 64
      const T* row = S.tile + iy * SW + ix;
      uint32_t mn = row[0], mx = row[0];
      for (int d = 1; d < k; ++d) {
        const uint32_t v = row[d];
        mn = min(mn, v);
        mx = max(mx, v);
      }
      S.hmin[iy * TW + ix] = (T)mn;
      S.hmax[iy * TW + ix] = (T)mx;
    }
    __syncthreads();
    // 2b. vertical k-tall min / max, flag test, signal pixels out, flagged ones queued
    for (int i = tid; i < TH * TW; i += THREADS) {
      const int oy = i >> 6, ox = i & (TW - 1);
      const int y = y0 + oy, x = x0 + ox;
      const bool valid = y < g.row_end && x < g.width;
      bool queue = false;
      if (valid) {
        const uint32_t c = S.tile[(oy + r) * SW + ox + r];
        if (fnr) {
          uint32_t mn = S.hmin[oy * TW + ox], mx = S.hmax[oy * TW + ox];
          for (int d = 1; d < k; ++d) {
            mn = min(mn, (uint32_t)S.hmin[(oy + d) * TW + ox]);
            mx = max(mx, (uint32_t)S.hmax[(oy + d) * TW + ox]);
          }
          queue = c == mn || c == mx;
          if (!queue) oframe[(int64_t)(y - g.row_begin) * g.out_pitch + x] = (T)c;
        } else {
          queue = true;
        }
      }
      // warp-aggregated append to the queue
      const unsigned bal = __ballot_sync(0xffffffffu, queue);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(&S.nq, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (queue) S.q[base + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)((oy << 8) | ox);
    }
    __syncthreads();
    // 3. one warp per queued pixel: bitwise rank selection over the k x k window
    const int nq = S.nq;
    if (fnr) detected += tid == 0 ? (uint32_t)nq : 0u;
    replaced += select_queue<T, V>(S, nq, SW, r, off, rank, oframe, y0, x0, g, fnr, k);
    __syncthreads();  // the queue and tile are reused by the next frame
  }
  if (fnr) block_add_counts<THREADS>(detected, replaced, counts);
}

}  // namespace large
}  // namespace irdn
