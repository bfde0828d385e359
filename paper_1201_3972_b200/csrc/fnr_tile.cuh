// TMA tile kernel for the FNR / MF pass (sm_100a), persistent and double-buffered.
//
// Each CTA loops over TH x TW output tiles (tile t, t + gridDim.x, ...) of a
// [batch, rows, width] u8/u16 image stack:
//   1. TMA (cp.async.bulk.tensor.3d) stages the tile plus its halo into one of
//      two shared-memory stages; the load of tile i+1 is in flight while tile i
//      is filtered. TMA fills out-of-frame cells with zeros, so tiles touching
//      the frame border rewrite those cells from the nearest in-frame cell
//      (replicate edge, reference image.py:117-130).
//   2. Detector (filters.py:169-171): separable window min/max on packed u16x2
//      words (two horizontally adjacent pixels per 32-bit op): per input row a
//      horizontal K-wide min/max, then a vertical K-row min/max over a register
//      ring while each thread walks down its column pair. A pixel is noisy iff
//      centre == min or == max. Signal pixels go straight to the output tile;
//      noisy pixels set bits in a per-thread mask that is compacted into a
//      shared-memory queue with one warp scan and one atomic per warp.
//   3. Median (filters.py:172-176, sorting.py:51-56): each thread takes two
//      queued pixels, packs their K*K window values into u16x2 words and runs
//      one exact median-selection network (select_nets.cuh) for both.
//      MF (filters.py:179-180) runs the network on every pixel.
//   4. The output tile leaves through a TMA store (clipped at the frame edge);
//      detected / replacement counters go out with one atomic per CTA.
#pragma once
#include <cuda.h>
#include "fnr_common.cuh"
#include "select_nets.cuh"

namespace irdn {
namespace tile {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int TW = 128;                 // output tile width (pixels) = 2 warps x 32 pairs
constexpr int TH = 64;                  // output tile height (rows)
constexpr int BANDS = WARPS / 2;        // row bands per tile
constexpr int BAND = TH / BANDS;        // rows walked by one thread (<= 16: one flag bit per row and lane)
static_assert(BAND <= 16, "flag mask holds 16 rows");

template <typename T, int K>
struct Geo {
  static constexpr int r = K / 2;
  static constexpr int ALIGN = 16 / (int)sizeof(T);
  // Left halo of the smem box. The TMA box's innermost start coordinate must be a
  // multiple of 16 bytes (a misaligned start, in or out of bounds, raises
  // cudaErrorIllegalInstruction on sm_100a — measured, tools/microbench/tma_probe.cu),
  // so the box starts ALIGN elements left of the tile; this also keeps output
  // pixel pairs 4-byte aligned in shared memory.
  static constexpr int R = ALIGN;
  static_assert(r <= R, "window radius exceeds the aligned halo");
  static constexpr int BOXW = ((TW + R + r + ALIGN - 1) / ALIGN) * ALIGN;
  static constexpr int BOXH = TH + 2 * r;
  static constexpr int IN_BYTES = BOXW * BOXH * (int)sizeof(T);
  static constexpr int IN_STRIDE = (IN_BYTES + 127) & ~127;
  static constexpr int OUT_BYTES = TW * TH * (int)sizeof(T);
  static constexpr int OUT_OFF = 2 * IN_STRIDE;
  static constexpr int Q_OFF = (OUT_OFF + OUT_BYTES + 127) & ~127;
  static constexpr int BAR_OFF = Q_OFF + TW * TH * 2;
  static constexpr int SMEM = BAR_OFF + 64 + 128;  // +128: runtime base alignment
  static_assert(BOXW <= 256 && BOXH <= 256, "TMA box limit");
};

struct TileParams {
  int32_t width;      // frame width
  int32_t height;     // GLOBAL frame height (clamp bound)
  int32_t in_row0;    // global row of input-map row 0
  int32_t row_begin;  // first output row (global); output-map row 0
  int32_t row_end;
  int32_t tiles_x;
  int32_t tiles_y;
  int32_t batch;
  int32_t method;     // 0 fnr, 1 mf
  unsigned long long* counts;
};

// ---- PTX helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Two adjacent pixels of smem row `row` starting at (even) column `col`, as u16x2.
template <typename T>
__device__ __forceinline__ uint32_t load_pair(const T* row, int col) {
  if constexpr (sizeof(T) == 2) {
    return *reinterpret_cast<const uint32_t*>(row + col);
  } else {
    const uint32_t b = *reinterpret_cast<const uint16_t*>(row + col);
    return prmt(b, 0u, 0x4140u);  // bytes (b0, 0, b1, 0)
  }
}
template <typename T>
__device__ __forceinline__ void store_pair(T* row, int col, uint32_t v) {
  if constexpr (sizeof(T) == 2) {
    *reinterpret_cast<uint32_t*>(row + col) = v;
  } else {
    *reinterpret_cast<uint16_t*>(row + col) = (uint16_t)prmt(v, 0u, 0x0020u);
  }
}

template <int NV>
__device__ __forceinline__ uint32_t median_dispatch(uint32_t (&v)[NV]) {
  if constexpr (NV == 9) return median_net_9(v);
  else if constexpr (NV == 25) return median_net_25(v);
  else if constexpr (NV == 49) return median_net_49(v);
  else if constexpr (NV == 81) return median_net_81(v);
  else return median_net_121(v);
}

// Replicate-edge fix-up of the smem cells of a box that fall outside the frame.
template <typename T, int K>
__device__ __forceinline__ void fix_edges(T* s_in, int gx_lo, int gy_lo, int width, int height) {
  using G = Geo<T, K>;
  constexpr int BOXW = G::BOXW, BOXH = G::BOXH;
  const int tid = threadIdx.x;
  const int c_lo = max(0, -gx_lo), c_hi = min(BOXW, width - gx_lo);   // in-frame columns
  const int y_lo = max(0, -gy_lo), y_hi = min(BOXH, height - gy_lo);  // in-frame rows
  const int ncl = c_lo, ncr = BOXW - c_hi;
  const int nc = ncl + ncr;
  if (nc) {  // (a) left / right margins of in-frame rows
    for (int i = tid; i < (y_hi - y_lo) * nc; i += THREADS) {
      const int row = y_lo + i / nc;
      const int j = i % nc;
      const int col = j < ncl ? j : c_hi + (j - ncl);
      s_in[row * BOXW + col] = s_in[row * BOXW + (j < ncl ? c_lo : c_hi - 1)];
    }
    __syncthreads();
  }
  const int nrt = y_lo, nrb = BOXH - y_hi;
  // (b) rows above / below the frame copy the nearest in-frame row (corners included)
  for (int i = tid; i < (nrt + nrb) * BOXW; i += THREADS) {
    const int j = i / BOXW, col = i % BOXW;
    const int row = j < nrt ? j : y_hi + (j - nrt);
    s_in[row * BOXW + col] = s_in[(j < nrt ? y_lo : y_hi - 1) * BOXW + col];
  }
}

// ---- the kernel ----------------------------------------------------------------
template <typename T, int K>
__global__ void __launch_bounds__(THREADS) fnr_tile_kernel(const __grid_constant__ CUtensorMap in_map,
                                                           const __grid_constant__ CUtensorMap out_map,
                                                           const TileParams p) {
  using G = Geo<T, K>;
  constexpr int r = G::r, R = G::R, BOXW = G::BOXW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // TMA needs 128-byte aligned shared-memory boxes: align the dynamic base explicitly.
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* s_out = reinterpret_cast<T*>(smem + G::OUT_OFF);
  uint16_t* s_q = reinterpret_cast<uint16_t*>(smem + G::Q_OFF);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + G::BAR_OFF);  // [2] full barriers
  int* s_qn = reinterpret_cast<int*>(smem + G::BAR_OFF + 16);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tiles_per_frame = p.tiles_x * p.tiles_y;
  const int ntiles = tiles_per_frame * p.batch;
  uint32_t replaced = 0, detected = 0;

  auto tile_origin = [&](int t, int& b, int& tx0, int& ty0) {
    b = t / tiles_per_frame;
    const int tt = t - b * tiles_per_frame;
    const int ty = tt / p.tiles_x;
    tx0 = (tt - ty * p.tiles_x) * TW;
    ty0 = p.row_begin + ty * TH;
  };
  auto issue_load = [&](int t, int stage) {
    int b, tx0, ty0;
    tile_origin(t, b, tx0, ty0);
    mbar_expect_tx(&s_bar[stage], G::IN_BYTES);
    tma_load_3d(smem + stage * G::IN_STRIDE, &in_map, &s_bar[stage], tx0 - R, ty0 - r - p.in_row0, b);
  };

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    *s_qn = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int t0 = blockIdx.x, t1 = blockIdx.x + gridDim.x;
    if (t0 < ntiles) issue_load(t0, 0);
    if (t1 < ntiles) issue_load(t1, 1);
  }
  __syncthreads();

  // detector geometry: warp -> (column half, row band); thread -> one column pair
  const int w = (warp & 1) * 32 + lane;  // pair index: pixels 2w, 2w+1 of the tile row
  const int band0 = (warp >> 1) * BAND;  // first output row of this thread's band
  const int c0 = 2 * w + R;              // smem column of lane 0's pixel

  int iter = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++iter) {
    const int stage = iter & 1;
    T* s_in = reinterpret_cast<T*>(smem + stage * G::IN_STRIDE);
    int b, tx0, ty0;
    tile_origin(t, b, tx0, ty0);
    mbar_wait(&s_bar[stage], (iter >> 1) & 1);
    const int gx_lo = tx0 - R, gy_lo = ty0 - r;  // global coords of smem (0, 0)
    if (gx_lo < 0 || gy_lo < 0 || gx_lo + BOXW > p.width || gy_lo + G::BOXH > p.height)
      fix_edges<T, K>(s_in, gx_lo, gy_lo, p.width, p.height);
    if (tid == 0) tma_store_wait_read();  // the previous tile's store has left s_out
    __syncthreads();

    const int valid_w = min(TW, p.width - tx0);    // valid output columns in this tile
    const int valid_h = min(TH, p.row_end - ty0);  // valid output rows

    if (p.method == 0) {
      // ---- detector ----
      constexpr int J = (r + 1) / 2;
      uint32_t rmin[K], rmax[K], rcen[r + 1];
      uint32_t flags = 0;
#pragma unroll
      for (int s = 0; s < BAND + 2 * r; ++s) {
        const T* row = s_in + (band0 + s) * BOXW;
        uint32_t wd[2 * J + 1];
#pragma unroll
        for (int j = -J; j <= J; ++j) wd[j + J] = load_pair<T>(row, c0 + 2 * j);
        uint32_t mn = wd[J], mx = wd[J];
#pragma unroll
        for (int d = -r; d <= r; ++d) {
          if (d == 0) continue;
          uint32_t op;
          if ((d & 1) == 0) op = wd[J + d / 2];
          else op = prmt(wd[J + (d - 1) / 2], wd[J + (d + 1) / 2], 0x5432u);
          mn = vmin2(mn, op);
          mx = vmax2(mx, op);
        }
        rmin[s % K] = mn;
        rmax[s % K] = mx;
        rcen[s % (r + 1)] = wd[J];
        if (s >= 2 * r) {
          const int y = s - 2 * r;  // output row within the band
          uint32_t vmn = rmin[0], vmx = rmax[0];
#pragma unroll
          for (int i = 1; i < K; ++i) {
            vmn = vmin2(vmn, rmin[i]);
            vmx = vmax2(vmx, rmax[i]);
          }
          const uint32_t c = rcen[(s - r) % (r + 1)];
          // lane of m == 0  <=>  centre equals the window min or max (no borrow: vmn <= c <= vmx)
          const uint32_t m = vmin2(c - vmn, vmx - c);
          // m < 0x8000 per lane (it is at most (max-min)/2), so +0x7FFF sets bit 15 iff m != 0
          const uint32_t e = m + 0x7FFF7FFFu;
          flags |= (~e & 0x80008000u) >> (15 - y);
          store_pair<T>(s_out + (band0 + y) * TW, 2 * w, c);
        }
      }
      // mask out pixels beyond the frame / strip, then compact into the queue
      const int vr = min(BAND, max(0, valid_h - band0));
      const uint32_t rowm = vr >= 16 ? 0xFFFFu : ((1u << vr) - 1u);
      const uint32_t colm = (2 * w < valid_w ? rowm : 0u) | (2 * w + 1 < valid_w ? (rowm << 16) : 0u);
      flags &= colm;
      const int cnt = __popc(flags);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      int base = 0;
      if (lane == 31 && total) base = atomicAdd(s_qn, total);
      base = __shfl_sync(0xffffffffu, base, 31);
      int pos = base + incl - cnt;
      while (flags) {
        const int bit = __ffs(flags) - 1;
        flags &= flags - 1u;
        const int y = band0 + (bit & 15);
        s_q[pos++] = (uint16_t)((y << 8) | (2 * w + (bit >> 4)));
      }
      __syncthreads();
    }

    // ---- median of queued (FNR) or all (MF) pixels, two per thread ----
    const int n = p.method == 0 ? *s_qn : TW * TH;
    if (p.method == 0) detected += (tid == 0) ? (uint32_t)n : 0u;
    for (int i = tid; 2 * i < n; i += THREADS) {
      uint32_t e0, e1;
      if (p.method == 0) {
        e0 = s_q[2 * i];
        e1 = (2 * i + 1 < n) ? s_q[2 * i + 1] : e0;
      } else {
        e0 = ((uint32_t)((2 * i) / TW) << 8) | (uint32_t)((2 * i) % TW);
        e1 = e0 + 1u;
      }
      const int y0 = (int)(e0 >> 8), x0 = (int)(e0 & 0xFFu);
      const int y1 = (int)(e1 >> 8), x1 = (int)(e1 & 0xFFu);
      const T* a = s_in + y0 * BOXW + x0 + (R - r);
      const T* bb = s_in + y1 * BOXW + x1 + (R - r);
      uint32_t v[K * K];
#pragma unroll
      for (int dy = 0; dy < K; ++dy)
#pragma unroll
        for (int dx = 0; dx < K; ++dx)
          v[dy * K + dx] = (uint32_t)a[dy * BOXW + dx] | ((uint32_t)bb[dy * BOXW + dx] << 16);
      const uint32_t med = median_dispatch<K * K>(v);
      const uint32_t m0 = med & 0xFFFFu, m1 = med >> 16;
      s_out[y0 * TW + x0] = (T)m0;
      if (p.method == 0) {
        replaced += (m0 != (uint32_t)a[r * BOXW + r]);
        if (2 * i + 1 < n) {
          s_out[y1 * TW + x1] = (T)m1;
          replaced += (m1 != (uint32_t)bb[r * BOXW + r]);
        }
      } else {
        s_out[y1 * TW + x1] = (T)m1;
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tma_store_3d(&out_map, s_out, tx0, ty0 - p.row_begin, b);
      *s_qn = 0;
      const int tn = t + 2 * gridDim.x;  // this stage is free again: prefetch two tiles ahead
      if (tn < ntiles) issue_load(tn, stage);
    }
  }
  if (tid == 0) tma_store_wait_all();
  if (p.method == 0) block_add_counts<THREADS>(detected, replaced, p.counts);
}

}  // namespace tile
}  // namespace irdn
