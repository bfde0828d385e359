// TMA tile kernel for the FNR / MF pass (sm_100a): persistent, per-warp work queues.
//
// Each CTA (4 warps) loops over TH x TW output tiles (t, t + gridDim.x, ...) of a
// [batch, rows, width] u8/u16 image stack:
//   1. TMA (cp.async.bulk.tensor.3d) stages the tile plus its halo into one of
//      NSTAGE shared-memory stages; with two stages the load of the next tile is
//      in flight while this one is filtered. TMA fills out-of-frame cells with
//      zeros, so tiles touching the frame border rewrite those cells from the
//      nearest in-frame cell (replicate edge, reference image.py:117-130).
//   2. Detector (filters.py:169-171): each warp owns a 64 x 32 strip; each thread
//      one column pair (two horizontally adjacent pixels packed as u16x2) walking
//      down the strip. Per input row a horizontal K-wide min/max, then a vertical
//      K-row min/max over a register ring. A pixel is noisy iff centre == min or
//      == max. Signal pixels are stored straight to global memory (one coalesced
//      128-byte row segment per warp); noisy pixels set bits in per-thread masks.
//   3. Median (filters.py:172-176, sorting.py:51-56): per 16-row half strip, the
//      warp compacts its noisy pixels into a warp-private queue (one warp scan),
//      then each lane takes two queued pixels, packs their K*K window values into
//      u16x2 words and runs one exact median-selection network (select_nets.cuh)
//      for both; medians overwrite the copied centres in global memory.
//      MF (filters.py:179-180) runs the network on every pixel.
//   4. Detected / replacement counters leave with one atomic per CTA at the end.
#pragma once
#include <cuda.h>
#include "fnr_common.cuh"
#include "select_nets.cuh"

#ifndef IRDN_NSTAGE
#define IRDN_NSTAGE 2
#endif

namespace irdn {
namespace tile {

constexpr int THREADS = 128;
constexpr int WARPS = THREADS / 32;
constexpr int TW = 128;                 // output tile width (pixels) = 2 warps x 32 pixel pairs
#ifndef IRDN_TH
#define IRDN_TH 32
#endif
constexpr int TH = IRDN_TH;             // output tile height (rows)
constexpr int BAND = TH / (WARPS / 2);  // rows walked by one thread
constexpr int NFW = BAND / 16;          // 16-row flag words per thread
constexpr int STRIP_PX = 64 * BAND;     // pixels of one warp strip (queue capacity)
constexpr int NSTAGE = IRDN_NSTAGE;     // input stages (2 = double-buffered TMA)
static_assert(BAND % 16 == 0 && NFW >= 1, "whole 16-row flag words per thread");

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
  static constexpr int Q_OFF = NSTAGE * IN_STRIDE;
  static constexpr int BAR_OFF = Q_OFF + WARPS * STRIP_PX * 2;
  static constexpr int TILE_OFF = BAR_OFF + 8 * NSTAGE;  // TileInfo staged with each buffer
  static constexpr int SMEM = TILE_OFF + 16 * NSTAGE + 128;  // +128: runtime base alignment
  static_assert(BOXW <= 256 && BOXH <= 256, "TMA box limit");
};

struct TileParams {
  void* out;          // output pixel (row_begin, 0) of frame 0
  int64_t out_pitch;  // elements
  int64_t out_frame;  // elements between output frames
  int32_t width;      // frame width
  int32_t height;     // GLOBAL frame height (clamp bound)
  int32_t in_row0;    // global row of input-map row 0
  int32_t row_begin;  // first output row (global)
  int32_t row_end;
  int32_t tiles_x;
  int32_t tiles_y;
  int32_t batch;
  int32_t method;     // 0 fnr, 1 mf
  unsigned long long* counts;
  unsigned int* sched;  // [0] next tile to hand out, [1] finished warps/CTAs (reset to 0 by the last)
  uint32_t one;         // 1, opaque to the compiler (keeps adds as IMAD on the FMA pipe)
  int32_t debug;        // experiments only: 1 = skip the median stage, 2 = skip the network
  int32_t full_tiles;   // warp kernel: tiles [0, full_tiles) are full height, the rest half-height halves
  int32_t static_rounds;  // warp kernel: warp w takes tiles w + k * nwarps for k < static_rounds, then dynamic
  // multi-pass warp kernel (fnr_warp_mp_kernel): `passes` passes in one launch
  int32_t passes;
  void* tmp;              // ping-pong buffer (same geometry as out)
  unsigned int* flags;    // [0] launch epoch of the stream; from [32]: (passes - 1) x tiles-per-pass flags
  uint32_t epoch;         // unused on the host (the kernel derives the epoch from flags[0])
  unsigned long long* debug_buf;  // experiments only (IRDN_TIMELINE builds): per-warp timeline
  // warp kernel, k = 5 / 7 (fnr_dense.cuh): FNR tiles with more than dense_min flagged
  // pixels take the dense median stage; dense_min < 0 keeps MF on the queue path too
  int32_t dense_min;
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
// Store a packed pixel pair to global memory (lanes beyond the frame are dropped).
template <typename T>
__device__ __forceinline__ void store_pair_g(T* dst, uint32_t v, bool ok0, bool ok1) {
  if constexpr (sizeof(T) == 2) {
    if (ok0 && ok1) *reinterpret_cast<uint32_t*>(dst) = v;
    else if (ok0) dst[0] = (T)(v & 0xFFFFu);
  } else {
    if (ok0 && ok1) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)prmt(v, 0u, 0x0020u);
    else if (ok0) dst[0] = (T)(v & 0xFFu);
  }
}

template <int NV>
__device__ __forceinline__ uint32_t median_dispatch(uint32_t (&v)[NV], uint32_t m1) {
  if constexpr (NV == 9) return median_net_9(v, m1);
  else if constexpr (NV == 25) return median_net_25(v, m1);
  else if constexpr (NV == 49) return median_net_49(v, m1);
  else if constexpr (NV == 81) return median_net_81(v, m1);
  else return median_net_121(v, m1);
}

// Min / max of N packed words with 3-input VIMNMX3 (N odd: (N-1)/2 instructions).
template <int N>
__device__ __forceinline__ uint32_t reduce_min(const uint32_t (&a)[N]) {
  uint32_t m = a[0];
  int i = 1;
#pragma unroll
  for (; i + 1 < N; i += 2) m = vmin3(m, a[i], a[i + 1]);
  if (i < N) m = vmin2(m, a[i]);
  return m;
}
template <int N>
__device__ __forceinline__ uint32_t reduce_max(const uint32_t (&a)[N]) {
  uint32_t m = a[0];
  int i = 1;
#pragma unroll
  for (; i + 1 < N; i += 2) m = vmax3(m, a[i], a[i + 1]);
  if (i < N) m = vmax2(m, a[i]);
  return m;
}

// Replicate-edge fix-up of the smem cells of a box that fall outside the frame.
// Common case (frame wider than the box's halo on that side): the margin is exactly
// ALIGN elements = 16 bytes per row, written with one 16-byte store per row.
template <typename T, int K>
__device__ __forceinline__ void fix_edges(T* s_in, int gx_lo, int gy_lo, int width, int height) {
  using G = Geo<T, K>;
  constexpr int BOXW = G::BOXW, BOXH = G::BOXH, A = G::ALIGN;
  const int tid = threadIdx.x;
  const int c_lo = max(0, -gx_lo), c_hi = min(BOXW, width - gx_lo);   // in-frame columns
  const int y_lo = max(0, -gy_lo), y_hi = min(BOXH, height - gy_lo);  // in-frame rows
  const int ncl = c_lo, ncr = BOXW - c_hi;
  const int lane = tid & 31, warp = tid >> 5;
  if (ncl | ncr) {
    if ((ncl == 0 || ncl == A) && (ncr == 0 || ncr == A)) {
      // (a) one thread per (row, side): replicate the edge pixel over a 16-byte margin
      for (int i = tid; i < 2 * (y_hi - y_lo); i += THREADS) {
        const int row = y_lo + (i >> 1);
        const bool left = (i & 1) == 0;
        if (left ? ncl == 0 : ncr == 0) continue;
        T* rp = s_in + row * BOXW;
        uint32_t v = (uint32_t)rp[left ? c_lo : c_hi - 1];
        if constexpr (sizeof(T) == 1) v *= 0x01010101u;
        else v *= 0x00010001u;
        const uint4 q = make_uint4(v, v, v, v);
        *reinterpret_cast<uint4*>(rp + (left ? 0 : BOXW - A)) = q;
      }
    } else {
      // (a') general margins: warps over rows, lanes over columns
      const int nc = ncl + ncr;
      for (int row = y_lo + warp; row < y_hi; row += WARPS) {
        T* rp = s_in + row * BOXW;
        for (int j = lane; j < nc; j += 32) {
          const int col = j < ncl ? j : c_hi + (j - ncl);
          rp[col] = rp[j < ncl ? c_lo : c_hi - 1];
        }
      }
    }
    __syncthreads();
  }
  // (b) rows above / below the frame copy the nearest in-frame row (corners included), 16 B at a time
  const int nrt = y_lo, nrb = BOXH - y_hi;
  constexpr int V = BOXW / A;  // 16-byte vectors per row
  for (int i = tid; i < (nrt + nrb) * V; i += THREADS) {
    const int j = i / V, col = (i - j * V) * A;
    const int row = j < nrt ? j : y_hi + (j - nrt);
    *reinterpret_cast<uint4*>(s_in + row * BOXW + col) =
        *reinterpret_cast<const uint4*>(s_in + (j < nrt ? y_lo : y_hi - 1) * BOXW + col);
  }
}

// Median of the pixels listed in q[0..n) (tile coords y << 8 | x), two per lane; the
// medians overwrite the copied centres at out_tile. Returns this lane's replacements.
template <typename T, int K>
__device__ __forceinline__ uint32_t median_queue(const T* s_in, const uint16_t* q, int n, T* out_tile,
                                                 int64_t pitch, int lane, bool fnr, uint32_t m1) {
  using G = Geo<T, K>;
  constexpr int r = G::r, R = G::R, BOXW = G::BOXW;
  uint32_t replaced = 0;
  const bool skip_net = n < 0;
  if (skip_net) n = -n;
  for (int i = lane; 2 * i < n; i += 32) {
    const uint32_t e0 = q[2 * i];
    const bool two = 2 * i + 1 < n;
    const uint32_t e1 = two ? q[2 * i + 1] : e0;
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
    const uint32_t med = skip_net ? (v[0] ^ v[K * K - 1] ^ v[K * K / 2]) : median_dispatch<K * K>(v, m1);
    const uint32_t med0 = med & 0xFFFFu, med1 = med >> 16;
    out_tile[y0 * pitch + x0] = (T)med0;
    if (two) out_tile[y1 * pitch + x1] = (T)med1;
    if (fnr) replaced += (med0 != (uint32_t)a[r * BOXW + r]) + (two && med1 != (uint32_t)bb[r * BOXW + r]);
  }
  return replaced;
}

// Detector over one warp strip (see the file comment). FULL: the strip lies entirely
// inside the frame, so no per-row / per-column validity checks are needed.
template <typename T, int K, bool FULL>
__device__ __forceinline__ void detect_strip(const T* s_in, int band0, int c0, T* outp, int64_t pitch, int valid_rows,
                                             bool ok0, bool ok1, uint32_t (&flags)[NFW], uint32_t one) {
  const uint32_t m1 = 0u - one, k65536 = one << 16, k2p31 = one << 31;
  using G = Geo<T, K>;
  constexpr int r = G::r, BOXW = G::BOXW;
  constexpr int J = (r + 1) / 2;
  uint32_t rmin[K], rmax[K], rcen[r + 1];
#pragma unroll
  for (int h = 0; h < NFW; ++h) flags[h] = 0u;
  const T* rowp = s_in + band0 * BOXW + c0;
#pragma unroll
  for (int s = 0; s < BAND + 2 * r; ++s) {
    uint32_t wd[2 * J + 1];
#pragma unroll
    for (int j = -J; j <= J; ++j) wd[j + J] = load_pair<T>(rowp + s * BOXW, 2 * j);
    uint32_t ops[K];  // lane-aligned operands for horizontal offsets -r..r
#pragma unroll
    for (int d = -r; d <= r; ++d)
      ops[d + r] = (d & 1) == 0 ? wd[J + d / 2] : shift_pair(wd[J + (d - 1) / 2], wd[J + (d + 1) / 2], k65536);
    rmin[s % K] = reduce_min<K>(ops);
    rmax[s % K] = reduce_max<K>(ops);
    rcen[s % (r + 1)] = wd[J];
    if (s >= 2 * r) {
      const int y = s - 2 * r;  // output row within the strip
      const uint32_t vmn = reduce_min<K>(rmin), vmx = reduce_max<K>(rmax);
      const uint32_t c = rcen[(s - r) % (r + 1)];
      // lane of m == 0  <=>  centre equals the window min or max (no borrow: vmn <= c <= vmx)
      const uint32_t m = vmin2(fma_sub(c, m1, vmn), fma_sub(vmx, m1, c));
      // m < 0x8000 per lane (it is at most (max-min)/2), so +0x7FFF sets bit 15 iff m != 0
      const uint32_t e = fma_add(m, one, 0x7FFF7FFFu);
      // shift the row history down one bit (IMAD.HI on the FMA pipe) and insert this
      // row's "noisy" bits at 15 / 31; after 16 rows row i sits at bits i and 16 + i
      uint32_t sh;
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(sh) : "r"(flags[y >> 4]), "r"(k2p31));
      flags[y >> 4] = (sh & 0x7FFF7FFFu) | (~e & 0x80008000u);
      if (FULL) store_pair_g<T>(outp, c, true, true);
      else if (y < valid_rows) store_pair_g<T>(outp, c, ok0, ok1);
      outp += pitch;
    }
  }
}

// ---- the kernel ----------------------------------------------------------------
struct TileInfo {
  int t, b, tx0, ty0;
};

template <typename T, int K>
__global__ void __launch_bounds__(THREADS) fnr_tile_kernel(const __grid_constant__ CUtensorMap in_map,
                                                           const TileParams p) {
  using G = Geo<T, K>;
  constexpr int r = G::r, R = G::R, BOXW = G::BOXW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // TMA needs 128-byte aligned shared-memory boxes: align the dynamic base explicitly.
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + G::BAR_OFF);  // [NSTAGE] stage-full barriers
  TileInfo* s_tile = reinterpret_cast<TileInfo*>(smem + G::TILE_OFF);

  pdl_wait_and_trigger();
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint16_t* s_q = reinterpret_cast<uint16_t*>(smem + G::Q_OFF) + warp * STRIP_PX;  // this warp's queue
  const int tiles_per_frame = p.tiles_x * p.tiles_y;
  const int ntiles = tiles_per_frame * p.batch;
  uint32_t replaced = 0, detected = 0;

  // Dynamic tile scheduler (thread 0): grab the next tile, publish it next to the stage,
  // then arrive on the stage barrier (with the TMA bytes, or empty past the end). The
  // barrier's release/acquire makes the TileInfo visible to every waiting thread.
  auto origin = [&](int t) {
    TileInfo ti;
    ti.t = t;
    ti.b = t / tiles_per_frame;
    const int tt = t - ti.b * tiles_per_frame;
    const int ty = tt / p.tiles_x;
    ti.tx0 = (tt - ty * p.tiles_x) * TW;
    ti.ty0 = p.row_begin + ty * TH;
    return ti;
  };
  // Thread 0 keeps the id of the tile it will load next (`ahead`) and asks the TMA unit to
  // pull that tile into L2 while the current one is filtered, so the smem load that
  // follows the end-of-tile barrier is served from L2.
  int ahead = 0;
  auto grab_ahead = [&]() {
    ahead = (int)atomicAdd(p.sched, 1u);
    if (ahead < ntiles) {
      const TileInfo ti = origin(ahead);
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(&in_map),
                   "r"(ti.tx0 - R), "r"(ti.ty0 - r - p.in_row0), "r"(ti.b)
                   : "memory");
    }
  };
  auto refill = [&](int stage) {
    const int t = ahead;
    TileInfo ti;
    if (t < ntiles) {
      ti = origin(t);
      s_tile[stage] = ti;
      mbar_expect_tx(&s_bar[stage], G::IN_BYTES);
      tma_load_3d(smem + stage * G::IN_STRIDE, &in_map, &s_bar[stage], ti.tx0 - R, ti.ty0 - r - p.in_row0, ti.b);
    } else {
      ti.t = t;
      s_tile[stage] = ti;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_bar[stage])) : "memory");
    }
    grab_ahead();
  };

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&s_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    grab_ahead();
    for (int s = 0; s < NSTAGE; ++s) refill(s);
  }
  __syncthreads();

  const int cpair = (warp & 1) * 32 + lane;  // pixel pair: tile columns 2*cpair, 2*cpair+1
  const int band0 = (warp >> 1) * BAND;      // first tile row of this warp's strip
  const int c0 = 2 * cpair + R;              // smem column of lane 0's pixel
  T* const out_base = reinterpret_cast<T*>(p.out);

  for (int iter = 0;; ++iter) {
    const int stage = NSTAGE == 1 ? 0 : (iter % NSTAGE);
    T* s_in = reinterpret_cast<T*>(smem + stage * G::IN_STRIDE);
    mbar_wait(&s_bar[stage], (iter / NSTAGE) & 1);
    const TileInfo ti = s_tile[stage];
    if (ti.t >= ntiles) break;
    const int gx_lo = ti.tx0 - R, gy_lo = ti.ty0 - r;  // global coords of smem (0, 0)
    if (gx_lo < 0 || gy_lo < 0 || gx_lo + BOXW > p.width || gy_lo + G::BOXH > p.height) {
      fix_edges<T, K>(s_in, gx_lo, gy_lo, p.width, p.height);
      __syncthreads();
    }

    const int valid_w = min(TW, p.width - ti.tx0);    // valid output columns in this tile
    const int valid_h = min(TH, p.row_end - ti.ty0);  // valid output rows
    T* const out_tile =
        out_base + (int64_t)ti.b * p.out_frame + (int64_t)(ti.ty0 - p.row_begin) * p.out_pitch + ti.tx0;
    const bool ok0 = 2 * cpair < valid_w, ok1 = 2 * cpair + 1 < valid_w;

    if (p.method == 0) {
      uint32_t flags[NFW];
      T* outp = out_tile + (int64_t)band0 * p.out_pitch + 2 * cpair;
      const int vr = min(BAND, max(0, valid_h - band0));
      if (valid_w == TW && valid_h == TH) {
        detect_strip<T, K, true>(s_in, band0, c0, outp, p.out_pitch, BAND, true, true, flags, p.one);
      } else {
        detect_strip<T, K, false>(s_in, band0, c0, outp, p.out_pitch, vr, ok0, ok1, flags, p.one);
        // mask out pixels beyond the frame / strip
        const uint32_t colm = (ok0 ? 0xFFFFu : 0u) | (ok1 ? 0xFFFF0000u : 0u);
#pragma unroll
        for (int h = 0; h < NFW; ++h) {
          const int v = min(16, max(0, vr - 16 * h));
          const uint32_t rowm = v >= 16 ? 0xFFFFu : ((1u << v) - 1u);
          flags[h] &= colm & (rowm | (rowm << 16));
        }
      }
      // compact the strip's noisy pixels into the warp queue
      int cnt = 0;
#pragma unroll
      for (int h = 0; h < NFW; ++h) cnt += __popc(flags[h]);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const int n = __shfl_sync(0xffffffffu, incl, 31);
      detected += (uint32_t)cnt;
      uint16_t* qp = s_q + (incl - cnt);
      const uint32_t ebase = ((uint32_t)band0 << 8) | (uint32_t)(2 * cpair);
#pragma unroll
      for (int h = 0; h < NFW; ++h) {
        uint32_t f = flags[h];
        while (f) {
          const int bit = __ffs(f) - 1;
          f &= f - 1u;
          // bit = lane*16 + row: entry = ((band0 + 16h + row) << 8) | (2*cpair + lane)
          *qp++ = (uint16_t)(ebase + ((uint32_t)(16 * h + (bit & 15)) << 8) + (uint32_t)(bit >> 4));
        }
      }
      __syncwarp();  // queue visible; centre stores ordered before the median stores
      if (p.debug != 1) replaced += median_queue<T, K>(s_in, s_q, p.debug == 2 ? -n : n, out_tile, p.out_pitch, lane, true,
                                                          0u - p.one);
      __syncwarp();
    } else {
      // MF: every valid pixel of the strip through the same queue
      const int cols = max(0, min(64, valid_w - (warp & 1) * 64));
      const int rows = min(BAND, max(0, valid_h - band0));
      const int n = rows * cols;
      for (int j = lane; j < n; j += 32) {
        const int y = j / cols, x = j - y * cols;
        s_q[j] = (uint16_t)(((band0 + y) << 8) | ((warp & 1) * 64 + x));
      }
      __syncwarp();
      median_queue<T, K>(s_in, s_q, n, out_tile, p.out_pitch, lane, false, 0u - p.one);
      __syncwarp();
    }
    // all warps are done with this stage: refill it with the next tile
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) refill(stage);
  }
  // the last CTA out resets the scheduler for the next launch on this slot
  if (tid == 0 && atomicAdd(p.sched + 1, 1u) == gridDim.x - 1) {
    p.sched[0] = 0u;
    p.sched[1] = 0u;
  }
  if (p.method == 0) block_add_counts<THREADS>(detected, replaced, p.counts);
}

}  // namespace tile
}  // namespace irdn
