// Dense 3x3 FNR / MF kernel for u8 frames (BASELINE configs c1, c5), sm_100a.
//
// For k = 3 the median network is cheap enough to evaluate for EVERY pixel, so
// this kernel has no queue: detector, median and select all run branch-free on
// packed words and the result goes straight to HBM.
//
// Packing: "vertical pair keys". A 32-bit word holds one column's pixels of two
// consecutive rows, each as the 16-bit key v*257 (= byte v in both halves, built
// by one PRMT from two row words). Keys are monotone in v and equality preserving,
// so min/max/median on keys are min/max/median on pixels, and with two rows per
// word the vertical neighbour comes from one PRMT and horizontal neighbours are
// just other registers.
//
// Per two output rows y, y+1 and column x (reference filters.py:156-180):
//   column sort   lo/hi = min3/max3(A, S, B), mid = A+S+B-lo-hi   (A = rows y-1,y;
//                 S = rows y,y+1; B = rows y+1,y+2: lanewise the 3-row window)
//   median of 9   med3(max3(lo), med3(mid), min3(hi))  over columns x-1, x, x+1
//                 (exact for 3x3: the classic sorted-columns identity)
//   detector      c == min9 || c == max9, min9 = min3(lo), max9 = max3(hi)
//   select        out = noisy ? median : c    (FNR)   /   out = median   (MF)
// Sums a+b+c-min-max are exact in 32-bit arithmetic, so the IADDs run on the
// FMA pipe while VIMNMX3 and PRMT use the ALU pipe.
#pragma once
#include "fnr_tile.cuh"

namespace irdn {
namespace k3 {

constexpr int THREADS = 128;
constexpr int TW = 128;                 // tile width (pixels)
constexpr int COLS = 8;                 // columns per thread (one 8-byte row segment)
constexpr int TPR = TW / COLS;          // threads per row band (16)
constexpr int BANDS = THREADS / TPR;    // row bands per tile (8)
constexpr int NSTAGE = 2;
// Tile height: 128 rows (16 per thread) for large frames, 32 rows (4 per thread) when a
// frame has too few 128-row tiles to fill the GPU, 16 rows (2 per thread) when even
// 32-row tiles leave SMs idle (BASELINE c1: 512x512 -> 128 tiles).

template <int TH>
struct Geo {
  static constexpr int r = 1;
  static constexpr int A = 16;  // TMA box x start must be 16-byte aligned
  static constexpr int R = A;
  static constexpr int BOXW = ((TW + R + r + A - 1) / A) * A;  // 160
  static constexpr int BOXH = TH + 2 * r;                      // 130
  static constexpr int IN_BYTES = BOXW * BOXH;
  static constexpr int IN_STRIDE = (IN_BYTES + 127) & ~127;
  static constexpr int BAR_OFF = NSTAGE * IN_STRIDE;
  static constexpr int TILE_OFF = BAR_OFF + 8 * NSTAGE;
  static constexpr int SMEM = TILE_OFF + 16 * NSTAGE + 128;
};

// Median of three packed keys: a + b + c - min - max (exact in 32-bit: the true median
// fits each lane). The 3-input sum stays one IADD3; the subtraction goes to the FMA pipe.
__device__ __forceinline__ uint32_t med3(uint32_t a, uint32_t b, uint32_t c, uint32_t m1) {
  return fma_sub(fma_sub(a + b + c, m1, vmin3(a, b, c)), m1, vmax3(a, b, c));
}

// Replicate-edge fix-up (see tile::fix_edges) for this kernel's box.
template <int TH>
__device__ __forceinline__ void fix_edges(uint8_t* s_in, int gx_lo, int gy_lo, int width, int height) {
  constexpr int BOXW = Geo<TH>::BOXW, BOXH = Geo<TH>::BOXH, A = Geo<TH>::A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c_lo = max(0, -gx_lo), c_hi = min(BOXW, width - gx_lo);
  const int y_lo = max(0, -gy_lo), y_hi = min(BOXH, height - gy_lo);
  const int ncl = c_lo, ncr = BOXW - c_hi;
  if (ncl | ncr) {
    if ((ncl == 0 || ncl == A) && (ncr == 0 || ncr == A)) {
      for (int i = tid; i < 2 * (y_hi - y_lo); i += THREADS) {
        const int row = y_lo + (i >> 1);
        const bool left = (i & 1) == 0;
        if (left ? ncl == 0 : ncr == 0) continue;
        uint8_t* rp = s_in + row * BOXW;
        const uint32_t v = (uint32_t)rp[left ? c_lo : c_hi - 1] * 0x01010101u;
        *reinterpret_cast<uint4*>(rp + (left ? 0 : BOXW - A)) = make_uint4(v, v, v, v);
      }
    } else {
      const int nc = ncl + ncr;
      for (int row = y_lo + warp; row < y_hi; row += THREADS / 32) {
        uint8_t* rp = s_in + row * BOXW;
        for (int j = lane; j < nc; j += 32) {
          const int col = j < ncl ? j : c_hi + (j - ncl);
          rp[col] = rp[j < ncl ? c_lo : c_hi - 1];
        }
      }
    }
    __syncthreads();
  }
  const int nrt = y_lo, nrb = BOXH - y_hi;
  constexpr int V = BOXW / A;
  for (int i = tid; i < (nrt + nrb) * V; i += THREADS) {
    const int j = i / V, col = (i - j * V) * A;
    const int row = j < nrt ? j : y_hi + (j - nrt);
    *reinterpret_cast<uint4*>(s_in + row * BOXW + col) =
        *reinterpret_cast<const uint4*>(s_in + (j < nrt ? y_lo : y_hi - 1) * BOXW + col);
  }
}

// Keys of the 10 columns x-1 .. x+8 for smem rows `ra` and `ra + 1` (lane 0 = row ra).
template <int BOXW>
__device__ __forceinline__ void load_keys(const uint8_t* s_row, uint32_t (&key)[COLS + 2]) {
  const uint8_t* p1 = s_row;
  const uint8_t* p2 = s_row + BOXW;
  const uint32_t l1 = *reinterpret_cast<const uint32_t*>(p1 - 4), l2 = *reinterpret_cast<const uint32_t*>(p2 - 4);
  const uint2 m1 = *reinterpret_cast<const uint2*>(p1), m2 = *reinterpret_cast<const uint2*>(p2);
  const uint32_t r1 = *reinterpret_cast<const uint32_t*>(p1 + 8), r2 = *reinterpret_cast<const uint32_t*>(p2 + 8);
  key[0] = tile::prmt(l1, l2, 0x7733u);  // column x-1 = byte 3 of the left word
  key[1] = tile::prmt(m1.x, m2.x, 0x4400u);
  key[2] = tile::prmt(m1.x, m2.x, 0x5511u);
  key[3] = tile::prmt(m1.x, m2.x, 0x6622u);
  key[4] = tile::prmt(m1.x, m2.x, 0x7733u);
  key[5] = tile::prmt(m1.y, m2.y, 0x4400u);
  key[6] = tile::prmt(m1.y, m2.y, 0x5511u);
  key[7] = tile::prmt(m1.y, m2.y, 0x6622u);
  key[8] = tile::prmt(m1.y, m2.y, 0x7733u);
  key[9] = tile::prmt(r1, r2, 0x4400u);  // column x+8 = byte 0 of the right word
}

template <int TH, bool FULL_W>
__global__ void __launch_bounds__(THREADS) fnr_k3_kernel(const __grid_constant__ CUtensorMap in_map,
                                                         const tile::TileParams p) {
  using G = Geo<TH>;
  constexpr int BAND = TH / BANDS;  // rows per thread
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tile::smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + G::BAR_OFF);
  tile::TileInfo* s_tile = reinterpret_cast<tile::TileInfo*>(smem + G::TILE_OFF);

  pdl_wait_and_trigger();
  const int tid = threadIdx.x;
  const int tiles_per_frame = p.tiles_x * p.tiles_y;
  const int ntiles = tiles_per_frame * p.batch;
  const bool fnr = p.method == 0;
  const uint32_t one = p.one, m1 = 0u - p.one, k65536 = p.one << 16;  // opaque constants for the FMA pipe
  uint32_t det_total = 0, rep_total = 0;

  auto refill = [&](int stage) {
    tile::TileInfo ti;
    ti.t = (int)atomicAdd(p.sched, 1u);
    if (ti.t < ntiles) {
      ti.b = ti.t / tiles_per_frame;
      const int tt = ti.t - ti.b * tiles_per_frame;
      const int ty = tt / p.tiles_x;
      ti.tx0 = (tt - ty * p.tiles_x) * TW;
      ti.ty0 = p.row_begin + ty * TH;
      s_tile[stage] = ti;
      tile::mbar_expect_tx(&s_bar[stage], G::IN_BYTES);
      tile::tma_load_3d(smem + stage * G::IN_STRIDE, &in_map, &s_bar[stage], ti.tx0 - G::R, ti.ty0 - 1 - p.in_row0,
                        ti.b);
    } else {
      s_tile[stage] = ti;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tile::smem_u32(&s_bar[stage])) : "memory");
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) tile::mbar_init(&s_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) refill(s);
  }
  __syncthreads();

  const int tc = tid % TPR, band = tid / TPR;
  const int x0 = tc * COLS;       // first tile column of this thread
  const int y0 = band * BAND;     // first tile row of this thread
  uint8_t* const out_base = reinterpret_cast<uint8_t*>(p.out);

  for (int iter = 0;; ++iter) {
    const int stage = iter % NSTAGE;
    const uint8_t* s_in = smem + stage * G::IN_STRIDE;
    tile::mbar_wait(&s_bar[stage], (iter / NSTAGE) & 1);
    const tile::TileInfo ti = s_tile[stage];
    if (ti.t >= ntiles) break;
    const int gx_lo = ti.tx0 - G::R, gy_lo = ti.ty0 - 1;
    if (gx_lo < 0 || gy_lo < 0 || gx_lo + G::BOXW > p.width || gy_lo + G::BOXH > p.height) {
      fix_edges<TH>(smem + stage * G::IN_STRIDE, gx_lo, gy_lo, p.width, p.height);
      __syncthreads();
    }
    const int valid_w = min(TW, p.width - ti.tx0);
    const int valid_h = min(TH, p.row_end - ti.ty0);
    uint8_t* outp = out_base + (int64_t)ti.b * p.out_frame + (int64_t)(ti.ty0 - p.row_begin + y0) * p.out_pitch +
                    ti.tx0 + x0;
    // column validity (only when the frame width is not a multiple of the tile)
    uint32_t colkeep[COLS];
#pragma unroll
    for (int i = 0; i < COLS; ++i) colkeep[i] = (FULL_W || x0 + i < valid_w) ? 0u : 0xFFFFFFFFu;

    // smem row of output row y is y + 1; the first pair A covers smem rows y0, y0+1
    const uint8_t* srow = s_in + y0 * G::BOXW + x0 + G::R;
    uint32_t A[COLS + 2];
    load_keys<G::BOXW>(srow, A);
    uint32_t keep_acc = 0, rep_acc = 0;
#pragma unroll (BAND >= 8 ? 2 : 1)
    for (int s = 0; s < BAND / 2; ++s) {
      uint32_t B[COLS + 2];
      load_keys<G::BOXW>(srow + (2 * s + 2) * G::BOXW, B);
      uint32_t lo[COLS + 2], hi[COLS + 2], mid[COLS + 2], S[COLS + 2];
#pragma unroll
      for (int c = 0; c < COLS + 2; ++c) {
        S[c] = shift_pair(A[c], B[c], k65536);  // rows y, y+1
        lo[c] = vmin3(A[c], S[c], B[c]);
        hi[c] = vmax3(A[c], S[c], B[c]);
        mid[c] = fma_sub(fma_sub(A[c] + S[c] + B[c], m1, lo[c]), m1, hi[c]);
        A[c] = B[c];
      }
      const int yr = y0 + 2 * s;  // tile row of lane 0
      const uint32_t rowkeep = (yr < valid_h ? 0u : 0x0000FFFFu) | (yr + 1 < valid_h ? 0u : 0xFFFF0000u);
      uint32_t out[COLS];
#pragma unroll
      for (int i = 0; i < COLS; ++i) {
        const uint32_t med = med3(vmax3(lo[i], lo[i + 1], lo[i + 2]), med3(mid[i], mid[i + 1], mid[i + 2], m1),
                                  vmin3(hi[i], hi[i + 1], hi[i + 2]), m1);
        if (fnr) {
          const uint32_t c = S[i + 1];
          const uint32_t mn = vmin3(lo[i], lo[i + 1], lo[i + 2]), mx = vmax3(hi[i], hi[i + 1], hi[i + 2]);
          // lane of m == 0 <=> centre is the window min or max; m <= 0x7FFF so +0x7FFF sets bit 15 iff m != 0
          const uint32_t e = fma_add(vmin2(fma_sub(c, m1, mn), fma_sub(mx, m1, c)), one, 0x7FFF7FFFu);
          uint32_t keep = tile::prmt(e, e, 0xBB99u);  // 0xFFFF lanes: signal pixel, keep the centre
          keep |= rowkeep | colkeep[i];
          out[i] = (c & keep) | (med & ~keep);
          keep_acc = fma_add(keep, one, keep_acc);                          // decoded per tile (see below)
          rep_acc = fma_add(vmin2((med ^ c) & ~keep, 0x00010001u), one, rep_acc);  // noisy and changed
        } else {
          out[i] = med;
        }
      }
      // keys -> bytes: both halves of a key hold the pixel value
      const uint32_t q01 = tile::prmt(out[0], out[1], 0x6240u), q23 = tile::prmt(out[2], out[3], 0x6240u);
      const uint32_t q45 = tile::prmt(out[4], out[5], 0x6240u), q67 = tile::prmt(out[6], out[7], 0x6240u);
      const uint2 row_a = make_uint2(tile::prmt(q01, q23, 0x5410u), tile::prmt(q45, q67, 0x5410u));
      const uint2 row_b = make_uint2(tile::prmt(q01, q23, 0x7632u), tile::prmt(q45, q67, 0x7632u));
      if (FULL_W) {
        if (yr < valid_h) *reinterpret_cast<uint2*>(outp) = row_a;
        if (yr + 1 < valid_h) *reinterpret_cast<uint2*>(outp + p.out_pitch) = row_b;
      } else {
        const uint8_t* ba = reinterpret_cast<const uint8_t*>(&row_a);
        const uint8_t* bb = reinterpret_cast<const uint8_t*>(&row_b);
#pragma unroll
        for (int i = 0; i < COLS; ++i) {
          if (x0 + i < valid_w) {
            if (yr < valid_h) outp[i] = ba[i];
            if (yr + 1 < valid_h) outp[p.out_pitch + i] = bb[i];
          }
        }
      }
      outp += 2 * p.out_pitch;
    }
    if (fnr) {
      // keep_acc = sum of lane masks 0xFFFF: as integers it is 65535*K0 - 65536*K1 (mod 2^32)
      // for K0 / K1 kept lane-0 / lane-1 pixels, K0, K1 <= BAND/2*COLS
      const uint32_t k0 = (0u - keep_acc) & 0xFFFFu;
      const int diff = (int)(int16_t)(uint16_t)((keep_acc + k0) >> 16);  // K0 - K1
      const uint32_t kept = 2u * k0 - (uint32_t)diff;
      det_total += (uint32_t)(BAND * COLS) - kept;
      rep_total += (rep_acc & 0xFFFFu) + (rep_acc >> 16);
    }
    tile::fence_proxy_async();
    __syncthreads();
    if (tid == 0) refill(stage);
  }
  if (tid == 0 && atomicAdd(p.sched + 1, 1u) == gridDim.x - 1) {
    p.sched[0] = 0u;
    p.sched[1] = 0u;
  }
  if (fnr) block_add_counts<THREADS>(det_total, rep_total, p.counts);
}

}  // namespace k3
}  // namespace irdn
