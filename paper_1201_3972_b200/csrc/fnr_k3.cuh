// Dense 3x3 FNR / MF kernel for u8 frames (BASELINE configs c1, c5), sm_100a.
//
// For k = 3 the median is cheap enough to evaluate for EVERY pixel, so this kernel has
// no queue: detector, median, select and counters run branch-free on packed words and
// the result goes straight to HBM (reference filters.py:156-180).
//
// Keys. One 32-bit word holds one column's pixels of two consecutive rows, each as the
// 16-bit key 0x6400 | v: as an unsigned integer it is monotone in v (so VIMNMX.U16x2
// min / max / median on keys are min / max / median on pixels), and as an fp16 number it
// is exactly 1024 + v (so differences of keys are exact small integers in f16x2
// arithmetic). A word's lane 0 is the upper row. Keys are built from two row words with
// two PRMTs per pair of columns plus one per column (interleave the rows, then insert
// the 0x64 exponent byte).
//
// Per step (two output rows y, y+1; A = keys of rows y-1,y; B = rows y+1,y+2;
// S = rows y,y+1 = one PRMT of A and B), for each of COLS + 2 columns:
//   column sort    lo = min3(A,S,B), hi = max3(A,S,B), mid = A+S+B-lo-hi   (lanewise the
//                  sorted 3-row column of both output rows; the integer sum is exact in 32
//                  bits because every lane of the result is in range)
// and for each output column (columns j-1, j, j+1):
//   median of 9    med3(max3(lo), med3(mid), min3(hi))  (the sorted-columns identity);
//                  med3(mid) shares the sorted middle pair between horizontal neighbours:
//                  p,q = sort(mid[j], mid[j+1]) serves outputs j-1 and j as clamp(., p, q)
//   detector       min9 = min3(lo), max9 = max3(hi); noisy iff c == min9 or c == max9
//   select (FNR)   in f16x2 on the FMA pipe: s = sat(1 + (min9 - c)(max9 - c)) is 1.0 for a
//                  noisy lane and 0 otherwise; out = c + (med - c) s
//   counters       detected += s, replaced += sat(|med - c| s), f16x2 accumulators
//                  flushed to integers once per tile
// The min/max network and the key shuffles issue on the ALU pipe, the f16x2 select and
// counters and the sums on the FMA pipe (measured half-rate each, dual-issuing:
// profiles/pipe_probe_r02.txt).
// MF (every pixel replaced, no detector, select or counters) takes the row-first body
// below: its work is almost all on the ALU pipe, where that layout needs fewer shuffles.
#pragma once
#include <cuda_fp16.h>
#include <type_traits>
#include "fnr_tile.cuh"

namespace irdn {
namespace k3 {

constexpr int THREADS = 128;
constexpr int COLS = 16;                // output columns per thread (one 16-byte row segment)
constexpr int TPR = 8;                  // threads per row band
constexpr int TW = COLS * TPR;          // tile width: 128 pixels
constexpr int BANDS = THREADS / TPR;    // 16 row bands per tile
#ifndef IRDN_K3_NSTAGE
#define IRDN_K3_NSTAGE 1  // measured: 1 stage x 8 CTAs/SM beats 2 stages x 4 (c5 0.789 vs 0.797 ms)
#endif
constexpr int NSTAGE = IRDN_K3_NSTAGE;

// Pipe placement of the integer helper arithmetic (A/B switches; the defaults are the
// measured best): the row-pair shift S and the column middle on the FMA pipe (IMADs), the
// final median-of-3 sum on the ALU pipe (IADD3).
#ifndef IRDN_K3_S_FMA
#define IRDN_K3_S_FMA 0
#endif
#ifndef IRDN_K3_MID_FMA
#define IRDN_K3_MID_FMA 1
#endif
#ifndef IRDN_K3_UNROLL
#define IRDN_K3_UNROLL 1
#endif
#ifndef IRDN_K3_FIN_FMA
#define IRDN_K3_FIN_FMA 0
#endif
constexpr int kStepUnroll = IRDN_K3_UNROLL;

// Tile height TH = BANDS * BAND (BAND = rows per thread, even): 160 (BAND 10), 128, 64 or 32.
template <int BAND>
struct Geo {
  static_assert(BAND % 2 == 0, "two output rows per step");
  static constexpr int TH = BANDS * BAND;
  static constexpr int R = 16;          // left halo: TMA box x start must be 16-byte aligned
  static constexpr int BOXW = TW + 2 * R;  // 160: tile columns -16 .. 143
  static constexpr int BOXH = TH + 2;
  static constexpr int IN_BYTES = BOXW * BOXH;
  static constexpr int IN_STRIDE = (IN_BYTES + 127) & ~127;
  static constexpr int BAR_OFF = NSTAGE * IN_STRIDE;
  static constexpr int TILE_OFF = BAR_OFF + 8 * NSTAGE;
  static constexpr int SMEM = TILE_OFF + 16 * NSTAGE + 128;
  static_assert(BOXH <= 256, "TMA box limit");
};

// ---- f16x2 helpers (FMA pipe) ----------------------------------------------------
__device__ __forceinline__ uint32_t hsub(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t hadd(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t hfma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t hfma_sat(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.sat.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// sat(|a| * b)
__device__ __forceinline__ uint32_t hmul_sat_abs(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{.reg .b32 t; abs.f16x2 t, %1; mul.rn.sat.f16x2 %0, t, %2;}" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// Both f16 lanes of an accumulator as one integer (each lane holds an exact count <= 2048).
__device__ __forceinline__ uint32_t hsum_lanes(uint32_t h) {
  const __half2 v = *reinterpret_cast<const __half2*>(&h);
  return (uint32_t)(__half2float(__low2half(v)) + __half2float(__high2half(v)));
}

constexpr uint32_t KEY_BYTE = 0x64646464u;  // f16 exponent byte of 1024 + v
constexpr uint32_t F16_ONE = 0x3C003C00u;

// A row segment of one thread: 16 pixels at tile columns x0 .. x0+15 plus the words
// holding columns x0-1 (byte 3 of `l`) and x0+16 (byte 0 of `r`).
struct RowSeg {
  uint4 m;
  uint32_t l, r;
};
__device__ __forceinline__ void load_seg(const uint8_t* p, RowSeg& s) {
  s.m = *reinterpret_cast<const uint4*>(p);
  s.l = *reinterpret_cast<const uint32_t*>(p - 4);
  s.r = *reinterpret_cast<const uint32_t*>(p + 16);
}
// Keys of columns x0-1 .. x0+16 (k[0] .. k[COLS+1]) for rows (t, b): lane 0 = row t.
__device__ __forceinline__ void make_keys(const RowSeg& t, const RowSeg& b, uint32_t (&k)[COLS + 2]) {
  k[0] = tile::prmt(tile::prmt(t.l, b.l, 0x7733u), KEY_BYTE, 0x4240u);  // (t3, t3, b3, b3) -> (t3, 64, b3, 64)
  const uint32_t tw[4] = {t.m.x, t.m.y, t.m.z, t.m.w}, bw[4] = {b.m.x, b.m.y, b.m.z, b.m.w};
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t i0 = tile::prmt(tw[w], bw[w], 0x5140u);  // (t0, b0, t1, b1)
    const uint32_t i1 = tile::prmt(tw[w], bw[w], 0x7362u);  // (t2, b2, t3, b3)
    k[1 + 4 * w] = tile::prmt(i0, KEY_BYTE, 0x4140u);
    k[2 + 4 * w] = tile::prmt(i0, KEY_BYTE, 0x4342u);
    k[3 + 4 * w] = tile::prmt(i1, KEY_BYTE, 0x4140u);
    k[4 + 4 * w] = tile::prmt(i1, KEY_BYTE, 0x4342u);
  }
  k[COLS + 1] = tile::prmt(tile::prmt(t.r, b.r, 0x4400u), KEY_BYTE, 0x4240u);
}

// ---- Row-first layout (MF) ---------------------------------------------------------
// A word holds two pixels of ONE row two columns apart (the even or the odd bytes of an
// input word, zero-extended in place), so the three rows of a window are three registers
// and only the raw input needs shifted copies. A thread owns 8 columns x RB rows:
//   widen      per row and input word w = (c0 c1 c2 c3): E = (c0, c2), O = (c1, c3),
//              L = (c-1, c1) from the previous O, R = (c2, c4) from the next E: 4 PRMT / 4 px
//   row sort   outputs (c0, c2): sort3(L, E, O); outputs (c1, c3): sort3(E, O, R):
//              lo = min3, hi = max3, mid = sum - lo - hi (IMADs), once per input row
//   vertical   for output rows y, y+1 from sorted rows y-1 .. y+2 (registers):
//              max3(lo), min3(hi), med3(mid) with the sorted middle pair (rows y, y+1) shared
//              between the two output rows, then the final median of the three.
// Against the column-first body: 1.0 instead of 1.9 PRMT per pixel and no column halo
// (18 / 16) for a row halo of (RB + 2) / RB: 6.0 instead of 8.1 ALU-pipe instructions per
// pixel. MF c5 0.622 -> 0.541 ms (0.72 of the HBM roofline). For FNR the same layout needs
// 72 registers (the centre words ride along) and measured within 1 % of the column-first
// body, so FNR keeps that one.
namespace rows {
constexpr int RCOLS = 8;                 // output columns per thread
constexpr int RTPR = TW / RCOLS;         // 16 threads per row band
constexpr int RBANDS = THREADS / RTPR;   // 8 row bands per tile
struct Sorted {
  uint32_t lo[4], mid[4], hi[4];         // words: columns (0,2), (1,3), (4,6), (5,7)
};
// Sorted horizontal triples of one input row; p = the thread's first column in that row.
__device__ __forceinline__ void sort_row(const uint8_t* p, Sorted& s, uint32_t one, uint32_t m1) {
  const uint2 m = *reinterpret_cast<const uint2*>(p);
  const uint32_t l = *reinterpret_cast<const uint32_t*>(p - 4);
  const uint32_t r = *reinterpret_cast<const uint32_t*>(p + 8);
  const uint32_t E0 = tile::prmt(m.x, 0u, 0x4240u), O0 = tile::prmt(m.x, 0u, 0x4341u);
  const uint32_t E1 = tile::prmt(m.y, 0u, 0x4240u), O1 = tile::prmt(m.y, 0u, 0x4341u);
  const uint32_t L0 = tile::prmt(l, O0, 0x5453u);   // (c-1, c1)
  const uint32_t L1 = tile::prmt(O0, O1, 0x5432u);  // (c3, c5)
  const uint32_t R0 = tile::prmt(E0, E1, 0x5432u);  // (c2, c4)
  const uint32_t R1 = tile::prmt(E1, r, 0x3432u);   // (c6, c8)
  const uint32_t a[4] = {L0, E0, L1, E1}, b[4] = {E0, O0, E1, O1}, c[4] = {O0, R0, O1, R1};
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    s.lo[w] = vmin3(a[w], b[w], c[w]);
    s.hi[w] = vmax3(a[w], b[w], c[w]);
    s.mid[w] = fma_sub(fma_sub(fma_add(c[w], one, fma_add(a[w], one, b[w])), m1, s.lo[w]), m1, s.hi[w]);
  }
}
}  // namespace rows

// Replicate-edge fix-up of the box cells outside the frame (TMA zero-fills them).
template <int BAND>
__device__ __forceinline__ void fix_edges(uint8_t* s_in, int gx_lo, int gy_lo, int width, int height) {
  constexpr int BOXW = Geo<BAND>::BOXW, BOXH = Geo<BAND>::BOXH, A = Geo<BAND>::R;
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

// FULL: every tile of the launch is whole (width % TW == 0, rows % TH == 0): one unmasked
// tile body. Otherwise the whole tiles still take the unmasked body and only the last
// column / row of tiles the masked one (a CTA-uniform branch). FNR: method "fnr" (else "mf").
#ifndef IRDN_K3_MINBLOCKS
#define IRDN_K3_MINBLOCKS 8  // whole-tile launches: <= 64 registers, 8 CTAs per SM (c5 0.783 -> 0.771 ms; 7 fit at the natural 65)
#endif
template <int BAND, bool FULL, bool FNR>
__global__ void __launch_bounds__(THREADS, FULL ? IRDN_K3_MINBLOCKS : 5) fnr_k3_kernel(const __grid_constant__ CUtensorMap in_map,
                                                         const tile::TileParams p) {
  using G = Geo<BAND>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (tile::smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + G::BAR_OFF);
  tile::TileInfo* s_tile = reinterpret_cast<tile::TileInfo*>(smem + G::TILE_OFF);

  pdl_wait_and_trigger();
  const int tid = threadIdx.x;
  const int tiles_per_frame = p.tiles_x * p.tiles_y;
  const int ntiles = tiles_per_frame * p.batch;
  uint32_t det_total = 0, rep_total = 0;
  const uint32_t one = p.one, m1 = 0u - p.one, k65536 = p.one << 16;  // opaque: keeps IMADs on the FMA pipe

  // (claiming the next tile's index when a tile starts, to overlap the atomic's round trip,
  // measured 0.5 % slower on c5: 0.7839 vs 0.7831 ms)
  auto refill = [&](int stage) {
    tile::TileInfo ti;
    ti.t = (int)atomicAdd(p.sched, 1u);
    if (ti.t < ntiles) {
      ti.b = tile::udiv(ti.t, tiles_per_frame, p.tpf_magic);
      const int tt = ti.t - ti.b * tiles_per_frame;
      const int ty = tile::udiv(tt, p.tiles_x, p.tx_magic);
      ti.tx0 = (tt - ty * p.tiles_x) * TW;
      ti.ty0 = p.row_begin + ty * G::TH;
      s_tile[stage] = ti;
      tile::mbar_expect_tx(&s_bar[stage], G::IN_BYTES);
      tile::tma_load_3d(smem + stage * G::IN_STRIDE, &in_map, &s_bar[stage], ti.tx0 - G::R,
                        ti.ty0 - 1 - p.in_row0, ti.b);
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

  // FNR: column-first body, 16 columns x BAND rows per thread; MF: row-first, 8 columns x 2 BAND rows
  constexpr int RB = FNR ? BAND : G::TH / rows::RBANDS;
  const int tc = FNR ? tid % TPR : tid % rows::RTPR, band = FNR ? tid / TPR : tid / rows::RTPR;
  const int x0 = tc * (FNR ? COLS : rows::RCOLS);  // first tile column of this thread
  const int y0 = band * RB;                        // first tile row of this thread
  uint8_t* const out_base = reinterpret_cast<uint8_t*>(p.out);

  for (int iter = 0;; ++iter) {
    const int stage = iter % NSTAGE;
    const uint8_t* s_in = smem + stage * G::IN_STRIDE;
    tile::mbar_wait(&s_bar[stage], (iter / NSTAGE) & 1);
    const tile::TileInfo ti = s_tile[stage];
    if (ti.t >= ntiles) break;
    const int gx_lo = ti.tx0 - G::R, gy_lo = ti.ty0 - 1;
    if (gx_lo < 0 || gy_lo < 0 || gx_lo + G::BOXW > p.width || gy_lo + G::BOXH > p.height) {
      fix_edges<BAND>(smem + stage * G::IN_STRIDE, gx_lo, gy_lo, p.width, p.height);
      __syncthreads();
    }
    uint32_t dacc = 0, racc = 0;  // f16x2 counters of this tile
    // MF: row-first body (header of namespace rows)
    auto body_mf = [&](auto masked) {
      constexpr bool MASKED = decltype(masked)::value;
      int valid_w = TW, valid_h = G::TH;
      if constexpr (MASKED) {
        valid_w = min(TW, p.width - ti.tx0);
        valid_h = min(G::TH, p.row_end - ti.ty0);
      }
      uint8_t* outp = out_base + (int64_t)ti.b * p.out_frame + (int64_t)(ti.ty0 - p.row_begin + y0) * p.out_pitch +
                      ti.tx0 + x0;
      // smem row of tile row y is y + 1; the thread's segment starts at box column R + x0
      const uint8_t* srow = s_in + y0 * G::BOXW + G::R + x0;
      rows::Sorted ring[4];
      rows::sort_row(srow, ring[0], one, m1);
      rows::sort_row(srow + G::BOXW, ring[1], one, m1);
      // one output row from the sorted rows u (above), v, w (below); pm / qm = the sorted pair
      // of the two middle rows this step's output rows share, t = the third row's middles
      auto out_row = [&](const rows::Sorted& u, const rows::Sorted& v, const rows::Sorted& w, const uint32_t (&pm)[4],
                         const uint32_t (&qm)[4], const uint32_t (&t)[4], int yr) {
        uint32_t out[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t md = vmax2(pm[i], vmin2(qm[i], t[i]));
          const uint32_t mxlo = vmax3(u.lo[i], v.lo[i], w.lo[i]);
          const uint32_t mnhi = vmin3(u.hi[i], v.hi[i], w.hi[i]);
          const uint32_t mn3 = vmin3(mxlo, md, mnhi), mx3 = vmax3(mxlo, md, mnhi);
          out[i] = fma_sub(fma_sub(fma_add(mnhi, one, fma_add(mxlo, one, md)), m1, mn3), m1, mx3);
        }
        // (c0, c2) and (c1, c3) interleave to one output word
        const uint32_t w0 = tile::prmt(out[0], out[1], 0x6240u), w1 = tile::prmt(out[2], out[3], 0x6240u);
        uint8_t* const orow = outp;
        outp += p.out_pitch;
        if constexpr (!MASKED) {
          *reinterpret_cast<uint2*>(orow) = make_uint2(w0, w1);
        } else if (yr < valid_h) {
          if (x0 + rows::RCOLS <= valid_w) {
            *reinterpret_cast<uint2*>(orow) = make_uint2(w0, w1);
          } else {
#pragma unroll
            for (int i = 0; i < rows::RCOLS; ++i)
              if (x0 + i < valid_w) orow[i] = (uint8_t)((i < 4 ? w0 : w1) >> (8 * (i & 3)));
          }
        }
      };
      // output rows 2s, 2s + 1 of the thread: r0, r1 = sorted rows above / at 2s (carried), r2, r3 new
      auto step = [&](int s, rows::Sorted& r0, rows::Sorted& r1, rows::Sorted& r2, rows::Sorted& r3) {
        rows::sort_row(srow + (2 * s + 2) * G::BOXW, r2, one, m1);
        uint32_t pm[4], qm[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          pm[i] = vmin2(r1.mid[i], r2.mid[i]);
          qm[i] = vmax2(r1.mid[i], r2.mid[i]);
        }
        out_row(r0, r1, r2, pm, qm, r0.mid, y0 + 2 * s);
        rows::sort_row(srow + (2 * s + 3) * G::BOXW, r3, one, m1);
        out_row(r1, r2, r3, pm, qm, r3.mid, y0 + 2 * s + 1);
      };
      // two steps per iteration: the ring's roles swap without register moves
#pragma unroll 1
      for (int s = 0; s < RB / 2; s += 2) {
        step(s, ring[0], ring[1], ring[2], ring[3]);
        step(s + 1, ring[2], ring[3], ring[0], ring[1]);
      }
    };
    // FNR: column-first body (header of this file)
    auto body_fnr = [&](auto masked) {
      constexpr bool MASKED = decltype(masked)::value;
      int valid_w = TW, valid_h = G::TH;
      if constexpr (MASKED) {
        valid_w = min(TW, p.width - ti.tx0);
        valid_h = min(G::TH, p.row_end - ti.ty0);
      }
      uint8_t* outp = out_base + (int64_t)ti.b * p.out_frame + (int64_t)(ti.ty0 - p.row_begin + y0) * p.out_pitch +
                      ti.tx0 + x0;
      // smem row of tile row y is y + 1; the thread's segment starts at box column R + x0
      const uint8_t* srow = s_in + y0 * G::BOXW + G::R + x0;
      uint32_t A[COLS + 2];
      {
        RowSeg r0, r1;
        load_seg(srow, r0);
        load_seg(srow + G::BOXW, r1);
        make_keys(r0, r1, A);
      }
  #pragma unroll (kStepUnroll)
      for (int s = 0; s < BAND / 2; ++s) {
        uint32_t B[COLS + 2];
        {
          RowSeg r1, r2;
          load_seg(srow + (2 * s + 2) * G::BOXW, r1);
          load_seg(srow + (2 * s + 3) * G::BOXW, r2);
          make_keys(r1, r2, B);
        }
        uint32_t lo[COLS + 2], hi[COLS + 2], mid[COLS + 2], S[COLS + 2];
  #pragma unroll
        for (int c = 0; c < COLS + 2; ++c) {
          if (IRDN_K3_S_FMA == 1 || (IRDN_K3_S_FMA == 2 && (c & 1)))
            S[c] = shift_pair(A[c], B[c], k65536);  // rows y, y+1 (IMAD.HI + IMAD)
          else
            S[c] = tile::prmt(A[c], B[c], 0x5432u);  // rows y, y+1
          lo[c] = vmin3(A[c], S[c], B[c]);
          hi[c] = vmax3(A[c], S[c], B[c]);
  #if IRDN_K3_MID_FMA
          mid[c] = fma_sub(fma_sub(fma_add(B[c], one, fma_add(A[c], one, S[c])), m1, lo[c]), m1, hi[c]);
  #else
          mid[c] = A[c] + S[c] + B[c] - lo[c] - hi[c];
  #endif
          A[c] = B[c];
        }
        uint32_t rowmask = 0xFFFFFFFFu;  // partial tiles: lanes of rows inside the tile
        if constexpr (MASKED) {
          const int yr = y0 + 2 * s;
          rowmask = (yr < valid_h ? 0x0000FFFFu : 0u) | (yr + 1 < valid_h ? 0xFFFF0000u : 0u);
        }
        uint32_t out[COLS];
  #pragma unroll
        for (int j = 0; j < COLS; j += 2) {
          const uint32_t pm = vmin2(mid[j + 1], mid[j + 2]), qm = vmax2(mid[j + 1], mid[j + 2]);
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int o = j + h;  // output column o: key columns o, o+1, o+2
            const uint32_t md = vmax2(pm, vmin2(qm, mid[h == 0 ? j : j + 3]));
            const uint32_t mxlo = vmax3(lo[o], lo[o + 1], lo[o + 2]);
            const uint32_t mnhi = vmin3(hi[o], hi[o + 1], hi[o + 2]);
            const uint32_t mn3 = vmin3(mxlo, md, mnhi), mx3 = vmax3(mxlo, md, mnhi);
            uint32_t med;
            if (IRDN_K3_FIN_FMA == 1 || (IRDN_K3_FIN_FMA == 2 && h == 1))
              med = fma_sub(fma_sub(fma_add(mnhi, one, fma_add(mxlo, one, md)), m1, mn3), m1, mx3);
            else
              med = mxlo + md + mnhi - mn3 - mx3;
            const uint32_t c = S[o + 1];
            const uint32_t mn = vmin3(lo[o], lo[o + 1], lo[o + 2]), mx = vmax3(hi[o], hi[o + 1], hi[o + 2]);
            uint32_t sflag = hfma_sat(hsub(mn, c), hsub(mx, c), F16_ONE);  // 1.0: noisy lane
            const uint32_t dm = hsub(med, c);
            out[o] = hfma(dm, sflag, c);
            if constexpr (MASKED) {
              const bool colok = x0 + o < valid_w;
              sflag &= colok ? rowmask : 0u;
            }
            racc = hadd(racc, hmul_sat_abs(dm, sflag));
            dacc = hadd(dacc, sflag);
          }
        }
        // keys -> bytes: byte 0 of a key is the upper row's pixel, byte 2 the lower row's
        uint32_t row_a[COLS / 4], row_b[COLS / 4];
  #pragma unroll
        for (int w = 0; w < COLS / 4; ++w) {
          const uint32_t q01 = tile::prmt(out[4 * w], out[4 * w + 1], 0x6240u);
          const uint32_t q23 = tile::prmt(out[4 * w + 2], out[4 * w + 3], 0x6240u);
          row_a[w] = tile::prmt(q01, q23, 0x5410u);
          row_b[w] = tile::prmt(q01, q23, 0x7632u);
        }
        if constexpr (!MASKED) {
          *reinterpret_cast<uint4*>(outp) = make_uint4(row_a[0], row_a[1], row_a[2], row_a[3]);
          *reinterpret_cast<uint4*>(outp + p.out_pitch) = make_uint4(row_b[0], row_b[1], row_b[2], row_b[3]);
        } else {
          const int yr = y0 + 2 * s;
          const uint8_t* ba = reinterpret_cast<const uint8_t*>(row_a);
          const uint8_t* bb = reinterpret_cast<const uint8_t*>(row_b);
          if (x0 + COLS <= valid_w) {
            if (yr < valid_h) *reinterpret_cast<uint4*>(outp) = make_uint4(row_a[0], row_a[1], row_a[2], row_a[3]);
            if (yr + 1 < valid_h)
              *reinterpret_cast<uint4*>(outp + p.out_pitch) = make_uint4(row_b[0], row_b[1], row_b[2], row_b[3]);
          } else {
  #pragma unroll
            for (int i = 0; i < COLS; ++i) {
              if (x0 + i < valid_w) {
                if (yr < valid_h) outp[i] = ba[i];
                if (yr + 1 < valid_h) outp[p.out_pitch + i] = bb[i];
              }
            }
          }
        }
        outp += 2 * p.out_pitch;
      }
    };
    auto run = [&](auto& body) {
      if (FULL || (ti.tx0 + TW <= p.width && ti.ty0 + G::TH <= p.row_end)) body(std::false_type{});
      else if constexpr (!FULL) body(std::true_type{});
    };
    if constexpr (FNR) run(body_fnr);
    else run(body_mf);
    if constexpr (FNR) {
      det_total += hsum_lanes(dacc);
      rep_total += hsum_lanes(racc);
    }
    tile::fence_proxy_async();
    __syncthreads();
    if (tid == 0) refill(stage);
  }
  if (tid == 0 && atomicAdd(p.sched + 1, 1u) == gridDim.x - 1) {
    p.sched[0] = 0u;
    p.sched[1] = 0u;
  }
  if constexpr (FNR) block_add_counts<THREADS>(det_total, rep_total, p.counts);
}

}  // namespace k3
}  // namespace irdn
