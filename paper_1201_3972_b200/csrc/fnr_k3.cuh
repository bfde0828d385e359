// Dense 3x3 FNR / MF kernel for u8 frames (BASELINE configs c1, c5), sm_100a.
//
// For k = 3 the median is cheap enough to evaluate for EVERY pixel, so this kernel has
// no queue: detector, median, select and counters run branch-free on packed words and
// the result goes straight to HBM (reference filters.py:156-180).
//
// Layout (row-first). One 32-bit word holds two pixels of ONE row two columns apart: the
// even or the odd bytes of an input word, widened in place, so the three rows of a window
// are three registers and only the raw input needs shifted copies. FNR widens each pixel to
// the 16-bit key 0x6400 | v: as an unsigned integer it is monotone in v (VIMNMX.U16x2 min /
// max / median on keys are those of the pixels), and as an fp16 number it is exactly
// 1024 + v (differences of keys are exact small integers in f16x2 arithmetic). MF
// zero-extends. A thread owns NW output words (FNR: 2 = one input word = 4 columns, MF: 4 =
// 8 columns) and walks RB rows down its tile:
//   widen      per row and input word (c0 c1 c2 c3): E = (c0, c2), O = (c1, c3), L = (c-1, c1)
//              from the previous O, R = (c2, c4) from the next E: 4 PRMT per 4 pixels
//   row sort   outputs (c0, c2): sort3(L, E, O); outputs (c1, c3): sort3(E, O, R): lo = min3,
//              hi = max3, mid = sum - lo - hi (IMADs: the integer sum is exact in 32 bits
//              because every lane of the result is in range), once per input row
//   vertical   output rows y, y+1 per step from the sorted rows y-1 .. y+2 (a ring of four in
//              registers; two steps per loop iteration so the roles swap without moves):
//   median of 9    med3(max3(lo), med3(mid), min3(hi))  (the sorted-rows identity); med3(mid)
//                  shares the sorted middle pair p, q = sort(mid[y], mid[y+1]) between the
//                  step's two output rows as clamp(., p, q)
//   detector       min9 = min3(lo), max9 = max3(hi); noisy iff c == min9 or c == max9
//   select (FNR)   in f16x2 on the FMA pipe: s = sat(1 + (min9 - c)(max9 - c)) is 1.0 for a
//                  noisy lane and 0 otherwise; out = c + (med - c) s
//   counters       detected += s, replaced += sat(|med - c| s), f16x2 accumulators
//                  flushed to integers once per tile
//   MF             out = med (no detector, select or counters)
// The min/max network and the byte shuffles issue on the ALU pipe, the f16x2 select and
// counters and the sums on the FMA pipe (measured half-rate each, dual-issuing:
// profiles/pipe_probe_r02.txt). Round 2 measured this layout against a column-first one
// (one word = one column's pixels of two consecutive rows, 16 columns per thread): FNR
// 0.754 vs 0.770 ms and MF 0.539 vs 0.622 ms on c5.
#pragma once
#include <cuda_fp16.h>
#include <type_traits>
#include "fnr_tile.cuh"

namespace irdn {
namespace k3 {

constexpr int THREADS = 128;
constexpr int TW = 128;                 // tile width in pixels
constexpr int BANDS = 16;               // tile height unit: TH = BANDS * BAND rows
#ifndef IRDN_K3_NSTAGE
#define IRDN_K3_NSTAGE 1  // measured: 1 stage x 8 CTAs/SM beats 2 stages x 4 (c5 0.789 vs 0.797 ms)
#endif
constexpr int NSTAGE = IRDN_K3_NSTAGE;

// Pipe placement of the integer helper arithmetic (A/B switches; the defaults are the
// measured best for FNR, profiles/r02/k3_rows/ab_5_fnr4.txt): the row-sort middle on the FMA
// pipe (IMADs), the final median-of-3 sum on the ALU pipe (IADD3). MF puts both on the FMA pipe.
#ifndef IRDN_K3_MID_FMA
#define IRDN_K3_MID_FMA 1
#endif
#ifndef IRDN_K3_FIN_FMA
#define IRDN_K3_FIN_FMA 0
#endif

// Tile height TH = BANDS * BAND (BAND even): 160 (BAND 10), 128, 96, 64 or 32.
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

// Words per thread and row: FNR 2 (4 columns: 56 registers, 8 CTAs per SM; with 4 words the
// carried centre words push it to 72 registers and 7 CTAs), MF 4 (8 columns, 60 registers).
template <bool FNR>
constexpr int kWords = FNR ? 2 : 4;

// The sorted horizontal triples of one input row for the thread's NW output words — word 2i:
// columns (4i, 4i+2), word 2i+1: columns (4i+1, 4i+3) — and the row's own pixels (centres).
template <int NW>
struct Sorted {
  uint32_t lo[NW], mid[NW], hi[NW], c[NW];
};
// p = the thread's first column in that smem row; hi_byte = the byte widened pixels carry
// above them (KEY_BYTE for FNR, 0 for MF).
template <int NW, bool FMA_SUM>
__device__ __forceinline__ void sort_row(const uint8_t* p, Sorted<NW>& s, uint32_t hi_byte, uint32_t one,
                                         uint32_t m1) {
  constexpr int NI = NW / 2;  // input words
  uint32_t in[NI];
  if constexpr (NI == 1) {
    in[0] = *reinterpret_cast<const uint32_t*>(p);
  } else {
    static_assert(NI == 2, "one or two input words per thread and row");
    const uint2 m = *reinterpret_cast<const uint2*>(p);
    in[0] = m.x;
    in[1] = m.y;
  }
  const uint32_t l = *reinterpret_cast<const uint32_t*>(p - 4);       // byte 3: column -1
  const uint32_t r = *reinterpret_cast<const uint32_t*>(p + 4 * NI);  // byte 0: column 4 NI
  uint32_t E[NI], O[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    E[i] = tile::prmt(in[i], hi_byte, 0x4240u);  // (c0, c2)
    O[i] = tile::prmt(in[i], hi_byte, 0x4341u);  // (c1, c3)
  }
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    // (c-1, c1): the high byte of the widened c-1 is O's own high byte
    const uint32_t L = i == 0 ? tile::prmt(l, O[0], 0x5453u) : tile::prmt(O[i - 1], O[i], 0x5432u);
    // (c2, c4)
    const uint32_t R = i == NI - 1 ? tile::prmt(E[i], r, 0x3432u) : tile::prmt(E[i], E[i + 1], 0x5432u);
    const uint32_t a[2] = {L, E[i]}, b[2] = {E[i], O[i]}, c[2] = {O[i], R};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int w = 2 * i + h;
      s.lo[w] = vmin3(a[h], b[h], c[h]);
      s.hi[w] = vmax3(a[h], b[h], c[h]);
      if constexpr (FMA_SUM)
        s.mid[w] = fma_sub(fma_sub(fma_add(c[h], one, fma_add(a[h], one, b[h])), m1, s.lo[w]), m1, s.hi[w]);
      else
        s.mid[w] = a[h] + b[h] + c[h] - s.lo[w] - s.hi[w];
      s.c[w] = b[h];
    }
  }
}

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
  const uint32_t one = p.one, m1 = 0u - p.one;  // opaque: keeps IMADs on the FMA pipe

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

  constexpr int NW = kWords<FNR>, NC = 2 * NW;  // words / columns per thread
  constexpr int TPR = TW / NC;                   // threads per row band
  constexpr int RB = G::TH / (THREADS / TPR);    // rows per thread (FNR: 4 BAND, MF: 2 BAND)
  static_assert(RB % 4 == 0, "two steps of two output rows per loop iteration");
  const int x0 = (tid % TPR) * NC;  // first tile column of this thread
  const int y0 = (tid / TPR) * RB;  // first tile row of this thread
  const uint32_t hi_byte = FNR ? KEY_BYTE : 0u;
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
    auto body = [&](auto masked) {
      constexpr bool MASKED = decltype(masked)::value;
      int valid_w = TW, valid_h = G::TH;
      uint32_t colmask[NW];  // partial tiles: lanes of columns inside the tile
#pragma unroll
      for (int w = 0; w < NW; ++w) colmask[w] = 0xFFFFFFFFu;
      if constexpr (MASKED) {
        valid_w = min(TW, p.width - ti.tx0);
        valid_h = min(G::TH, p.row_end - ti.ty0);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const int cw = x0 + (w & 1) + 4 * (w >> 1);  // columns cw and cw + 2
          colmask[w] = (cw < valid_w ? 0x0000FFFFu : 0u) | (cw + 2 < valid_w ? 0xFFFF0000u : 0u);
        }
      }
      uint8_t* outp = out_base + (int64_t)ti.b * p.out_frame + (int64_t)(ti.ty0 - p.row_begin + y0) * p.out_pitch +
                      ti.tx0 + x0;
      // smem row of tile row y is y + 1; the thread's segment starts at box column R + x0
      const uint8_t* srow = s_in + y0 * G::BOXW + G::R + x0;
      constexpr bool MID_FMA = !FNR || IRDN_K3_MID_FMA;
      using Row = Sorted<NW>;
      Row ring[4];
      sort_row<NW, MID_FMA>(srow, ring[0], hi_byte, one, m1);
      sort_row<NW, MID_FMA>(srow + G::BOXW, ring[1], hi_byte, one, m1);
      // one output row (tile row yr) from the sorted rows u (above), v, w (below); pm / qm = the
      // sorted pair of the two middle rows this step's output rows share, t = the third middles
      auto out_row = [&](const Row& u, const Row& v, const Row& w, const uint32_t (&pm)[NW], const uint32_t (&qm)[NW],
                         const uint32_t (&t)[NW], int yr) {
        uint32_t out[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const uint32_t md = vmax2(pm[i], vmin2(qm[i], t[i]));
          const uint32_t mxlo = vmax3(u.lo[i], v.lo[i], w.lo[i]);
          const uint32_t mnhi = vmin3(u.hi[i], v.hi[i], w.hi[i]);
          const uint32_t mn3 = vmin3(mxlo, md, mnhi), mx3 = vmax3(mxlo, md, mnhi);
          uint32_t med;
          if (!FNR || IRDN_K3_FIN_FMA == 1 || (IRDN_K3_FIN_FMA == 2 && (i & 1)))
            med = fma_sub(fma_sub(fma_add(mnhi, one, fma_add(mxlo, one, md)), m1, mn3), m1, mx3);
          else
            med = mxlo + md + mnhi - mn3 - mx3;
          if constexpr (FNR) {
            const uint32_t c = v.c[i];
            const uint32_t mn = vmin3(u.lo[i], v.lo[i], w.lo[i]), mx = vmax3(u.hi[i], v.hi[i], w.hi[i]);
            uint32_t sflag = hfma_sat(hsub(mn, c), hsub(mx, c), F16_ONE);  // 1.0: noisy lane
            const uint32_t dm = hsub(med, c);
            out[i] = hfma(dm, sflag, c);
            if constexpr (MASKED) sflag &= yr < valid_h ? colmask[i] : 0u;
            racc = hadd(racc, hmul_sat_abs(dm, sflag));
            dacc = hadd(dacc, sflag);
          } else {
            out[i] = med;
          }
        }
        // widened pixels -> bytes: (c0, c2) and (c1, c3) interleave to one output word
        uint32_t ow[NW / 2];
#pragma unroll
        for (int i = 0; i < NW / 2; ++i) ow[i] = tile::prmt(out[2 * i], out[2 * i + 1], 0x6240u);
        uint8_t* const orow = outp;
        outp += p.out_pitch;
        auto store_row = [&]() {
          if constexpr (NW == 2) *reinterpret_cast<uint32_t*>(orow) = ow[0];
          else *reinterpret_cast<uint2*>(orow) = make_uint2(ow[0], ow[NW / 2 - 1]);
        };
        if constexpr (!MASKED) {
          store_row();
        } else if (yr < valid_h) {
          if (x0 + NC <= valid_w) {
            store_row();
          } else {
#pragma unroll
            for (int i = 0; i < NC; ++i)
              if (x0 + i < valid_w) orow[i] = (uint8_t)(ow[i >> 2] >> (8 * (i & 3)));
          }
        }
      };
      // output rows 2s, 2s + 1 of the thread: r0, r1 = sorted rows above / at 2s (carried), r2, r3 new
      auto step = [&](int s, Row& r0, Row& r1, Row& r2, Row& r3) {
        sort_row<NW, MID_FMA>(srow + (2 * s + 2) * G::BOXW, r2, hi_byte, one, m1);
        uint32_t pm[NW], qm[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          pm[i] = vmin2(r1.mid[i], r2.mid[i]);
          // MF (ALU-pipe bound): the pair's max as a + b - min on the FMA pipe (c5 0.538 -> 0.531 ms)
          if constexpr (FNR) qm[i] = vmax2(r1.mid[i], r2.mid[i]);
          else qm[i] = fma_sub(fma_add(r1.mid[i], one, r2.mid[i]), m1, pm[i]);
        }
        out_row(r0, r1, r2, pm, qm, r0.mid, y0 + 2 * s);
        sort_row<NW, MID_FMA>(srow + (2 * s + 3) * G::BOXW, r3, hi_byte, one, m1);
        out_row(r1, r2, r3, pm, qm, r3.mid, y0 + 2 * s + 1);
      };
      // two steps per iteration: the ring's roles swap without register moves
#pragma unroll 1
      for (int s = 0; s < RB / 2; s += 2) {
        step(s, ring[0], ring[1], ring[2], ring[3]);
        step(s + 1, ring[2], ring[3], ring[0], ring[1]);
      }
    };
    if (FULL || (ti.tx0 + TW <= p.width && ti.ty0 + G::TH <= p.row_end)) body(std::false_type{});
    else if constexpr (!FULL) body(std::true_type{});
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
