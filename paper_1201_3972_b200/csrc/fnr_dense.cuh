// Dense median stage of the warp kernel (fnr_warp.cuh) for k = 5 and 7: the median of
// EVERY pixel of a warp tile from shared sorted rows, for MF (reference filters.py:179-180)
// and for FNR tiles where many pixels are flagged (filters.py:172-176: 49 % of c3's).
//
// The queue path pays a full k*k selection network per flagged pixel (7x7: 514 VIMNMX
// per two pixels) plus a k*k gather. Here each lane walks its column pair (one u16x2
// word per row: two horizontally adjacent pixels) down the tile and
//   1. sorts each window ROW once (the k values at columns x-r .. x+r of one row, for both
//      pixels of the pair: the detector's word loads plus PRMT/IMAD-shifted odd offsets),
//   2. merges sorted rows into blocks that vertically adjacent outputs share, pruned to the
//      ranks that can still be the median (sep_nets.cuh, generated and checked by
//      tools/netgen/sepgen.py; structure after Adams, "Fast median filters using separable
//      sorting networks", 2021):
//        k = 7, output rows a..a+3:  P = pairs of sorted rows, C4 = rows a..a+3 (ranks 3..24),
//              C6 = C4 + the pair above / below (ranks 17..24), median = rank 7 of C6 + 1 row
//        k = 5, output rows a, a+1:  C4 = rows a-1..a+2 (ranks 7..12), median = rank 5 of C4 + 1 row
//      60.75 (k = 7) / 28 (k = 5) VIMNMX instructions per pixel instead of 257 / 86 per
//      queued pixel;
//   3. stores the medians of the flagged pixels (FNR; the detector already stored the
//      others) or of all pixels (MF), and counts replacements (median != centre).
// The median is a selected input value, so the result is bit-identical to the introsort's.
#pragma once
#ifdef IRDN_SEP_NETS_H  // A/B builds with another generated header
#include IRDN_SEP_NETS_H
#else
#include "sep_nets.cuh"
#endif

// Group loops unrolled by two: half of the carried state's register moves between groups
// disappear (MF c3 0.301 -> 0.292 ms, MF c2 51.9 -> 50.2 us, FNR c3 / c2 -0.3 % / -0.7 %); by
// four the loop outgrows the instruction cache (FNR c3 0.347 ms).
#ifndef IRDN_DENSE_UNROLL7
#define IRDN_DENSE_UNROLL7 2
#endif
#ifndef IRDN_DENSE_UNROLL5
#define IRDN_DENSE_UNROLL5 2
#endif

namespace irdn {
namespace wk {

constexpr int kDenseUnroll7 = IRDN_DENSE_UNROLL7, kDenseUnroll5 = IRDN_DENSE_UNROLL5;

// Sorted window row of smem row `rowp` (pointing at the lane's first pixel): v[i] is the
// i-th smallest of the k values around each pixel of the pair (u16x2 lanes).
template <typename T, int K>
__device__ __forceinline__ void sorted_row(const T* rowp, uint32_t (&v)[K], uint32_t k65536, uint32_t m1) {
  constexpr int r = K / 2, J = (r + 1) / 2;
  uint32_t wd[2 * J + 1];
#pragma unroll
  for (int j = -J; j <= J; ++j) wd[j + J] = tile::load_pair<T>(rowp, 2 * j);
#pragma unroll
  for (int d = -r; d <= r; ++d)
    v[d + r] = (d & 1) == 0 ? wd[J + d / 2] : shift_pair(wd[J + (d - 1) / 2], wd[J + (d + 1) / 2], k65536);
  if constexpr (K == 7) sep::sort7(v, m1);
  else sep::sort5(v, m1);
}

// Store the medians `med` of output row y (tile coordinates): FNR stores only the flagged
// pixels (flag bits: row y at bit y % 16 and 16 + y % 16 of flags[y / 16], already masked
// to the valid part of the tile) and counts the ones that change; MF stores every valid one.
template <typename T>
__device__ __forceinline__ uint32_t put_row(T* rowp, const T* crow, uint32_t med, int y, int valid_rows, bool ok0,
                                            bool ok1, const uint32_t (&flags)[2], bool fnr) {
  if (!fnr) {
    if (y < valid_rows) tile::store_pair_g<T>(rowp, med, ok0, ok1);
    return 0u;
  }
  const uint32_t f = flags[y >> 4] >> (y & 15);
  const bool f0 = f & 1u, f1 = (f >> 16) & 1u;
  if (!(f0 | f1)) return 0u;
  const uint32_t c = tile::load_pair<T>(crow, 0);
  const uint32_t lo = med & 0xFFFFu, hi = med >> 16;
  uint32_t rep = 0;
  if (f0 && f1) {
    tile::store_pair_g<T>(rowp, med, true, true);
  } else if (f0) {
    rowp[0] = (T)lo;
  } else {
    rowp[1] = (T)hi;
  }
  rep += (f0 && lo != (c & 0xFFFFu)) + (f1 && hi != (c >> 16));
  return rep;
}

// Dense medians of one warp tile (rows 0 .. rows-1, rows a multiple of the group size);
// k = 5 or 7 only (other windows never call it: wk::kDense).
// s_in: the staged box (box row b = tile row b - r); c0: smem column of the lane's first
// pixel; outp: output pixel (0, 2 * lane) of the tile. Returns the replacements (FNR).
//
// FUSED (FNR on a whole tile that is predicted dense, i.e. the detector did not run): the
// detector comes from the same sorted rows — a window's min / max is the min / max of its
// rows' first / last sorted elements, shared between the rows of a group — and every pixel
// is stored once as  noisy ? median : centre  (branch-free on packed words:
// m = min(c - min, max - c) is 0 exactly in noisy lanes). *detected receives the tile's
// noisy pixels (whole tiles only: no row / column masking).
template <typename T, int K, int BOXW, bool FUSED = false>
__device__ __forceinline__ uint32_t dense_tile(const T* s_in, int c0, T* outp, int64_t pitch, int rows,
                                               int valid_rows, bool ok0, bool ok1, const uint32_t (&flags)[2],
                                               bool fnr, uint32_t one, uint32_t* detected = nullptr) {
  constexpr int r = K / 2;
  const uint32_t k65536 = one << 16, m1 = 0u - one;
  const uint32_t ones = one * 0x00010001u, kffff = one * 0xFFFFu;
  const T* base = s_in + c0 + r * BOXW;  // window row q of the tile = base + q * BOXW
  uint32_t replaced = 0;
  uint32_t sacc = 0, racc = 0;  // FUSED: per-lane counts of signal / replaced pixels (u16 lanes, <= rows)
  auto S = [&](int q, uint32_t (&v)[K]) {
    if constexpr (K == 5 || K == 7) sorted_row<T, K>(base + q * BOXW, v, k65536, m1);
  };
  auto put = [&](int y, uint32_t med) {
    replaced += put_row<T>(outp + (int64_t)y * pitch, base + y * BOXW, med, y, valid_rows, ok0, ok1, flags, fnr);
  };
  // FUSED store of output row y: window min mn, max mx
  auto put_f = [&](int y, uint32_t med, uint32_t mn, uint32_t mx) {
    const uint32_t c = tile::load_pair<T>(base + y * BOXW, 0);
    const uint32_t m = vmin2(fma_sub(c, m1, mn), fma_sub(mx, m1, c));  // lane 0 <=> noisy
    const uint32_t z = vmin2(m, ones);                                  // 1 signal, 0 noisy
    const uint32_t keep = fma_add(z, kffff, 0u);                        // 0xFFFF in signal lanes
    const uint32_t out = (c & keep) | (med & ~keep);
    tile::store_pair_g<T>(outp + (int64_t)y * pitch, out, true, true);
    sacc = fma_add(z, one, sacc);
    racc = fma_add(vmin2(out ^ c, ones), one, racc);
  };
  if constexpr (K == 7) {
    // state at group a: Pm2 = P[a-2], P0 = P[a], Sm3 = S[a-3], Sm1 = S[a-1], S1 = S[a+1], S2 = S[a+2]
    uint32_t Pm2[14], P0[14], Sm3[7], Sm1[7], S1[7], S2[7];
    {
      uint32_t t[7];
      S(-3, Sm3);
      S(-2, t);
      S(-1, Sm1);
      sep::merge7(t, Sm1, Pm2, m1);
      S(0, t);
      S(1, S1);
      sep::merge7(t, S1, P0, m1);
      S(2, S2);
    }
#pragma unroll (kDenseUnroll7)
    for (int a = 0; a < rows; a += 4) {
      uint32_t S3[7], S4[7], S5[7], S6[7], P2[14], P4[14];
      S(a + 3, S3);
      S(a + 4, S4);
      S(a + 5, S5);
      S(a + 6, S6);
      sep::merge7(S2, S3, P2, m1);
      sep::merge7(S4, S5, P4, m1);
      uint32_t c4[22], cA[8], cB[8];
      sep::core4_7(P0, P2, c4, m1);
      sep::core6_7(c4, Pm2, cA, m1);
      sep::core6_7(c4, P4, cB, m1);
      if constexpr (FUSED) {
        // window rows: a-3 | a-2, a-1 | a .. a+3 (shared) | a+4 | a+5 | a+6
        const uint32_t tn = vmin2(P0[0], P2[0]), tx = vmax2(P0[13], P2[13]);
        put_f(a, sep::final7(cA, Sm3, m1), vmin3(tn, Sm3[0], Pm2[0]), vmax3(tx, Sm3[6], Pm2[13]));
        put_f(a + 1, sep::final7(cA, S4, m1), vmin3(tn, Pm2[0], S4[0]), vmax3(tx, Pm2[13], S4[6]));
        put_f(a + 2, sep::final7(cB, Sm1, m1), vmin3(tn, Sm1[0], P4[0]), vmax3(tx, Sm1[6], P4[13]));
        put_f(a + 3, sep::final7(cB, S6, m1), vmin3(tn, P4[0], S6[0]), vmax3(tx, P4[13], S6[6]));
      } else {
        put(a, sep::final7(cA, Sm3, m1));
        put(a + 1, sep::final7(cA, S4, m1));
        put(a + 2, sep::final7(cB, Sm1, m1));
        put(a + 3, sep::final7(cB, S6, m1));
      }
#pragma unroll
      for (int i = 0; i < 14; ++i) {
        Pm2[i] = P2[i];
        P0[i] = P4[i];
      }
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        Sm3[i] = S1[i];
        Sm1[i] = S3[i];
        S1[i] = S5[i];
        S2[i] = S6[i];
      }
    }
  } else if constexpr (K == 5) {
    // state at group a: Pm1 = P[a-1], Sm2 = S[a-2], S0 = S[a], S1 = S[a+1]
    uint32_t Pm1[10], Sm2[5], S0[5], S1[5];
    {
      uint32_t t[5];
      S(-2, Sm2);
      S(-1, t);
      S(0, S0);
      sep::merge5(t, S0, Pm1, m1);
      S(1, S1);
    }
#pragma unroll (kDenseUnroll5)
    for (int a = 0; a < rows; a += 2) {
      uint32_t S2[5], S3[5], P1[10], c[6];
      S(a + 2, S2);
      S(a + 3, S3);
      sep::merge5(S1, S2, P1, m1);
      sep::core4_5(Pm1, P1, c, m1);
      if constexpr (FUSED) {
        // window rows: a-2 | a-1 .. a+2 (shared) | a+3
        const uint32_t tn = vmin2(Pm1[0], P1[0]), tx = vmax2(Pm1[9], P1[9]);
        put_f(a, sep::final5(c, Sm2, m1), vmin2(tn, Sm2[0]), vmax2(tx, Sm2[4]));
        put_f(a + 1, sep::final5(c, S3, m1), vmin2(tn, S3[0]), vmax2(tx, S3[4]));
      } else {
        put(a, sep::final5(c, Sm2, m1));
        put(a + 1, sep::final5(c, S3, m1));
      }
#pragma unroll
      for (int i = 0; i < 10; ++i) Pm1[i] = P1[i];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        Sm2[i] = S0[i];
        S0[i] = S2[i];
        S1[i] = S3[i];
      }
    }
  }
  if constexpr (FUSED) {
    *detected = (uint32_t)(2 * rows) - ((sacc & 0xFFFFu) + (sacc >> 16));
    replaced = (racc & 0xFFFFu) + (racc >> 16);
  }
  return replaced;
}

}  // namespace wk
}  // namespace irdn
