// Warp-autonomous FNR / MF kernel (sm_100a): every warp streams its own 64 x 32 tiles.
//
// The flagged-pixel median work is irregular (2-50 % of pixels, clustered by scene
// content), so CTA-wide tiles leave warps waiting at barriers for the slowest warp
// and for the next tile's load. Here each warp is its own pipeline:
//   * a dynamic scheduler hands out 64 x 32 warp tiles (one atomic per tile);
//   * lane 0 stages the tile plus halo with TMA (cp.async.bulk.tensor.3d) into the
//     warp's own shared-memory ring (NSTAGE deep, one mbarrier per stage), issuing
//     the load of the warp's next tile as soon as a stage is released — so the load
//     runs while the current tile is filtered, and no CTA barrier exists at all;
//   * detector (filters.py:169-171) and median (filters.py:172-176) exactly as in
//     fnr_tile.cuh: each lane owns one column pair (u16x2) walking the 32 rows, noisy
//     pixels are compacted with one warp scan into the warp's queue, and each lane
//     runs one median-selection network per two queued pixels.
// Frame borders: TMA zero-fills out-of-frame cells; the warp overwrites them with the
// nearest in-frame cell (replicate edge, image.py:117-130) before filtering.
#pragma once
#include <type_traits>
#include "fnr_tile.cuh"
#include "fnr_dense.cuh"

namespace irdn {
namespace wk {

// Windows with a dense-median stage (fnr_dense.cuh): MF always (unless p.dense_min < 0),
// FNR for tiles with more than p.dense_min flagged pixels.
template <int K>
constexpr bool kDense = K == 5 || K == 7;

#ifndef IRDN_WARPS
#define IRDN_WARPS 4  // round-2 re-sweep: 2 / 4 warps per CTA c2 37.3 / 36.9 us (packaging only)
#endif
constexpr int WARPS = IRDN_WARPS;      // warps per CTA (packaging only: no CTA barriers)
constexpr int THREADS = 32 * WARPS;
constexpr int WW = 64;                 // warp tile width: 32 lanes x 2 pixels
#ifndef IRDN_WH
#define IRDN_WH 32
#endif
#ifndef IRDN_DET_FMA
#define IRDN_DET_FMA 0  // odd-offset shifts as PRMT (ALU): round-2 re-sweep c2 37.3 -> 36.4 us (round 1: IMAD)
#endif
#ifndef IRDN_WSTAGE
#define IRDN_WSTAGE 1
#endif
constexpr int WH = IRDN_WH;            // warp tile height, k <= 9 (16 or 32: one flag word per 16 rows)
constexpr int NSTAGE = IRDN_WSTAGE;
// k >= 11: taller tiles. The median stage runs one 121-input network per lane for up to 64
// queued pixels whatever their number, and BASELINE c4 flags ~1.7 % of its pixels: a 64 x 32
// tile queues ~34 (17 of 32 lanes busy), a 64 x 48 tile ~51 (26 lanes) and still fits one
// round; the halo rows fall from 42 / 32 to 58 / 48.
#ifndef IRDN_WH11
#define IRDN_WH11 48
#endif
template <int K>
constexpr int WHK = K >= 11 ? IRDN_WH11 : WH;
#ifndef IRDN_QCAP
#define IRDN_QCAP 2048
#endif
// Queue entries per round: a warp tile with more noisy pixels than QCAP is filtered in
// several rounds of QCAP pixels (keeps shared memory per warp small -> more warps/SM).
constexpr int QCAP = IRDN_QCAP;

template <typename T, int K>
struct Geo {
  static constexpr int r = K / 2;
  static constexpr int A = 16 / (int)sizeof(T);  // TMA x start: 16-byte aligned
  static constexpr int R = A;
  static_assert(r <= R, "window radius exceeds the aligned halo");
  static constexpr int BOXW = ((WW + R + r + A - 1) / A) * A;
  static constexpr int TH = WHK<K>;      // warp tile height
  static constexpr int NF = (TH + 15) / 16;  // flag words per lane (16 rows x 2 pixels each)
  static_assert(TH % 16 == 0 && TH >= 16 && TH <= 64, "whole 16-row flag words, 8-bit queue rows");
  static constexpr int BOXH = TH + 2 * r;
  static constexpr int IN_BYTES = BOXW * BOXH * (int)sizeof(T);
  static constexpr int STAGE = (IN_BYTES + 127) & ~127;
  static constexpr int Q_OFF = NSTAGE * STAGE;
  static constexpr int BAR_OFF = Q_OFF + QCAP * 2;
  static constexpr int INFO_OFF = BAR_OFF + 8 * NSTAGE;
  static constexpr int WARP_BYTES = (INFO_OFF + 32 * NSTAGE + 127) & ~127;
  static constexpr int SMEM = WARPS * WARP_BYTES + 128;
};

struct WTile {
  int t, b, x0, y0, rows, pass;
};

// Tile t of the pass. The pool ends in half-height tiles (the halves of the last
// ntiles - full_tiles full tiles, p.full_tiles.. onwards), so the warps that finish
// last finish a short tile: with ~3.5 tiles per warp the tail of a 64 x 32 pool is
// about one tile time.
template <int TH>
__device__ __forceinline__ WTile tile_of(const tile::TileParams& p, int t, int tiles_per_frame) {
  WTile ti;
  ti.t = t;
  int f = t, rows = TH, dy = 0;
  if (t >= p.full_tiles) {
    const int h = t - p.full_tiles;
    f = p.full_tiles + (h >> 1);
    rows = TH / 2;
    dy = (h & 1) * (TH / 2);
  }
  ti.b = tile::udiv(f, tiles_per_frame, p.tpf_magic);
  const int tt = f - ti.b * tiles_per_frame;
  const int ty = tile::udiv(tt, p.tiles_x, p.tx_magic);
  ti.x0 = (tt - ty * p.tiles_x) * WW;
  ti.y0 = p.row_begin + ty * TH + dy;
  ti.rows = rows;
  return ti;
}

// Multi-pass launch: tiles [0, (P-1) N) are the full tiles of passes 0 .. P-2 in order
// (N tiles per pass), the rest is the last pass with its half-height tail (tile_of).
template <int TH>
__device__ __forceinline__ WTile tile_of_mp(const tile::TileParams& p, int t, int tiles_per_frame) {
  const int N = tiles_per_frame * p.batch;
  const int early = (p.passes - 1) * N;
  if (t >= early) {
    WTile ti = tile_of<TH>(p, t - early, tiles_per_frame);
    ti.t = t;
    ti.pass = p.passes - 1;
    return ti;
  }
  WTile ti;
  ti.t = t;
  ti.pass = t / N;
  const int u = t - ti.pass * N;
  ti.b = u / tiles_per_frame;
  const int tt = u - ti.b * tiles_per_frame;
  const int ty = tt / p.tiles_x;
  ti.x0 = (tt - ty * p.tiles_x) * WW;
  ti.y0 = p.row_begin + ty * TH;
  ti.rows = TH;
  return ti;
}

// replicate-edge fix-up of one warp's box (cells outside the frame)
template <typename T, int K, int BOXW = Geo<T, K>::BOXW, int BOXH = Geo<T, K>::BOXH>
__device__ __forceinline__ void fix_edges_warp(T* s_in, int gx_lo, int gy_lo, int width, int height, int lane) {
  using G = Geo<T, K>;
  constexpr int A = G::A;
  const int c_lo = max(0, -gx_lo), c_hi = min(BOXW, width - gx_lo);
  const int y_lo = max(0, -gy_lo), y_hi = min(BOXH, height - gy_lo);
  const int ncl = c_lo, ncr = BOXW - c_hi;
  if (ncl | ncr) {
    if ((ncl == 0 || ncl == A) && (ncr == 0 || ncr == A)) {
      for (int i = lane; i < 2 * (y_hi - y_lo); i += 32) {
        const int row = y_lo + (i >> 1);
        const bool left = (i & 1) == 0;
        if (left ? ncl == 0 : ncr == 0) continue;
        T* rp = s_in + row * BOXW;
        uint32_t v = (uint32_t)rp[left ? c_lo : c_hi - 1];
        v *= sizeof(T) == 1 ? 0x01010101u : 0x00010001u;
        *reinterpret_cast<uint4*>(rp + (left ? 0 : BOXW - A)) = make_uint4(v, v, v, v);
      }
    } else {
      const int nc = ncl + ncr;
      for (int i = lane; i < (y_hi - y_lo) * nc; i += 32) {
        const int row = y_lo + i / nc, j = i % nc;
        T* rp = s_in + row * BOXW;
        rp[j < ncl ? j : c_hi + (j - ncl)] = rp[j < ncl ? c_lo : c_hi - 1];
      }
    }
    __syncwarp();
  }
  const int nrt = y_lo, nrb = BOXH - y_hi;
  constexpr int V = BOXW / A;
  for (int i = lane; i < (nrt + nrb) * V; i += 32) {
    const int j = i / V, col = (i - j * V) * A;
    const int row = j < nrt ? j : y_hi + (j - nrt);
    *reinterpret_cast<uint4*>(s_in + row * BOXW + col) =
        *reinterpret_cast<const uint4*>(s_in + (j < nrt ? y_lo : y_hi - 1) * BOXW + col);
  }
  __syncwarp();
}

// K-wide horizontal min / max of one smem row for the lane's column pair (u16x2), and the
// centre word. Odd r (k = 3, 7, 11): with aligned words w_j = columns (x+2j, x+2j+1),
// pixel x needs the low halves of w_-(r-1)/2 .. w_(r-1)/2 and the high halves of
// w_-(r+1)/2 .. w_(r-1)/2, pixel x+1 the mirror image, so one word-wise reduction M over
// the r middle words serves both: min(x) = min(M.lo, M.hi, w_-(r+1)/2.hi) and
// min(x+1) = min(M.hi, M.lo, w_(r+1)/2.lo), i.e. vmin3(M, swap(M), C) with one shared
// PRMT for C — 6 VIMNMX3 + 3 PRMT for 11x11 min and max instead of 10 VIMNMX3 + 6 shifted
// words (12 IMAD). Even r (k = 5, 9): the k words at every offset (odd ones shifted in).
template <typename T, int K>
__device__ __forceinline__ void row_minmax(const T* rowp, uint32_t& mn, uint32_t& mx, uint32_t& cen,
                                           uint32_t k65536) {
  constexpr int r = K / 2, J = (r + 1) / 2;
  uint32_t wd[2 * J + 1];
#pragma unroll
  for (int j = -J; j <= J; ++j) wd[j + J] = tile::load_pair<T>(rowp, 2 * j);
  cen = wd[J];
  if constexpr ((r & 1) == 1) {
    uint32_t mid[2 * J - 1];
#pragma unroll
    for (int i = 0; i < 2 * J - 1; ++i) mid[i] = wd[i + 1];
    const uint32_t a = tile::reduce_min<2 * J - 1>(mid), b = tile::reduce_max<2 * J - 1>(mid);
    const uint32_t c = tile::prmt(wd[0], wd[2 * J], 0x5432u);  // (w_-J.hi, w_J.lo)
    mn = vmin3(a, tile::prmt(a, a, 0x1032u), c);
    mx = vmax3(b, tile::prmt(b, b, 0x1032u), c);
  } else {
    uint32_t ops[K];
#pragma unroll
    for (int d = -r; d <= r; ++d)
      ops[d + r] = (d & 1) == 0 ? wd[J + d / 2]
                   : (IRDN_DET_FMA ? shift_pair(wd[J + (d - 1) / 2], wd[J + (d + 1) / 2], k65536)
                                   : tile::prmt(wd[J + (d - 1) / 2], wd[J + (d + 1) / 2], 0x5432u));
    mn = tile::reduce_min<K>(ops);
    mx = tile::reduce_max<K>(ops);
  }
}

// Detector over the warp tile.
//
// Per input row: the K-wide horizontal min / max of the lane's column pair (2J+1 aligned
// words, odd offsets shifted in). Vertically, output rows are produced in pairs (j, j+1)
// that share the K-2 input rows j+1 .. j+2r-1: one reduction over those, then one
// 3-input op per output for the two rows each adds — (K-3)/2 + 2 ops per two rows instead
// of K-1. Measured (tools/ab.sh): c3 (7x7) 689.7 -> 684.5 us, but c2 (5x5) 40.2 -> 40.5 us
// and c4 (11x11) 251.2 -> 253.8 us, so by default only K = 7 pairs its rows
// (IRDN_VPAIR=0: never, 1: every K).
#ifndef IRDN_ROWADDR
#define IRDN_ROWADDR 0  // per-row pointer increments (round-2 re-sweep: c2 -0.7 %; -1: k <= 5 only, 1 always)
#endif
#ifndef IRDN_VPAIR
#define IRDN_VPAIR -1
#endif
template <typename T, int K, bool FULL, int ROWS = WHK<K>>
__device__ __forceinline__ void detect(const T* s_in, int c0, T* outp, int64_t pitch, int valid_rows, bool ok0,
                                       bool ok1, uint32_t (&flags)[2], uint32_t one) {
  static_assert(ROWS <= 32, "one or two 16-row flag words (taller tiles: detect_rolled)");
  static_assert(ROWS % 2 == 0, "output rows are produced in pairs");
  using G = Geo<T, K>;
  constexpr int r = G::r, BOXW = G::BOXW;
  constexpr bool VPAIR = IRDN_VPAIR < 0 ? K == 7 : IRDN_VPAIR != 0;
  constexpr int KR = VPAIR ? K + 1 : K;  // ring of per-row horizontal results
  constexpr int CR = r + 2;                   // ring of centre words
  const uint32_t m1 = 0u - one, k65536 = one << 16, ones = one * 0x00010001u;
  uint32_t rmin[KR], rmax[KR], rcen[CR];
  const T* rowp = s_in + c0;
  constexpr bool ROWADDR = IRDN_ROWADDR < 0 ? K <= 5 : IRDN_ROWADDR != 0;
  const uint32_t pitch_b = (uint32_t)(pitch * (int64_t)sizeof(T));  // < 2^32: rows of at most 2^31 pixels
  // flag test and signal-pixel store of output row y (window min vmn, max vmx, centre c)
  uint32_t sig[2] = {0u, 0u};  // signal (not noisy) bits: row y at bits y % 16 and 16 + y % 16 of sig[y / 16]
  auto emit = [&](int y, uint32_t vmn, uint32_t vmx, uint32_t c) {
    // z = min(c - vmn, vmx - c, 1) per lane: 0 <=> centre is the window min or max (no
    // borrow: vmn <= c <= vmx), 1 otherwise; shifted into the row's bit position
    const uint32_t z = vmin3(fma_sub(c, m1, vmn), fma_sub(vmx, m1, c), ones);
    sig[y >> 4] += z << (y & 15);
    if constexpr (ROWADDR) {
      // row address = base + y * pitch (one wide multiply-add per row, y is a constant)
      T* const rp = reinterpret_cast<T*>(reinterpret_cast<char*>(outp) + (uint64_t)(uint32_t)y * pitch_b);
      if (FULL) tile::store_pair_g<T>(rp, c, true, true);
      else if (y < valid_rows) tile::store_pair_g<T>(rp, c, ok0, ok1);
    } else {
      if (FULL) tile::store_pair_g<T>(outp, c, true, true);
      else if (y < valid_rows) tile::store_pair_g<T>(outp, c, ok0, ok1);
      outp += pitch;
    }
  };
#pragma unroll
  for (int s = 0; s < ROWS + 2 * r; ++s) {
    row_minmax<T, K>(rowp + s * BOXW, rmin[s % KR], rmax[s % KR], rcen[s % CR], k65536);
    if constexpr (VPAIR) {
      if (s >= 2 * r + 1 && ((s - 2 * r - 1) & 1) == 0) {
        const int y = s - 2 * r - 1;  // output rows y, y + 1 = input rows y .. y + 2r + 1 (= s)
        uint32_t am[K - 2], ax[K - 2];
#pragma unroll
        for (int q = 0; q < K - 2; ++q) {
          am[q] = rmin[(y + 1 + q) % KR];
          ax[q] = rmax[(y + 1 + q) % KR];
        }
        const uint32_t amn = tile::reduce_min<K - 2>(am), amx = tile::reduce_max<K - 2>(ax);
        const uint32_t e_mn = rmin[(y + 2 * r) % KR], e_mx = rmax[(y + 2 * r) % KR];
        emit(y, vmin3(amn, rmin[y % KR], e_mn), vmax3(amx, rmax[y % KR], e_mx), rcen[(y + r) % CR]);
        emit(y + 1, vmin3(amn, e_mn, rmin[s % KR]), vmax3(amx, e_mx, rmax[s % KR]), rcen[(y + 1 + r) % CR]);
      }
    } else if (s >= 2 * r) {
      const int y = s - 2 * r;
      emit(y, tile::reduce_min<KR>(rmin), tile::reduce_max<KR>(rmax), rcen[(s - r) % CR]);
    }
  }
  flags[0] = ~sig[0];
  flags[1] = ROWS > 16 ? ~sig[1] : 0u;
}

// Detector for large windows (k >= 11): the same per-row horizontal min / max, but the
// vertical K-row min / max by blocks of K input rows (van Herk / Gil-Werman): within a
// block a running prefix, at its end the suffixes, and an output row whose window ends in
// row i of block b is min(suffix_{b-1}[i+1], prefix_b[i]) — 6 two-input ops per row for
// min and max instead of 2 (K-1)/2 three-input ones. The block loop is rolled (one block
// of K rows unrolled, ~8 KB of SASS for 11x11 instead of ~27 KB for the 42 unrolled rows),
// so the detector and the 121-input median network no longer evict each other from the
// instruction cache (c4's top stall was no_instruction).
#ifndef IRDN_ROLLED_MIN_K
#define IRDN_ROLLED_MIN_K 11
#endif
template <typename T, int K, bool FULL, int ROWS = WHK<K>>
__device__ __forceinline__ void detect_rolled(const T* s_in, int c0, T* outp, int64_t pitch, int valid_rows,
                                              bool ok0, bool ok1, uint32_t (&flags)[Geo<T, K>::NF], uint32_t one) {
  static_assert(ROWS <= 64, "flag streams hold 64 rows");
  using G = Geo<T, K>;
  constexpr int r = G::r, BOXW = G::BOXW;
  constexpr int NIN = ROWS + 2 * r;          // box rows
  constexpr int NB = (ROWS + K - 1) / K;     // output blocks of K rows
  const uint32_t m1 = 0u - one, k65536 = one << 16, ones = one * 0x00010001u;
  const T* rowb = s_in + c0;
  // horizontal K-wide min / max (and the centre word) of box row s
  auto hrow = [&](int s, uint32_t& mn, uint32_t& mx, uint32_t& cen) {
    row_minmax<T, K>(rowb + min(s, NIN - 1) * BOXW, mn, mx, cen, k65536);  // rows past the box feed no output
  };
  // Previous block: suffix min / max from position j to K-1, and centre words, position j
  // <-> box row 2r + (b-1)K + j. Prologue: box rows 0 .. 2r-1 at positions 1 .. K-1.
  uint32_t hn[K], hx[K], cp[K];
  {
    uint32_t cn[K], cx[K];
#pragma unroll
    for (int j = 1; j < K; ++j) hrow(j - 1, cn[j], cx[j], cp[j]);
    hn[K - 1] = cn[K - 1];
    hx[K - 1] = cx[K - 1];
#pragma unroll
    for (int j = K - 2; j >= 1; --j) {
      hn[j] = vmin2(cn[j], hn[j + 1]);
      hx[j] = vmax2(cx[j], hx[j + 1]);
    }
    hn[0] = hx[0] = cp[0] = 0u;
  }
  // signal streams: bit y = row y of pixel 0 / pixel 1 is not noisy
  using Stream = std::conditional_t<(ROWS > 32), uint64_t, uint32_t>;
  Stream st0 = 0u, st1 = 0u;
  T* orow = outp;
#pragma unroll 1
  for (int b = 0; b < NB; ++b) {
    // block b: box rows 2r + bK + i (output row y = bK + i ends its window there)
    uint32_t cn[K], cx[K], cc[K], gn = 0u, gx = 0u, blk = 0u;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      hrow(2 * r + b * K + i, cn[i], cx[i], cc[i]);
      gn = i == 0 ? cn[0] : vmin2(gn, cn[i]);
      gx = i == 0 ? cx[0] : vmax2(gx, cx[i]);
      const uint32_t vmn = i == K - 1 ? gn : vmin2(hn[i + 1], gn);
      const uint32_t vmx = i == K - 1 ? gx : vmax2(hx[i + 1], gx);
      const uint32_t c = i >= r ? cc[i - r] : cp[i + K - r];  // centre: box row y + r
      // z = min(c - min, max - c, 1): 0 in noisy lanes; row i of the block at bits i, 16 + i
      blk += vmin3(fma_sub(c, m1, vmn), fma_sub(vmx, m1, c), ones) << i;
      if (b * K + i < ROWS) {
        if (FULL) tile::store_pair_g<T>(orow, c, true, true);
        else if (b * K + i < valid_rows) tile::store_pair_g<T>(orow, c, ok0, ok1);
        orow += pitch;
      }
    }
    constexpr uint32_t kBlk = (1u << K) - 1u;
    st0 |= (Stream)(blk & kBlk) << (b * K);
    st1 |= (Stream)((blk >> 16) & kBlk) << (b * K);
    hn[K - 1] = cn[K - 1];
    hx[K - 1] = cx[K - 1];
#pragma unroll
    for (int i = K - 2; i >= 0; --i) {
      hn[i] = vmin2(cn[i], hn[i + 1]);
      hx[i] = vmax2(cx[i], hx[i + 1]);
    }
#pragma unroll
    for (int i = 0; i < K; ++i) cp[i] = cc[i];
  }
  constexpr Stream kRows = ROWS >= 8 * (int)sizeof(Stream) ? ~(Stream)0 : ((Stream)1 << (ROWS % 64)) - 1u;
  st0 = ~st0 & kRows;  // noisy streams
  st1 = ~st1 & kRows;
  // detect()'s layout: row y at bits y % 16 (pixel 0) and 16 + y % 16 (pixel 1) of flags[y / 16]
#pragma unroll
  for (int h = 0; h < Geo<T, K>::NF; ++h) {
    const uint32_t a = (uint32_t)((uint64_t)st0 >> (32 * (h >> 1))), b = (uint32_t)((uint64_t)st1 >> (32 * (h >> 1)));
    flags[h] = 16 * h >= ROWS ? 0u : tile::prmt(a, b, (h & 1) ? 0x7632u : 0x5410u);
  }
}

// Median of queued pixels (entries y << 8 | x in warp-tile coords), two per lane.
template <typename T, int K>
__device__ __forceinline__ uint32_t medians(const T* s_in, const uint16_t* q, int n, T* out_tile, int64_t pitch,
                                            int lane, bool fnr, uint32_t m1) {
  using G = Geo<T, K>;
  constexpr int r = G::r, R = G::R, BOXW = G::BOXW;
  uint32_t replaced = 0;
  // Pair p = (entry p, entry p + P). Lane i takes pairs i*rounds .. i*rounds+rounds-1, so in one round the
  // 32 lanes touch entries ~n/64 apart: queue order is lane-major (a column pair's noisy
  // pixels are adjacent), and consecutive entries would hit the same smem banks (TMA rows
  // are multiples of 16 bytes, so a column's rows share few banks).
  const int P = (n + 1) >> 1;
  const int rounds = (P + 31) >> 5;
  for (int k = 0; k < rounds; ++k) {
    const int pi = lane * rounds + k;
    if (pi >= P) break;
    const uint32_t e0 = q[pi];
    const bool two = pi + P < n;
    const uint32_t e1 = two ? q[pi + P] : e0;
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
    const uint32_t cen = v[(K * K) / 2];  // both centres, packed (the network may reuse v)
    const uint32_t med = tile::median_dispatch<K * K>(v, m1);
    const uint32_t med0 = med & 0xFFFFu, med1 = med >> 16;
    out_tile[y0 * pitch + x0] = (T)med0;
    if (two) out_tile[y1 * pitch + x1] = (T)med1;
    if (fnr) replaced += (med0 != (cen & 0xFFFFu)) + (two && med1 != (cen >> 16));
  }
  return replaced;
}

// MP = false: one pass from map0 into p.out. MP = true: p.passes passes in one persistent
// launch (pass 0 reads map0 = input; pass q > 0 reads the output of pass q-1 through map1
// (= p.tmp) or map2 (= p.out); the last pass writes p.out). A tile of pass q > 0 starts
// once the (up to) 3 x 3 tiles of pass q-1 under its box have published their flags, so
// the passes overlap tile by tile instead of meeting at a kernel boundary.
template <typename T, int K, bool MP>
__device__ __forceinline__ void warp_body(const CUtensorMap* map0, const CUtensorMap* map1, const CUtensorMap* map2,
                                          const tile::TileParams& p) {
  static_assert(!MP || NSTAGE == 1, "a warp waiting on pass dependencies must hold no other tile");
  using G = Geo<T, K>;
  constexpr int r = G::r, R = G::R, BOXW = G::BOXW;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((128u - (tile::smem_u32(smem_raw) & 127u)) & 127u);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* wsm = base + warp * G::WARP_BYTES;
  uint16_t* s_q = reinterpret_cast<uint16_t*>(wsm + G::Q_OFF);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(wsm + G::BAR_OFF);
  WTile* s_info = reinterpret_cast<WTile*>(wsm + G::INFO_OFF);

  const int tiles_per_frame = p.tiles_x * p.tiles_y;
  const int npass = tiles_per_frame * p.batch;  // full tiles per pass
  const int ntiles = (MP ? (p.passes - 1) * npass : 0) + p.full_tiles + 2 * (npass - p.full_tiles);
  const bool fnr = p.method == 0;
  // pass q writes out when (P-1-q) is even, else tmp (the last pass lands in out)
  auto dst_is_out = [&](int q) { return !MP || ((p.passes - 1 - q) & 1) == 0; };
  constexpr int TH = G::TH, NF = G::NF;
  auto tile_at = [&](int t) {
    return MP ? tile_of_mp<TH>(p, t, tiles_per_frame) : tile_of<TH>(p, t, tiles_per_frame);
  };
  uint32_t replaced = 0, detected = 0;
  bool pred_dense = false;  // k = 5 / 7 FNR: this warp's last tile took the dense stage

  // lane 0: grab a warp tile, publish it beside the stage, start its TMA load (or
  // arrive empty past the end); the mbarrier's release/acquire publishes the info.
  uint32_t epoch = 0;  // MP: this launch's flag value (lane 0; read after griddepcontrol.wait)
  const int nwarps = (int)gridDim.x * WARPS, gwarp = (int)blockIdx.x * WARPS + warp;
  int taken = 1;  // tiles this warp has taken (the first one below)
  auto refill = [&](int stage, int pre = -1) {
    int t = pre;
    if (t < 0) {
      t = taken < p.static_rounds ? gwarp + taken * nwarps
                                  : (int)atomicAdd(p.sched, 1u) + p.static_rounds * nwarps;
      ++taken;
    }
    WTile ti;
    ti.t = t;
    if (t < ntiles) {
      ti = tile_at(t);
      const CUtensorMap* src = map0;
      if (MP && ti.pass > 0) {
        // wait for the pass-(q-1) tiles under this tile's box, then read their output
        const int tx = ti.x0 / WW, ty = (ti.y0 - p.row_begin) / TH;
        const unsigned int* fl = p.flags + 32 + (size_t)(ti.pass - 1) * npass + (size_t)ti.b * tiles_per_frame;
        // the (up to) 9 flags with independent relaxed loads, one fence once all match
        // (chained acquire loads would serialise nine L2 round trips per tile)
        const int y_lo = max(ty - 1, 0), y_hi = min(ty + 1, p.tiles_y - 1);
        const int x_lo = max(tx - 1, 0), x_hi = min(tx + 1, p.tiles_x - 1);
        for (;;) {
          bool ready = true;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
              const int y = min(y_lo + dy, y_hi), x = min(x_lo + dx, x_hi);
              uint32_t v;
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl + y * p.tiles_x + x) : "memory");
              ready &= v == epoch;
            }
          if (ready) break;
          __nanosleep(64);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: the flags' release stores
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy writes -> TMA reads
        src = dst_is_out(ti.pass - 1) ? map2 : map1;
      }
      s_info[stage] = ti;
      tile::mbar_expect_tx(&s_bar[stage], G::IN_BYTES);
      tile::tma_load_3d(wsm + stage * G::STAGE, src, &s_bar[stage], ti.x0 - R, ti.y0 - r - p.in_row0, ti.b);
    } else {
      s_info[stage] = ti;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tile::smem_u32(&s_bar[stage])) : "memory");
    }
  };
  // Before waiting for the previous grid (PDL): take the first tile and pull it into L2.
  // A prefetch is only a hint (L2 stays coherent with the previous grid's writes), so it
  // is safe even when that grid produces this kernel's input; the smem load itself is
  // issued after griddepcontrol.wait.
  // The scheduler slot is shared with the previous launch on this stream, which may still be
  // draining under PDL (its last warp resets the slot), so a dynamically scheduled first tile
  // (static_rounds == 0: the multi-pass kernel) is claimed only after griddepcontrol.wait.
  int first = -1;
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map0) : "memory");
    if (p.static_rounds > 0) first = gwarp;
    if (first >= 0 && first < ntiles) {
      const WTile f = tile_at(first);
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(map0),
                   "r"(f.x0 - R), "r"(f.y0 - r - p.in_row0), "r"(f.b)
                   : "memory");
    }
  }
  pdl_wait_and_trigger();
  if (lane == 0) {
    if (MP) {
      epoch = *reinterpret_cast<volatile unsigned int*>(p.flags) + 1u;
      if (epoch == 0u) epoch = 1u;
    }
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) tile::mbar_init(&s_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) refill(s, s == 0 ? first : -1);  // first < 0: from the scheduler
  }
  __syncwarp();

  const int c0 = 2 * lane + R;  // smem column of this lane's first pixel

#ifdef IRDN_TIMELINE
  uint64_t t_wait, t_ready, t_det = 0, t_done;
#define IRDN_TL_NOW(v) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#endif
  for (int iter = 0;; ++iter) {
    const int stage = iter % NSTAGE;
    T* s_in = reinterpret_cast<T*>(wsm + stage * G::STAGE);
#ifdef IRDN_TIMELINE
    IRDN_TL_NOW(t_wait);
#endif
    tile::mbar_wait(&s_bar[stage], (iter / NSTAGE) & 1);
    const WTile ti = s_info[stage];
    if (ti.t >= ntiles) break;
#ifdef IRDN_TIMELINE
    IRDN_TL_NOW(t_ready);
#endif
    const int valid_w = min(WW, p.width - ti.x0);
    const int valid_h = min(ti.rows, p.row_end - ti.y0);
    if (valid_h <= 0) {  // lower half of a bottom-edge tile with <= WH / 2 rows
      __syncwarp();
      if (lane == 0) refill(stage);
      continue;
    }
    const int gx_lo = ti.x0 - R, gy_lo = ti.y0 - r;
    if (gx_lo < 0 || gy_lo < 0 || gx_lo + BOXW > p.width || gy_lo + G::BOXH > p.height)
      fix_edges_warp<T, K>(s_in, gx_lo, gy_lo, p.width, p.height, lane);
    T* const out_base = reinterpret_cast<T*>(dst_is_out(MP ? ti.pass : 0) ? p.out : p.tmp);
    T* const out_tile = out_base + (int64_t)ti.b * p.out_frame + (int64_t)(ti.y0 - p.row_begin) * p.out_pitch + ti.x0;
    const bool ok0 = 2 * lane < valid_w, ok1 = 2 * lane + 1 < valid_w;
    int n;
    bool fused = false;
    if constexpr (kDense<K>) {
      // the previous tile of this warp was dense: skip the detector, take the detector from
      // the dense stage's sorted rows (whole tiles only), and re-predict from this tile
      if (fnr && pred_dense && valid_w == WW && valid_h == ti.rows) {
        fused = true;
        const uint32_t none[2] = {0u, 0u};
        uint32_t det_t = 0;
        replaced += dense_tile<T, K, BOXW, true>(s_in, c0, out_tile + 2 * lane, p.out_pitch, ti.rows, valid_h,
                                                 true, true, none, true, p.one, &det_t);
        detected += det_t;
        n = (int)__reduce_add_sync(0xffffffffu, det_t);
        pred_dense = n * TH > p.dense_min * ti.rows;
      }
    }
    if (fused) {
    } else if (fnr) {
      uint32_t flags[NF];
      T* outp = out_tile + 2 * lane;
      if (valid_w == WW && valid_h == TH) {
        if constexpr (K >= IRDN_ROLLED_MIN_K) detect_rolled<T, K, true>(s_in, c0, outp, p.out_pitch, TH, true, true, flags, p.one);
        else detect<T, K, true>(s_in, c0, outp, p.out_pitch, TH, true, true, flags, p.one);
      } else if (TH % 32 == 0 && valid_w == WW && valid_h == TH / 2 && ti.rows == TH / 2) {
        if constexpr (K >= IRDN_ROLLED_MIN_K)
          detect_rolled<T, K, true, TH / 2>(s_in, c0, outp, p.out_pitch, TH / 2, true, true, flags, p.one);
        else detect<T, K, true, TH / 2>(s_in, c0, outp, p.out_pitch, TH / 2, true, true, flags, p.one);
#pragma unroll
        for (int h = TH / 32; h < NF; ++h) flags[h] = 0u;
      } else {
        if constexpr (K >= IRDN_ROLLED_MIN_K)
          detect_rolled<T, K, false>(s_in, c0, outp, p.out_pitch, valid_h, ok0, ok1, flags, p.one);
        else detect<T, K, false>(s_in, c0, outp, p.out_pitch, valid_h, ok0, ok1, flags, p.one);
        const uint32_t colm = (ok0 ? 0xFFFFu : 0u) | (ok1 ? 0xFFFF0000u : 0u);
#pragma unroll
        for (int h = 0; h < NF; ++h) {
          const int v = min(16, max(0, valid_h - 16 * h));
          const uint32_t rowm = v >= 16 ? 0xFFFFu : ((1u << v) - 1u);
          flags[h] &= colm & (rowm | (rowm << 16));
        }
      }
      if (TH == 16 && NF > 1) flags[NF - 1] = 0u;
#ifdef IRDN_TIMELINE
      IRDN_TL_NOW(t_det);
#endif
      int cnt = 0;
#pragma unroll
      for (int h = 0; h < NF; ++h) cnt += __popc(flags[h]);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      n = __shfl_sync(0xffffffffu, incl, 31);
      detected += (uint32_t)cnt;
      const int off = incl - cnt;  // index of this lane's first queue entry
      const uint32_t ebase = (uint32_t)(2 * lane);
      bool dense = false;
      if constexpr (kDense<K>) {
        // many flagged pixels: every pixel's median from shared sorted rows (fnr_dense.cuh)
        if (p.dense_min >= 0 && n * TH > p.dense_min * ti.rows) {  // dense_min: per full-height tile
          dense = true;
          replaced += dense_tile<T, K, BOXW>(s_in, c0, out_tile + 2 * lane, p.out_pitch, ti.rows, valid_h, ok0,
                                             ok1, flags, true, p.one);
        }
        pred_dense = dense;
      }
      for (int q0 = 0; q0 < (dense ? 0 : n); q0 += QCAP) {
        if (off < q0 + QCAP && off + cnt > q0) {
          int idx = off - q0;
#pragma unroll
          for (int h = 0; h < NF; ++h) {
            uint32_t f = flags[h];
            while (f) {
              const int bit = __ffs(f) - 1;
              f &= f - 1u;
              if (QCAP >= WW * TH || (unsigned)idx < (unsigned)QCAP)
                s_q[idx] = (uint16_t)(ebase + ((uint32_t)(16 * h + (bit & 15)) << 8) + (uint32_t)(bit >> 4));
              ++idx;
            }
          }
        }
        __syncwarp();  // queue visible; centre stores ordered before the median stores
        replaced += medians<T, K>(s_in, s_q, min(QCAP, n - q0), out_tile, p.out_pitch, lane, true, 0u - p.one);
        __syncwarp();  // queue reads done before the next round overwrites it
      }
    } else if (kDense<K> && p.dense_min >= 0) {
      const uint32_t none[2] = {0u, 0u};
      n = valid_h * valid_w;
      dense_tile<T, K, BOXW>(s_in, c0, out_tile + 2 * lane, p.out_pitch, ti.rows, valid_h, ok0, ok1, none, false,
                             p.one);
    } else {
      const int cols = max(0, valid_w), rows = max(0, valid_h);
      n = rows * cols;
      for (int q0 = 0; q0 < n; q0 += QCAP) {
        for (int j = lane; j < min(QCAP, n - q0); j += 32) {
          const int y = (q0 + j) / cols, x = (q0 + j) - y * cols;
          s_q[j] = (uint16_t)((y << 8) | x);
        }
        __syncwarp();
        medians<T, K>(s_in, s_q, min(QCAP, n - q0), out_tile, p.out_pitch, lane, false, 0u - p.one);
        __syncwarp();
      }
    }
#ifdef IRDN_TIMELINE
    IRDN_TL_NOW(t_done);
    if (lane == 0 && p.debug_buf) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* d = p.debug_buf + (size_t)ti.t * 6;
      d[0] = t_wait;
      d[1] = t_ready;
      d[2] = t_det;
      d[3] = t_done;
      d[4] = (unsigned long long)n;
      d[5] = ((unsigned long long)(blockIdx.x * WARPS + warp) << 16) | smid;
    }
#endif
    if (MP && ti.pass < p.passes - 1) {
      // publish this tile's output to the next pass: every lane's stores, then the flag
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        const int tx = ti.x0 / WW, ty = (ti.y0 - p.row_begin) / TH;
        unsigned int* f =
            p.flags + 32 + (size_t)ti.pass * npass + (size_t)ti.b * tiles_per_frame + ty * p.tiles_x + tx;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
      }
    }
    // this stage is free: load the warp's next tile into it
    tile::fence_proxy_async();
    __syncwarp();
    if (lane == 0) refill(stage);
  }
  if (lane == 0 && atomicAdd(p.sched + 1, 1u) == gridDim.x * WARPS - 1) {
    p.sched[0] = 0u;
    p.sched[1] = 0u;
    if (MP) *reinterpret_cast<volatile unsigned int*>(p.flags) = epoch;  // every warp has read the old one
  }
  if (fnr) block_add_counts<THREADS>(detected, replaced, p.counts);
}

template <typename T, int K>
__global__ void __launch_bounds__(THREADS) fnr_warp_kernel(const __grid_constant__ CUtensorMap in_map,
                                                           const tile::TileParams p) {
  warp_body<T, K, false>(&in_map, &in_map, &in_map, p);
}

// `p.passes` passes in one launch: in_map = input, tmp_map = p.tmp, out_map = p.out.
template <typename T, int K>
__global__ void __launch_bounds__(THREADS) fnr_warp_mp_kernel(const __grid_constant__ CUtensorMap in_map,
                                                              const __grid_constant__ CUtensorMap tmp_map,
                                                              const __grid_constant__ CUtensorMap out_map,
                                                              const tile::TileParams p) {
  warp_body<T, K, true>(&in_map, &tmp_map, &out_map, p);
}

}  // namespace wk
}  // namespace irdn
