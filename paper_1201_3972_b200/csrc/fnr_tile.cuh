// Shared pieces of the TMA tile kernels (sm_100a): launch parameters, PTX helpers
// (mbarrier, cp.async.bulk.tensor, PRMT), packed-pixel loads / stores and 3-input
// min / max reductions. The kernels are fnr_warp.cuh (k = 5..11, warp tiles),
// fnr_dense.cuh (its dense median stage) and fnr_k3.cuh (dense 3x3 u8).
//
// Round 1 also kept a CTA-tile kernel family here (4-warp CTAs, per-warp queues),
// selectable with IRDN_KERNEL=tile for comparison; the warp-autonomous kernel replaced
// it (c2 52 -> 39 us) and it was retired in round 2.
#pragma once
#include <cuda.h>
#include "fnr_common.cuh"
#include "select_nets.cuh"

namespace irdn {
namespace tile {

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
  // warp kernel: ceil(2^32 / d) for d = tiles per frame and tiles_x (wk::udiv)
  uint32_t tpf_magic, tx_magic;
};

inline uint32_t udiv_magic(uint32_t d) {
  return d <= 1u ? 0xFFFFFFFFu : (uint32_t)((((uint64_t)1 << 32) + d - 1) / d);
}

// n / d for 0 <= n < 2^31, 1 <= d < 2^31, with the launch-invariant magic = ceil(2^32 / d)
// (0xFFFFFFFF for d = 1): the multiply-high estimate is off by at most one either way and
// one remainder check fixes it — a few instructions instead of the integer-division
// sequence, in the path from the tile scheduler's atomic to the tile's TMA issue.
__device__ __forceinline__ int udiv(int n, int d, uint32_t magic) {
  int q = (int)__umulhi((uint32_t)n, magic);
  const int rem = n - q * d;
  q += rem < 0 ? -1 : (rem >= d ? 1 : 0);
  return q;
}

struct TileInfo {
  int t, b, tx0, ty0;
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

}  // namespace tile
}  // namespace irdn
