// Seeded salt-and-pepper injection on the GPU, bit-identical to the reference's
// sequential generator (pkg/src/irdenoise/noise.py:89-106).
//
// The reference walks pixels in row-major order drawing from one SplitMix64 stream
// (noise.py:17-34): one uniform per pixel decides corruption (u < density) and, only
// for a corrupted pixel, a second uniform picks salt (255) or pepper (0). Draw p of
// the stream is mix(seed + (p + 1) * gamma), so any draw can be computed directly; what
// is sequential is which draw belongs to which pixel, because corrupted pixels consume
// two draws. Seen as a parse of the draw stream into tokens of length 1 or 2, each
// draw position is a two-state transfer function on "does a token start here?":
//     start (state 0): one token, next state = corrupted(p) ? 1 : 0
//     continuation (1): no token,  next state = 0
// and composing those functions is associative, so the token index of every draw is
// a parallel scan:
//   K1 (draws)  one thread per 32 draw positions: 32 SplitMix64 draws -> corruption
//               and salt bit words, the word's transfer function, composed per CTA;
//   K2 (chunks) one CTA scans the per-CTA functions -> entry state + token offset;
//   K3 (emit)   per CTA: recompose the word functions, scan them from the chunk's
//               entry, walk the bits and write pixel i = token i (out, flags, count).
// 2n draw positions always hold the first n tokens (a token is at most 2 draws).
//
// Comparison against a double: the reference tests (x >> 11) / 2^53 < d; with
// x' = x >> 11 < 2^53 that is x' < d * 2^53 <=> x' < ceil(d * 2^53) (d * 2^53 is exact).
#pragma once
#include <cstdint>

namespace irdn {
namespace noise {

constexpr int THREADS = 256;                  // words per chunk (one per thread)
constexpr int WORD = 32;                      // draw positions per word
constexpr int64_t CHUNK = (int64_t)THREADS * WORD;

__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t p) {
  uint64_t z = seed + (p + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Transfer function over a run of draws, for both entry states: n = tokens started,
// e = exit state (1: the next position continues a corrupted token).
struct Fn {
  uint32_t n0, n1;
  uint32_t e0, e1;
};

__device__ __forceinline__ Fn fn_identity() { return Fn{0u, 0u, 0u, 1u}; }

// f then g
__device__ __forceinline__ Fn fn_then(const Fn& f, const Fn& g) {
  Fn r;
  r.n0 = f.n0 + (f.e0 ? g.n1 : g.n0);
  r.e0 = f.e0 ? g.e1 : g.e0;
  r.n1 = f.n1 + (f.e1 ? g.n1 : g.n0);
  r.e1 = f.e1 ? g.e1 : g.e0;
  return r;
}

// Function of one 32-draw word with corruption bits c (bit b = draw b of the word).
// Tokens start where the state is 0; the state after a start at b is c_b, after a
// continuation 0. Walking the 32 bits for both entries costs ~4 ops per bit.
__device__ __forceinline__ Fn fn_word(uint32_t c) {
  uint32_t x0 = 0u, x1 = 1u, n0 = 0u, n1 = 0u;
#pragma unroll
  for (int b = 0; b < WORD; ++b) {
    const uint32_t cb = (c >> b) & 1u;
    n0 += x0 ^ 1u;
    n1 += x1 ^ 1u;
    x0 = (x0 ^ 1u) & cb;
    x1 = (x1 ^ 1u) & cb;
  }
  return Fn{n0, n1, x0, x1};
}

__device__ __forceinline__ Fn shfl_fn(const Fn& f, int src_lane_delta, bool up) {
  Fn r;
  if (up) {
    r.n0 = __shfl_up_sync(0xffffffffu, f.n0, src_lane_delta);
    r.n1 = __shfl_up_sync(0xffffffffu, f.n1, src_lane_delta);
    r.e0 = __shfl_up_sync(0xffffffffu, f.e0, src_lane_delta);
    r.e1 = __shfl_up_sync(0xffffffffu, f.e1, src_lane_delta);
  } else {
    r.n0 = __shfl_sync(0xffffffffu, f.n0, src_lane_delta);
    r.n1 = __shfl_sync(0xffffffffu, f.n1, src_lane_delta);
    r.e0 = __shfl_sync(0xffffffffu, f.e0, src_lane_delta);
    r.e1 = __shfl_sync(0xffffffffu, f.e1, src_lane_delta);
  }
  return r;
}

// Inclusive scan (composition in thread order) over the CTA; returns the inclusive
// prefix of this thread and writes the CTA total to *total.
template <int NT>
__device__ __forceinline__ Fn block_scan(Fn f, Fn* s_warp, Fn* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Fn prev = shfl_fn(f, o, true);
    if (lane >= o) f = fn_then(prev, f);
  }
  if (lane == 31) s_warp[warp] = f;
  __syncthreads();
  if (warp == 0) {
    Fn w = lane < NT / 32 ? s_warp[lane] : fn_identity();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Fn prev = shfl_fn(w, o, true);
      if (lane >= o) w = fn_then(prev, w);
    }
    if (lane < NT / 32) s_warp[lane] = w;  // inclusive prefix over warps
  }
  __syncthreads();
  if (warp > 0) f = fn_then(s_warp[warp - 1], f);
  *total = s_warp[NT / 32 - 1];
  return f;
}

struct Params {
  const uint8_t* in;
  uint8_t* out;
  uint8_t* flags;                // may be null
  unsigned long long* count;     // may be null: number of corrupted pixels
  uint32_t* cbits;               // [nwords] corruption bit per draw
  uint32_t* sbits;               // [nwords] salt bit per draw (used as a token's second draw)
  Fn* chunk_fn;                  // [nchunks]
  uint2* chunk_entry;            // [nchunks] {entry state, unused}
  unsigned long long* chunk_off; // [nchunks] token index of the chunk's first token
  int64_t n;                     // pixels
  int64_t nwords;                // ceil(2n / 32)
  int64_t nchunks;
  uint64_t seed;
  uint64_t thr_density;          // ceil(density * 2^53)
  uint64_t thr_salt;             // ceil(salt_fraction * 2^53)
};

__global__ void __launch_bounds__(THREADS) noise_draws_kernel(const Params p) {
  __shared__ Fn s_warp[THREADS / 32];
  const int64_t w = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  uint32_t c = 0u, s = 0u;
  if (w < p.nwords) {
    const uint64_t p0 = (uint64_t)w * WORD;
#pragma unroll 4
    for (int b = 0; b < WORD; ++b) {
      const uint64_t u = splitmix_draw(p.seed, p0 + b) >> 11;
      c |= (uint32_t)(u < p.thr_density) << b;
      s |= (uint32_t)(u < p.thr_salt) << b;
    }
    p.cbits[w] = c;
    p.sbits[w] = s;
  }
  Fn f = w < p.nwords ? fn_word(c) : fn_identity();
  Fn total;
  block_scan<THREADS>(f, s_warp, &total);
  if (threadIdx.x == 0) p.chunk_fn[blockIdx.x] = total;
}

// One CTA: sequential over tiles of THREADS chunk functions.
__global__ void __launch_bounds__(THREADS) noise_chunks_kernel(const Params p) {
  __shared__ Fn s_warp[THREADS / 32];
  __shared__ uint32_t s_state;
  __shared__ unsigned long long s_off;
  if (threadIdx.x == 0) {
    s_state = 0u;
    s_off = 0ull;
  }
  __syncthreads();
  for (int64_t base = 0; base < p.nchunks; base += THREADS) {
    const int64_t j = base + threadIdx.x;
    const Fn f = j < p.nchunks ? p.chunk_fn[j] : fn_identity();
    Fn total;
    const Fn incl = block_scan<THREADS>(f, s_warp, &total);
    const uint32_t a = s_state;
    const unsigned long long o = s_off;
    // exclusive prefix = inclusive prefix of the previous thread
    Fn excl = shfl_fn(incl, 1, true);
    if ((threadIdx.x & 31) == 0) excl = threadIdx.x ? s_warp[(threadIdx.x >> 5) - 1] : fn_identity();
    if (j < p.nchunks) {
      p.chunk_entry[j] = make_uint2(a ? excl.e1 : excl.e0, 0u);
      p.chunk_off[j] = o + (a ? excl.n1 : excl.n0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_off = o + (a ? total.n1 : total.n0);
      s_state = a ? total.e1 : total.e0;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(THREADS) noise_emit_kernel(const Params p) {
  __shared__ Fn s_warp[THREADS / 32];
  __shared__ unsigned long long s_cnt;
  const int64_t w = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  const uint32_t c = w < p.nwords ? p.cbits[w] : 0u;
  const Fn f = w < p.nwords ? fn_word(c) : fn_identity();
  if (threadIdx.x == 0) s_cnt = 0ull;
  Fn total;
  const Fn incl = block_scan<THREADS>(f, s_warp, &total);
  Fn excl = shfl_fn(incl, 1, true);
  if ((threadIdx.x & 31) == 0) excl = threadIdx.x ? s_warp[(threadIdx.x >> 5) - 1] : fn_identity();
  const uint32_t a = p.chunk_entry[blockIdx.x].x;
  uint32_t x = a ? excl.e1 : excl.e0;
  int64_t i = (int64_t)p.chunk_off[blockIdx.x] + (a ? excl.n1 : excl.n0);
  uint32_t corrupted = 0u;
  if (w < p.nwords && i < p.n) {
    const uint32_t s = p.sbits[w];
    const uint32_t s_next = w + 1 < p.nwords ? p.sbits[w + 1] : 0u;
    for (int b = 0; b < WORD && i < p.n; ++b) {
      if (x == 0u) {
        const uint32_t cb = (c >> b) & 1u;
        const uint8_t v = p.in[i];
        uint8_t o = v;
        if (cb) {
          const uint32_t salt = b + 1 < WORD ? (s >> (b + 1)) & 1u : s_next & 1u;
          o = salt ? (uint8_t)255 : (uint8_t)0;
          ++corrupted;
        }
        p.out[i] = o;
        if (p.flags) p.flags[i] = (uint8_t)cb;
        ++i;
        x = cb;
      } else {
        x = 0u;
      }
    }
  }
  if (p.count) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) corrupted += __shfl_xor_sync(0xffffffffu, corrupted, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && corrupted) atomicAdd(&s_cnt, (unsigned long long)corrupted);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) atomicAdd(p.count, s_cnt);
  }
}

}  // namespace noise
}  // namespace irdn
