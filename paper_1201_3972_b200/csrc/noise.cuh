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
// and composing those functions is associative, so the token (= pixel) index of every
// draw is a prefix scan over draw positions.
//
// One persistent kernel does it in a single pass (chained scan with decoupled
// look-back): a CTA takes the next chunk of CHUNK draw positions in order (ticket),
//   1. computes its CHUNK = 32768 draws (1024 threads x 32: corruption + salt bit words),
//   2. composes the per-word functions (warp shuffles + one smem step) and publishes
//      the chunk's function, then the whole CTA looks back over the predecessors'
//      published functions / inclusive prefixes, 1024 chunks per step (one per thread:
//      with ~300 chunks in flight one step nearly always finds a prefix), to get its
//      entry state and first token index, and publishes its own inclusive prefix;
//   3. writes one action code per token to shared memory and emits its contiguous
//      range of output pixels with 16-byte loads/stores (noisy image + mask flags).
// Chunks stop being taken once a published prefix covers all n pixels, so only the
// ~(1 + density) n draws that the reference itself consumes are computed.
//
// Comparison against a double: the reference tests (x >> 11) / 2^53 < d; with
// x' = x >> 11 < 2^53 that is x' < d * 2^53 <=> x' < ceil(d * 2^53) (d * 2^53 is exact).
#pragma once
#include <cstdint>

namespace irdn {
namespace noise {

constexpr int THREADS = 1024;                 // words per chunk (one per thread)
constexpr int WORD = 32;                      // draw positions per word
constexpr int CHUNK = THREADS * WORD;         // 32768 draw positions per chunk
constexpr int WARPS = THREADS / 32;

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
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

// Corrupted token starts of one 32-draw word (bit b = draw b) given its entry state x
// (1: draw 0 is the second draw of a token started in the previous word). Within a
// run of consecutive corrupted draws, starts alternate from the run's first start; a
// run's parity is found with one carry-propagating add (the odd/even-run trick used
// by SIMD JSON scanners): c + (even run starts) flips exactly the runs that begin at
// even bit positions. A run entered in the continuation state begins at virtual
// position -1 (odd). Then continuations = corrupted starts << 1 (| x), tokens = the
// other positions, and the exit state is the corrupted-start bit 31.
__device__ __forceinline__ uint32_t corrupted_starts(uint32_t c, uint32_t x) {
  constexpr uint32_t kEven = 0x55555555u;
  const uint32_t run_start = c & ~((c << 1) | x);
  const uint32_t even_runs = ((c + (run_start & kEven)) ^ c) & c;  // runs starting at even bits
  const uint32_t odd_runs = c & ~even_runs;
  return (even_runs & kEven) | (odd_runs & ~kEven);
}

__device__ __forceinline__ Fn fn_word(uint32_t c) {
  const uint32_t cs0 = corrupted_starts(c, 0u), cs1 = corrupted_starts(c, 1u);
  const uint32_t cont0 = cs0 << 1, cont1 = (cs1 << 1) | 1u;
  return Fn{32u - (uint32_t)__popc(cont0), 32u - (uint32_t)__popc(cont1), cs0 >> 31, cs1 >> 31};
}

__device__ __forceinline__ Fn shfl_up_fn(const Fn& f, int d) {
  return Fn{__shfl_up_sync(0xffffffffu, f.n0, d), __shfl_up_sync(0xffffffffu, f.n1, d),
            __shfl_up_sync(0xffffffffu, f.e0, d), __shfl_up_sync(0xffffffffu, f.e1, d)};
}

// Chunk status words (one u64 per chunk, zeroed before the launch):
//   [63:62] 0 = not ready, 1 = function published, 2 = inclusive prefix published
//   function:  n0 [15:0], n1 [31:16], e0 [32], e1 [33]   (n <= CHUNK = 32768 < 2^16)
//   inclusive: tokens before the next chunk [40:0], exit state [41]
constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kFlagMask = 3ull << 62;

__device__ __forceinline__ unsigned long long pack_fn(const Fn& f) {
  return kAgg | (unsigned long long)f.n0 | ((unsigned long long)f.n1 << 16) | ((unsigned long long)f.e0 << 32) |
         ((unsigned long long)f.e1 << 33);
}
__device__ __forceinline__ Fn unpack_fn(unsigned long long w) {
  return Fn{(uint32_t)(w & 0xFFFFu), (uint32_t)((w >> 16) & 0xFFFFu), (uint32_t)((w >> 32) & 1u),
            (uint32_t)((w >> 33) & 1u)};
}

// Inclusive scan (composition in thread order) of one Fn per thread over the CTA;
// s_warp receives the inclusive prefix per warp ([WARPS - 1] = the CTA total).
__device__ __forceinline__ Fn block_scan_fn(Fn f, Fn* s_warp, int lane, int warp) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Fn prev = shfl_up_fn(f, o);
    if (lane >= o) f = fn_then(prev, f);
  }
  if (lane == 31) s_warp[warp] = f;
  __syncthreads();
  if (warp == 0) {
    Fn w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Fn prev = shfl_up_fn(w, o);
      if (lane >= o) w = fn_then(prev, w);
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  if (warp > 0) f = fn_then(s_warp[warp - 1], f);
  return f;
}

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct Params {
  const uint8_t* in;
  uint8_t* out;
  uint8_t* flags;                 // may be null
  unsigned long long* count;      // may be null: number of corrupted pixels (added)
  unsigned long long* status;     // [max_chunks] zeroed
  unsigned int* ctl;              // [0] chunk ticket, [1] done flag (zeroed)
  int64_t n;                      // pixels
  int64_t max_chunks;             // ceil(2n / CHUNK): 2n draws always hold n tokens
  uint64_t seed;
  uint64_t z_density;             // ceil(density * 2^53) << 11 (compare the raw 64-bit output)
  uint64_t z_salt;                // ceil(salt_fraction * 2^53) << 11
  int32_t all_density;            // density threshold is 2^53 (density 1.0): always corrupt
  int32_t all_salt;
  int32_t vec;                    // in / out / flags 16-byte aligned: vector body
};

__global__ void __launch_bounds__(THREADS, 2) noise_kernel(const Params p) {
  __shared__ Fn s_warp[WARPS];
  __shared__ Fn s_look[WARPS];
  __shared__ uint8_t s_code[CHUNK];   // per token of the chunk: 0 keep, 1 pepper, 2 salt
  __shared__ int64_t s_chunk;
  __shared__ int s_hi;
  __shared__ unsigned long long s_incl;
  __shared__ unsigned long long s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  volatile unsigned int* ctl = p.ctl;
  uint32_t corrupted = 0u;

  for (;;) {
    if (tid == 0) s_chunk = ctl[1] ? -1 : (int64_t)atomicAdd(p.ctl, 1u);
    __syncthreads();
    const int64_t chunk = s_chunk;
    if (chunk < 0 || chunk >= p.max_chunks) break;

    // 1. draws: 32 positions per thread, SplitMix64 state advanced by gamma per draw
    const uint64_t p0 = (uint64_t)chunk * CHUNK + (uint64_t)tid * WORD;
    uint64_t st = p.seed + (p0 + 1ull) * 0x9E3779B97F4A7C15ull;
    uint32_t c = 0u, s = 0u;
#pragma unroll 8
    for (int b = 0; b < WORD; ++b) {
      const uint64_t z = splitmix_mix(st);  // (z >> 11) < T  <=>  z < T << 11
      st += 0x9E3779B97F4A7C15ull;
      c |= (uint32_t)(z < p.z_density) << b;
      s |= (uint32_t)(z < p.z_salt) << b;
    }
    if (p.all_density) c = ~0u;  // T = 2^53: T << 11 overflows, every draw passes
    if (p.all_salt) s = ~0u;
    // salt bit of a token whose first draw is this word's last position: next word's bit 0
    uint32_t s_next = __shfl_down_sync(0xffffffffu, s, 1);
    if (lane == 31) s_next = p.all_salt || splitmix_mix(st) < p.z_salt;  // st = draw p0 + 32

    // 2. chunk function, published before the look-back
    Fn f = block_scan_fn(fn_word(c), s_warp, lane, warp);
    const Fn w = s_warp[WARPS - 1];
    if (tid == 0 && chunk > 0) st_status(p.status + chunk, pack_fn(w));
    // look-back: thread t reads chunk base - (THREADS - 1 - t)
    unsigned long long pre = 0ull;  // tokens before the chunk, entry state in bit 63
    Fn acc = fn_identity();         // composition of the chunks between the prefix and this one
    for (int64_t base = chunk - 1; base >= 0; base -= THREADS) {
      const int64_t j = base - (THREADS - 1 - tid);
      unsigned long long v = kIncl;  // j < 0: virtual prefix (0 tokens, state 0)
      if (j >= 0)
        while (((v = ld_status(p.status + j)) & kFlagMask) == 0ull) __nanosleep(256);  // leave issue slots to the SM's other CTA
      const bool incl = (v & kFlagMask) == kIncl;
      if (tid == 0) s_hi = -1;
      __syncthreads();
      const unsigned bal = __ballot_sync(0xffffffffu, incl);
      if (lane == 0 && bal) atomicMax(&s_hi, warp * 32 + 31 - __clz((int)bal));
      __syncthreads();
      const int hi = s_hi;
      if (tid == hi) s_incl = v;
      const Fn g = block_scan_fn(tid > hi ? unpack_fn(v) : fn_identity(), s_look, lane, warp);
      (void)g;
      acc = fn_then(s_look[WARPS - 1], acc);
      if (hi >= 0) {
        const unsigned long long vi = s_incl;
        const uint32_t a0 = (uint32_t)((vi >> 41) & 1u);
        const unsigned long long off = vi & ((1ull << 41) - 1);
        pre = (off + (a0 ? acc.n1 : acc.n0)) | ((unsigned long long)(a0 ? acc.e1 : acc.e0) << 63);
        break;
      }
      __syncthreads();  // s_hi / s_look reused by the next window
    }
    if (tid == 0) {
      const uint32_t a = (uint32_t)(pre >> 63);
      const unsigned long long off = pre & ~(1ull << 63);
      const unsigned long long end = off + (a ? w.n1 : w.n0);
      st_status(p.status + chunk, kIncl | end | ((unsigned long long)(a ? w.e1 : w.e0) << 41));
      if (end >= (unsigned long long)p.n) ctl[1] = 1u;
    }
    Fn excl = shfl_up_fn(f, 1);
    if (lane == 0) excl = warp ? s_warp[warp - 1] : fn_identity();
    const uint32_t a = (uint32_t)(pre >> 63);
    const int64_t chunk_tok0 = (int64_t)(pre & ~(1ull << 63));
    const int64_t chunk_ntok = a ? w.n1 : w.n0;

    // 3. action codes per token (local token index within the chunk): one per set bit
    //    of the token-start mask; a corrupted token's salt bit is its next draw's
    {
      const uint32_t x = a ? excl.e1 : excl.e0;
      const uint32_t cs = corrupted_starts(c, x);
      uint32_t starts = ~((cs << 1) | x);
      const uint32_t salt_next = (s >> 1) | (s_next << 31);  // bit b = salt bit of draw b + 1
      int t = (int)(a ? excl.n1 : excl.n0);
      const int64_t lim = p.n - chunk_tok0;  // tokens at local index >= lim are past the image
      const uint32_t ncorr = __popc(cs);
      if (t + __popc(starts) <= lim) {
        corrupted += ncorr;
      } else {
        // the image ends inside this word: count corrupted tokens below lim only
        uint32_t m = starts;
        for (int tt = t; m; ++tt) {
          const int b = __ffs(m) - 1;
          m &= m - 1u;
          if (tt < lim && ((cs >> b) & 1u)) ++corrupted;
        }
      }
      // code of the token starting at draw b: 0 keep, 1 pepper, 2 salt (cs bit * (1 + salt bit))
      const uint32_t code_lo = cs & ~salt_next, code_hi = cs & salt_next;  // code 1 / code 2
#pragma unroll
      for (int b = 0; b < WORD; ++b) {
        if ((starts >> b) & 1u) s_code[t] = (uint8_t)(((code_lo >> b) & 1u) | (((code_hi >> b) & 1u) << 1));
        t += (starts >> b) & 1u;
      }
    }
    __syncthreads();
    // emit pixels [tok0, tok1) of the image: 16-byte aligned body, scalar head / tail
    const int64_t tok0 = chunk_tok0, tok1 = min(chunk_tok0 + chunk_ntok, p.n);
    if (tok0 < tok1) {
      int64_t body0 = min(tok1, (tok0 + 15) & ~(int64_t)15), body1 = max(body0, tok1 & ~(int64_t)15);
      if (!p.vec) body0 = body1 = tok1;
      auto emit1 = [&](int64_t i) {
        const uint32_t code = s_code[i - tok0];
        p.out[i] = code ? (code == 2u ? (uint8_t)255 : (uint8_t)0) : p.in[i];
        if (p.flags) p.flags[i] = (uint8_t)(code != 0u);
      };
      for (int64_t i = tok0 + tid; i < body0; i += THREADS) emit1(i);
      for (int64_t i = body1 + tid; i < tok1; i += THREADS) emit1(i);
      for (int64_t v = body0 + 16 * (int64_t)tid; v < body1; v += 16 * THREADS) {
        uint4 px = *reinterpret_cast<const uint4*>(p.in + v);
        uint32_t* pw = reinterpret_cast<uint32_t*>(&px);
        uint32_t fw[4];
        const uint8_t* sc = s_code + (v - tok0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o = pw[q], fl = 0u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t code = sc[4 * q + j];
            if (code) {
              o = (o & ~(0xFFu << (8 * j))) | ((code == 2u ? 0xFFu : 0u) << (8 * j));
              fl |= 1u << (8 * j);
            }
          }
          pw[q] = o;
          fw[q] = fl;
        }
        *reinterpret_cast<uint4*>(p.out + v) = px;
        if (p.flags) *reinterpret_cast<uint4*>(p.flags + v) = make_uint4(fw[0], fw[1], fw[2], fw[3]);
      }
    }
    __syncthreads();  // s_code / s_warp / s_look / s_chunk reused by the next chunk
  }
  if (p.count) {
    if (tid == 0) s_cnt = 0ull;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) corrupted += __shfl_xor_sync(0xffffffffu, corrupted, o);
    if (lane == 0 && corrupted) atomicAdd(&s_cnt, (unsigned long long)corrupted);
    __syncthreads();
    if (tid == 0 && s_cnt) atomicAdd(p.count, s_cnt);
  }
}

}  // namespace noise
}  // namespace irdn
