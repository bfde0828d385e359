// Host half of the sparse result return (format in delta.cuh):
// out = in with the changed pixels of every block expanded from the packed values.
//
// The per-block counts make every block independent, so blocks are split over an
// OpenMP team. On CPUs with AVX-512 VBMI2 each 64-byte vector of output is one load of
// the caller's input, one masked expand-load of the packed values and one store
// (vpexpandw / vpexpandb), i.e. the decode runs at host memory-copy speed; elsewhere it
// is a memcpy plus a loop over the set mask bits.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <immintrin.h>
#include <omp.h>

namespace irdn {
namespace delta_host {

constexpr int64_t BLK = 4096;

// region layout: delta.cuh
static inline int64_t nblocks(int64_t n) { return (n + BLK - 1) / BLK; }
static inline int64_t table_bytes(int64_t n) { return ((nblocks(n) * 4) + 15) & ~int64_t(15); }
static inline int64_t mask_offset(int64_t n) { return 16 + 2 * table_bytes(n); }
static inline int64_t values_offset(int64_t n) { return mask_offset(n) + nblocks(n) * (BLK / 8); }

template <typename T>
static void block_scalar(const T* in, T* out, int64_t m, const uint32_t* mask, const T* vals, uint32_t cnt) {
  memcpy(out, in, (size_t)m * sizeof(T));
  if (!cnt) return;
  const int64_t words = (m + 31) / 32;
  for (int64_t w = 0; w < words; ++w) {
    uint32_t x = mask[w];
    while (x) {
      const int j = __builtin_ctz(x);
      x &= x - 1u;
      out[w * 32 + j] = *vals++;
    }
  }
}

__attribute__((target("avx512f,avx512bw,avx512vbmi2"))) static void block_avx512_u16(
    const uint16_t* in, uint16_t* out, int64_t m, const uint32_t* mask, const uint16_t* vals, uint32_t cnt) {
  if (!cnt) {
    memcpy(out, in, (size_t)m * 2);
    return;
  }
  const int64_t full = m / 32;
  // (streaming stores were measured slower here: c2 1.11 vs 1.00 ms per call)
  for (int64_t w = 0; w < full; ++w) {
    const uint32_t x = mask[w];
    __m512i v = _mm512_loadu_si512(in + 32 * w);
    v = _mm512_mask_expandloadu_epi16(v, (__mmask32)x, vals);
    _mm512_storeu_si512(out + 32 * w, v);
    vals += __builtin_popcount(x);
  }
  if (m > full * 32) block_scalar<uint16_t>(in + full * 32, out + full * 32, m - full * 32, mask + full, vals, 1);
}

__attribute__((target("avx512f,avx512bw,avx512vbmi2"))) static void block_avx512_u8(
    const uint8_t* in, uint8_t* out, int64_t m, const uint32_t* mask, const uint8_t* vals, uint32_t cnt) {
  if (!cnt) {
    memcpy(out, in, (size_t)m);
    return;
  }
  const int64_t full = m / 64;
  for (int64_t w = 0; w < full; ++w) {
    const uint64_t x = (uint64_t)mask[2 * w] | ((uint64_t)mask[2 * w + 1] << 32);
    __m512i v = _mm512_loadu_si512(in + 64 * w);
    v = _mm512_mask_expandloadu_epi8(v, (__mmask64)x, vals);
    _mm512_storeu_si512(out + 64 * w, v);
    vals += __builtin_popcountll(x);
  }
  if (m > full * 64) block_scalar<uint8_t>(in + full * 64, out + full * 64, m - full * 64, mask + 2 * full, vals, 1);
}

static bool has_vbmi2() {
  static const int v = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512vbmi2") && __builtin_cpu_supports("avx512bw") ? 1 : 0;
  }();
  return v != 0;
}

// Decode one chunk region `src` (n pixels) into out[0, n) from in[0, n). Returns the
// bytes of the region that carry data (fixed part + total values).
template <typename T>
static uint64_t decode(const uint8_t* src, const T* in, T* out, int64_t n, int threads, int simd) {
  const int64_t nb = nblocks(n);
  const uint32_t total = reinterpret_cast<const uint32_t*>(src)[0];
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(src + 16);
  const uint32_t* offsets = reinterpret_cast<const uint32_t*>(src + 16 + table_bytes(n));
  const uint32_t* mask = reinterpret_cast<const uint32_t*>(src + mask_offset(n));
  const T* vals = reinterpret_cast<const T*>(src + values_offset(n));
  const bool vec = simd && has_vbmi2();
#pragma omp parallel for schedule(static) num_threads(threads) if (nb > 4)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t p = b * BLK, m = (n - p) < BLK ? (n - p) : BLK;
    const uint32_t c = counts[b];
    const uint32_t* mk = mask + b * (BLK / 32);
    const T* v = vals + (c ? offsets[b] : 0);
    if (vec) {
      if (sizeof(T) == 2)
        block_avx512_u16(reinterpret_cast<const uint16_t*>(in + p), reinterpret_cast<uint16_t*>(out + p), m, mk,
                         reinterpret_cast<const uint16_t*>(v), c);
      else
        block_avx512_u8(reinterpret_cast<const uint8_t*>(in + p), reinterpret_cast<uint8_t*>(out + p), m, mk,
                        reinterpret_cast<const uint8_t*>(v), c);
    } else {
      block_scalar<T>(in + p, out + p, m, mk, v, c);
    }
  }
  return (uint64_t)values_offset(n) + (uint64_t)total * sizeof(T);
}

}  // namespace delta_host
}  // namespace irdn

// Internal entry points for irdn_api.cu (and the exported irdn_delta_decode_* in irdn.h).
uint64_t irdn_delta_decode_host_u8(const uint8_t* src, const uint8_t* in, uint8_t* out, int64_t n, int threads,
                                   int simd) {
  return irdn::delta_host::decode<uint8_t>(src, in, out, n, threads, simd);
}
uint64_t irdn_delta_decode_host_u16(const uint8_t* src, const uint16_t* in, uint16_t* out, int64_t n, int threads,
                                    int simd) {
  return irdn::delta_host::decode<uint16_t>(src, in, out, n, threads, simd);
}
