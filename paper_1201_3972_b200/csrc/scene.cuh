// On-device rendering of the seeded BASELINE scenes (second half).
//
// csrc/scene.c defines the scenes. Its per-pixel work is IEEE double
// arithmetic — the blob sum, sensor noise, scaling, hot lines, rectangles, rint, clip —
// plus SplitMix64 counter hashes; only the per-frame parameters need exp / sin / cos.
// The host computes those parameters with scene.c's own code (scene_tables():
// O(nblobs * (W + H)) values per frame) and this kernel does the O(W * H) part with the
// same operations in the same order, each rounded on its own (__dadd_rn / __dmul_rn /
// __dsub_rn: no FMA contraction, matching the host build's -ffp-contract=off and x86-64
// SSE2 doubles). So the device writes exactly scene_generate()'s bytes
// (tests/test_scene_device.py compares every config).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/irdn.h"

namespace irdn {
namespace scene {

enum : uint64_t { ST_SENSOR = 4, ST_IMP = 5, ST_IMPV = 6 };

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double u01(uint64_t h) { return __dmul_rn((double)(h >> 11), 1.0 / 9007199254740992.0); }

constexpr int THREADS = 128;
constexpr int PX = 4;  // consecutive pixels of one row per thread

// grid: x = row segments of THREADS * PX pixels, y = row, z = frame of the call.
template <typename T>
__global__ void __launch_bounds__(THREADS) render_kernel(const irdn_scene_desc d, T* __restrict__ out) {
  const int W = d.width, H = d.height, y = blockIdx.y;
  const int64_t fi = blockIdx.z, f = d.frame0 + fi;
  const int x0 = (blockIdx.x * THREADS + threadIdx.x) * PX;
  if (x0 >= W) return;
  // key(p, f, stream, idx) = sm64(prefix(f, stream) ^ idx)  (scene.c key())
  uint64_t h = sm64(d.seed ^ ((uint64_t)(uint32_t)d.config_id << 56));
  h = sm64(h ^ ((uint64_t)f * 0xD1B54A32D192ED03ull));
  const uint64_t h_sens = sm64(h ^ (ST_SENSOR * 0xABC98388FB8FAC03ull));
  const uint64_t h_imp = sm64(h ^ (ST_IMP * 0xABC98388FB8FAC03ull));
  const uint64_t h_impv = sm64(h ^ (ST_IMPV * 0xABC98388FB8FAC03ull));

  double v[PX];
#pragma unroll
  for (int i = 0; i < PX; ++i) v[i] = 60.0;
  const double* gx = d.gx + (size_t)fi * d.nblobs * W;
  const double* gy = d.gy + (size_t)fi * d.nblobs * H;
  for (int j = 0; j < d.nblobs; ++j) {
    const double g = __ldg(gy + (size_t)j * H + y);
    if (g < 1e-6) continue;
    const double* gr = gx + (size_t)j * W;
#pragma unroll
    for (int i = 0; i < PX; ++i)
      if (x0 + i < W) v[i] = __dadd_rn(v[i], __dmul_rn(g, __ldg(gr + x0 + i)));
  }
  const double* lines = d.lines + (size_t)fi * d.nlines * 5;
  const int32_t* rects = d.rects + (size_t)fi * d.nrects * 4;
  const double yd = (double)y;
  uint32_t q[PX];
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int x = x0 + i;
    const uint64_t idx = (uint64_t)y * (uint64_t)W + (uint64_t)x;
    double val = v[i];
    if (d.sensor) {
      const uint64_t hs = sm64(h_sens ^ idx);
      const double s4 = __dadd_rn(__dadd_rn(__dadd_rn((double)(hs & 0xFFFF), (double)((hs >> 16) & 0xFFFF)),
                                            (double)((hs >> 32) & 0xFFFF)),
                                  (double)(hs >> 48));
      // s4 / 65536.0 is an exact power-of-two scaling: the same double as the host's division
      val = __dadd_rn(val, __dmul_rn(__dsub_rn(__dmul_rn(s4, 1.0 / 65536.0), 2.0), d.sensor_mul));
    }
    val = __dmul_rn(val, d.scale);
    const double xd = (double)x;
    for (int l = 0; l < d.nlines; ++l) {
      const double* L = lines + 5 * l;
      const double dd = __dsub_rn(__dmul_rn(__dsub_rn(xd, __ldg(L + 2)), __ldg(L + 0)),
                                  __dmul_rn(__dsub_rn(yd, __ldg(L + 3)), __ldg(L + 1)));
      if (fabs(dd) < __ldg(L + 4)) val = __dadd_rn(val, d.line_amp);
    }
    for (int k = 0; k < d.nrects; ++k) {
      const int4 rc = __ldg(reinterpret_cast<const int4*>(rects) + k);
      if (x >= rc.x && x < rc.z && y >= rc.y && y < rc.w) val = __dadd_rn(val, d.rect_amp);
    }
    double r = rint(val);
    if (r < 0) r = 0;
    if (r > d.maxval) r = d.maxval;
    uint32_t o = (uint32_t)r;
    if (d.impulse_kind && u01(sm64(h_imp ^ idx)) < d.density) {
      const uint64_t hv = sm64(h_impv ^ idx);
      o = d.impulse_kind == 1 ? ((hv >> 63) ? (uint32_t)d.maxval : 0u) : (uint32_t)(hv % (uint64_t)(d.maxval + 1));
    }
    q[i] = o;
  }
  T* row = out + (size_t)fi * W * H + (size_t)y * W + x0;
  if (x0 + PX <= W && (reinterpret_cast<uintptr_t>(row) % (PX * sizeof(T))) == 0) {
    if constexpr (sizeof(T) == 1) {
      *reinterpret_cast<uint32_t*>(row) = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
    } else {
      *reinterpret_cast<uint2*>(row) = make_uint2(q[0] | (q[1] << 16), q[2] | (q[3] << 16));
    }
  } else {
#pragma unroll
    for (int i = 0; i < PX; ++i)
      if (x0 + i < W) row[i] = (T)q[i];
  }
}

inline int render(const irdn_scene_desc* d, void* d_out, cudaStream_t s, cudaError_t* err) {
  if (!d || !d_out || d->width < 1 || d->height < 1 || d->height > 65535 || d->nframes < 0 || d->nframes > 65535 ||
      (d->bytes_per_pixel != 1 && d->bytes_per_pixel != 2) || d->nblobs < 0 || d->nlines < 0 || d->nlines > 64 ||
      d->nrects < 0 || d->nrects > 256 || (d->nblobs > 0 && (!d->gx || !d->gy)) || (d->nlines > 0 && !d->lines) ||
      (d->nrects > 0 && (!d->rects || (reinterpret_cast<uintptr_t>(d->rects) & 15))))
    return IRDN_EINVAL;
  if (d->nframes == 0) return IRDN_OK;
  const dim3 grid((unsigned)((d->width + THREADS * PX - 1) / (THREADS * PX)), (unsigned)d->height, (unsigned)d->nframes);
  if (d->bytes_per_pixel == 1)
    render_kernel<uint8_t><<<grid, THREADS, 0, s>>>(*d, static_cast<uint8_t*>(d_out));
  else
    render_kernel<uint16_t><<<grid, THREADS, 0, s>>>(*d, static_cast<uint16_t*>(d_out));
  *err = cudaGetLastError();
  return *err == cudaSuccess ? IRDN_OK : IRDN_ECUDA;
}

}  // namespace scene
}  // namespace irdn
