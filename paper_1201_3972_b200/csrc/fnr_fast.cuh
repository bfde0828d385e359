// Host-side dispatch of the specialised TMA tile kernels (fnr_tile.cuh).
//
// The tile path is taken when the window side has a generated selection
// network (k = 3, 5, 7, 9, 11) and the buffers satisfy TMA's rules (16-byte
// aligned base, row pitch and frame stride multiples of 16 bytes). Anything
// else goes to the generic kernel (fnr_generic.cuh) — still sm_100a code.
#pragma once
#include <cuda.h>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>
#include "fnr_common.cuh"
#include "fnr_tile.cuh"
#include "fnr_k3.cuh"
#include "fnr_warp.cuh"

namespace irdn {
void note_launch();
namespace fast {

static thread_local std::string g_fast_err;
inline const char* last_error() { return g_fast_err.c_str(); }

inline uint64_t window_mask(int32_t) {
  return (1ull << 3) | (1ull << 5) | (1ull << 7) | (1ull << 9) | (1ull << 11);
}

// Launch with programmatic dependent launch (PDL): the next kernel in the stream may be
// scheduled while this one drains its last tiles; every kernel starts with
// griddepcontrol.wait (pdl_wait), so it still observes all memory written by the
// previous kernel before touching global memory — safe for dependent passes.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

// Small cache of encoded tensor maps (the host path and the benchmarks re-launch on the same
// buffers every call; encoding costs a few microseconds of host time per launch).
struct MapKey {
  const void* base;
  int64_t width, rows, batch, pitch, frame_stride;
  int box_w, box_h, bpp, dev;
  bool operator==(const MapKey& o) const {
    return base == o.base && width == o.width && rows == o.rows && batch == o.batch && pitch == o.pitch &&
           frame_stride == o.frame_stride && box_w == o.box_w && box_h == o.box_h && bpp == o.bpp && dev == o.dev;
  }
};
template <typename T>
inline bool make_map_uncached(CUtensorMap* map, const void* base, int64_t width, int64_t rows, int64_t batch,
                              int64_t pitch, int64_t frame_stride, int box_w, int box_h);
template <typename T>
inline bool make_map(CUtensorMap* map, const void* base, int64_t width, int64_t rows, int64_t batch,
                     int64_t pitch, int64_t frame_stride, int box_w, int box_h) {
  constexpr int kEntries = 32;
  static std::mutex mu;
  static MapKey keys[kEntries];
  static CUtensorMap maps[kEntries];
  static int used = 0, next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const MapKey k{base, width, rows, batch, pitch, frame_stride, box_w, box_h, (int)sizeof(T), dev};
  {
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < used; ++i)
      if (keys[i] == k) {
        *map = maps[i];
        return true;
      }
  }
  if (!make_map_uncached<T>(map, base, width, rows, batch, pitch, frame_stride, box_w, box_h)) return false;
  std::lock_guard<std::mutex> lock(mu);
  keys[next] = k;
  maps[next] = *map;
  next = (next + 1) % kEntries;
  if (used < kEntries) ++used;
  return true;
}

template <typename T>
inline bool make_map_uncached(CUtensorMap* map, const void* base, int64_t width, int64_t rows, int64_t batch,
                              int64_t pitch, int64_t frame_stride, int box_w, int box_h) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)width, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)(pitch * (int64_t)sizeof(T)),
                                 (cuuint64_t)(frame_stride * (int64_t)sizeof(T))};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  const CUtensorMapDataType dt = sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  CUresult res = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) return false;
  // Drivers up to 13.1 encode tensors spanning < 128 KiB with descriptor bit 85
  // (word 1, bit 21) set, which faults (cudaErrorIllegalInstruction) on sm_100;
  // clear it, as CUTLASS does for the same driver range.
  int drv = 0;
  if (cudaDriverGetVersion(&drv) == cudaSuccess && drv <= 13010) {
    const int64_t span = ((batch - 1) * frame_stride + (rows - 1) * pitch + width) * (int64_t)sizeof(T);
    if (span < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  }
  return true;
}

// Multiprocessor count of a device (cached: queried once per device).
inline int sm_count(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev] = n;
  }
  return cache[dev];
}

// Tile-scheduler slots ({next tile, finished CTAs}, 128 B apart), one per (device, stream).
// Launches on one stream are ordered (every kernel starts with griddepcontrol.wait, and
// the last CTA of a launch resets its slot to {0, 0} before the grid completes), so a slot
// is never used by two grids at once as long as distinct streams get distinct slots. The
// pool is allocated on first use per device, in relaxed capture mode so that a first call
// made inside a CUDA-graph capture still works. Streams beyond kSchedSlots per device
// share slots round-robin (not expected: one slot per concurrently used stream).
constexpr int kSchedSlots = 256;

// Warp kernel, k = 5 / 7: flagged pixels per 64 x 32 tile above which the tile takes the
// dense median stage (fnr_dense.cuh) instead of the per-pixel queue; MF is always dense.
// The crossover is where the queue's per-pixel network (plus gather) costs as much as
// the dense stage does for the whole tile. IRDN_DENSE_FRAC overrides
// the fraction (A/B experiments; < 0 disables the dense stage, MF included).
template <int K>
inline int dense_min_for() {
  if (K != 5 && K != 7) return -1;
  static const double env = getenv("IRDN_DENSE_FRAC") ? atof(getenv("IRDN_DENSE_FRAC")) : -2.0;
  // measured crossovers (tools/dense_threshold_probe.py, profiles/r02/dense_threshold_probe.jsonl:
  // 64 x 640x512 frames, salt-and-pepper density swept): 5x5 ~20 % flagged, 7x7 ~18 %
  const double frac = env > -2.0 ? env : (K == 7 ? 0.18 : 0.20);
  if (frac < 0.0) return -1;
  return (int)(frac * wk::WW * wk::WHK<K>);
}
inline unsigned int* sched_slot(int dev, cudaStream_t s) {
  struct Entry { int dev; cudaStream_t s; unsigned int slot; };
  static std::mutex mu;
  static unsigned int* pool[64] = {nullptr};
  static unsigned int next[64] = {0};
  static std::vector<Entry> assigned;
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pool[dev]) {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    void* p = nullptr;
    bool ok = cudaMalloc(&p, (size_t)kSchedSlots * 128) == cudaSuccess;
    if (ok) ok = cudaMemset(p, 0, (size_t)kSchedSlots * 128) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (!ok) {
      cudaGetLastError();
      return nullptr;
    }
    pool[dev] = static_cast<unsigned int*>(p);
  }
  for (const Entry& e : assigned)
    if (e.dev == dev && e.s == s) return pool[dev] + e.slot * 32;
  const unsigned int slot = next[dev]++ % kSchedSlots;
  assigned.push_back({dev, s, slot});
  return pool[dev] + slot * 32;
}

#ifdef IRDN_TIMELINE
// Experiments only: per-tile (wait, ready, detected, done, n, warp << 16 | smid) of the last warp-kernel launch.
inline unsigned long long* g_timeline = nullptr;
#endif

// Warp-autonomous kernel (fnr_warp.cuh): 64 x 32 warp tiles, per-warp TMA ring.
template <typename T, int K>
inline int launch_warp(const T* d_in, T* d_out, const PassGeom& g, int method, unsigned long long* counts,
                       cudaStream_t s, bool* taken) {
  using G = wk::Geo<T, K>;
  *taken = false;
  CUtensorMap in_map;
  const int out_rows = g.row_end - g.row_begin;
  if (!make_map<T>(&in_map, d_in, g.width, g.in_rows, g.batch, g.in_pitch, g.in_frame_stride, G::BOXW, G::BOXH))
    return 0;
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaFuncSetAttribute(wk::fnr_warp_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, wk::fnr_warp_kernel<T, K>, wk::THREADS, G::SMEM) !=
            cudaSuccess ||
        n < 1) {
      cudaGetLastError();
      n = 1;
    }
    if (getenv("IRDN_WARP_CTAS")) n = std::min(n, atoi(getenv("IRDN_WARP_CTAS")));  // experiments
    blocks_per_sm = n;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  sms = sm_count(dev);
  unsigned int* sched = sched_slot(dev, s);
  if (!sched) return 0;
  tile::TileParams p;
  p.out = d_out;
  p.out_pitch = g.out_pitch;
  p.out_frame = g.out_frame_stride;
  p.width = g.width;
  p.height = g.height;
  p.in_row0 = g.in_row0;
  p.row_begin = g.row_begin;
  p.row_end = g.row_end;
  p.tiles_x = (g.width + wk::WW - 1) / wk::WW;
  p.tiles_y = (out_rows + G::TH - 1) / G::TH;
  p.batch = g.batch;
  p.method = method;
  p.counts = counts;
  p.sched = sched;
  p.one = 1u;
  p.dense_min = dense_min_for<K>();
  p.tpf_magic = tile::udiv_magic((uint32_t)(p.tiles_x * p.tiles_y));
  p.tx_magic = tile::udiv_magic((uint32_t)p.tiles_x);
  p.debug_buf = nullptr;
#ifdef IRDN_TIMELINE
  if (!g_timeline) cudaMalloc(&g_timeline, 8 << 20);
  cudaMemsetAsync(g_timeline, 0, 8 << 20, s);
  p.debug_buf = g_timeline;
#endif
  const long long ntiles = (long long)p.tiles_x * p.tiles_y * g.batch;
  if (2 * ntiles > 0x7fffffffLL) return 0;
  const long long ctas = std::max<long long>(1, std::min<long long>((ntiles + wk::WARPS - 1) / wk::WARPS,
                                                                    (long long)sms * blocks_per_sm));
  // Tail: the last `split` full tiles are handed out as two half-height tiles each
  // (about one tile per warp; none when the pool is a single wave).
  // (round 1 kept one wave of halves; with the round-2 kernels they cost c2 39.3 vs 37.4 us
  // and are off by default: IRDN_TAIL=1 restores them)
  static const double tail_waves = getenv("IRDN_TAIL") ? atof(getenv("IRDN_TAIL")) : 0.0;
  // (a short pool only: with many tiles per warp the tail is a small share and the
  // halves' extra halo rows cost more than they save - c4: 18 tiles/warp, +2 %)
  long long split = G::TH % 32 == 0 ? (long long)(tail_waves * ctas * wk::WARPS) : 0;
  if (ntiles <= ctas * wk::WARPS || ntiles >= 8LL * ctas * wk::WARPS) split = 0;
  split = std::min(split, ntiles);
  p.full_tiles = (int)(ntiles - split);
  // Static rounds: warp w takes tiles w, w + nwarps, ... without the scheduler atomic (its
  // round trip stalls the warp before every tile's TMA issue); the rest of the pool is
  // handed out dynamically so the tail stays balanced.
  {
    static const int srounds_env = getenv("IRDN_STATIC_ROUNDS") ? atoi(getenv("IRDN_STATIC_ROUNDS")) : -1;
    const long long nwarps = ctas * wk::WARPS;
    long long sr = srounds_env >= 0 ? srounds_env : 2;  // measured: 2 rounds c2 37.36 -> 37.27 us (3: 38.6)
    p.static_rounds = (int)std::max<long long>(0, std::min<long long>(sr, ntiles / nwarps));
    if (srounds_env < 0 && p.static_rounds == 0) p.static_rounds = 1;  // a short pool: one static round
  }
  *taken = true;
  cudaError_t e = launch_pdl(wk::fnr_warp_kernel<T, K>, dim3((unsigned)ctas), dim3(wk::THREADS), G::SMEM, s, in_map, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_fast_err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// Completion flags of the multi-pass kernel: one grow-only buffer per (device, stream).
// Word 0 is the stream's launch epoch: a launch reads it after griddepcontrol.wait (the
// previous launch on the stream has completed), tags its flags with epoch + 1 and its last
// warp stores epoch + 1 back, so stale flags never match — also across CUDA-graph
// replays, whose kernel parameters are frozen. Distinct streams never share a buffer.
constexpr size_t kMpFlagsOff = 32;  // tile flags start one 128-byte line after the epoch
inline unsigned int* mp_flags(int dev, cudaStream_t s, size_t words) {
  struct Entry { int dev; cudaStream_t s; unsigned int* p; size_t cap; };
  static std::mutex mu;
  static std::vector<Entry> pool;
  std::lock_guard<std::mutex> lock(mu);
  Entry* e = nullptr;
  for (Entry& x : pool)
    if (x.dev == dev && x.s == s) e = &x;
  if (!e) {
    pool.push_back({dev, s, nullptr, 0});
    e = &pool.back();
  }
  words += kMpFlagsOff;
  if (e->cap < words) {
    // a larger buffer for this stream: free the old one once the stream has drained it
    if (e->p) {
      cudaStreamSynchronize(s);
      cudaFree(e->p);
    }
    e->p = nullptr;
    e->cap = 0;
    void* q = nullptr;
    if (cudaMalloc(&q, words * sizeof(unsigned int)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    cudaMemset(q, 0, words * sizeof(unsigned int));
    cudaDeviceSynchronize();
    e->p = static_cast<unsigned int*>(q);
    e->cap = words;
  }
  return e->p;
}

// All `passes` passes of run_filter in one persistent launch of the warp kernel
// (fnr_warp_mp_kernel); d_tmp has the geometry of d_out.
template <typename T, int K>
inline int launch_warp_mp(const T* d_in, T* d_out, T* d_tmp, const PassGeom& g, int method, int passes,
                          unsigned long long* counts, cudaStream_t s, bool* taken) {
  using G = wk::Geo<T, K>;
  *taken = false;
  CUtensorMap maps[3];
  if (!make_map<T>(&maps[0], d_in, g.width, g.in_rows, g.batch, g.in_pitch, g.in_frame_stride, G::BOXW, G::BOXH) ||
      !make_map<T>(&maps[1], d_tmp, g.width, g.in_rows, g.batch, g.out_pitch, g.out_frame_stride, G::BOXW,
                   G::BOXH) ||
      !make_map<T>(&maps[2], d_out, g.width, g.in_rows, g.batch, g.out_pitch, g.out_frame_stride, G::BOXW,
                   G::BOXH))
    return 0;
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaFuncSetAttribute(wk::fnr_warp_mp_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, wk::fnr_warp_mp_kernel<T, K>, wk::THREADS, G::SMEM) !=
            cudaSuccess ||
        n < 1) {
      cudaGetLastError();
      n = 1;
    }
    blocks_per_sm = n;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  sms = sm_count(dev);
  unsigned int* sched = sched_slot(dev, s);
  if (!sched) return 0;
  tile::TileParams p;
  p.out = d_out;
  p.out_pitch = g.out_pitch;
  p.out_frame = g.out_frame_stride;
  p.width = g.width;
  p.height = g.height;
  p.in_row0 = g.in_row0;
  p.row_begin = g.row_begin;
  p.row_end = g.row_end;
  p.tiles_x = (g.width + wk::WW - 1) / wk::WW;
  p.tiles_y = (g.row_end - g.row_begin + G::TH - 1) / G::TH;
  p.batch = g.batch;
  p.method = method;
  p.counts = counts;
  p.sched = sched;
  p.one = 1u;
  p.dense_min = dense_min_for<K>();
  p.tpf_magic = tile::udiv_magic((uint32_t)(p.tiles_x * p.tiles_y));
  p.tx_magic = tile::udiv_magic((uint32_t)p.tiles_x);
  p.debug_buf = nullptr;
  p.passes = passes;
  p.tmp = d_tmp;
  const long long npass = (long long)p.tiles_x * p.tiles_y * g.batch;
  if ((long long)passes * npass + npass > 0x7fffffffLL) return 0;
  p.flags = mp_flags(dev, s, (size_t)(passes - 1) * (size_t)npass);
  if (!p.flags) return 0;
  p.epoch = 0;  // read on the device
  const long long ctas = std::max<long long>(1, std::min<long long>((npass + wk::WARPS - 1) / wk::WARPS,
                                                                    (long long)sms * blocks_per_sm));
  const long long nwarps = ctas * wk::WARPS;
  long long split = G::TH % 32 == 0 ? nwarps : 0;  // half-height tail: about one tile per warp
  if ((long long)passes * npass <= nwarps || (long long)passes * npass >= 8LL * nwarps) split = 0;
  split = std::min(split, npass);
  p.full_tiles = (int)(npass - split);
  // Every tile is handed out dynamically: a tile is then always owned by a running warp,
  // and a warp only waits on tiles of the previous pass, all handed out before its own,
  // so the launch makes progress even when another grid holds part of the GPU (a static
  // first tile could belong to a CTA that is not resident yet).
  p.static_rounds = 0;
  *taken = true;
  cudaError_t e = launch_pdl(wk::fnr_warp_mp_kernel<T, K>, dim3((unsigned)ctas), dim3(wk::THREADS), G::SMEM, s,
                             maps[0], maps[1], maps[2], p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_fast_err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

// Multi-pass launch for the warp-kernel family (u16: k = 3..11; u8: k = 5..11), whole
// frames only; false when the layout or k does not qualify (the caller then runs the
// passes as separate launches). Opt-in (irdn_set_multipass / IRDN_MULTIPASS=1): measured
// slower than back-to-back single-pass launches on B200.
template <typename T>
inline bool try_launch_mp(const T* d_in, T* d_out, T* d_tmp, const PassGeom& g, int k, int method, int passes,
                          unsigned long long* counts, cudaStream_t s, int* rc) {
  if (passes < 2) return false;
  const size_t bpp = sizeof(T);
  if (((uintptr_t)d_in & 15) || ((uintptr_t)d_out & 15) || ((uintptr_t)d_tmp & 15)) return false;
  if ((g.in_pitch * bpp) % 16 || (g.out_pitch * bpp) % 16) return false;
  if ((g.in_frame_stride * bpp) % 16 || (g.out_frame_stride * bpp) % 16) return false;
  if (g.width < 16 || g.height < 1 || g.row_begin != 0 || g.row_end != g.height || g.in_rows != g.height) return false;
  bool taken = false;
  int e = 0;
  switch (k) {
    case 3:
      if constexpr (sizeof(T) == 2) e = launch_warp_mp<T, 3>(d_in, d_out, d_tmp, g, method, passes, counts, s, &taken);
      else return false;
      break;
    case 5: e = launch_warp_mp<T, 5>(d_in, d_out, d_tmp, g, method, passes, counts, s, &taken); break;
    case 7: e = launch_warp_mp<T, 7>(d_in, d_out, d_tmp, g, method, passes, counts, s, &taken); break;
    case 9: e = launch_warp_mp<T, 9>(d_in, d_out, d_tmp, g, method, passes, counts, s, &taken); break;
    case 11: e = launch_warp_mp<T, 11>(d_in, d_out, d_tmp, g, method, passes, counts, s, &taken); break;
    default: return false;
  }
  if (!taken) return false;
  *rc = e ? 2 : 0;
  return true;
}

template <int BAND, bool FULL, bool FNR>
inline int launch_k3_kern(const uint8_t* d_in, uint8_t* d_out, const PassGeom& g, int method,
                          unsigned long long* counts, cudaStream_t s, bool* taken) {
  using G = k3::Geo<BAND>;
  *taken = false;
  CUtensorMap in_map;
  const int out_rows = g.row_end - g.row_begin;
  if (!make_map<uint8_t>(&in_map, d_in, g.width, g.in_rows, g.batch, g.in_pitch, g.in_frame_stride, G::BOXW,
                         G::BOXH))
    return 0;
  auto kern = k3::fnr_k3_kernel<BAND, FULL, FNR>;
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, k3::THREADS, G::SMEM) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 1;
    }
    blocks_per_sm = n;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  sms = sm_count(dev);
  unsigned int* sched = sched_slot(dev, s);
  if (!sched) return 0;
  tile::TileParams p = {};
  p.out = d_out;
  p.out_pitch = g.out_pitch;
  p.out_frame = g.out_frame_stride;
  p.width = g.width;
  p.height = g.height;
  p.in_row0 = g.in_row0;
  p.row_begin = g.row_begin;
  p.row_end = g.row_end;
  p.tiles_x = (g.width + k3::TW - 1) / k3::TW;
  p.tiles_y = (out_rows + G::TH - 1) / G::TH;
  p.batch = g.batch;
  p.method = method;
  p.counts = counts;
  p.sched = sched;
  p.one = 1u;
  p.dense_min = -1;
  p.tpf_magic = tile::udiv_magic((uint32_t)(p.tiles_x * p.tiles_y));
  p.tx_magic = tile::udiv_magic((uint32_t)p.tiles_x);
  const long long ntiles = (long long)p.tiles_x * p.tiles_y * g.batch;
  if (ntiles > 0x7fffffffLL) return 0;
  dim3 grid((unsigned)std::min<long long>(ntiles, (long long)sms * blocks_per_sm));
  *taken = true;
  cudaError_t e = launch_pdl(kern, grid, dim3(k3::THREADS), G::SMEM, s, in_map, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_fast_err = cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

template <int BAND>
inline int launch_k3_band(const uint8_t* d_in, uint8_t* d_out, const PassGeom& g, int method,
                          unsigned long long* counts, cudaStream_t s, bool* taken) {
  const bool full = g.width % k3::TW == 0 && (g.row_end - g.row_begin) % k3::Geo<BAND>::TH == 0;
  if (full)
    return method == 0 ? launch_k3_kern<BAND, true, true>(d_in, d_out, g, method, counts, s, taken)
                       : launch_k3_kern<BAND, true, false>(d_in, d_out, g, method, counts, s, taken);
  return method == 0 ? launch_k3_kern<BAND, false, true>(d_in, d_out, g, method, counts, s, taken)
                     : launch_k3_kern<BAND, false, false>(d_in, d_out, g, method, counts, s, taken);
}

// Dense 3x3 kernel for u8 frames (fnr_k3.cuh). Tile height 160 / 128 / 96 / 64 / 32 rows:
// the tallest one that divides the rows (then no tile needs validity masks) while leaving
// at least two tiles per SM; else 128-row tiles (masked last row of tiles) for large jobs
// and 32-row tiles for small ones (BASELINE c1: 64 tiles of 128 x 32).
inline int launch_k3(const uint8_t* d_in, uint8_t* d_out, const PassGeom& g, int method,
                     unsigned long long* counts, cudaStream_t s, bool* taken) {
  const long long rows = g.row_end - g.row_begin;
  const long long tx = (g.width + k3::TW - 1) / k3::TW;
  auto tiles = [&](int th) { return tx * ((rows + th - 1) / th) * g.batch; };
  const long long enough = 2LL * 148;
#ifdef IRDN_K3_BAND
  return launch_k3_band<IRDN_K3_BAND>(d_in, d_out, g, method, counts, s, taken);
#endif
  if (rows % 160 == 0 && tiles(160) >= enough) return launch_k3_band<10>(d_in, d_out, g, method, counts, s, taken);
  if (rows % 128 == 0 && tiles(128) >= enough) return launch_k3_band<8>(d_in, d_out, g, method, counts, s, taken);
  if (rows % 96 == 0 && tiles(96) >= enough) return launch_k3_band<6>(d_in, d_out, g, method, counts, s, taken);
  if (rows % 64 == 0 && tiles(64) >= enough) return launch_k3_band<4>(d_in, d_out, g, method, counts, s, taken);
  if (tiles(128) >= 4 * enough) return launch_k3_band<8>(d_in, d_out, g, method, counts, s, taken);
  return launch_k3_band<2>(d_in, d_out, g, method, counts, s, taken);
}

template <typename T>
inline bool try_launch(const T* d_in, T* d_out, const PassGeom& g, int k, int method, unsigned long long* counts,
                       cudaStream_t s, int* rc) {
  const size_t bpp = sizeof(T);
  if (((uintptr_t)d_in & 15) || ((uintptr_t)d_out & 15)) return false;
  if ((g.in_pitch * bpp) % 16 || (g.out_pitch * bpp) % 16) return false;
  if ((g.in_frame_stride * bpp) % 16 || (g.out_frame_stride * bpp) % 16) return false;
  if (g.width < 16 || g.height < 1) return false;
  bool taken = false;
  int e = 0;
#define IRDN_LAUNCH_K(KK) launch_warp<T, KK>(d_in, d_out, g, method, counts, s, &taken)
  switch (k) {
    case 3:
      if constexpr (sizeof(T) == 1) e = launch_k3(d_in, d_out, g, method, counts, s, &taken);
      else e = IRDN_LAUNCH_K(3);
      break;
    case 5: e = IRDN_LAUNCH_K(5); break;
    case 7: e = IRDN_LAUNCH_K(7); break;
    case 9: e = IRDN_LAUNCH_K(9); break;
    case 11: e = IRDN_LAUNCH_K(11); break;
    default: return false;
  }
#undef IRDN_LAUNCH_K
  if (!taken) return false;
  *rc = e ? 2 : 0;
  return true;
}

}  // namespace fast
}  // namespace irdn
