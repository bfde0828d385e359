// C-ABI of the B200 FNR filter (declared in include/irdn.h).
//
// Host-side mirror of the reference driver (pkg/src/irdenoise/filters.py):
//   run_filter        filters.py:79-102   -> irdn_run_filter_{u8,u16} (host buffers)
//                                            irdn_run_filter_device_{u8,u16} (device buffers)
//   fnr_pass/mf_pass  filters.py:69-76    -> irdn_filter_pass_{u8,u16}
//   _filter_rows(y0,y1) filters.py:130    -> irdn_filter_strip_{u8,u16}
// There is no CPU fallback anywhere in this file: every compute entry point
// launches sm_100a kernels or fails with IRDN_ENODEV / IRDN_ECUDA.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <omp.h>
#include <sched.h>
#include <string>
#include <vector>

#include "../../include/irdn.h"
#include "fnr_common.cuh"
#include "fnr_generic.cuh"
#include "fnr_fast.cuh"
#include "metrics.cuh"
#include "noise.cuh"
#include "scene.cuh"
#include "delta.cuh"
#include "fnr_large.cuh"

// delta_host.cpp (host decode of the sparse result return, compiled by the host compiler)
uint64_t irdn_delta_decode_host_u8(const uint8_t* src, const uint8_t* in, uint8_t* out, int64_t n, int threads,
                                   int simd);
uint64_t irdn_delta_decode_host_u16(const uint8_t* src, const uint16_t* in, uint16_t* out, int64_t n, int threads,
                                    int simd);

namespace irdn {

static thread_local std::string g_err;
static thread_local uint64_t g_launches = 0;
static thread_local uint64_t g_xfer_h2d = 0, g_xfer_d2h = 0;  // bytes moved by the last irdn_run_filter_* call
static int32_t g_force_generic = 0;
// passes > 1 in one multi-pass launch (fnr_warp_mp_kernel); off by default
static int32_t g_multipass = getenv("IRDN_MULTIPASS") ? (atoi(getenv("IRDN_MULTIPASS")) != 0) : 0;
// Host-buffer result return: 0 = auto (sparse for FNR on u16, else the full copy), 1 = full copy,
// 2 = sparse (delta.cuh). IRDN_HOST_RETURN=full|delta|auto sets the initial value.
static int32_t g_host_return = [] {
  const char* e = getenv("IRDN_HOST_RETURN");
  if (!e) return 0;
  return e[0] == 'f' ? 1 : e[0] == 'd' ? 2 : 0;
}();

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define IRDN_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(IRDN_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),        \
                  __FILE__, __LINE__);                                                       \
  } while (0)

void note_launch() { ++g_launches; }

// Cached per-device check: only compute capability 10.x runs the sm_100a code.
static int check_device(int* dev_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(IRDN_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  static int cc_major[64] = {0};
  if (dev < 64 && cc_major[dev] == 0) {
    int major = -1;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return fail(IRDN_ENODEV, "device query failed: %s", cudaGetErrorString(e));
    cc_major[dev] = major;
  }
  if (dev >= 64 || cc_major[dev] != 10)
    return fail(IRDN_ENODEV, "device %d is not an sm_100 (B200) device", dev);
  if (dev_out) *dev_out = dev;
  return IRDN_OK;
}

// Validation mirroring the reference's ValueErrors.
static int validate(int64_t batch, int64_t height, int64_t width, int32_t k, int32_t method) {
  if (method != IRDN_METHOD_FNR && method != IRDN_METHOD_MF)  // filters.py:90-91
    return fail(IRDN_EINVAL, "unknown method %d, expected 'fnr' or 'mf'", method);
  if (k < 3 || k % 2 == 0)  // image.py:63-65
    return fail(IRDN_EINVAL, "window side must be an odd integer >= 3, got %d", k);
  if (width < 1 || height < 1)  // image.py:30-31
    return fail(IRDN_EINVAL, "image dimensions must be >= 1, got %lldx%lld", (long long)width,
                (long long)height);
  if (batch < 1) return fail(IRDN_EINVAL, "batch must be >= 1, got %lld", (long long)batch);
  if (height > INT32_MAX / 2 || width > INT32_MAX / 2 || k > 4095)
    return fail(IRDN_EINVAL, "frame %lldx%lld or window %d too large", (long long)width,
                (long long)height, k);
  return IRDN_OK;
}

static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

template <typename T>
static int launch_pass(const T* d_in, T* d_out, const PassGeom& g, int k, int method,
                       unsigned long long* d_counts, cudaStream_t s) {
  if (!g_force_generic) {
    int rc = -1;
    if (fast::try_launch<T>(d_in, d_out, g, k, method, d_counts, s, &rc)) {
      if (rc != IRDN_OK) return fail(IRDN_ECUDA, "fast kernel launch failed: %s", fast::last_error());
      note_launch();
      return IRDN_OK;
    }
  }
  const int rows = g.row_end - g.row_begin;
  if (!g_force_generic && k / 2 <= large::LMAX_R) {
    // shared-memory tiled kernel: k >= 13, or layouts the TMA kernels cannot take
    const long long tiles = (long long)((g.width + large::TW - 1) / large::TW) * ((rows + large::TH - 1) / large::TH);
    if (tiles <= 0x7fffffffLL) {
      // median search with the window in registers: up to V elements per lane (k^2 <= 32 V)
      const int kk = k * k;
      auto kern = kk <= 32 * 8 ? large::fnr_large_kernel<T, 8>
                  : kk <= 32 * 16 ? large::fnr_large_kernel<T, 16>
                  : kk <= 32 * 32 ? large::fnr_large_kernel<T, 32> : large::fnr_large_kernel<T, 0>;
      const size_t smem = sizeof(large::Smem<T>);
      IRDN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<dim3((unsigned)tiles, (unsigned)std::min<int>(g.batch, 65535)), large::THREADS, smem, s>>>(
          d_in, d_out, g, k, method, d_counts);
      IRDN_CUDA(cudaGetLastError());
      note_launch();
      return IRDN_OK;
    }
  }
  dim3 grid((g.width + 31) / 32, (rows + 7) / 8, std::min<int>(g.batch, 65535));
  if (grid.y > 65535u) return fail(IRDN_EINVAL, "frame too tall for the generic kernel");
  fnr_generic_kernel<T><<<grid, 256, 0, s>>>(d_in, d_out, g, k, method, d_counts);
  IRDN_CUDA(cudaGetLastError());
  note_launch();
  return IRDN_OK;
}

template <typename T>
static int filter_pass(const T* d_in, T* d_out, int64_t batch, int64_t height, int64_t width,
                       int64_t in_pitch, int64_t out_pitch, int32_t k, int32_t method,
                       unsigned long long* d_counts, void* stream) {
  int rc = validate(batch, height, width, k, method);
  if (rc) return rc;
  if (!d_in || !d_out) return fail(IRDN_EINVAL, "null buffer");
  if (in_pitch < width || out_pitch < width) return fail(IRDN_EINVAL, "pitch smaller than width");
  if (method == IRDN_METHOD_FNR && !d_counts) return fail(IRDN_EINVAL, "FNR needs d_counts[2]");
  const size_t in_bytes = (size_t)((batch - 1) * height * in_pitch + (height - 1) * in_pitch + width) * sizeof(T);
  const size_t out_bytes = (size_t)((batch - 1) * height * out_pitch + (height - 1) * out_pitch + width) * sizeof(T);
  if (overlaps(d_in, in_bytes, d_out, out_bytes))
    return fail(IRDN_EINVAL, "input and output buffers overlap (a pass never sees its own writes)");
  if ((rc = check_device(nullptr))) return rc;
  PassGeom g;
  g.in_frame_stride = height * in_pitch;
  g.out_frame_stride = height * out_pitch;
  g.in_pitch = in_pitch;
  g.out_pitch = out_pitch;
  g.height = (int32_t)height;
  g.width = (int32_t)width;
  g.in_row0 = 0;
  g.in_rows = (int32_t)height;
  g.row_begin = 0;
  g.row_end = (int32_t)height;
  g.batch = (int32_t)batch;
  return launch_pass<T>(d_in, d_out, g, k, method, d_counts, (cudaStream_t)stream);
}

template <typename T>
static int filter_strip(const T* d_in, int64_t in_row0, int64_t in_rows, T* d_out,
                        int64_t row_begin, int64_t row_end, int64_t height, int64_t width,
                        int64_t in_pitch, int64_t out_pitch, int32_t k, int32_t method,
                        unsigned long long* d_counts, void* stream) {
  int rc = validate(1, height, width, k, method);
  if (rc) return rc;
  if (!d_in || !d_out) return fail(IRDN_EINVAL, "null buffer");
  if (in_pitch < width || out_pitch < width) return fail(IRDN_EINVAL, "pitch smaller than width");
  if (method == IRDN_METHOD_FNR && !d_counts) return fail(IRDN_EINVAL, "FNR needs d_counts[2]");
  if (row_begin < 0 || row_end > height || row_begin >= row_end)
    return fail(IRDN_EINVAL, "bad output row range [%lld, %lld) for height %lld",
                (long long)row_begin, (long long)row_end, (long long)height);
  const int64_t r = k / 2;
  const int64_t need0 = std::max<int64_t>(0, row_begin - r);
  const int64_t need1 = std::min<int64_t>(height, row_end + r);
  if (in_row0 > need0 || in_row0 + in_rows < need1 || in_row0 < 0 || in_row0 + in_rows > height)
    return fail(IRDN_EINVAL,
                "input strip rows [%lld, %lld) do not cover the clamped window rows [%lld, %lld)",
                (long long)in_row0, (long long)(in_row0 + in_rows), (long long)need0, (long long)need1);
  if ((rc = check_device(nullptr))) return rc;
  PassGeom g;
  g.in_frame_stride = in_rows * in_pitch;
  g.out_frame_stride = (row_end - row_begin) * out_pitch;
  g.in_pitch = in_pitch;
  g.out_pitch = out_pitch;
  g.height = (int32_t)height;
  g.width = (int32_t)width;
  g.in_row0 = (int32_t)in_row0;
  g.in_rows = (int32_t)in_rows;
  g.row_begin = (int32_t)row_begin;
  g.row_end = (int32_t)row_end;
  g.batch = 1;
  return launch_pass<T>(d_in, d_out, g, k, method, d_counts, (cudaStream_t)stream);
}

// passes > 1: pass i reads pass i-1's output (filters.py:96-100). Buffers are
// chosen so the LAST pass lands in d_out.
template <typename T>
static int run_device(const T* d_in, T* d_out, T* d_tmp, int64_t batch, int64_t height,
                      int64_t width, int32_t k, int32_t method, int32_t passes,
                      unsigned long long* d_counts, void* stream, int64_t pitch = 0) {
  if (pitch <= 0) pitch = width;
  if (passes < 1) return fail(IRDN_EINVAL, "passes must be >= 1, got %d", passes);  // filters.py:92-93
  if (passes > 1 && !d_tmp) return fail(IRDN_EINVAL, "passes > 1 needs a d_tmp buffer");
  if (passes > 1 && !g_force_generic && g_multipass) {
    // all passes in one persistent launch of the warp kernel (tile-level pass dependencies)
    int rc = validate(batch, height, width, k, method);
    if (rc) return rc;
    if (!d_in || !d_out) return fail(IRDN_EINVAL, "null buffer");
    if (method == IRDN_METHOD_FNR && !d_counts) return fail(IRDN_EINVAL, "FNR needs d_counts[2]");
    const size_t bytes = (size_t)(batch * height * pitch) * sizeof(T);
    if (overlaps(d_in, bytes, d_out, bytes) || overlaps(d_in, bytes, d_tmp, bytes) ||
        overlaps(d_out, bytes, d_tmp, bytes))
      return fail(IRDN_EINVAL, "input, output and scratch buffers overlap");
    if ((rc = check_device(nullptr))) return rc;
    PassGeom g;
    g.in_frame_stride = height * pitch;
    g.out_frame_stride = height * pitch;
    g.in_pitch = pitch;
    g.out_pitch = pitch;
    g.height = (int32_t)height;
    g.width = (int32_t)width;
    g.in_row0 = 0;
    g.in_rows = (int32_t)height;
    g.row_begin = 0;
    g.row_end = (int32_t)height;
    g.batch = (int32_t)batch;
    int lrc = 0;
    if (fast::try_launch_mp<T>(d_in, d_out, d_tmp, g, k, method, passes, d_counts, (cudaStream_t)stream, &lrc)) {
      if (lrc != IRDN_OK) return fail(IRDN_ECUDA, "multi-pass kernel launch failed: %s", fast::last_error());
      note_launch();
      return IRDN_OK;
    }
  }
  const T* src = d_in;
  for (int p = 0; p < passes; ++p) {
    T* dst = ((passes - 1 - p) % 2 == 0) ? d_out : d_tmp;
    int rc = filter_pass<T>(src, dst, batch, height, width, pitch, pitch, k, method, d_counts, stream);
    if (rc) return rc;
    src = dst;
  }
  return IRDN_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer run_filter with copy/compute pipelining.
//
// The batch is cut into ~8 MB chunks of whole frames (row strips for one large frame).
// Per chunk: H2D on s_h2d (from pinned staging slots when the caller's buffer is
// pageable), the passes on s_comp once its H2D event fires, then the result back on s_d2h:
// either a full D2H copy, or — FNR on 16-bit frames — the sparse return (delta.cuh:
// encode + one DMA of counts, masks and a value budget; the host rebuilds the chunk from
// its own input, delta_host.cpp), with the last chunk split between the two. The
// counters come back last (FilterStats accounting: filters.py:121-126).
// ---------------------------------------------------------------------------
// Rows of row_bytes from src (pitch spitch bytes) to dst (pitch dpitch bytes): the host
// path's padding of unaligned rows to the TMA kernels' 16-byte pitch and back. A DMA
// engine moves 364-byte rows at ~4 GB/s (2-D cudaMemcpy, measured), this at HBM speed.
__global__ void copy_rows_kernel(const uint8_t* __restrict__ src, int64_t spitch, uint8_t* __restrict__ dst,
                                 int64_t dpitch, int64_t row_bytes, int64_t rows) {
  const bool w4 = ((row_bytes | spitch | dpitch | (int64_t)(uintptr_t)src | (int64_t)(uintptr_t)dst) & 3) == 0;
  const int64_t n = w4 ? row_bytes / 4 : row_bytes;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    if (w4) reinterpret_cast<uint32_t*>(dst + r * dpitch)[c] = reinterpret_cast<const uint32_t*>(src + r * spitch)[c];
    else dst[r * dpitch + c] = src[r * spitch + c];
  }
}
static void copy_rows(const void* src, int64_t spitch, void* dst, int64_t dpitch, int64_t row_bytes, int64_t rows,
                      cudaStream_t st) {
  const bool w4 = ((row_bytes | spitch | dpitch | (int64_t)(uintptr_t)src | (int64_t)(uintptr_t)dst) & 3) == 0;
  const int64_t n = w4 ? row_bytes / 4 : row_bytes;
  const dim3 grid((unsigned)((n + 255) / 256), (unsigned)std::min<int64_t>(rows, 16384));
  copy_rows_kernel<<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(src), spitch, static_cast<uint8_t*>(dst), dpitch,
                                         row_bytes, rows);
}

struct DeviceWorkspace {
  std::mutex mu;
  void* buf = nullptr;  // [in | out | tmp] regions
  size_t cap = 0;
  unsigned long long* counts = nullptr;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done;  // grow-only pools (created once, reused per call)
  // pageable host buffers: pinned staging slots (in / out), CPU copies run in parallel
  // (OpenMP) while the DMA engines move the neighbouring chunks
  void* stage_in = nullptr;
  void* stage_out = nullptr;
  size_t stage_cap = 0;  // bytes per direction (kStageSlots slots)
  cudaEvent_t ev_out[4] = {nullptr, nullptr, nullptr, nullptr};
  // sparse result return: mapped pinned region the encode kernel writes over PCIe
  uint8_t* delta_h = nullptr;  // pinned host copy of the regions
  uint8_t* delta_d = nullptr;  // device regions (encode target)
  size_t delta_cap = 0;
  double delta_ratio = 0.25;   // changed-pixel fraction the value budget assumes (last call's max)
  bool ready = false;
};
constexpr int kStageSlots = 3;
static DeviceWorkspace g_ws[64];

static int ensure_staging(DeviceWorkspace& ws, size_t slot_bytes) {
  const size_t need = slot_bytes * kStageSlots;
  if (ws.stage_cap < need) {
    if (ws.stage_in) IRDN_CUDA(cudaFreeHost(ws.stage_in));
    if (ws.stage_out) IRDN_CUDA(cudaFreeHost(ws.stage_out));
    ws.stage_in = ws.stage_out = nullptr;
    ws.stage_cap = 0;
    IRDN_CUDA(cudaHostAlloc(&ws.stage_in, need, cudaHostAllocDefault));
    IRDN_CUDA(cudaHostAlloc(&ws.stage_out, need, cudaHostAllocDefault));
    ws.stage_cap = need;
  }
  for (int i = 0; i < kStageSlots; ++i)
    if (!ws.ev_out[i]) IRDN_CUDA(cudaEventCreateWithFlags(&ws.ev_out[i], cudaEventDisableTiming));
  return IRDN_OK;
}

// Host threads for copies and the sparse-return decode: the host's cores shared out between
// the processes on this node (LOCAL_WORLD_SIZE under torchrun, else one per visible GPU),
// capped at 16 (16 threads: 113 GB/s memcpy on the 16-core B200 box vs 90 GB/s with 8,
// tools/microbench/host_probe.cu). Counted from the CPU affinity mask, not from
// OMP_NUM_THREADS (torchrun sets that to 1 per rank); IRDN_COPY_THREADS overrides.
static int copy_threads() {
  static const int nt = [] {
    const char* e = getenv("IRDN_COPY_THREADS");
    if (e) return std::max(1, atoi(e));
    int hw = 0;
    cpu_set_t cs;
    if (sched_getaffinity(0, sizeof(cs), &cs) == 0) hw = CPU_COUNT(&cs);
    if (hw <= 0) hw = std::max(1, omp_get_num_procs());
    int ranks = 0;
    if (const char* l = getenv("LOCAL_WORLD_SIZE")) ranks = atoi(l);
    if (ranks <= 0) {
      if (cudaGetDeviceCount(&ranks) != cudaSuccess || ranks < 1) {
        cudaGetLastError();
        ranks = 1;
      }
    }
    return std::max(1, std::min(16, hw / ranks));
  }();
  return nt;
}

// memcpy split over the OpenMP team (host DRAM bandwidth, not one core, bounds it)
static void par_copy(void* dst, const void* src, size_t n) {
  constexpr size_t kPart = 256 << 10;
  const long long parts = (long long)((n + kPart - 1) / kPart);
  if (parts <= 1) {
    memcpy(dst, src, n);
    return;
  }
  const int nt = copy_threads();
#pragma omp parallel for schedule(static) num_threads(nt)
  for (long long i = 0; i < parts; ++i) {
    const size_t off = (size_t)i * kPart;
    memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(kPart, n - off));
  }
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static int ensure_workspace(DeviceWorkspace& ws, size_t bytes) {
  if (!ws.ready) {
    IRDN_CUDA(cudaStreamCreateWithFlags(&ws.s_h2d, cudaStreamNonBlocking));
    IRDN_CUDA(cudaStreamCreateWithFlags(&ws.s_comp, cudaStreamNonBlocking));
    IRDN_CUDA(cudaStreamCreateWithFlags(&ws.s_d2h, cudaStreamNonBlocking));
    IRDN_CUDA(cudaMalloc(&ws.counts, 2 * sizeof(unsigned long long)));
    ws.ready = true;
  }
  if (ws.cap < bytes) {
    if (ws.buf) IRDN_CUDA(cudaFree(ws.buf));
    ws.buf = nullptr;
    ws.cap = 0;
    IRDN_CUDA(cudaMalloc(&ws.buf, bytes));
    ws.cap = bytes;
  }
  return IRDN_OK;
}

template <typename T>
static int run_host(const T* h_in, T* h_out, int64_t batch, int64_t height, int64_t width,
                    int32_t k, int32_t method, int32_t passes, int32_t device, irdn_stats* stats) {
  auto t0 = std::chrono::steady_clock::now();
  int rc = validate(batch, height, width, k, method);
  if (rc) return rc;
  if (passes < 1) return fail(IRDN_EINVAL, "passes must be >= 1, got %d", passes);
  if (!h_in || !h_out) return fail(IRDN_EINVAL, "null buffer");
  // IRDN_HOST_TRACE: host timestamps per chunk and device event times (experiments only)
  static const bool trace = getenv("IRDN_HOST_TRACE") != nullptr;
  static std::vector<cudaEvent_t> tev;
  auto tmark = [&](size_t idx, cudaStream_t st) {
    if (!trace) return;
    while (tev.size() <= idx) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      tev.push_back(e);
    }
    cudaEventRecord(tev[idx], st);
  };
  const int64_t frame = height * width;
  const size_t nbytes = (size_t)(batch * frame) * sizeof(T);
  if (overlaps(h_in, nbytes, h_out, nbytes)) return fail(IRDN_EINVAL, "input and output buffers overlap");
  if (device < 0 || device >= 64) return fail(IRDN_EINVAL, "bad device %d", device);
  int prev = 0;
  {
    const cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return fail(IRDN_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (prev != device) IRDN_CUDA(cudaSetDevice(device));
  struct Restore {
    int d, p;
    ~Restore() { if (d != p) cudaSetDevice(p); }
  } restore{device, prev};
  if ((rc = check_device(nullptr))) return rc;

  DeviceWorkspace& ws = g_ws[device];
  std::lock_guard<std::mutex> lock(ws.mu);
  // Device rows are padded to a multiple of 16 bytes (pitch dp) when the caller's are not
  // (the reference's own 364-pixel rows): the TMA kernels need 16-byte aligned rows, and a
  // 2-D copy pads them on the way in and strips the padding on the way out.
  const int64_t align = 16 / (int64_t)sizeof(T);
  const int64_t dp = (width % align == 0 || width < 16) ? width : (width + align - 1) / align * align;
  const int64_t dframe = height * dp;
  const size_t dbytes = (size_t)(batch * dframe) * sizeof(T);
  const int nbuf = passes > 1 ? 3 : 2;
  if ((rc = ensure_workspace(ws, dbytes * nbuf + (dp == width ? 0 : 2 * nbytes)))) return rc;
  T* d_in = (T*)ws.buf;
  T* d_out = d_in + batch * dframe;
  T* d_tmp = passes > 1 ? d_out + batch * dframe : nullptr;
  T* lin_in = d_in + nbuf * batch * dframe;  // padded rows only: contiguous landing / leaving zones
  T* lin_out = lin_in + batch * frame;
  IRDN_CUDA(cudaMemsetAsync(ws.counts, 0, 2 * sizeof(unsigned long long), ws.s_comp));

  // Chunking: frames for a batch; row strips for a single frame with one pass.
  const int r = k / 2;
  struct Chunk { int64_t f0, nf, y0, y1; };
  std::vector<Chunk> chunks;
  if (batch >= 2) {
    static const int64_t chunk_bytes = [] {
      const char* e = getenv("IRDN_CHUNK_MB");
      return (int64_t)((e ? atof(e) : 8.0) * (1 << 20));
    }();
    const int64_t target = std::max<int64_t>(1, chunk_bytes / (int64_t)sizeof(T) / frame);  // ~8 MB of frames (measured optimum for c2: tools/pcie_probe.py)
    const int64_t nchunks = std::min<int64_t>(std::max<int64_t>(1, batch / target), 256);
    // (halving chunk sizes towards the end was measured neutral)
    for (int64_t i = 0; i < nchunks; ++i) {
      int64_t a = batch * i / nchunks, b = batch * (i + 1) / nchunks;
      if (b > a) chunks.push_back({a, b - a, 0, height});
    }
  } else if (passes == 1 && height >= 4 * (int64_t)(r + 1) && frame * (int64_t)sizeof(T) >= (16 << 20)) {
    const int64_t nchunks = std::min<int64_t>(16, height / (4 * (r + 1)));
    for (int64_t i = 0; i < nchunks; ++i) {
      int64_t a = height * i / nchunks, b = height * (i + 1) / nchunks;
      chunks.push_back({0, 1, a, b});
    }
  } else {
    chunks.push_back({0, batch, 0, height});
  }

  while (ws.ev_in.size() < chunks.size()) {
    cudaEvent_t a, b;
    IRDN_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    IRDN_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    ws.ev_in.push_back(a);
    ws.ev_done.push_back(b);
  }
  std::vector<cudaEvent_t>& ev_in = ws.ev_in;
  std::vector<cudaEvent_t>& ev_done = ws.ev_done;

  const bool row_mode = batch == 1 && chunks.size() > 1;
  auto chunk_off = [&](const Chunk& c) { return c.f0 * frame + c.y0 * width; };
  auto chunk_cnt = [&](const Chunk& c) { return row_mode ? (c.y1 - c.y0) * width : c.nf * frame; };
  auto dev_off = [&](const Chunk& c) { return c.f0 * dframe + c.y0 * dp; };     // device layout (pitch dp)
  auto chunk_rows = [&](const Chunk& c) { return row_mode ? c.y1 - c.y0 : c.nf * height; };
  // copies between the caller's contiguous rows (host offset hoff) and the device's possibly
  // padded rows: padded ones land contiguous in lin_in and are spread by copy_rows on the
  // same stream (and gathered into lin_out before leaving)
  auto h2d = [&](T* dst, const T* src, int64_t rows, int64_t hoff, cudaStream_t st) {
    const size_t b = (size_t)(rows * width) * sizeof(T);
    if (dp == width) return cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, st);
    cudaError_t e = cudaMemcpyAsync(lin_in + hoff, src, b, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      copy_rows(lin_in + hoff, width * (int64_t)sizeof(T), dst, dp * (int64_t)sizeof(T), width * (int64_t)sizeof(T),
                rows, st);
      e = cudaGetLastError();
    }
    return e;
  };
  auto d2h = [&](T* dst, const T* src, int64_t rows, int64_t hoff, cudaStream_t st) {
    const size_t b = (size_t)(rows * width) * sizeof(T);
    if (dp == width) return cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, st);
    copy_rows(src, dp * (int64_t)sizeof(T), lin_out + hoff, width * (int64_t)sizeof(T), width * (int64_t)sizeof(T),
              rows, st);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst, lin_out + hoff, b, cudaMemcpyDeviceToHost, st);
    return e;
  };
  // Pageable caller buffers: DMA from / to pinned staging slots; the CPU copies chunk
  // i into a slot (parallel memcpy) while the copy engines move chunks i-1 and i-2.
  // Result return: sparse (only the pixels that differ from the input, delta.cuh; the
  // host rebuilds the output from its own input) or the full D2H copy of the output.
  // auto: sparse for FNR on 16-bit frames (c2 1.23-1.27 -> 1.01 ms, c4 4.6 -> 3.3 ms per call,
  // tools/e2e_probe.py); 8-bit frames keep the full copy: rebuilding 1 B/px on the host costs
  // about what the D2H saves (c3 2.06 -> 1.98 ms, but c5 31.8 -> 37.4 ms, c1 0.050 -> 0.067 ms)
  // (and only with >= 6 host threads for the rebuild: ~13 GB/s per thread, the full copy's
  // extra cost over the H2D is ~0.2-0.4 ms per 42 MB)
  // (and only for a pinned input: with a pageable one the host threads are busy staging it,
  // and the full copy wins — pageable c2 1.42-1.46 vs 1.46-1.59 ms, c4 4.12 vs 5.1-5.7 ms)
  const bool in_pinned = is_pinned(h_in);
  const bool use_delta = dp == width &&  // the region encoder reads contiguous rows
                         (g_host_return == 2 || (g_host_return == 0 && method == IRDN_METHOD_FNR &&
                                                 sizeof(T) == 2 && copy_threads() >= 6 && in_pinned));
  // Sparse return: the last chunk is rebuilt on the host after everything else has landed,
  // so its second half comes back by a plain D2H copy into the (pinned) caller buffer
  // instead, while the host rebuilds the first half (IRDN_SPLIT_LAST=0 disables).
  size_t full_chunk = chunks.size();  // index of the chunk returned by a full copy (none)
  {
    static const int split_last = getenv("IRDN_SPLIT_LAST") ? atoi(getenv("IRDN_SPLIT_LAST")) : 1;
    if (use_delta && split_last && chunks.size() >= 2 && is_pinned(h_out)) {
      const Chunk c = chunks.back();
      if (row_mode && c.y1 - c.y0 >= 2) {
        const int64_t m = c.y0 + (c.y1 - c.y0) / 2;
        chunks.back().y1 = m;
        chunks.push_back({0, 1, m, c.y1});
        full_chunk = chunks.size() - 1;
      } else if (!row_mode && c.nf >= 2) {
        const int64_t a = c.nf / 2;
        chunks.back().nf = a;
        chunks.push_back({c.f0 + a, c.nf - a, 0, height});
        full_chunk = chunks.size() - 1;
      }
    }
    while (ws.ev_in.size() < chunks.size()) {
      cudaEvent_t a, b;
      IRDN_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      IRDN_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      ws.ev_in.push_back(a);
      ws.ev_done.push_back(b);
    }
  }
  std::vector<int64_t> delta_off(chunks.size() + 1, 0);
  if (use_delta) {
    for (size_t i = 0; i < chunks.size(); ++i)
      delta_off[i + 1] = delta_off[i] + (i == full_chunk ? 0
                                         : row_mode ? delta::region_bytes<T>((chunks[i].y1 - chunks[i].y0) * width)
                                                    : delta::region_bytes<T>(chunks[i].nf * frame));
    if ((size_t)delta_off.back() > ws.delta_cap) {
      if (ws.delta_h) IRDN_CUDA(cudaFreeHost(ws.delta_h));
      if (ws.delta_d) IRDN_CUDA(cudaFree(ws.delta_d));
      ws.delta_h = nullptr;
      ws.delta_d = nullptr;
      ws.delta_cap = 0;
      IRDN_CUDA(cudaHostAlloc((void**)&ws.delta_h, (size_t)delta_off.back(), cudaHostAllocDefault));
      IRDN_CUDA(cudaMalloc((void**)&ws.delta_d, (size_t)delta_off.back()));
      ws.delta_cap = (size_t)delta_off.back();
    }
  }
  // values copied with the fixed part of each region: the last call's changed fraction + 15 %
  auto delta_budget = [&](int64_t n) {
    return std::min<int64_t>(n, (int64_t)((double)n * ws.delta_ratio * 1.15) + 2 * delta::BLK);
  };
  uint64_t d2h_bytes = 16;  // the counters
  const bool staged_in = !in_pinned, staged_out = !use_delta && !is_pinned(h_out);
  const bool staged = staged_in || staged_out;
  int64_t max_cnt = 0;
  for (const Chunk& c : chunks) max_cnt = std::max(max_cnt, chunk_cnt(c));
  const size_t slot_bytes = ((size_t)max_cnt * sizeof(T) + 255) & ~(size_t)255;
  if (staged && (rc = ensure_staging(ws, slot_bytes))) return rc;
  auto stage_in = [&](size_t i) { return reinterpret_cast<T*>(static_cast<char*>(ws.stage_in) + (i % kStageSlots) * slot_bytes); };
  auto stage_out = [&](size_t i) { return reinterpret_cast<T*>(static_cast<char*>(ws.stage_out) + (i % kStageSlots) * slot_bytes); };
  auto drain_out = [&](size_t i) -> int {  // chunk i's D2H into its slot -> caller's buffer
    IRDN_CUDA(cudaEventSynchronize(ws.ev_out[i % kStageSlots]));
    par_copy(h_out + chunk_off(chunks[i]), stage_out(i), (size_t)chunk_cnt(chunks[i]) * sizeof(T));
    return IRDN_OK;
  };
  auto us = [&] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(); };
  // Sparse return: rebuild chunk i on the host from h_in and the chunk's region.
  const int nt = copy_threads();
  double delta_ratio = 0.0;
  size_t decoded = 0;
  auto decode_chunk = [&](size_t i) -> int {
    if (i == full_chunk) {  // came back by a full copy (synchronised with s_d2h at the end)
      d2h_bytes += (uint64_t)chunk_cnt(chunks[i]) * sizeof(T);
      return IRDN_OK;
    }
    IRDN_CUDA(cudaEventSynchronize(ev_done[i]));
    if (trace) fprintf(stderr, "[irdn]   chunk %zu ready %.1f us", i, us());
    const int64_t off = chunk_off(chunks[i]), cnt = chunk_cnt(chunks[i]);
    uint8_t* src = ws.delta_h + delta_off[i];
    const int64_t total = *reinterpret_cast<const uint32_t*>(src), budget = delta_budget(cnt);
    if (total > budget) {  // more changed pixels than budgeted: fetch the rest of the values
      const int64_t vo = delta::values_offset(cnt) + budget * (int64_t)sizeof(T);
      const size_t extra = (size_t)(total - budget) * sizeof(T);
      IRDN_CUDA(cudaMemcpyAsync(src + vo, ws.delta_d + delta_off[i] + vo, extra, cudaMemcpyDeviceToHost,
                                ws.s_d2h));
      IRDN_CUDA(cudaStreamSynchronize(ws.s_d2h));
      d2h_bytes += extra;
    }
    delta_ratio = std::max(delta_ratio, (double)total / (double)cnt);
    if constexpr (sizeof(T) == 1)
      irdn_delta_decode_host_u8(src, h_in + off, h_out + off, cnt, nt, 1);
    else
      irdn_delta_decode_host_u16(src, h_in + off, h_out + off, cnt, nt, 1);
    if (trace) fprintf(stderr, " decoded %.1f us (%lld px, %lld changed)\n", us(), (long long)cnt, (long long)total);
    return IRDN_OK;
  };
  // One chunk without the sparse return (small frames: c1, the paper's 364 x 244 image):
  // copies and kernel on ONE stream, so the call pays no cross-stream event hops.
  const bool one_stream = chunks.size() == 1 && !use_delta;
  cudaStream_t s_h2d = one_stream ? ws.s_comp : ws.s_h2d;
  cudaStream_t s_d2h = one_stream ? ws.s_comp : ws.s_d2h;
  // H2D: each chunk's own rows (row mode: strips, in order).
  if (!staged_in) {
    for (size_t i = 0; i < chunks.size(); ++i) {
      const int64_t off = chunk_off(chunks[i]);
      if (i == 0) tmark(0, s_h2d);
      IRDN_CUDA(h2d(d_in + dev_off(chunks[i]), h_in + off, chunk_rows(chunks[i]), off, s_h2d));
      tmark(1 + 4 * i, s_h2d);
      IRDN_CUDA(cudaEventRecord(ev_in[i], s_h2d));
    }
  }
  size_t drained = 0, issued = 0;
  // staged H2D of chunks [issued, upto]: slot j % kStageSlots was last used by chunk
  // j - kStageSlots, whose H2D must be done before the slot is refilled and whose output
  // must be copied out before the D2H reuses the slot (its D2H is already enqueued: a
  // row strip looks ahead at most one strip, kStageSlots >= 3)
  auto issue_h2d = [&](size_t upto) -> int {
    for (; issued <= upto && issued < chunks.size(); ++issued) {
      const size_t j = issued;
      if (j >= (size_t)kStageSlots) {
        IRDN_CUDA(cudaEventSynchronize(ev_in[j - kStageSlots]));
        if (staged_out && drained <= j - kStageSlots) {
          int e = drain_out(j - kStageSlots);
          if (e) return e;
          drained = j - kStageSlots + 1;
        }
      }
      const int64_t off = chunk_off(chunks[j]), cnt = chunk_cnt(chunks[j]);
      par_copy(stage_in(j), h_in + off, (size_t)cnt * sizeof(T));
      IRDN_CUDA(h2d(d_in + dev_off(chunks[j]), stage_in(j), chunk_rows(chunks[j]), off, s_h2d));
      IRDN_CUDA(cudaEventRecord(ev_in[j], s_h2d));
    }
    return IRDN_OK;
  };
  for (size_t i = 0; i < chunks.size(); ++i) {
    const Chunk& c = chunks[i];
    if (staged_in) {
      size_t need = i;
      if (row_mode)
        while (need + 1 < chunks.size() && chunks[need].y1 < std::min<int64_t>(height, c.y1 + r)) ++need;
      if ((rc = issue_h2d(need))) return rc;
    }
    if (row_mode) {
      // A strip needs the input rows up to y1 + r, i.e. possibly the next chunk's copy.
      size_t last = i;
      while (last + 1 < chunks.size() && chunks[last].y1 < std::min<int64_t>(height, c.y1 + r)) ++last;
      IRDN_CUDA(cudaStreamWaitEvent(ws.s_comp, ev_in[last], 0));
      const int64_t in0 = std::max<int64_t>(0, c.y0 - r);
      const int64_t in1 = std::min<int64_t>(height, c.y1 + r);
      rc = filter_strip<T>(d_in + in0 * dp, in0, in1 - in0, d_out + c.y0 * dp, c.y0, c.y1,
                           height, width, dp, dp, k, method, ws.counts, ws.s_comp);
      if (rc) return rc;
    } else {
      IRDN_CUDA(cudaStreamWaitEvent(ws.s_comp, ev_in[i], 0));
      tmark(2 + 4 * i, ws.s_comp);
      const int64_t off = c.f0 * dframe;
      rc = run_device<T>(d_in + off, d_out + off, d_tmp ? d_tmp + off : nullptr, c.nf, height,
                         width, k, method, passes, ws.counts, ws.s_comp, dp);
      if (rc) return rc;
    }
    const int64_t off = chunk_off(c), cnt = chunk_cnt(c);  // host layout (delta: dp == width)
    if (use_delta && i != full_chunk) {  // encode out vs in into the device region, DMA its fixed part + budget
      const T* a = d_in + off;
      const T* o = d_out + off;
      const int vec = (((uintptr_t)a | (uintptr_t)o) & 15) == 0;
      uint8_t* dreg = ws.delta_d + delta_off[i];
      // the encode runs on the D2H stream, so the next chunk's filter does not queue behind it
      // (measured neutral against the compute stream; kept off the filter's path)
      IRDN_CUDA(cudaEventRecord(ev_done[i], ws.s_comp));
      IRDN_CUDA(cudaStreamWaitEvent(s_d2h, ev_done[i], 0));
      IRDN_CUDA(cudaMemsetAsync(dreg, 0, 16, s_d2h));
      tmark(3 + 4 * i, s_d2h);
      delta::encode_kernel<T><<<(unsigned)delta::nblocks(cnt), delta::THREADS, 0, s_d2h>>>(a, o, cnt, dreg, vec);
      IRDN_CUDA(cudaGetLastError());
      note_launch();
      const size_t bytes = (size_t)(delta::values_offset(cnt) + delta_budget(cnt) * (int64_t)sizeof(T));
      IRDN_CUDA(cudaMemcpyAsync(ws.delta_h + delta_off[i], dreg, bytes, cudaMemcpyDeviceToHost, s_d2h));
      d2h_bytes += bytes;
      tmark(4 + 4 * i, s_d2h);
      IRDN_CUDA(cudaEventRecord(ev_done[i], s_d2h));
      continue;
    }
    IRDN_CUDA(cudaEventRecord(ev_done[i], ws.s_comp));
    IRDN_CUDA(cudaStreamWaitEvent(s_d2h, ev_done[i], 0));
    if (staged_out && !staged_in && i >= (size_t)kStageSlots && drained <= i - kStageSlots) {
      if ((rc = drain_out(i - kStageSlots))) return rc;  // the slot's previous chunk
      drained = i - kStageSlots + 1;
    }
    IRDN_CUDA(d2h(staged_out ? stage_out(i) : h_out + off, d_out + dev_off(c), chunk_rows(c), off, s_d2h));
    if (staged_out) IRDN_CUDA(cudaEventRecord(ws.ev_out[i % kStageSlots], s_d2h));
  }
  if (staged_out)
    for (size_t i = drained; i < chunks.size(); ++i)
      if ((rc = drain_out(i))) return rc;
  if (trace) fprintf(stderr, "[irdn] %zu chunks enqueued at %.1f us\n", chunks.size(), us());
  if (use_delta) {
    for (; decoded < chunks.size(); ++decoded)
      if ((rc = decode_chunk(decoded))) return rc;
    ws.delta_ratio = delta_ratio;
  } else {
    d2h_bytes += nbytes;
  }
  g_xfer_h2d = nbytes;
  g_xfer_d2h = d2h_bytes;
  unsigned long long counts[2] = {0, 0};
  IRDN_CUDA(cudaStreamWaitEvent(s_d2h, ev_done[chunks.size() - 1], 0));
  IRDN_CUDA(cudaMemcpyAsync(counts, ws.counts, sizeof(counts), cudaMemcpyDeviceToHost, s_d2h));
  IRDN_CUDA(cudaStreamSynchronize(s_d2h));
  IRDN_CUDA(cudaStreamSynchronize(ws.s_comp));
  IRDN_CUDA(cudaGetLastError());
  if (trace) {
    fprintf(stderr, "[irdn] done %.1f us; device (us from the first H2D): ", us());
    for (size_t i = 0; i < chunks.size() && 4 * i + 4 < tev.size(); ++i) {
      float a = 0, b = 0, c = 0, d = 0;
      cudaEventElapsedTime(&a, tev[0], tev[1 + 4 * i]);
      cudaEventElapsedTime(&b, tev[0], tev[2 + 4 * i]);
      cudaEventElapsedTime(&c, tev[0], tev[3 + 4 * i]);
      cudaEventElapsedTime(&d, tev[0], tev[4 + 4 * i]);
      fprintf(stderr, "[%zu h2d %.0f filt %.0f-%.0f enc -%.0f] ", i, a * 1e3, b * 1e3, c * 1e3, d * 1e3);
    }
    cudaGetLastError();
    fprintf(stderr, "\n");
  }

  if (stats) {
    const uint64_t pixels = (uint64_t)(batch * frame) * (uint64_t)passes;
    // FilterStats accounting (filters.py:121-126).
    stats->passes = (uint64_t)passes;
    if (method == IRDN_METHOD_FNR) {
      stats->minmax_scans = pixels;
      stats->detected = counts[0];
      stats->sorts = counts[0];
      stats->replacements = counts[1];
    } else {
      stats->minmax_scans = 0;
      stats->detected = 0;
      stats->sorts = pixels;
      stats->replacements = 0;
    }
    stats->elapsed_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return IRDN_OK;
}

// ---- inject_impulse (noise.py:89-106), csrc/noise.cuh ------------------------
static int inject_impulse(const uint8_t* d_in, uint8_t* d_out, uint8_t* d_flags, int64_t n, uint64_t seed,
                          double density, double salt, unsigned long long* d_count, void* stream) {
  if (!(density >= 0.0 && density <= 1.0))  // noise.py:47-48
    return fail(IRDN_EINVAL, "density must be in [0, 1], got %g", density);
  if (!(salt >= 0.0 && salt <= 1.0))  // noise.py:49-52
    return fail(IRDN_EINVAL, "salt_fraction must be in [0, 1], got %g", salt);
  if (n < 0) return fail(IRDN_EINVAL, "pixel count must be >= 0, got %lld", (long long)n);
  if (n > ((int64_t)1 << 40)) return fail(IRDN_EINVAL, "too many pixels (%lld)", (long long)n);
  if (n > 0 && (!d_in || !d_out)) return fail(IRDN_EINVAL, "null image pointer");
  if (n > 0 && d_in == d_out) return fail(IRDN_EINVAL, "in-place injection is not supported (d_out == d_in)");
  int rc = check_device(nullptr);
  if (rc != IRDN_OK) return rc;
  if (n == 0) return IRDN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  noise::Params p;
  p.in = d_in;
  p.out = d_out;
  p.flags = d_flags;
  p.count = d_count;
  p.n = n;
  p.max_chunks = (2 * n + noise::CHUNK - 1) / noise::CHUNK;
  p.seed = seed;
  // (x >> 11) / 2^53 < d  <=>  (x >> 11) < ceil(d * 2^53): d * 2^53 is exact in binary64
  const uint64_t thr_density = (uint64_t)std::ceil(std::ldexp(density, 53));
  const uint64_t thr_salt = (uint64_t)std::ceil(std::ldexp(salt, 53));
  p.all_density = thr_density >= (1ull << 53);
  p.all_salt = thr_salt >= (1ull << 53);
  p.z_density = p.all_density ? 0ull : thr_density << 11;
  p.z_salt = p.all_salt ? 0ull : thr_salt << 11;
  p.vec = ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out) |
            reinterpret_cast<uintptr_t>(d_flags)) & 15) == 0;
  const size_t ws_bytes = 16 + (size_t)p.max_chunks * sizeof(unsigned long long);
  void* ws = nullptr;
  IRDN_CUDA(cudaMallocAsync(&ws, ws_bytes, s));
  IRDN_CUDA(cudaMemsetAsync(ws, 0, ws_bytes, s));
  p.ctl = static_cast<unsigned int*>(ws);
  p.status = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + 16);
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, noise::noise_kernel, noise::THREADS, 0) !=
            cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
  }
  const long long grid = std::min<long long>(p.max_chunks, (long long)sms * per_sm);
  noise::noise_kernel<<<(unsigned)grid, noise::THREADS, 0, s>>>(p);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return fail(IRDN_ECUDA, "inject_impulse launch failed: %s", cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(IRDN_ECUDA, "cudaFreeAsync failed: %s", cudaGetErrorString(e2));
  return IRDN_OK;
}

// ---- exact squared-error sum (metrics.py:22-32), csrc/metrics.cuh -------------
template <typename T>
static int sq_err_sum(const T* d_a, const T* d_b, int64_t n, unsigned long long* d_sum, void* stream) {
  if (n < 0) return fail(IRDN_EINVAL, "element count must be >= 0, got %lld", (long long)n);
  if (sizeof(T) == 2 && n > (int64_t)0xFFFFFFFFLL)
    return fail(IRDN_EINVAL, "u16 squared-error sum takes at most 2^32-1 elements per call, got %lld",
                (long long)n);
  if (!d_sum || (n > 0 && (!d_a || !d_b))) return fail(IRDN_EINVAL, "null pointer");
  int dev = 0;
  int rc = check_device(&dev);
  if (rc != IRDN_OK) return rc;
  if (n == 0) return IRDN_OK;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = ((reinterpret_cast<uintptr_t>(d_a) | reinterpret_cast<uintptr_t>(d_b)) & 15) == 0;
  const int64_t per_cta = (int64_t)metrics::THREADS * 16 / (int64_t)sizeof(T) * 4;
  const int64_t want = (n + per_cta - 1) / per_cta;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
  metrics::sq_err_kernel<T><<<grid, metrics::THREADS, 0, static_cast<cudaStream_t>(stream)>>>(d_a, d_b, n, vec,
                                                                                                d_sum);
  ++g_launches;
  IRDN_CUDA(cudaGetLastError());
  return IRDN_OK;
}

// Device half of the sparse result return as a public entry point (delta.cuh format);
// d_region is device-accessible (device memory or mapped pinned host memory).
template <typename T>
static int delta_encode(const T* d_in, const T* d_out, int64_t n, void* d_region, void* stream) {
  if (n < 0 || (n > 0 && (!d_in || !d_out || !d_region))) return fail(IRDN_EINVAL, "bad delta_encode arguments");
  if (((uintptr_t)d_region & 15)) return fail(IRDN_EINVAL, "delta region must be 16-byte aligned");
  if (n == 0) return IRDN_OK;
  int rc = check_device(nullptr);
  if (rc) return rc;
  const int vec = (((uintptr_t)d_in | (uintptr_t)d_out) & 15) == 0;
  IRDN_CUDA(cudaMemsetAsync(d_region, 0, 16, static_cast<cudaStream_t>(stream)));
  delta::encode_kernel<T><<<(unsigned)delta::nblocks(n), delta::THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
      d_in, d_out, n, static_cast<uint8_t*>(d_region), vec);
  IRDN_CUDA(cudaGetLastError());
  note_launch();
  return IRDN_OK;
}

}  // namespace irdn

using namespace irdn;

extern "C" {

const char* irdn_version(void) { return "irdn-b200 0.1.0 (sm_100a)"; }
const char* irdn_last_error(void) { return g_err.c_str(); }

int irdn_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int count = 0;
  for (int d = 0; d < n; ++d) {
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10)
      ++count;
  }
  return count;
}

uint64_t irdn_fast_window_mask(int32_t bytes_per_pixel) { return fast::window_mask(bytes_per_pixel); }

int irdn_filter_pass_u8(const uint8_t* d_in, uint8_t* d_out, int64_t batch, int64_t height,
                        int64_t width, int64_t in_pitch, int64_t out_pitch, int32_t k,
                        int32_t method, unsigned long long* d_counts, void* stream) {
  return filter_pass<uint8_t>(d_in, d_out, batch, height, width, in_pitch, out_pitch, k, method,
                              d_counts, stream);
}
int irdn_filter_pass_u16(const uint16_t* d_in, uint16_t* d_out, int64_t batch, int64_t height,
                         int64_t width, int64_t in_pitch, int64_t out_pitch, int32_t k,
                         int32_t method, unsigned long long* d_counts, void* stream) {
  return filter_pass<uint16_t>(d_in, d_out, batch, height, width, in_pitch, out_pitch, k, method,
                               d_counts, stream);
}
int irdn_filter_strip_u8(const uint8_t* d_in, int64_t in_row0, int64_t in_rows, uint8_t* d_out,
                         int64_t row_begin, int64_t row_end, int64_t height, int64_t width,
                         int64_t in_pitch, int64_t out_pitch, int32_t k, int32_t method,
                         unsigned long long* d_counts, void* stream) {
  return filter_strip<uint8_t>(d_in, in_row0, in_rows, d_out, row_begin, row_end, height, width,
                               in_pitch, out_pitch, k, method, d_counts, stream);
}
int irdn_filter_strip_u16(const uint16_t* d_in, int64_t in_row0, int64_t in_rows,
                          uint16_t* d_out, int64_t row_begin, int64_t row_end, int64_t height,
                          int64_t width, int64_t in_pitch, int64_t out_pitch, int32_t k,
                          int32_t method, unsigned long long* d_counts, void* stream) {
  return filter_strip<uint16_t>(d_in, in_row0, in_rows, d_out, row_begin, row_end, height, width,
                                in_pitch, out_pitch, k, method, d_counts, stream);
}
int irdn_run_filter_u8(const uint8_t* h_in, uint8_t* h_out, int64_t batch, int64_t height,
                       int64_t width, int32_t k, int32_t method, int32_t passes, int32_t device,
                       irdn_stats* stats) {
  return run_host<uint8_t>(h_in, h_out, batch, height, width, k, method, passes, device, stats);
}
int irdn_run_filter_u16(const uint16_t* h_in, uint16_t* h_out, int64_t batch, int64_t height,
                        int64_t width, int32_t k, int32_t method, int32_t passes,
                        int32_t device, irdn_stats* stats) {
  return run_host<uint16_t>(h_in, h_out, batch, height, width, k, method, passes, device, stats);
}
int irdn_run_filter_device_u8(const uint8_t* d_in, uint8_t* d_out, uint8_t* d_tmp,
                              int64_t batch, int64_t height, int64_t width, int32_t k,
                              int32_t method, int32_t passes, unsigned long long* d_counts,
                              void* stream) {
  return run_device<uint8_t>(d_in, d_out, d_tmp, batch, height, width, k, method, passes,
                             d_counts, stream);
}
int irdn_run_filter_device_u16(const uint16_t* d_in, uint16_t* d_out, uint16_t* d_tmp,
                               int64_t batch, int64_t height, int64_t width, int32_t k,
                               int32_t method, int32_t passes, unsigned long long* d_counts,
                               void* stream) {
  return run_device<uint16_t>(d_in, d_out, d_tmp, batch, height, width, k, method, passes,
                              d_counts, stream);
}
int irdn_inject_impulse_u8(const uint8_t* d_in, uint8_t* d_out, uint8_t* d_flags, int64_t n, uint64_t seed,
                           double density, double salt_fraction, unsigned long long* d_count, void* stream) {
  return inject_impulse(d_in, d_out, d_flags, n, seed, density, salt_fraction, d_count, stream);
}
int irdn_sq_err_sum_u8(const uint8_t* d_a, const uint8_t* d_b, int64_t n, unsigned long long* d_sum,
                       void* stream) {
  return sq_err_sum<uint8_t>(d_a, d_b, n, d_sum, stream);
}
int irdn_sq_err_sum_u16(const uint16_t* d_a, const uint16_t* d_b, int64_t n, unsigned long long* d_sum,
                        void* stream) {
  return sq_err_sum<uint16_t>(d_a, d_b, n, d_sum, stream);
}
int irdn_scene_render(const irdn_scene_desc* desc, void* d_out, void* stream) {
  int rc = check_device(nullptr);
  if (rc != IRDN_OK) return rc;
  cudaError_t err = cudaSuccess;
  rc = scene::render(desc, d_out, static_cast<cudaStream_t>(stream), &err);
  if (rc == IRDN_EINVAL) return fail(rc, "invalid scene descriptor");
  if (rc != IRDN_OK) return fail(rc, "scene render launch failed: %s", cudaGetErrorString(err));
  return IRDN_OK;
}
int32_t irdn_set_multipass(int32_t on) {
  int32_t prev = g_multipass;
  g_multipass = on ? 1 : 0;
  return prev;
}
int32_t irdn_set_host_return(int32_t mode) {
  int32_t prev = g_host_return;
  g_host_return = (mode >= 0 && mode <= 2) ? mode : 0;
  return prev;
}
void irdn_last_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  if (h2d_bytes) *h2d_bytes = g_xfer_h2d;
  if (d2h_bytes) *d2h_bytes = g_xfer_d2h;
}
uint64_t irdn_delta_region_bytes(int64_t n, int32_t bytes_per_pixel) {
  if (n < 1) return 0;
  return (uint64_t)(bytes_per_pixel == 1 ? delta::region_bytes<uint8_t>(n) : delta::region_bytes<uint16_t>(n));
}
uint64_t irdn_delta_decode_u8(const void* region, const uint8_t* h_in, uint8_t* h_out, int64_t n, int32_t simd) {
  return n < 1 ? 0 : irdn_delta_decode_host_u8(static_cast<const uint8_t*>(region), h_in, h_out, n, copy_threads(),
                                               simd);
}
uint64_t irdn_delta_decode_u16(const void* region, const uint16_t* h_in, uint16_t* h_out, int64_t n, int32_t simd) {
  return n < 1 ? 0 : irdn_delta_decode_host_u16(static_cast<const uint8_t*>(region), h_in, h_out, n,
                                                copy_threads(), simd);
}
int irdn_delta_encode_u8(const uint8_t* d_in, const uint8_t* d_out, int64_t n, void* d_region, void* stream) {
  return delta_encode<uint8_t>(d_in, d_out, n, d_region, stream);
}
int irdn_delta_encode_u16(const uint16_t* d_in, const uint16_t* d_out, int64_t n, void* d_region, void* stream) {
  return delta_encode<uint16_t>(d_in, d_out, n, d_region, stream);
}
uint64_t irdn_launch_count(void) { return g_launches; }
void irdn_reset_launch_count(void) { g_launches = 0; }
int32_t irdn_set_force_generic(int32_t on) {
  int32_t prev = g_force_generic;
  g_force_generic = on ? 1 : 0;
  return prev;
}

// ---- fused gather: CUDA IPC of the owner's output allocation ----------------------------
typedef CUresult (*MemGetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
static MemGetAddressRangeFn address_range_fn() {
  static MemGetAddressRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<MemGetAddressRangeFn>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

int irdn_ipc_export(const void* d_ptr, void* handle64, uint64_t* offset) {
  if (!d_ptr || !handle64 || !offset) return fail(IRDN_EINVAL, "null argument");
  MemGetAddressRangeFn range = address_range_fn();
  if (!range) return fail(IRDN_ECUDA, "cuMemGetAddressRange is not available");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)(uintptr_t)d_ptr) != CUDA_SUCCESS)
    return fail(IRDN_EINVAL, "pointer is not in a device allocation");
  cudaIpcMemHandle_t h;
  IRDN_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>((uintptr_t)base)));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  *offset = (uint64_t)((uintptr_t)d_ptr - (uintptr_t)base);
  return IRDN_OK;
}

int irdn_ipc_open(const void* handle64, uint64_t offset, void** d_ptr) {
  if (!handle64 || !d_ptr) return fail(IRDN_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  IRDN_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_ptr = static_cast<char*>(base) + offset;
  return IRDN_OK;
}

int irdn_ipc_close(void* d_ptr, uint64_t offset) {
  if (!d_ptr) return fail(IRDN_EINVAL, "null argument");
  IRDN_CUDA(cudaIpcCloseMemHandle(static_cast<char*>(d_ptr) - offset));
  return IRDN_OK;
}

#ifdef IRDN_TIMELINE
IRDN_API int irdn_debug_timeline(void* host, int64_t bytes) {
  if (!irdn::fast::g_timeline) return IRDN_EINVAL;
  return cudaMemcpy(host, irdn::fast::g_timeline, std::min<int64_t>(bytes, 8 << 20), cudaMemcpyDeviceToHost) ==
                 cudaSuccess ? IRDN_OK : IRDN_ECUDA;
}
#endif
}  // extern "C"
