/*
 * irdn.h — C ABI of the B200-native FNR (Fast Noise Reduction) filter.
 *
 * This is the drop-in boundary for the reference's filter entry points
 * (irdenoise v0.1.0, pure Python). Every function here replaces one
 * reference interface; the citation is given beside each declaration
 * (paths relative to the reference checkout, pkg/src/irdenoise/...):
 *
 *   irdn_run_filter_u8 / _u16     <- filters.py:79-102   run_filter(img, spec, method, passes, threads)
 *   irdn_filter_pass_u8 / _u16    <- filters.py:69-76    fnr_pass / mf_pass  (one pass, caller's stats)
 *                                    filters.py:105-127  _run_rows_threaded  (fresh out buffer, counter merge)
 *                                    filters.py:130-181  _filter_rows        (gather, detect, median, write)
 *   irdn_filter_strip_u8 / _u16   <- filters.py:130      _filter_rows(img, k, y0, y1, ...) row range [y0, y1)
 *                                    of a frame whose rows are clamped against the GLOBAL image height
 *   irdn_stats                    <- filters.py:33-52    FilterStats (same field meaning and key order)
 *   IRDN_METHOD_FNR / _MF         <- filters.py:23-24    METHOD_FNR = "fnr", METHOD_MF = "mf"
 *   irdn_inject_impulse_u8        <- noise.py:89-106     inject_impulse(img, NoiseSpec) (SplitMix64 stream,
 *                                    noise.py:17-34; bit-identical output image, mask and count)
 *   irdn_sq_err_sum_u8 / _u16     <- metrics.py:22-32    the exact integer sum inside mse() (and psnr(),
 *                                    quality_report(), build_comparison())
 *   irdn_scene_render             <- (no reference interface) the seeded BASELINE scenes of
 *                                    csrc/scene.c rendered on the device (bench / test input)
 *
 * Semantics (bit-exact with the reference):
 *   - row-major frames, origin top-left; replicate-edge (clamp) window gather;
 *   - FNR: a pixel is noisy iff it equals the min or the max of its k x k
 *     window (centre included); noisy pixels become the window median
 *     (element (k*k-1)/2 of the sorted window), signal pixels are copied;
 *   - MF: every pixel becomes the window median;
 *   - a pass reads an immutable input and writes a distinct output buffer.
 *
 * Counters: the device pass entry points ADD to d_counts[0] (= detected,
 * which also equals FNR sorts) and d_counts[1] (= replacements). For MF both
 * stay untouched (sorts = pixels x passes, as the reference counts them).
 *
 * Error handling: every entry point returns IRDN_OK (0) or an error code;
 * irdn_last_error() returns the thread-local message of the last failure.
 * Argument errors (IRDN_EINVAL) mirror the reference's ValueErrors
 * (filters.py:90-93 bad method / passes; image.py:63-65 bad k;
 * image.py:30-36 bad image dimensions). There is no CPU fallback: without a
 * usable sm_100 device every compute call fails with IRDN_ENODEV.
 *
 * Streams are passed as void* (a cudaStream_t / CUstream; NULL = legacy
 * default stream). Device pointers must be device-resident (cudaMalloc /
 * torch); host pointers in irdn_run_filter_* may be pageable or pinned.
 */
#ifndef IRDN_H_
#define IRDN_H_

#include <stdint.h>

#if defined(__GNUC__)
#define IRDN_API __attribute__((visibility("default")))
#else
#define IRDN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define IRDN_OK 0
#define IRDN_EINVAL 1   /* invalid argument: the reference raises ValueError */
#define IRDN_ECUDA 2    /* CUDA runtime / launch failure */
#define IRDN_ENODEV 3   /* no usable sm_100 device */

#define IRDN_METHOD_FNR 0  /* filters.py:23  METHOD_FNR = "fnr" */
#define IRDN_METHOD_MF 1   /* filters.py:24  METHOD_MF = "mf"   */

/* Mirrors FilterStats (filters.py:33-52). elapsed_ms is wall time of the call. */
typedef struct irdn_stats {
  uint64_t minmax_scans;
  uint64_t sorts;
  uint64_t replacements;
  uint64_t detected;
  double elapsed_ms;
  uint64_t passes;
} irdn_stats;

/* Library identity / capability queries. */
IRDN_API const char* irdn_version(void);
IRDN_API const char* irdn_last_error(void);
/* Number of visible CUDA devices of compute capability 10.x (0 when none). */
IRDN_API int irdn_device_count(void);
/* Bit mask of window sides with a specialised kernel (bit k set => k fast path). */
IRDN_API uint64_t irdn_fast_window_mask(int32_t bytes_per_pixel);

/*
 * One filter pass over `batch` frames of height x width, device-resident,
 * stream-ordered and asynchronous (no host sync).
 *   in_pitch / out_pitch: row pitch in ELEMENTS; frames are contiguous blocks
 *   of height*pitch elements. d_in and d_out must not overlap.
 * Replaces fnr_pass / mf_pass (filters.py:69-76) for one frame per batch entry.
 */
IRDN_API int irdn_filter_pass_u8(const uint8_t* d_in, uint8_t* d_out, int64_t batch, int64_t height,
                        int64_t width, int64_t in_pitch, int64_t out_pitch, int32_t k,
                        int32_t method, unsigned long long* d_counts, void* stream);
IRDN_API int irdn_filter_pass_u16(const uint16_t* d_in, uint16_t* d_out, int64_t batch, int64_t height,
                         int64_t width, int64_t in_pitch, int64_t out_pitch, int32_t k,
                         int32_t method, unsigned long long* d_counts, void* stream);

/*
 * Row-strip pass for one frame of GLOBAL size height x width (multi-GPU row
 * strips, BASELINE config 4): computes output rows [row_begin, row_end).
 *   d_in   points at global row in_row0 and holds in_rows rows; it must cover
 *          [max(0,row_begin-k/2), min(height,row_end+k/2)) — window rows are
 *          clamped against the global image, exactly like _filter_rows(y0, y1)
 *          (filters.py:130-157), never against the strip.
 *   d_out  points at the output row row_begin (row_end-row_begin rows).
 */
IRDN_API int irdn_filter_strip_u8(const uint8_t* d_in, int64_t in_row0, int64_t in_rows, uint8_t* d_out,
                         int64_t row_begin, int64_t row_end, int64_t height, int64_t width,
                         int64_t in_pitch, int64_t out_pitch, int32_t k, int32_t method,
                         unsigned long long* d_counts, void* stream);
IRDN_API int irdn_filter_strip_u16(const uint16_t* d_in, int64_t in_row0, int64_t in_rows,
                          uint16_t* d_out, int64_t row_begin, int64_t row_end, int64_t height,
                          int64_t width, int64_t in_pitch, int64_t out_pitch, int32_t k,
                          int32_t method, unsigned long long* d_counts, void* stream);

/*
 * Whole run_filter (filters.py:79-102) over HOST buffers: validation, H2D,
 * `passes` passes on `device` (each pass reading the previous output), D2H,
 * and the FilterStats counters. Copies are pipelined against the filter in
 * frame chunks (or row strips for a single frame) on internal streams.
 * h_in and h_out must not overlap; batch frames are contiguous (pitch=width).
 */
IRDN_API int irdn_run_filter_u8(const uint8_t* h_in, uint8_t* h_out, int64_t batch, int64_t height,
                       int64_t width, int32_t k, int32_t method, int32_t passes,
                       int32_t device, irdn_stats* stats);
IRDN_API int irdn_run_filter_u16(const uint16_t* h_in, uint16_t* h_out, int64_t batch, int64_t height,
                        int64_t width, int32_t k, int32_t method, int32_t passes,
                        int32_t device, irdn_stats* stats);

/*
 * run_filter over DEVICE buffers, stream-ordered: `passes` passes from d_in
 * to d_out, ping-ponging through d_tmp (required when passes > 1, same size
 * as d_out). Counters are added to d_counts[0..1] (see above).
 */
IRDN_API int irdn_run_filter_device_u8(const uint8_t* d_in, uint8_t* d_out, uint8_t* d_tmp,
                              int64_t batch, int64_t height, int64_t width, int32_t k,
                              int32_t method, int32_t passes, unsigned long long* d_counts,
                              void* stream);
IRDN_API int irdn_run_filter_device_u16(const uint16_t* d_in, uint16_t* d_out, uint16_t* d_tmp,
                               int64_t batch, int64_t height, int64_t width, int32_t k,
                               int32_t method, int32_t passes, unsigned long long* d_counts,
                               void* stream);

/*
 * inject_impulse (noise.py:89-106) over n row-major u8 pixels, device buffers,
 * stream-ordered. Draw p of SplitMix64(seed) (noise.py:17-34) is mix(seed +
 * (p+1) * 0x9E3779B97F4A7C15); per pixel one uniform (top 53 bits / 2^53) < density
 * decides corruption and, only then, a second one < salt_fraction picks 255 over 0.
 * d_out receives the noisy image (d_out != d_in), d_flags (optional, may be NULL)
 * the NoiseMask flags (1 = corrupted), *d_count (optional) is INCREMENTED by the
 * number of corrupted pixels. density / salt_fraction outside [0, 1] -> IRDN_EINVAL
 * (NoiseSpec.__post_init__, noise.py:45-55). Uses ~n/4 bytes of stream-ordered
 * scratch (cudaMallocAsync).
 */
IRDN_API int irdn_inject_impulse_u8(const uint8_t* d_in, uint8_t* d_out, uint8_t* d_flags, int64_t n,
                                    uint64_t seed, double density, double salt_fraction,
                                    unsigned long long* d_count, void* stream);

/*
 * Exact sum over i of (a[i] - b[i])^2 (metrics.py:29-32), ADDED to *d_sum, device
 * buffers, stream-ordered. u16: n <= 2^32 - 1 per call (the sum must fit 64 bits).
 */
IRDN_API int irdn_sq_err_sum_u8(const uint8_t* d_a, const uint8_t* d_b, int64_t n,
                                unsigned long long* d_sum, void* stream);
IRDN_API int irdn_sq_err_sum_u16(const uint16_t* d_a, const uint16_t* d_b, int64_t n,
                                 unsigned long long* d_sum, void* stream);

/*
 * Seeded BASELINE scene rendering on the device (bench / test input, SURVEY §8f rank 2;
 * not a reference interface: the reference evaluates on one IR photograph, SPEC.md:309,
 * that these scenes stand in for). Renders frames [frame0, frame0 +
 * nframes) of the scene csrc/scene.c's scene_generate() defines into d_out (contiguous
 * [nframes][height][width] pixels of bytes_per_pixel bytes), stream-ordered, byte for byte
 * equal to scene_generate(). The tables are scene_tables()' output (the per-frame
 * parameters that need exp / sin / cos, computed by the host code), copied to the device.
 */
typedef struct irdn_scene_desc {
  int32_t width, height, bytes_per_pixel, maxval;
  int32_t nblobs, nlines, nrects;  /* nlines <= 64, nrects <= 256 (scene.c's caps) */
  int32_t impulse_kind;            /* 0 none, 1 salt & pepper, 2 uniform random */
  int32_t config_id, sensor;       /* sensor: 1 iff sensor_sigma > 0 */
  double scale;                    /* maxval / 255.0 */
  double sensor_mul;               /* sensor_sigma * 1.7320508075688772 */
  double line_amp, rect_amp, density;
  uint64_t seed;
  int64_t frame0, nframes;         /* height and nframes <= 65535 per call */
  const double* gx;                /* [nframes][nblobs][width]  device */
  const double* gy;                /* [nframes][nblobs][height] device */
  const double* lines;             /* [nframes][nlines][5]      device */
  const int32_t* rects;            /* [nframes][nrects][4]      device, 16-byte aligned */
} irdn_scene_desc;
IRDN_API int irdn_scene_render(const irdn_scene_desc* desc, void* d_out, void* stream);

/*
 * passes > 1 (irdn_run_filter_*, irdn_run_filter_device_*): 1 = all passes in ONE
 * persistent launch of the warp kernel, a tile of pass q starting as soon as the tiles of
 * pass q-1 under its window box have published their output (filters.py:96-100: every
 * pass still reads the complete previous output); 0 (default) = one launch per pass,
 * back to back with programmatic dependent launch — measured faster on B200 (DESIGN.md
 * §9). Returns the previous setting. Process-wide; IRDN_MULTIPASS=1 sets it initially.
 */
IRDN_API int32_t irdn_set_multipass(int32_t on);

/*
 * Result return of irdn_run_filter_*: 0 = auto (sparse for FNR on u16 frames from a pinned
 * input with >= 6 host threads per GPU process, else full copy),
 * 1 = full device->host copy of the output, 2 = sparse. Sparse: the device sends only
 * the output pixels that differ from the input (a per-4096-pixel count, a change
 * bit mask and the packed changed values, written by the encode kernel into mapped
 * pinned memory) and the host rebuilds the output from the caller's own input —
 * filters.py:108 / :127's fresh output buffer, with the unchanged pixels copied on the
 * host instead of over PCIe. Returns the previous mode. Process-wide. The environment
 * variable IRDN_HOST_RETURN=auto|full|delta sets the initial mode.
 */
IRDN_API int32_t irdn_set_host_return(int32_t mode);
/* Host->device and device->host bytes moved by this thread's last irdn_run_filter_* call. */
IRDN_API void irdn_last_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/*
 * The sparse return as separate halves (the format is documented in
 * paper_1201_3972_b200/csrc/delta.cuh). irdn_delta_encode_*: compare n device pixels
 * d_out against d_in and write the region (irdn_delta_region_bytes(n, bpp) bytes,
 * 16-byte aligned, device-accessible: device memory or mapped pinned host memory),
 * stream-ordered. irdn_delta_decode_*: h_out = h_in with the region's changed pixels
 * applied (host memory, OpenMP; simd = 0 forces the scalar decoder); returns the
 * region bytes the encoder wrote.
 */
IRDN_API uint64_t irdn_delta_region_bytes(int64_t n, int32_t bytes_per_pixel);
IRDN_API int irdn_delta_encode_u8(const uint8_t* d_in, const uint8_t* d_out, int64_t n, void* d_region,
                                  void* stream);
IRDN_API int irdn_delta_encode_u16(const uint16_t* d_in, const uint16_t* d_out, int64_t n, void* d_region,
                                   void* stream);
IRDN_API uint64_t irdn_delta_decode_u8(const void* region, const uint8_t* h_in, uint8_t* h_out, int64_t n,
                                       int32_t simd);
IRDN_API uint64_t irdn_delta_decode_u16(const void* region, const uint16_t* h_in, uint16_t* h_out, int64_t n,
                                        int32_t simd);

/*
 * Fused gather for multi-GPU shards (reference filters.py:110-126: the row bands' results
 * land in ONE output buffer). The rank that owns the full output exports it with
 * irdn_ipc_export (a 64-byte CUDA IPC handle of the allocation containing d_ptr, plus
 * d_ptr's byte offset in it, so pointers from caching allocators work); every other rank
 * maps it with irdn_ipc_open and passes (mapped pointer + its shard's offset) as d_out of
 * irdn_run_filter_device_* / irdn_filter_strip_*: the filter kernels then store their
 * output straight into the owner's memory over NVLink (peer stores from the same kernel,
 * no separate gather collective). irdn_ipc_close unmaps. Works between processes on the
 * same GPU too (the CPU test of the path).
 */
IRDN_API int irdn_ipc_export(const void* d_ptr, void* handle64, uint64_t* offset);
IRDN_API int irdn_ipc_open(const void* handle64, uint64_t offset, void** d_ptr);
IRDN_API int irdn_ipc_close(void* d_ptr, uint64_t offset);

/* Kernel launches issued by this thread since the last reset (for bench accounting). */
IRDN_API uint64_t irdn_launch_count(void);
IRDN_API void irdn_reset_launch_count(void);

/*
 * Force the generic (non-specialised) kernel for testing: 1 = generic only,
 * 0 = normal dispatch. Returns the previous value. Process-wide.
 */
IRDN_API int32_t irdn_set_force_generic(int32_t on);

#ifdef __cplusplus
}
#endif

#endif /* IRDN_H_ */
