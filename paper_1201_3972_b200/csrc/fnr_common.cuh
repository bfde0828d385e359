// Shared device helpers and launch geometry for the FNR kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace irdn {

// Geometry of one pass: `batch` frames, each frame of GLOBAL size height x width.
// The input pointer addresses global row `in_row0` of frame 0 and holds rows
// [in_row0, in_row0 + in_rows); the output pointer addresses global row
// `row_begin` of frame 0, and the pass writes rows [row_begin, row_end).
// Window rows are clamped to [0, height-1] (replicate edge, image.py:117-123),
// then re-based to the input's first row: the strip must cover the clamped rows.
struct PassGeom {
  int64_t in_frame_stride;   // elements between frames of the input
  int64_t out_frame_stride;  // elements between frames of the output
  int64_t in_pitch;          // elements between rows of the input
  int64_t out_pitch;         // elements between rows of the output
  int32_t height;            // global frame height (clamp bound)
  int32_t width;
  int32_t in_row0;
  int32_t in_rows;
  int32_t row_begin;
  int32_t row_end;
  int32_t batch;
};

// ---- FMA-pipe integer helpers -------------------------------------------------
// On sm_100a VIMNMX(3), PRMT, LOP3, SHF and IADD3 all issue on the ALU pipe (64
// lanes/clk/SM, measured: profiles/alu_probe_r01.txt) while IMAD issues on the FMA
// pipe at the same rate. The min/max-heavy kernels are ALU-bound, so adds, subtracts
// and shifts that are not min/max go to the FMA pipe as IMADs.
// Integer multiply-add on the FMA pipe. `one` is an opaque runtime 1 (a kernel argument), so
// ptxas keeps IMAD instead of turning the add into IADD3, which would compete with the
// VIMNMX3 / PRMT / LOP3 stream for the ALU pipe (measured ALU-bound at 92%).
__device__ __forceinline__ uint32_t fma_add(uint32_t a, uint32_t one, uint32_t b) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
  return r;
}
// a - b on the FMA pipe (b * 0xFFFFFFFF + a).
__device__ __forceinline__ uint32_t fma_sub(uint32_t a, uint32_t minus_one, uint32_t b) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(minus_one), "r"(a));
  return r;
}
// (a >> 16) | (b << 16) with two IMADs instead of one PRMT (moves the shift to the FMA pipe).
__device__ __forceinline__ uint32_t shift_pair(uint32_t a, uint32_t b, uint32_t k65536) {
  uint32_t hi, r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(k65536));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(k65536), "r"(hi));
  return r;
}
// PDL: wait for the previous grid in the stream (no-op without PDL), then let the next
// grid start launching (its CTAs fill SMs this grid has left and wait the same way).
__device__ __forceinline__ void pdl_wait_and_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Block-wide reduction of the two FNR counters followed by ONE 64-bit atomic
// per counter per block (filters.py:121-126 merges per-band counters the same way).
template <int NTHREADS>
__device__ __forceinline__ void block_add_counts(uint32_t detected, uint32_t replaced,
                                                 unsigned long long* counts) {
  __shared__ uint32_t s_det[NTHREADS / 32], s_rep[NTHREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    detected += __shfl_xor_sync(0xffffffffu, detected, o);
    replaced += __shfl_xor_sync(0xffffffffu, replaced, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_det[warp] = detected; s_rep[warp] = replaced; }
  __syncthreads();
  if (warp == 0) {
    uint32_t d = lane < NTHREADS / 32 ? s_det[lane] : 0u;
    uint32_t r = lane < NTHREADS / 32 ? s_rep[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d += __shfl_xor_sync(0xffffffffu, d, o);
      r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if (lane == 0) {
      if (d) atomicAdd(&counts[0], (unsigned long long)d);
      if (r) atomicAdd(&counts[1], (unsigned long long)r);
    }
  }
}

}  // namespace irdn
