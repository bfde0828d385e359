// Issue-rate probe for the instruction mix of the dense 3x3 kernel (round 2).
//
// Question it answers: which execution pipe (and at what rate) runs the packed
// f16x2 arithmetic (HADD2 / HMUL2 / HFMA2 incl. .SAT / .RELU and the |x| / -x
// operand modifiers) on sm_100a, and how it dual-issues beside VIMNMX3.U16x2
// (ALU pipe) and IMAD (FMA pipe). 16 independent chains per thread so latency
// never limits the rate; each probe reports thread-instructions / clk / SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
// Check the SASS (cuobjdump -sass) that every probe is the instruction it names.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 16;
constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t vmin3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("{.reg .b32 t; min.u16x2 t, %1, %2; min.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t hfma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t hfma_relu(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("fma.rn.relu.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t hfma_sat(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("fma.rn.sat.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t hadd(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t hsub(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t hmul_sat_abs(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("{.reg .b32 t; abs.f16x2 t, %1; mul.rn.sat.f16x2 %0, t, %2;}" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("{.reg .b32 t; add.u32 t, %1, %2; sub.u32 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t ffma(uint32_t a, uint32_t b, uint32_t c) {
  float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)), "f"(__uint_as_float(c))); return __float_as_uint(r);
}

// One op per chain per iteration; OPs that mix take chain parity / index mod 3 to alternate.
template <int OP>
__device__ __forceinline__ uint32_t step(int i, uint32_t v, uint32_t w, uint32_t b, uint32_t c) {
  switch (OP) {
    case 0: return vmin3(v, b, c);                     // VIMNMX3.U16x2   (ALU)
    case 1: return imad(v, b, c);                      // IMAD            (FMA)
    case 2: return hfma(v, b, c);                      // HFMA2
    case 3: return hfma_relu(v, b, c);                 // HFMA2.RELU
    case 4: return hfma_sat(v, b, c);                  // HFMA2.SAT
    case 5: return hadd(v, b);                         // HADD2
    case 6: return hmul_sat_abs(v, b);                 // HMUL2.SAT |x|
    case 7: return iadd3(v, b, c);                     // IADD3
    case 8: return ffma(v, b, c);                      // FFMA
    case 9: return prmt(v, b);                         // PRMT
    case 10: return (i & 1) ? hfma(v, b, c) : vmin3(v, b, c);        // HFMA2 : VIMNMX3 = 1:1
    case 11: return (i & 1) ? imad(v, b, c) : vmin3(v, b, c);        // IMAD : VIMNMX3 = 1:1
    case 12: return (i & 1) ? hfma(v, b, c) : imad(v, b, c);         // HFMA2 : IMAD = 1:1
    case 13: return (i % 3 == 0) ? vmin3(v, b, c) : hfma(v, b, c);   // VIMNMX3 : HFMA2 = 1:2
    case 14: return (i & 1) ? hsub(v, w) : vmin3(v, b, c);           // HADD2(sub) : VIMNMX3
    case 15: return (i & 1) ? iadd3(v, b, c) : hfma(v, b, c);        // IADD3 : HFMA2
    case 16: return (i & 1) ? prmt(v, b) : hfma(v, b, c);            // PRMT : HFMA2
    case 17: return (i & 1) ? ffma(v, b, c) : vmin3(v, b, c);        // FFMA : VIMNMX3
    case 18: return (i % 4 == 0) ? imad(v, b, c) : ((i & 1) ? hfma(v, b, c) : vmin3(v, b, c));  // mix 1:2:1
    default: return v;
  }
}

template <int OP>
__global__ void probe(uint32_t* out, uint32_t seed) {
  uint32_t v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = 0x64006400u + ((seed * (threadIdx.x + 1 + i * 77)) & 0x00FF00FFu);
  const uint32_t b = 0x3C003C00u ^ (seed & 1u), c = 0x00010001u + (seed & 2u);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = step<OP>(i, v[i], v[(i + 5) % CH], b, c);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc ^= v[i];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

template <int OP>
int run(const char* name, uint32_t* d, int sms, double clk_khz) {
  const int blocks = sms * 8, threads = 256;
  probe<OP><<<blocks, threads>>>(d, 1);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    probe<OP><<<blocks, threads>>>(d, 1);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double inst = (double)blocks * threads * ITERS * CH;  // thread-instructions
  const double per_clk_sm = inst / (best * 1e-3) / (clk_khz * 1e3) / sms;
  printf("{\"probe\": \"%s\", \"thread_inst_per_clk_per_sm\": %.2f, \"ms\": %.4f}\n", name, per_clk_sm, best);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"max_clk_khz\": %d}\n", p.name, p.multiProcessorCount, clk);
  uint32_t* d;
  CK(cudaMalloc(&d, 4096));
  const int s = p.multiProcessorCount;
  run<0>("VIMNMX3.U16x2", d, s, clk);
  run<1>("IMAD", d, s, clk);
  run<2>("HFMA2", d, s, clk);
  run<3>("HFMA2.RELU", d, s, clk);
  run<4>("HFMA2.SAT", d, s, clk);
  run<5>("HADD2", d, s, clk);
  run<6>("HMUL2.SAT|x|", d, s, clk);
  run<7>("IADD3", d, s, clk);
  run<8>("FFMA", d, s, clk);
  run<9>("PRMT", d, s, clk);
  run<10>("HFMA2+VIMNMX3 1:1", d, s, clk);
  run<11>("IMAD+VIMNMX3 1:1", d, s, clk);
  run<12>("HFMA2+IMAD 1:1", d, s, clk);
  run<13>("VIMNMX3+HFMA2 1:2", d, s, clk);
  run<14>("HADD2sub+VIMNMX3 1:1", d, s, clk);
  run<15>("IADD3+HFMA2 1:1", d, s, clk);
  run<16>("PRMT+HFMA2 1:1", d, s, clk);
  run<17>("FFMA+VIMNMX3 1:1", d, s, clk);
  run<18>("IMAD:HFMA2:VIMNMX3 1:2:1", d, s, clk);
  return 0;
}
