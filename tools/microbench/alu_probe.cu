// Microbenchmarks for the selection/detection kernels' building blocks on B200.
// Measures issue throughput of the packed integer min/max instructions the
// FNR kernels are made of (VIMNMX.U16x2, VIMNMX3.U16x2, IADD3, PRMT, LOP3),
// HBM copy bandwidth for u8 streams and back-to-back launch latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_probe alu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t min2(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t min3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("{.reg .b32 t; min.u16x2 t, %1, %2; min.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t max3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("{.reg .b32 t; max.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}

template <int OP>
__global__ void alu_kernel(uint32_t* out, uint32_t seed) {
  uint32_t v[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) v[i] = seed * (threadIdx.x + 1 + i * 77);
  uint32_t b = seed ^ 0x5bd1e995u, c = seed * 31u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      if (OP == 0) v[i] = min2(v[i], v[(i + 1) % CHAINS]);  // VIMNMX.U16x2 (no fusion)
      if (OP == 1) v[i] = min3(v[i], b, c);               // VIMNMX3.U16x2
      if (OP == 2) v[i] = max3(v[i], b, c) ;              // VIMNMX3.U16x2 (max)
      if (OP == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(b));   // IADD3
      if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(v[i]) : "r"(b));  // PRMT
      if (OP == 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[i]) : "r"(b), "r"(c));  // LOP3
      if (OP == 6) { uint32_t t = min3(v[i], b, c); v[i] = max3(t, b, c); }  // mixed min/max pair
      if (OP == 8) { uint32_t t; asm volatile("min.f16x2 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // HMNMX2
      if (OP == 9) { uint32_t t; asm volatile("min.bf16x2 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // bf16 min
      if (OP == 10) { uint32_t t; if (i & 1) asm volatile("min.f16x2 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); else asm volatile("min.u16x2 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // mixed
      if (OP == 11) { uint32_t t; asm volatile("min.f32 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // FMNMX
      if (OP == 12) { uint32_t t; if (i & 1) asm volatile("add.u32 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); else asm volatile("min.u16x2 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // VIMNMX + IADD mix
      if (OP == 13) { uint32_t t; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(v[i]), "r"(c), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // IMAD reg
      if (OP == 14) { uint32_t t; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(c)); v[i] = t ^ b; }  // IMAD.HI (+LOP3)
      if (OP == 15) { uint32_t t; if (i & 1) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(v[i]), "r"(c), "r"(v[(i + 1) % CHAINS])); else asm volatile("{.reg .b32 q; min.u16x2 q, %1, %2; min.u16x2 %0, q, %3;}" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS]), "r"(b)); v[i] = t; }  // VIMNMX3 + IMAD
      if (OP == 16) { uint32_t t; asm volatile("add.u32 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); asm volatile("add.u32 %0, %0, %1;" : "+r"(t) : "r"(b)); v[i] = t; }  // IADD3
      if (OP == 7) { uint32_t t; asm volatile("min.u32 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // IMNMX.U32
      if (OP == 17) { uint32_t t; if (i & 1) asm volatile("{.reg .b32 q; add.u32 q, %1, %2; sub.u32 %0, q, %3;}" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS]), "r"(b)); else asm volatile("min.u16x2 %0, %1, %2;" : "=r"(t) : "r"(v[i]), "r"(v[(i + 1) % CHAINS])); v[i] = t; }  // VIMNMX + IADD3 a+b-c
      if (OP == 18) { const uint32_t a = v[i], bb = v[(i + 1) % CHAINS]; uint32_t lo, hi; asm volatile("min.u16x2 %0, %1, %2;" : "=r"(lo) : "r"(a), "r"(bb)); asm volatile("{.reg .b32 q; add.u32 q, %1, %2; sub.u32 %0, q, %3;}" : "=r"(hi) : "r"(a), "r"(bb), "r"(lo)); v[i] = lo; v[(i + 1) % CHAINS] = hi; }  // cx as min + (a+b-min)
      if (OP == 19) { const uint32_t a = v[i], bb = v[(i + 1) % CHAINS]; uint32_t lo, hi; asm volatile("min.u16x2 %0, %1, %2;" : "=r"(lo) : "r"(a), "r"(bb)); asm volatile("max.u16x2 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(bb)); v[i] = lo; v[(i + 1) % CHAINS] = hi; }  // cx as min + max
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc ^= v[i];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

__global__ void copy_u8(const int4* __restrict__ in, int4* __restrict__ out, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n16; i += stride) out[i] = in[i];
}

__global__ void empty_kernel() {}

template <int OP>
int run_alu(const char* name, int insts_per_chain_iter) {
  uint32_t* d; CK(cudaMalloc(&d, 4096));
  int blocks = 148 * 8, threads = 256;
  alu_kernel<OP><<<blocks, threads>>>(d, 3);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) alu_kernel<OP><<<blocks, threads>>>(d, 3 + r);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  double lane_ops = 5.0 * blocks * threads * (double)ITERS * CHAINS * insts_per_chain_iter;
  double tops = lane_ops / (ms * 1e-3) / 1e12;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_sm_clk = lane_ops / (ms * 1e-3) / 148.0 / (clk * 1e3);
  printf("{\"probe\": \"%s\", \"Tlane_ops_per_s\": %.3f, \"lane_ops_per_clk_per_sm_at_max_clk\": %.2f, \"ms\": %.3f}\n",
         name, tops, per_sm_clk, ms);
  cudaFree(d);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"max_clk_khz\": %d, \"smem_optin\": %zu}\n",
         p.name, p.multiProcessorCount, l2, clk, p.sharedMemPerBlockOptin);
  run_alu<0>("vimnmx_u16x2", 1);
  run_alu<1>("vimnmx3_u16x2_min", 1);
  run_alu<2>("vimnmx3_u16x2_max", 1);
  run_alu<3>("iadd", 1);
  run_alu<4>("prmt", 1);
  run_alu<5>("lop3", 1);
  run_alu<6>("vimnmx3_minmax_pair", 2);
  run_alu<7>("imnmx_u32", 1);
  run_alu<8>("hmnmx2_f16x2", 1);
  run_alu<9>("hmnmx2_bf16x2", 1);
  run_alu<10>("mixed_vimnmx_hmnmx2", 1);
  run_alu<11>("fmnmx_f32", 1);
  run_alu<12>("mixed_vimnmx_iadd", 1);
  run_alu<13>("imad_reg", 1);
  run_alu<14>("imad_hi_plus_lop3", 2);
  run_alu<15>("mixed_vimnmx3_imad", 1);
  run_alu<16>("iadd3_3input", 1);
  run_alu<17>("mixed_vimnmx_iadd3_sub", 1);
  run_alu<18>("cx_min_plus_addsub", 2);
  run_alu<19>("cx_min_max", 2);

  // HBM copy: 2 GiB in + 2 GiB out
  size_t bytes = (size_t)2 << 30;
  int4 *din, *dout; CK(cudaMalloc(&din, bytes)); CK(cudaMalloc(&dout, bytes));
  cudaMemset(din, 1, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    copy_u8<<<g, 256>>>(din, dout, bytes / 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) copy_u8<<<g, 256>>>(din, dout, bytes / 16);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("{\"probe\": \"hbm_copy_int4\", \"grid\": %d, \"GBps_rw\": %.1f}\n", g, 10.0 * 2 * bytes / (ms * 1e-3) / 1e9);
  }
  // launch latency: back-to-back empty kernels
  empty_kernel<<<1, 32>>>(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < 1000; ++r) empty_kernel<<<148, 128>>>();
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\": \"empty_launch_back_to_back_us\", \"value\": %.3f}\n", ms * 1e3 / 1000);
  return 0;
}
