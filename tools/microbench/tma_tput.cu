// TMA box-load throughput on B200: persistent CTAs stream boxes of a given shape from a
// large u16 tensor into shared memory (no compute) — is the tile kernel's staging cheap?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_tput tma_tput.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream(const __grid_constant__ CUtensorMap map, int bw, int bh, int tiles_x, int tiles_y, int frames,
                       int nstage, unsigned int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  const int bytes = bw * bh * 2;
  const int stride = (bytes + 1023) & ~1023;
  const int ntiles = tiles_x * tiles_y * frames;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int t, int s) {
    const int f = t / (tiles_x * tiles_y), tt = t % (tiles_x * tiles_y);
    const int x = (tt % tiles_x) * (bw - 16) - 8, y = (tt / tiles_x) * (bh - 4) - 2;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(sm + s * stride)),
        "l"(&map), "r"(x & ~7), "r"(y), "r"(f), "r"(su32(&bar[s]))
        : "memory");
  };
  int it = 0;
  uint32_t acc = 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < nstage; ++s)
      if ((int)blockIdx.x + s * (int)gridDim.x < ntiles) issue(blockIdx.x + s * gridDim.x, s);
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % nstage;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar[s])),
        "r"((it / nstage) & 1)
        : "memory");
    acc += sm[s * stride + (threadIdx.x * 4) % bytes];
    __syncthreads();
    if (threadIdx.x == 0 && t + nstage * (int)gridDim.x < ntiles) issue(t + nstage * gridDim.x, s);
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
  const int W = 640, H = 512, F = 256;  // 256 frames of c2-sized u16
  uint16_t* d;
  cudaMalloc(&d, (size_t)W * H * F * 2);
  cudaMemset(d, 1, (size_t)W * H * F * 2);
  unsigned int* sink;
  cudaMalloc(&sink, 64);
  void* fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fnp;
  struct Shape { int bw, bh; } shapes[] = {{144, 68}, {272, 36}, {144, 132}, {256, 64}, {72, 132}};
  for (auto sh : shapes) {
    for (int nstage : {1, 2}) {
      for (int cps : {4, 8}) {
        CUtensorMap map;
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)F};
        cuuint64_t str[2] = {(cuuint64_t)W * 2, (cuuint64_t)W * H * 2};
        cuuint32_t box[3] = {(cuuint32_t)sh.bw, (cuuint32_t)sh.bh, 1}, es[3] = {1, 1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int tiles_x = (W + (sh.bw - 16) - 1) / (sh.bw - 16), tiles_y = (H + (sh.bh - 4) - 1) / (sh.bh - 4);
        const int smem = nstage * (((sh.bw * sh.bh * 2) + 1023) & ~1023) + 1024;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = 148 * cps;
        stream<<<grid, 128, smem>>>(map, sh.bw, sh.bh, tiles_x, tiles_y, F, nstage, sink);
        cudaDeviceSynchronize();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        stream<<<grid, 128, smem>>>(map, sh.bw, sh.bh, tiles_x, tiles_y, F, nstage, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)tiles_x * tiles_y * F * sh.bw * sh.bh * 2;
        printf("{\"box\": \"%dx%d u16\", \"nstage\": %d, \"ctas_per_sm\": %d, \"GBps_smem_fill\": %.0f, \"us\": %.1f, \"err\": \"%s\"}\n",
               sh.bw, sh.bh, nstage, cps, bytes / (ms * 1e-3) / 1e9, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
