// Isolation probe for the TMA / mbarrier building blocks (one variant per process).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VAR>
__global__ void k_load(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, uint8_t* out, int x, int y,
                       int bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const CUtensorMap* m = (VAR == 1) ? gmap : &map;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (VAR == 2) asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    if (VAR == 3) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(sm)),
          "l"(m), "r"(x), "r"(y), "r"(su32(&bar))
          : "memory");
    } else {
      const int off = VAR == 5 ? 128 : (VAR == 6 ? 16 : (VAR == 7 ? 256 : (VAR == 8 ? 512 : 0)));
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su32(sm + off)),
          "l"(m), "r"(x), "r"(y), "r"(0), "r"(su32(&bar))
          : "memory");
    }
  }
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(&bar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  int var = argc > 1 ? atoi(argv[1]) : 0;
  int bw = argc > 2 ? atoi(argv[2]) : 144, bh = argc > 3 ? atoi(argv[3]) : 34;
  int W = argc > 4 ? atoi(argv[4]) : 256, H = argc > 5 ? atoi(argv[5]) : 64;
  int l2 = argc > 6 ? atoi(argv[6]) : 0;
  int cx = argc > 7 ? atoi(argv[7]) : 16, cy = argc > 8 ? atoi(argv[8]) : 16;
  uint8_t *d_in, *d_dump;
  cudaMalloc(&d_in, (size_t)W * H);
  cudaMalloc(&d_dump, 65536);
  cudaMemset(d_in, 7, (size_t)W * H);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fnp;
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t strides[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[3] = {1, 1, 1};
  int rank = var == 3 ? 2 : 3;
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, d_in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int drv = 0;
  cudaDriverGetVersion(&drv);
  printf("xy=(%d,%d) var=%d box=%dx%d tensor=%dx%d l2=%d encode=%d drv=%d desc:", var, bw, bh, W, H, l2, (int)r, drv);
  for (int i = 0; i < 4; ++i) printf(" %016llx", (unsigned long long)((uint64_t*)&map)[i]);
  printf("\n");
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  cudaMemcpy(gmap, &map, sizeof(map), cudaMemcpyHostToDevice);
  int bytes = bw * bh;
  cudaFuncSetAttribute(k_load<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  switch (var) {
    case 0: case 4: k_load<0><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 1: k_load<1><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 2: k_load<2><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 3: k_load<3><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 5: k_load<5><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 6: k_load<6><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 7: k_load<7><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
    case 8: k_load<8><<<1, 128, bytes + 1024>>>(map, gmap, d_dump, cx, cy, bytes); break;
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("  -> %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
