// Host-side probe for the e2e path: can a sparse result return beat the
// full device->host copy of the filtered image?
//   1. host memcpy bandwidth (pinned -> pinned) with 1..T OpenMP threads, alone and while
//      the DMA engines run a concurrent H2D of the same size;
//   2. SM stores into mapped pinned host memory (zero-copy D2H): coalesced 16-byte stores;
//   3. DMA H2D / D2H reference figures.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp host_probe.cu -o host_probe
#include <cuda_runtime.h>
#include <omp.h>
#include <sched.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void par_copy(char* d, const char* s, size_t n, int nt) {
  const size_t part = 256 << 10;
  const long long parts = (n + part - 1) / part;
#pragma omp parallel for schedule(static) num_threads(nt)
  for (long long i = 0; i < parts; ++i) memcpy(d + i * part, s + i * part, std::min(part, n - (size_t)i * part));
}

__global__ void store_mapped(uint4* dst, size_t n16, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4(v, v + 1, v + 2, (uint32_t)i);
}
__global__ void store_mapped_u32(uint32_t* dst, size_t n4, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = v ^ (uint32_t)i;
}

int main() {
  cpu_set_t cs;
  sched_getaffinity(0, sizeof(cs), &cs);
  printf("host cpus (affinity) %d, omp max threads %d\n", CPU_COUNT(&cs), omp_get_max_threads());
  const size_t n = 42ull << 20;
  char *a, *b, *c;
  CK(cudaHostAlloc(&a, n, cudaHostAllocDefault));
  CK(cudaHostAlloc(&b, n, cudaHostAllocDefault));
  CK(cudaHostAlloc(&c, n, cudaHostAllocMapped));
  memset(a, 1, n); memset(b, 2, n); memset(c, 3, n);
  char* d;
  CK(cudaMalloc(&d, n));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // DMA reference
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    CK(cudaMemcpyAsync(d, a, n, cudaMemcpyHostToDevice, s)); CK(cudaStreamSynchronize(s));
    double t1 = now();
    CK(cudaMemcpyAsync(b, d, n, cudaMemcpyDeviceToHost, s)); CK(cudaStreamSynchronize(s));
    double t2 = now();
    if (rep == 2) printf("DMA 42 MiB: H2D %.1f GB/s  D2H %.1f GB/s\n", n / (t1 - t0) / 1e9, n / (t2 - t1) / 1e9);
  }
  int ths[] = {1, 2, 4, 8, 12, 16, 24, 32, 48, 64};
  for (int nt : ths) {
    if (nt > CPU_COUNT(&cs)) break;
    par_copy(b, a, n, nt);
    double best = 1e9, best_c = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      double t0 = now();
      par_copy(b, a, n, nt);
      best = std::min(best, now() - t0);
      // concurrently with an H2D DMA of the same size from a third buffer
      CK(cudaMemcpyAsync(d, c, n, cudaMemcpyHostToDevice, s));
      t0 = now();
      par_copy(b, a, n, nt);
      double tc = now() - t0;
      CK(cudaStreamSynchronize(s));
      best_c = std::min(best_c, tc);
    }
    printf("memcpy 42 MiB, %2d threads: %.1f GB/s alone, %.1f GB/s beside an H2D\n", nt, n / best / 1e9, n / best_c / 1e9);
  }
  // zero-copy stores
  char* cd;
  CK(cudaHostGetDevicePointer((void**)&cd, c, 0));
  size_t sizes[] = {1ull << 20, 4ull << 20, 16ull << 20, 42ull << 20};
  for (size_t sz : sizes) {
    for (int grid : {148, 296, 1184}) {
      store_mapped<<<grid, 256, 0, s>>>((uint4*)cd, sz / 16, 7);
      CK(cudaStreamSynchronize(s));
      double best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        double t0 = now();
        store_mapped<<<grid, 256, 0, s>>>((uint4*)cd, sz / 16, rep);
        CK(cudaStreamSynchronize(s));
        best = std::min(best, now() - t0);
      }
      double best32 = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        double t0 = now();
        store_mapped_u32<<<grid, 256, 0, s>>>((uint32_t*)cd, sz / 4, rep);
        CK(cudaStreamSynchronize(s));
        best32 = std::min(best32, now() - t0);
      }
      printf("SM stores to mapped host memory, %5.1f MiB, grid %4d: uint4 %.1f GB/s, u32 %.1f GB/s (incl. launch+sync)\n",
             sz / 1048576.0, grid, sz / best / 1e9, sz / best32 / 1e9);
    }
  }
  // zero-copy stores concurrent with an H2D DMA
  {
    double best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaStream_t s2; CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
      double t0 = now();
      CK(cudaMemcpyAsync(d, a, n, cudaMemcpyHostToDevice, s2));
      store_mapped<<<296, 256, 0, s>>>((uint4*)cd, (8ull << 20) / 16, rep);
      CK(cudaStreamSynchronize(s)); CK(cudaStreamSynchronize(s2));
      best = std::min(best, now() - t0);
      cudaStreamDestroy(s2);
    }
    printf("H2D 42 MiB + concurrent 8 MiB mapped stores: %.3f ms total\n", best * 1e3);
  }
  return 0;
}
