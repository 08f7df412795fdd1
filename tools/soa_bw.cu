// tools/soa_bw.cu -- does the update kernel's access shape (a 32 x 8 (i, j)
// tile marching k, one double from each of NA separate arrays per cell) lose
// DRAM bandwidth against the same bytes laid out row-interleaved (the NA rows
// of one (k, j) adjacent in memory)?  Prints GB/s for both layouts.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o soa_bw tools/soa_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256, P = 264, NA = 32, SEG = 16;

template <bool INTERLEAVED>
__global__ void __launch_bounds__(256) k_read(const double* __restrict__ a, double* __restrict__ out) {
  const int i = blockIdx.x * 32 + (threadIdx.x & 31), j = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int kb = blockIdx.z * SEG;
  double s = 0.0;
  for (int k = kb; k < kb + SEG; ++k) {
#pragma unroll 8
    for (int v = 0; v < NA; ++v) {
      size_t id;
      if (INTERLEAVED) id = ((size_t(k) * N + j) * NA + v) * P + i;
      else id = size_t(v) * N * N * P + (size_t(k) * N + j) * P + i;
      s += __ldg(a + id);
    }
    out[(size_t(k) * N + j) * P + i] = s;
  }
}

int main() {
  const size_t n = size_t(NA) * N * N * P;
  double *a, *o;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&o, size_t(N) * N * P * 8);
  cudaMemset(a, 0, n * 8);
  dim3 g(N / 32, N / 8, N / SEG);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep)
    for (int lay = 0; lay < 2; ++lay) {
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) {
        if (lay) k_read<true><<<g, 256>>>(a, o);
        else k_read<false><<<g, 256>>>(a, o);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = 5.0 * (double(NA) + 1) * N * N * N * 8;
      printf("%s: %.3f ms/launch, %.0f GB/s\n", lay ? "row-interleaved" : "separate arrays", ms / 5,
             bytes / (ms / 5 * 1e-3) / 1e9 / 5);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
