// tma_probe.cu -- standalone check of the TMA helpers (tma.cuh): one 34 x 10
// box of a pitched 3D double array into shared memory, copied back out.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#include "tma.cuh"

using namespace pmhd_gpu;

template <int SMEM_EXTRA>
__global__ void k_probe(const CUtensorMap* map, double* out, int x, int y, int z) {
  extern __shared__ __align__(16) unsigned char raw[];
  double* box = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(box + 340 + SMEM_EXTRA);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init_fence(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, 340 * 8);
    tma_load_3d(box, map, bar, x, y, z);
  }
  mbar_wait(bar, 0);
  for (int q = threadIdx.x; q < 340; q += blockDim.x) out[q] = box[q];
}

int main(int argc, char** argv) {
  const int n1 = 68, n2 = 68, n3 = 68, sx = 96, sy = sx * (n2 + 1);
  const size_t n = size_t(n3 + 1) * sy + 64;
  std::vector<double> h(n);
  for (size_t q = 0; q < n; ++q) h[q] = double(q);
  double *d = nullptr, *o = nullptr;
  cudaMalloc(&d, n * 8);
  cudaMalloc(&o, 340 * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int fails = 0;
  for (int variant = 0; variant < 4; ++variant) {
    const int xo = variant & 1;  // base one element early (8 B offset array)
    double* base = d + 32 + xo;  // "array" at element 32 (+1: 8 B misaligned)
    CUtensorMap map;
    const cuuint64_t dim[3] = {cuuint64_t(n1 + 1 + xo), cuuint64_t(n2 + 1), cuuint64_t(n3 + 1)};
    const cuuint64_t stride[2] = {cuuint64_t(sx) * 8, cuuint64_t(sy) * 8};
    const cuuint32_t bx[3] = {34, 10, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base - xo, dim, stride, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* dm = nullptr;
    cudaMalloc(&dm, sizeof(map));
    cudaMemcpy(dm, &map, sizeof(map), cudaMemcpyHostToDevice);
    const int i0 = 5, j0 = 3, k = 7;
    const int smem = 340 * 8 + 64 + 256 + ((variant & 2) ? 150000 : 0);
    cudaError_t e;
    if (variant & 2) {
      cudaFuncSetAttribute(k_probe<18750>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_probe<18750><<<1, 256, smem>>>(dm, o, i0 - 1 + xo, j0 - 1, k);
    } else {
      k_probe<0><<<1, 256, smem>>>(dm, o, i0 - 1 + xo, j0 - 1, k);
    }
    e = cudaDeviceSynchronize();
    std::vector<double> got(340);
    cudaMemcpy(got.data(), o, 340 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r2 = 0; r2 < 10; ++r2)
      for (int c = 0; c < 34; ++c) {
        const double want = h[32 + xo + size_t(k) * sy + size_t(j0 - 1 + r2) * sx + (i0 - 1 + c)];
        if (got[r2 * 34 + c] != want) ++bad;
      }
    printf("variant %d (xoff %d, big smem %d): encode %d, kernel %s, %d mismatches\n", variant, xo, (variant & 2) ? 1 : 0,
           (int)r, cudaGetErrorString(e), bad);
    if (e != cudaSuccess || bad) ++fails;
    if (e != cudaSuccess) break;
    cudaFree(dm);
  }
  return fails ? 1 : 0;
}
