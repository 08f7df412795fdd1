// divsqrt_check.cu -- test helper (not product code): compares the product
// build's branch-free ddiv / dsqrt (physics.cuh, PMHD_FAST_DIVSQRT) with the
// IEEE operators bit for bit on caller-supplied operands.
#include <cuda_runtime.h>

#include "physics.cuh"

namespace {
__global__ void k_check(const double* a, const double* b, long long n, unsigned long long* mism) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double x = a[t], y = b[t];
  const double q0 = x / y, q1 = pmhd_gpu::ddiv(x, y);
  const double s0 = sqrt(fabs(x)), s1 = pmhd_gpu::dsqrt(fabs(x));
  if (__double_as_longlong(q0) != __double_as_longlong(q1)) atomicAdd(&mism[0], 1ULL);
  if (__double_as_longlong(s0) != __double_as_longlong(s1)) atomicAdd(&mism[1], 1ULL);
}
}  // namespace

// Returns 0 and writes the division / sqrt mismatch counts, or a CUDA error code.
extern "C" int pmhd_test_divsqrt(const double* a, const double* b, long long n,
                                 unsigned long long out[2]) {
  double *da = nullptr, *db = nullptr;
  unsigned long long* dm = nullptr;
  cudaError_t e = cudaMalloc(&da, n * sizeof(double));
  if (!e) e = cudaMalloc(&db, n * sizeof(double));
  if (!e) e = cudaMalloc(&dm, 2 * sizeof(unsigned long long));
  if (!e) e = cudaMemcpy(da, a, n * sizeof(double), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(db, b, n * sizeof(double), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemset(dm, 0, 2 * sizeof(unsigned long long));
  if (!e) {
    k_check<<<(unsigned)((n + 255) / 256), 256>>>(da, db, n, dm);
    e = cudaGetLastError();
  }
  if (!e) e = cudaMemcpy(out, dm, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dm);
  return (int)e;
}
