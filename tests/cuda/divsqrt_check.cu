// divsqrt_check.cu -- test helper (not product code): compares the branch-free
// ddiv / dsqrt / drsqrt of physics.cuh with the IEEE operators on
// caller-supplied operands.  Built twice: with the product's flags
// (PMHD_DIVSQRT_1ULP: within 1 ulp; drsqrt(x) against the correctly rounded
// 1 / sqrt(x)) and with PMHD_FAST_DIVSQRT alone (bit-identical to IEEE; that
// build has no drsqrt).
#include <cuda_runtime.h>

#include "physics.cuh"

namespace {
// distance in units in the last place between two finite doubles of one sign
__device__ unsigned long long ulps(double p, double q) {
  const long long a = __double_as_longlong(p), b = __double_as_longlong(q);
  return (unsigned long long)(a > b ? a - b : b - a);
}

// mism[0..1]: division / sqrt results that differ from IEEE; mism[2..3]: the
// largest distance in ulps; mism[4..5]: the same for drsqrt against the IEEE
// expression it replaces, 1 / sqrt(x) (two roundings, itself up to ~1 ulp
// from the exact reciprocal root)
__global__ void k_check(const double* a, const double* b, long long n, unsigned long long* mism) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double x = a[t], y = b[t];
  const double q0 = x / y, q1 = pmhd_gpu::ddiv(x, y);
  const double s0 = sqrt(fabs(x)), s1 = pmhd_gpu::dsqrt(fabs(x));
  if (__double_as_longlong(q0) != __double_as_longlong(q1)) atomicAdd(&mism[0], 1ULL);
  if (__double_as_longlong(s0) != __double_as_longlong(s1)) atomicAdd(&mism[1], 1ULL);
  atomicMax(&mism[2], ulps(q0, q1));
  atomicMax(&mism[3], ulps(s0, s1));
#ifdef PMHD_HAVE_DRSQRT
  const double ax = fabs(x);
  if (ax > 0.0) {
    const double r0 = 1.0 / sqrt(ax), r1 = pmhd_gpu::drsqrt(ax);
    if (__double_as_longlong(r0) != __double_as_longlong(r1)) atomicAdd(&mism[4], 1ULL);
    atomicMax(&mism[5], ulps(r0, r1));
  }
#endif
}
}  // namespace

// Returns 0 and writes the division / sqrt / rsqrt mismatch counts and their
// largest ulp distances (out[0..5]; out[4..5] stay 0 in a build without
// drsqrt), or a CUDA error code.
extern "C" int pmhd_test_divsqrt(const double* a, const double* b, long long n,
                                 unsigned long long out[6]) {
  double *da = nullptr, *db = nullptr;
  unsigned long long* dm = nullptr;
  cudaError_t e = cudaMalloc(&da, n * sizeof(double));
  if (!e) e = cudaMalloc(&db, n * sizeof(double));
  if (!e) e = cudaMalloc(&dm, 6 * sizeof(unsigned long long));
  if (!e) e = cudaMemcpy(da, a, n * sizeof(double), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(db, b, n * sizeof(double), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemset(dm, 0, 6 * sizeof(unsigned long long));
  if (!e) {
    k_check<<<(unsigned)((n + 255) / 256), 256>>>(da, db, n, dm);
    e = cudaGetLastError();
  }
  if (!e) e = cudaMemcpy(out, dm, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dm);
  return (int)e;
}
