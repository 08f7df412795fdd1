// tools/fp64_peak.cu -- measures the B200 fp64 (DFMA) peak that the roofline
// of the fp64-pipe-bound MHD stage is quoted against (MEASURED_PEAKS.json has
// only HBM and bf16).  Writes one JSON line to stdout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 8192;

__global__ void dfma_loop(double* out, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the work live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8;
  dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * CHAINS * double(ITERS) * threads * blocks;
  const double tf = flops / (best * 1e-3) / 1e12;
  const double nominal = 2.0 * 64 * sms * (clk * 1e3) / 1e12;
  printf("{\"fp64_dfma_tflops\": %.3f, \"best_ms\": %.4f, \"sms\": %d, \"clock_khz_attr\": %d, "
         "\"nominal_64fma_per_sm_tflops\": %.3f, \"how\": \"%d blocks x %d threads, %d independent DFMA "
         "chains x %d iters, best of 10, CUDA events\"}\n",
         tf, best, sms, clk, nominal, blocks, threads, CHAINS, ITERS);
  return 0;
}
