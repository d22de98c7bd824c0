// FP64 FMA throughput of the device (the denominator of the elastomer
// kernel's fp64 compute fraction; MEASURED_PEAKS.json has no fp64 figure).
// Every thread runs 8 independent DFMA chains; the result is printed as one
// JSON line. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   tools/fp64_peak.cu -o paper_2301_08343_b200/_lib/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, mhz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int threads = 256, blocks = sms * 8, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * double(blocks) * threads;
  std::printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"clock_mhz_attr\": %d, "
              "\"how\": \"8 independent DFMA chains per thread, %d blocks x %d threads x %d "
              "iterations, best of 5, CUDA events\"}\n",
              flops / (best * 1e-3) / 1e12, best, sms, mhz / 1000, blocks, threads, iters);
  return 0;
}
