// FP64 FMA throughput microbenchmark: the roofline denominator for the fused
// N-1 sweep (MEASURED_PEAKS.json carries HBM and bf16 only). 16 independent
// DFMA chains per thread, grid a multiple of the SM count, timed with events.
#include <cuda_runtime.h>

namespace tgb {

namespace {

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

// Returns TFLOP/s (2 flops per DFMA); best of 5 runs.
double measure_fp64_peak(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  k_dfma<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm-up
  double best = 0.0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16.0 * iters * static_cast<double>(blocks) * threads;
    if (ms > 0.f) best = flops / (ms * 1e-3) / 1e12 > best ? flops / (ms * 1e-3) / 1e12 : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

}  // namespace tgb
