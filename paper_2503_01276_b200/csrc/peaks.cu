// Measured device peaks for the roofline denominators that MEASURED_PEAKS.json lacks (SURVEY.md
// §8(d): "measure [the FP64 peak] with a DFMA loop before claiming a bound"): FP64 FMA throughput
// and shared-memory load bandwidth of this GPU, timed with CUDA events, best of several runs.
// Standalone executable (lib/mch_peaks); prints one JSON line.  Not part of the hot path.
#include <cuda_runtime.h>

#include <cstdio>

// 8 independent FMA chains per thread, kIter rounds: 16 * kIter flops per thread
constexpr int kIter = 4096;
__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIter; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// every thread streams 8-byte loads over a 32 KB shared array (consecutive lanes, conflict-free)
constexpr int kSmemDoubles = 4096;
constexpr int kSmemIter = 2048;
__global__ void k_smem(double* out) {
  __shared__ double buf[kSmemDoubles];
  for (int i = threadIdx.x; i < kSmemDoubles; i += blockDim.x) buf[i] = i * 0.5;
  __syncthreads();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int idx = threadIdx.x;
  for (int it = 0; it < kSmemIter; it++) {
#pragma unroll
    for (int u = 0; u < 4; u++) acc[u] += buf[(idx + u * 1024) & (kSmemDoubles - 1)];
    idx = (idx + 256) & (kSmemDoubles - 1);
  }
  const double s = acc[0] + acc[1] + acc[2] + acc[3];
  if (s == -1.0) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 64) != cudaSuccess) {
    printf("{\"error\": \"no device\"}\n");
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  double best_fp64 = 0.0, best_smem = 0.0;
  for (int rep = 0; rep < 6; rep++) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * kIter * (double)blocks * threads;
    if (rep > 0 && flops / (ms * 1e-3) > best_fp64) best_fp64 = flops / (ms * 1e-3);
    cudaEventRecord(e0);
    k_smem<<<blocks, threads>>>(out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 8.0 * 4.0 * kSmemIter * (double)blocks * threads;
    if (rep > 0 && bytes / (ms * 1e-3) > best_smem) best_smem = bytes / (ms * 1e-3);
  }
  const cudaError_t err = cudaGetLastError();
  printf("{\"fp64_tflops\": %.3f, \"smem_tbs\": %.3f, \"sms\": %d, \"clock_mhz\": %.0f, \"how\": "
         "\"k_dfma: 8 independent fp64 FMA chains x %d per thread, %d CTAs x %d threads, best of 5; k_smem: "
         "conflict-free 8-byte shared loads, same grid, best of 5\", \"status\": \"%s\"}\n",
         best_fp64 * 1e-12, best_smem * 1e-12, sms, clk * 1e-3, kIter, blocks, threads,
         err == cudaSuccess ? "ok" : cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
