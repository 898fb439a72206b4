// fp64_peak.cu — measured FP64 multiply throughput of this B200 (the
// denominator of the DIS "pairs/s" row): every thread runs
// 8 independent dependent chains of DMUL (`__dmul_rn`, the instruction the
// DIS kernels issue), 148 x 8 blocks of 256 threads, CUDA events around a
// warm launch.  Prints one JSON object: dmul/s and the FLOP/s of the same
// rate counted as FMA pairs.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmul(double* out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __dmul_rn(x[j], a);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.0) out[0] = s;  // keep the chains live
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * 8, threads = 256, iters = 1 << 16;
  k_dmul<<<blocks, threads>>>(d, 1024, 0.9999999);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    k_dmul<<<blocks, threads>>>(d, iters, 0.9999999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double n = (double)blocks * threads * iters * 8.0;
  const double dmul_s = n / (best * 1e-3);
  printf("{\"dmul_per_s\": %.4e, \"fp64_fma_tflops_equiv\": %.2f, \"sms\": %d, \"ms\": %.3f, "
         "\"how\": \"8 independent __dmul_rn chains per thread, %d blocks x %d threads x %d iterations, "
         "best of 3\"}\n",
         dmul_s, 2.0 * dmul_s / 1e12, nsm, best, blocks, threads, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
