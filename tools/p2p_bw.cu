// NVLink peer-write bandwidth on one box (>= 2 GPUs, one process): what the
// product exchange of a flipping dressing step can reach.  Measures, for
// 1 GiB per direction between GPU 0 and GPU 1:
//   ce_1dir   cudaMemcpyPeerAsync 0 -> 1 (copy engine)
//   ce_2dir   both directions at once
//   sm_1dir   SM stores (16-byte, coalesced) from GPU 0 into GPU 1's memory
//   sm_2dir   both directions at once
// for several grid sizes of the SM kernel.  Prints one JSON line per case.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__global__ void k_copy16(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  const size_t bytes = (size_t)1 << 30;
  void *src[2], *dst[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes));
    CK(cudaMemset(src[d], d + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  auto run = [&](const char* name, int dirs, int grid, int reps) {
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      for (int d = 0; d < dirs; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < dirs; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        if (grid == 0)
          CK(cudaMemcpyPeerAsync(dst[1 - d], 1 - d, src[d], d, bytes, st[d]));
        else
          k_copy16<<<grid, 256, 0, st[d]>>>((const int4*)src[d], (int4*)dst[1 - d], bytes / 16);
        CK(cudaEventRecord(e1[d], st[d]));
      }
      float worst = 0.f;
      for (int d = 0; d < dirs; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = ms > worst ? ms : worst;
      }
      best = worst < best ? worst : best;
    }
    printf("{\"case\": \"%s\", \"grid\": %d, \"ms\": %.4f, \"GBps_per_dir\": %.1f}\n", name, grid, best,
           bytes / (best * 1e-3) / 1e9);
    fflush(stdout);
  };
  run("ce_1dir", 1, 0, 5);
  run("ce_2dir", 2, 0, 5);
  for (int g : {148, 296, 592, 1184, 2368}) {
    run("sm_1dir", 1, g, 5);
    run("sm_2dir", 2, g, 5);
  }
  return 0;
}
