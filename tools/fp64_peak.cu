// FP64 FMA peak probe: independent FMA chains per thread, all SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void fma_kernel(double *out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char **argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 8);
  const int threads = argc > 1 ? atoi(argv[1]) : 512;
  const int per_sm = argc > 2 ? atoi(argv[2]) : 4;
  const int blocks = sms * per_sm, iters = 20000;
  fma_kernel<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 16.0 * iters * (double)threads * blocks;
  printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"warps_per_sm\": %d}\n",
         flops / best / 1e9, best, sms, threads / 32 * per_sm);
  return 0;
}
