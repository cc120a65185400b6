// FP64 outer-product microbenchmark: TMxTN register tile, operands from shared
// memory each k-step (the k-means assign inner loop without global traffic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_outer tools/fp64_outer.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int TM, int TN>
__global__ void outer_kernel(double *out, int iters) {
  __shared__ double As[16][TM * 16 + 2];
  __shared__ double Bs[16][TN * 8 + 1];
  for (int i = threadIdx.x; i < 16 * (TM * 16 + 2); i += blockDim.x) (&As[0][0])[i] = i * 1e-3;
  for (int i = threadIdx.x; i < 16 * (TN * 8 + 1); i += blockDim.x) (&Bs[0][0])[i] = i * 2e-3;
  __syncthreads();
  const int tx = threadIdx.x & 7, ty = (threadIdx.x >> 3) & 15;
  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + 8 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) s += acc[i][j];
  if (s == 1.2345) out[0] = s;
}

template <int TM, int TN>
void run(int threads, int per_sm, int sms, double *out) {
  const int iters = 2000, blocks = sms * per_sm;
  outer_kernel<TM, TN><<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    outer_kernel<TM, TN><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * TM * TN * 16.0 * iters * (double)threads * blocks;
  cudaFuncAttributes attr;
  cudaFuncGetAttributes(&attr, outer_kernel<TM, TN>);
  printf("TM=%d TN=%d threads=%d blocks/SM=%d warps/SM=%d regs=%d: %.2f TFLOP/s\n", TM, TN, threads,
         per_sm, threads / 32 * per_sm, attr.numRegs, flops / best / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 8);
  run<8, 8>(128, 1, sms, out);
  run<8, 8>(128, 2, sms, out);
  run<8, 8>(128, 3, sms, out);
  run<8, 8>(128, 4, sms, out);
  run<8, 4>(128, 2, sms, out);
  run<8, 4>(128, 4, sms, out);
  run<8, 4>(128, 6, sms, out);
  run<4, 4>(128, 8, sms, out);
  return 0;
}
