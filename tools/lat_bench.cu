// Dependent-chain latencies on this GPU (clock64): DFMA, DADD, LDS.64 (pointer chase).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, int n) {
  __shared__ double sm[1024];
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; nxt[i] = (i * 37 + 11) & 1023; }
  __syncthreads();
  double a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { a = a + c; a = a + b; a = a + c; a = a + b; }
  long long t2 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) { p = nxt[p]; p = nxt[p]; p = nxt[p]; p = nxt[p]; }
  long long t3 = clock64();
  double s = 0; int q = p;
  for (int i = 0; i < n; ++i) { s = sm[q]; q = (int)(s * 1e9) & 1023; s = sm[q]; q = (int)(s * 1e9) & 1023; }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; out[3] = a + p + s; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  double h[4] = {1.0, 0.999999, 1e-9, 0}; cudaMemcpy(o, h, 32, cudaMemcpyHostToDevice);
  int n = 4096;
  lat<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, n); long long hc[4]; cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
  printf("DFMA dep latency %.1f cyc, DADD %.1f cyc, LDS.32 chase %.1f cyc, LDS.64+cvt chase %.1f cyc\n",
         hc[0] / (4.0 * n), hc[1] / (4.0 * n), hc[2] / (4.0 * n), hc[3] / (2.0 * n));
  return 0;
}
