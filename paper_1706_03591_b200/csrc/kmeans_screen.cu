// FP32 screen of the k-means assignment (kmeans.py:54-61, 96-97) with an exact
// FP64 fallback: labels are bit-identical to the pure FP64 path.
//
// The reference label of row i is the first argmin over j of the FP64
// GEMM-form distance D_ij = max(0, (|f|^2 - 2 f.c_j) + |c_j|^2). The screen
// computes the same form in FP32 from FP32-rounded features and centroids,
// E_ij, on the FP32 pipe (twice the FP64 rate on B200). For FP32-rounded
// inputs, a sum of d products, and three more roundings,
//   |E_ij - T_ij| <= (d + 4) u32 (|f_i| + |c_j|)^2 =: delta_ij
// (T = the exact distance; |D - T| is ~1e9 times smaller and covered by the
// extra term below), so if the FP32 gap between the best and the second best
// exceeds 2 delta_i with delta_i = (d + 5) u32 (|f_i| + max_j |c_j|)^2, every
// D_ij (j != best) exceeds D_i,best strictly (and is positive): the FP64
// first-argmin is the FP32 argmin. Such rows are decided here with Hamerly
// bounds widened by delta (ub = sqrt(E1 + delta), lb = sqrt(max(E2 - delta, 0)));
// every other row is appended to a list the FP64 assignment then recomputes.
// On configs[4]-shape features (tools/fp32_screen_sim.py) 99.9% of rows are
// decided and the largest observed |E - D| is 3% of delta.
//
// No tensor cores (north_star): SIMT FFMA, 64 rows x 64 centroids per pass,
// 4 x 4 per thread, row tiles double-buffered with cp.async.
#include "common.cuh"
#include "kmeans_screen.cuh"

namespace {

constexpr int kSRT = 16, kSCT = 16, kSTM = 4, kSTN = 4;
constexpr int kSThreads = kSRT * kSCT;  // 256
constexpr int kSBM = kSRT * kSTM;       // 64 rows per tile
constexpr int kSBN = kSCT * kSTN;       // 64 centroids per pass

// F (fp64, ld) -> F32 (ld32, zero padding to ld32), fn32 = |F32 row|^2 (fp32)
__global__ void f32_convert_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                                   float *__restrict__ f32, int64_t ld32, float *__restrict__ fn32) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < n; r += warps) {
    float s = 0.0f;
    for (int64_t t = lane; t < ld32; t += 32) {
      const float v = t < d ? (float)f[r * ld + t] : 0.0f;
      f32[r * ld32 + t] = v;
      s = fmaf(v, v, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) fn32[r] = s;
  }
}

// centroids -> transposed fp32 tile [d][kpad] (zero past k), cn32 (+inf past
// k), and cmax = max_j |c_j| (fp64, from cnorm) for the error bound
__global__ void c32_convert_kernel(const double *__restrict__ c, int64_t k, int64_t d,
                                   int64_t ldc, const double *__restrict__ cnorm, int kpad,
                                   float *__restrict__ c32t, float *__restrict__ cn32,
                                   double *__restrict__ cmax) {
  __shared__ double red[32];
  for (int64_t e = threadIdx.x; e < d * kpad; e += blockDim.x) {
    const int64_t t = e / kpad, j = e - t * kpad;
    c32t[e] = j < k ? (float)c[j * ldc + t] : 0.0f;
  }
  double m = 0.0;
  for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
    if (j < k) {
      float s = 0.0f;
      for (int64_t t = 0; t < d; ++t) {
        const float v = (float)c[j * ldc + t];
        s = fmaf(v, v, s);
      }
      cn32[j] = s;
      m = fmax(m, cnorm[j]);
    } else {
      cn32[j] = INFINITY;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) m = fmax(m, red[w]);
    cmax[0] = sqrt(fmax(m, red[0]));
  }
}

__device__ __forceinline__ void cp_async16_s(void *smem, const void *gmem, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit_s() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1_s() { asm volatile("cp.async.wait_group 1;\n" ::); }

// 64-row tiles, double-buffered with cp.async (rows stay row-major: 16-byte
// copies straight from the FP32 features); per thread 4 rows x 4 centroids,
// per 4 columns four float4 row loads and four float4 centroid loads feed 64
// FFMAs. Centroids resident, transposed [d][kpad].
__global__ void __launch_bounds__(kSThreads, 2)
    screen_kernel(const float *__restrict__ f32, int64_t ld32, const float *__restrict__ fn32,
                  const double *__restrict__ fn64, int64_t n, int d,
                  const float *__restrict__ c32t, const float *__restrict__ cn32, int k, int kpad,
                  const double *__restrict__ cmax_dev, const int32_t *__restrict__ rows,
                  const int32_t *__restrict__ nrows_dev, int32_t *__restrict__ labels,
                  double *__restrict__ ub, double *__restrict__ lb, int32_t *__restrict__ counts,
                  int32_t *__restrict__ amb, int32_t *__restrict__ namb) {
  extern __shared__ __align__(16) float ssm[];
  const int d4 = (d + 3) / 4, ldp = 4 * d4 + 4;   // padded row stride (floats)
  float *Cs = ssm;                                 // [4*d4][kpad] transposed centroids
  float *Cn = Cs + (int64_t)4 * d4 * kpad;         // [kpad]
  float *Fs = Cn + kpad;                           // [2][kSBM][ldp]
  float *Fn = Fs + 2 * kSBM * ldp;                 // [2][kSBM]
  int32_t *Rid = reinterpret_cast<int32_t *>(Fn + 2 * kSBM);  // [2][kSBM]
  int32_t *Hs = Rid + 2 * kSBM;                    // [kpad]
  const int tid = threadIdx.x, tx = tid % kSCT, ty = tid / kSCT;
  const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : n;
  const int64_t ntiles = (nr + kSBM - 1) / kSBM;
  if ((int64_t)blockIdx.x >= ntiles) return;
  for (int64_t e = tid; e < (int64_t)4 * d4 * kpad; e += kSThreads)
    Cs[e] = e < (int64_t)d * kpad ? c32t[e] : 0.0f;
  for (int j = tid; j < kpad; j += kSThreads) {
    Cn[j] = cn32[j];
    Hs[j] = 0;
  }
  const double cmax = *cmax_dev;
  const double dscale = (double)(d + 5) * 5.9604644775390625e-8;  // (d + 5) * 2^-24
  // stage tile t into buffer b: row ids / |f|^2 by plain loads, rows by cp.async
  auto prep = [&](int64_t t, int b) {
    int32_t *rid = Rid + b * kSBM;
    if (tid < kSBM) {
      const int64_t lr = t * kSBM + tid;
      const int64_t gr = lr < nr ? (rows ? (int64_t)rows[lr] : lr) : -1;
      rid[tid] = (int32_t)gr;
      Fn[b * kSBM + tid] = gr >= 0 ? fn32[gr] : 0.0f;
    }
    float *fs = Fs + (int64_t)b * kSBM * ldp;
    // kSThreads / kSBM threads per row (no division, one row id load each)
    constexpr int TPR = kSThreads / kSBM;
    const int row = tid / TPR, part = tid % TPR;
    const int64_t lr = t * kSBM + row;
    const int64_t gr = lr < nr ? (rows ? (int64_t)__ldg(rows + lr) : lr) : -1;
    const float *src = gr >= 0 ? f32 + gr * ld32 : f32;
    for (int q = part; q < d4; q += TPR) cp_async16_s(fs + row * ldp + 4 * q, src + 4 * q, gr >= 0);
  };
  int buf = 0;
  prep(blockIdx.x, 0);
  cp_async_commit_s();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (tile + gridDim.x < ntiles) prep(tile + gridDim.x, buf ^ 1);
    cp_async_commit_s();
    cp_async_wait1_s();
    __syncthreads();
    const float *fs = Fs + (int64_t)buf * kSBM * ldp + (ty * kSTM) * ldp;
    const float *fnb = Fn + buf * kSBM;
    float bv[kSTM], bv2[kSTM];
    int bi[kSTM];
#pragma unroll
    for (int i = 0; i < kSTM; ++i) {
      bv[i] = INFINITY;
      bv2[i] = INFINITY;
      bi[i] = 0x7fffffff;
    }
    for (int c0 = 0; c0 < kpad; c0 += kSBN) {
      float acc[kSTM][kSTN];
#pragma unroll
      for (int i = 0; i < kSTM; ++i)
#pragma unroll
        for (int j = 0; j < kSTN; ++j) acc[i][j] = 0.0f;
      const float *cb = Cs + c0 + tx * kSTN;
#pragma unroll 2
      for (int q = 0; q < d4; ++q) {
        float4 a[kSTM], b[4];
#pragma unroll
        for (int i = 0; i < kSTM; ++i) a[i] = *reinterpret_cast<const float4 *>(fs + i * ldp + 4 * q);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          b[u] = *reinterpret_cast<const float4 *>(cb + (int64_t)(4 * q + u) * kpad);
#pragma unroll
        for (int i = 0; i < kSTM; ++i) {
          const float av[4] = {a[i].x, a[i].y, a[i].z, a[i].w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc[i][0] = fmaf(av[u], b[u].x, acc[i][0]);
            acc[i][1] = fmaf(av[u], b[u].y, acc[i][1]);
            acc[i][2] = fmaf(av[u], b[u].z, acc[i][2]);
            acc[i][3] = fmaf(av[u], b[u].w, acc[i][3]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kSTM; ++i) {
        const float fni = fnb[ty * kSTM + i];
#pragma unroll
        for (int j = 0; j < kSTN; ++j) {
          const int cj = c0 + tx * kSTN + j;
          const float e = fmaf(-2.0f, acc[i][j], fni) + Cn[cj];
          if (e < bv[i]) {  // ascending centroid index within the thread
            bv2[i] = bv[i];
            bv[i] = e;
            bi[i] = cj;
          } else {
            bv2[i] = fminf(bv2[i], e);
          }
        }
      }
    }
    // across the 16 threads of a row group (a half warp), lowest index on ties
    const int32_t *rid = Rid + buf * kSBM;
#pragma unroll
    for (int i = 0; i < kSTM; ++i) {
#pragma unroll
      for (int o = 1; o < kSCT; o <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv[i], o);
        const float ov2 = __shfl_xor_sync(0xffffffffu, bv2[i], o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi[i], o);
        if (ov < bv[i] || (ov == bv[i] && oi < bi[i])) {
          bv2[i] = fminf(ov2, bv[i]);
          bv[i] = ov;
          bi[i] = oi;
        } else {
          bv2[i] = fminf(bv2[i], ov);
        }
      }
      if (tx == 0) {
        const int32_t r = rid[ty * kSTM + i];
        if (r >= 0) {
          const double fr = sqrt(fn64[r]) + cmax;
          const double delta = dscale * fr * fr * (1.0 + 1e-6);
          const double e1 = (double)bv[i], e2 = (double)bv2[i];
          if (e2 - e1 > 2.0 * delta) {
            labels[r] = bi[i];
            ub[r] = sqrt(fmax(e1 + delta, 0.0));
            lb[r] = sqrt(fmax(e2 - delta, 0.0));
            if (counts) atomicAdd(Hs + bi[i], 1);
          } else {
            amb[atomicAdd(namb, 1)] = r;
          }
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled two tiles later
    buf ^= 1;
  }
  if (counts) {
    __syncthreads();
    for (int j = tid; j < k; j += kSThreads)
      if (Hs[j]) atomicAdd(counts + j, Hs[j]);
  }
}

}  // namespace

namespace csc {

bool screen_supported(int64_t d, int64_t k) {
  const int64_t kpad = (k + kSBN - 1) / kSBN * kSBN;
  return d >= 1 && d <= 256 && k >= 2 && screen_smem(d, k) <=
         (size_t)csc::device_info().max_smem_optin && kpad <= 1024;
}

size_t screen_smem(int64_t d, int64_t k) {
  const int64_t kpad = (k + kSBN - 1) / kSBN * kSBN;
  const int64_t d4 = (d + 3) / 4, ldp = 4 * d4 + 4;
  return sizeof(float) * (4 * d4 * kpad + kpad + 2 * kSBM * ldp + 2 * kSBM) +
         sizeof(int32_t) * (2 * kSBM + kpad);
}

int64_t screen_kpad(int64_t k) { return (k + kSBN - 1) / kSBN * kSBN; }

int screen_convert_features(const double *f, int64_t n, int64_t d, int64_t ld, float *f32,
                            int64_t ld32, float *fn32, cudaStream_t st) {
  const int64_t grid = std::min<int64_t>(csc::device_info().sm_count * 8, ceil_div(n, 8));
  f32_convert_kernel<<<(unsigned)std::max<int64_t>(1, grid), 256, 0, st>>>(f, n, d, ld, f32, ld32,
                                                                          fn32);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int screen_convert_centroids(const double *c, int64_t k, int64_t d, int64_t ldc,
                             const double *cnorm, float *c32t, float *cn32, double *cmax,
                             cudaStream_t st) {
  c32_convert_kernel<<<1, 256, 0, st>>>(c, k, d, ldc, cnorm, (int)screen_kpad(k), c32t, cn32, cmax);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int screen_assign(const float *f32, int64_t ld32, const float *fn32, const double *fn64,
                  int64_t n, int64_t d, const float *c32t, const float *cn32, int64_t k,
                  const double *cmax, const int32_t *rows, const int32_t *nrows_dev,
                  int32_t *labels, double *ub, double *lb, int32_t *counts, int32_t *amb,
                  int32_t *namb, cudaStream_t st) {
  const size_t smem = screen_smem(d, k);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CSC_TRY_CUDA(cudaFuncSetAttribute(screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    configured = smem;
  }
  int occ = 0;
  CSC_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, screen_kernel, kSThreads, smem));
  const int64_t tiles = ceil_div(n, kSBM);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(occ, 1) *
                                                                  csc::device_info().sm_count,
                                                              tiles));
  screen_kernel<<<(unsigned)grid, kSThreads, smem, st>>>(
      f32, ld32, fn32, fn64, n, (int)d, c32t, cn32, (int)k, (int)screen_kpad(k), cmax, rows,
      nrows_dev, labels, ub, lb, counts, amb, namb);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

}  // namespace csc
