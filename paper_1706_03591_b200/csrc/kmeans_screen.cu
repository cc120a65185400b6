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
// No tensor cores (north_star): SIMT FFMA, 256 rows x 64 centroids per block
// pass, 8 x 8 per thread, 16-column row stages through a cp.async ring.
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kmeans_screen.cuh"

namespace {

constexpr int kSBN = 64;  // centroid padding unit (kpad)

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
  for (int64_t t = threadIdx.x / 32; t < d; t += blockDim.x / 32)  // warp per column of the transposed tile
    for (int64_t j = threadIdx.x % 32; j < kpad; j += 32) c32t[t * kpad + j] = j < k ? (float)c[j * ldc + t] : 0.0f;
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
template <int N>
__device__ __forceinline__ void cp_async_wait_s() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// 256 rows x 64 centroids per block pass, 32 x 8 threads, 8 x 8 per thread
// (rows ty + 32 i: the 4 row groups of a warp hit disjoint banks; centroids
// 8 tx .. 8 tx + 7). The row tile streams
// through a 3-stage cp.async ring of 16-column slices kept row-major ([row][20]
// floats: one float4 per row and 4 columns), so per 4 columns eight float4 row
// loads and eight float4 centroid loads feed 256 FFMAs; the centroid tile is
// resident, transposed [d][kpad].
constexpr int kS3RT = 32, kS3CT = 8, kS3TM = 8, kS3TN = 8;
constexpr int kS3Threads = kS3RT * kS3CT;  // 256
constexpr int kS3BM = kS3RT * kS3TM;       // 256 rows per tile
constexpr int kS3BN = kS3CT * kS3TN;       // 64 centroids per pass
constexpr int kS3KS = 32;                  // columns per stage
constexpr int kS3KP = kS3KS + 4;           // padded stage row (floats)
constexpr int kS3NS = 3;                   // stages in the ring

__global__ void __launch_bounds__(kS3Threads, 1)
    screen_kernel(const float *__restrict__ f32, int64_t ld32, const float *__restrict__ fn32,
                  const double *__restrict__ fn64, int64_t n, int d,
                  const float *__restrict__ c32t, const float *__restrict__ cn32, int k, int kpad,
                  const double *__restrict__ cmax_dev, const int32_t *__restrict__ rows,
                  const int32_t *__restrict__ nrows_dev, int32_t *__restrict__ labels,
                  double *__restrict__ ub, double *__restrict__ lb, int32_t *__restrict__ counts,
                  int32_t *__restrict__ amb, int32_t *__restrict__ namb) {
  extern __shared__ __align__(16) float ssm[];
  const int nst = (d + kS3KS - 1) / kS3KS, dpad = nst * kS3KS;
  float *Cs = ssm;                              // [dpad][kpad] transposed centroids
  float *Cn = Cs + (int64_t)dpad * kpad;        // [kpad]
  float *Fs = Cn + kpad;                        // [kS3NS][kS3BM][kS3KP] row stages
  float *Fn = Fs + kS3NS * kS3BM * kS3KP;       // [kS3BM]
  int32_t *Rid = reinterpret_cast<int32_t *>(Fn + kS3BM);  // [kS3BM]
  int32_t *Hs = Rid + kS3BM;                    // [kpad]
  const int tid = threadIdx.x, tx = tid % kS3CT, ty = tid / kS3CT;
  const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : n;
  const int64_t ntiles = (nr + kS3BM - 1) / kS3BM;
  if ((int64_t)blockIdx.x >= ntiles) return;
  for (int64_t e = tid; e < (int64_t)dpad * kpad; e += kS3Threads)
    Cs[e] = e < (int64_t)d * kpad ? c32t[e] : 0.0f;
  for (int j = tid; j < kpad; j += kS3Threads) {
    Cn[j] = cn32[j];
    Hs[j] = 0;
  }
  const double cmax = *cmax_dev;
  const double dscale = (double)(d + 5) * 5.9604644775390625e-8;  // (d + 5) * 2^-24
  // stage st of the current tile into ring slot b: 256 rows x KS/4 float4
  // (e = tid + 256 u: row e / (KS/4), column group e % (KS/4)); columns past d
  // (and padding rows) are zero-filled
  constexpr int kQ = kS3KS / 4, kU = kS3BM * kQ / kS3Threads;
  auto stage = [&](int st, int b) {
    float *fs = Fs + b * kS3BM * kS3KP;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = tid + kS3Threads * u, row = e / kQ, q = e % kQ;
      const int32_t gr = Rid[row];
      const int col = st * kS3KS + 4 * q;
      const bool ok = gr >= 0 && col < d;
      cp_async16_s(fs + row * kS3KP + 4 * q, ok ? f32 + (int64_t)gr * ld32 + col : f32, ok);
    }
  };
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();  // previous tile's Rid / Fn / stages consumed
    {
      const int64_t lr = tile * kS3BM + tid;
      const int64_t gr = lr < nr ? (rows ? (int64_t)rows[lr] : lr) : -1;
      Rid[tid] = (int32_t)gr;
      Fn[tid] = gr >= 0 ? fn32[gr] : 0.0f;
    }
    __syncthreads();
    float bv[kS3TM], bv2[kS3TM];
    int bi[kS3TM];
#pragma unroll
    for (int i = 0; i < kS3TM; ++i) {
      bv[i] = INFINITY;
      bv2[i] = INFINITY;
      bi[i] = 0x7fffffff;
    }
    for (int c0 = 0; c0 < kpad; c0 += kS3BN) {
      float acc[kS3TM][kS3TN];
#pragma unroll
      for (int i = 0; i < kS3TM; ++i)
#pragma unroll
        for (int j = 0; j < kS3TN; ++j) acc[i][j] = 0.0f;
#pragma unroll
      for (int p = 0; p < kS3NS - 1; ++p) {
        if (p < nst) stage(p, p);
        cp_async_commit_s();
      }
      for (int st = 0; st < nst; ++st) {
        if (st + kS3NS - 1 < nst) stage(st + kS3NS - 1, (st + kS3NS - 1) % kS3NS);
        cp_async_commit_s();
        cp_async_wait_s<kS3NS - 1>();
        __syncthreads();
        const float *fs = Fs + (st % kS3NS) * kS3BM * kS3KP + ty * kS3KP;
        const float *cb = Cs + (int64_t)st * kS3KS * kpad + c0 + tx * kS3TN;
#pragma unroll
        for (int k4 = 0; k4 < kS3KS / 4; ++k4) {
          float4 a[kS3TM];
#pragma unroll
          for (int i = 0; i < kS3TM; ++i)
            a[i] = *reinterpret_cast<const float4 *>(fs + i * kS3RT * kS3KP + 4 * k4);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 b0 = *reinterpret_cast<const float4 *>(cb + (int64_t)(4 * k4 + u) * kpad);
            const float4 b1 = *reinterpret_cast<const float4 *>(cb + (int64_t)(4 * k4 + u) * kpad + 4);
            const float bw[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < kS3TM; ++i) {
              const float av = u == 0 ? a[i].x : u == 1 ? a[i].y : u == 2 ? a[i].z : a[i].w;
#pragma unroll
              for (int j = 0; j < kS3TN; ++j) acc[i][j] = fmaf(av, bw[j], acc[i][j]);
            }
          }
        }
        __syncthreads();  // slot st % NS is refilled by the next iteration's stage()
      }
#pragma unroll
      for (int i = 0; i < kS3TM; ++i) {
        const float fni = Fn[ty + kS3RT * i];
#pragma unroll
        for (int j = 0; j < kS3TN; ++j) {
          const int cj = c0 + tx * kS3TN + j;
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
    // across the 8 threads of a row group (lanes 8m .. 8m+7), lowest index on
    // ties; afterwards every lane of the group holds all 8 rows' results and
    // lane tx settles row ty + 32 tx
    float myv = INFINITY, myv2 = INFINITY;
    int myi = 0;
#pragma unroll
    for (int i = 0; i < kS3TM; ++i) {
#pragma unroll
      for (int o = 1; o < kS3CT; o <<= 1) {
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
      if (tx == i) {
        myv = bv[i];
        myv2 = bv2[i];
        myi = bi[i];
      }
    }
    const int32_t r = Rid[ty + kS3RT * tx];
    if (r >= 0) {
      // |f| from the FP32 norm (relative error < 1e-5 for d <= 256), inflated
      const double fr = sqrt((double)Fn[ty + kS3RT * tx] * (1.0 + 2e-5)) + cmax;
      const double delta = dscale * fr * fr * (1.0 + 1e-6);
      const double e1 = (double)myv, e2 = (double)myv2;
      if (e2 - e1 > 2.0 * delta) {
        labels[r] = myi;
        ub[r] = sqrt(fmax(e1 + delta, 0.0));
        lb[r] = sqrt(fmax(e2 - delta, 0.0));
        if (counts) atomicAdd(Hs + myi, 1);
      } else {
        amb[atomicAdd(namb, 1)] = r;
      }
    }
  }
  if (counts) {
    __syncthreads();
    for (int j = tid; j < k; j += kS3Threads)
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
  const int64_t dpad = (d + kS3KS - 1) / kS3KS * kS3KS;
  return sizeof(float) * (dpad * kpad + kpad + kS3NS * kS3BM * kS3KP + kS3BM) +
         sizeof(int32_t) * (kS3BM + kpad);
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
  // per-device launch setup (dynamic shared memory opt-in, occupancy), cached
  static std::mutex mu;
  static std::vector<std::pair<size_t, int>> setup;  // [device] (configured smem, blocks/SM)
  int dev = 0;
  CSC_TRY_CUDA(cudaGetDevice(&dev));
  int occ = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if ((int)setup.size() <= dev) setup.resize(dev + 1, {0, 0});
    if (smem > setup[dev].first) {
      CSC_TRY_CUDA(cudaFuncSetAttribute(screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
      CSC_TRY_CUDA(
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, screen_kernel, kS3Threads, smem));
      setup[dev] = {smem, occ};
    }
    occ = setup[dev].second;
  }
  const int64_t tiles = ceil_div(n, kS3BM);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(occ, 1) *
                                                                  csc::device_info().sm_count,
                                                              tiles));
  screen_kernel<<<(unsigned)grid, kS3Threads, smem, st>>>(
      f32, ld32, fn32, fn64, n, (int)d, c32t, cn32, (int)k, (int)screen_kpad(k), cmax, rows,
      nrows_dev, labels, ub, lb, counts, amb, namb);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

}  // namespace csc
