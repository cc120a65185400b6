// Lloyd k-means on the filtered n x d features, fp64, sm_100a
// (cscluster.kmeans, kmeans.py:54-117).
//
// assign  : GEMM-form distances |f|^2 - 2 f.c + |c|^2 (kmeans.py:54-61, same
//           association), clamped at 0, first-index argmin. Register-tiled
//           SIMT FP64 (64 rows x 64 centroids per 256-thread block, 4x4 per
//           thread, 16-wide d chunks in shared memory). FP64 FMA bound at
//           k >= ~32; tensor cores are deliberately unused.
// repair  : empty-cluster reseeding (kmeans.py:99-108), single block, exits
//           immediately when no cluster is empty (no host sync needed).
// update  : means by label (kmeans.py:80-85). Each block owns a contiguous
//           row range and accumulates per-column sums sequentially in shared
//           memory; a finishing kernel adds the block partials in block order.
//           Deterministic; no floating-point atomics.
// cost    : sum |f_i - c_{l_i}|^2 (kmeans.py:111), fixed-order partials.
// k-means++: distance update + contiguous-chunk partial sums, then a
//           single-block D^2 draw for one host-supplied uniform
//           (Generator.choice(n, p) == searchsorted(cumsum(p), u, 'right')).
#include <cub/cub.cuh>

#include "common.cuh"

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kAssignThreads = 256;

__global__ void rownorm_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                               double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < n;
       r += warps) {
    const double *row = f + r * ld;
    double s = 0.0;
    for (int64_t c = lane; c < d; c += 32) s = fma(row[c], row[c], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
  }
}

__global__ void __launch_bounds__(kAssignThreads)
    assign_kernel(const double *__restrict__ f, const double *__restrict__ fnorm, int64_t n,
                  int64_t d, int64_t ld, const double *__restrict__ cent, int64_t ldc,
                  const double *__restrict__ cnorm, int64_t k, int32_t *__restrict__ labels,
                  double *__restrict__ own, int32_t *__restrict__ counts) {
  __shared__ __align__(16) double Fs[kBK][kBM];
  __shared__ __align__(16) double Cs[kBK][kBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15;  // centroid group
  const int ty = tid >> 4;  // row group
  const int64_t r0 = (int64_t)blockIdx.x * kBM;
  double best_v[4];
  int best_i[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    best_v[i] = INFINITY;
    best_i[i] = 0;
  }
  double fn[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty * 4 + i;
    fn[i] = r < n ? fnorm[r] : 0.0;
  }
  // tile loader mapping: 256 threads x 4 elements = 64 x 16
  const int lrow = tid >> 2;        // 0..63
  const int lcol = (tid & 3) * 4;   // 0,4,8,12
  for (int64_t c0 = 0; c0 < k; c0 += kBN) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t k0 = 0; k0 < d; k0 += kBK) {
      {
        const int64_t r = r0 + lrow, cc = c0 + lrow;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t col = k0 + lcol + e;
          Fs[lcol + e][lrow] = (r < n && col < d) ? f[r * ld + col] : 0.0;
          Cs[lcol + e][lrow] = (cc < k && col < d) ? cent[cc * ldc + col] : 0.0;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        const double2 a01 = *reinterpret_cast<const double2 *>(&Fs[kk][ty * 4]);
        const double2 a23 = *reinterpret_cast<const double2 *>(&Fs[kk][ty * 4 + 2]);
        const double2 b01 = *reinterpret_cast<const double2 *>(&Cs[kk][tx * 4]);
        const double2 b23 = *reinterpret_cast<const double2 *>(&Cs[kk][tx * 4 + 2]);
        const double a[4] = {a01.x, a01.y, a23.x, a23.y};
        const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
    // distances and argmin within this centroid tile
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double v = INFINITY;
      int vi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t c = c0 + tx * 4 + j;
        if (c < k) {
          const double t = __dsub_rn(fn[i], __dmul_rn(2.0, acc[i][j]));
          double d2 = __dadd_rn(t, cnorm[c]);
          d2 = d2 > 0.0 ? d2 : 0.0;
          if (d2 < v) {
            v = d2;
            vi = (int)c;
          }
        }
      }
      // reduce over the 16 centroid groups (lanes sharing ty sit in one half-warp)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o, 16);
        const int oi = __shfl_xor_sync(0xffffffffu, vi, o, 16);
        if (ov < v || (ov == v && oi < vi)) {
          v = ov;
          vi = oi;
        }
      }
      if (v < best_v[i] || (v == best_v[i] && vi < best_i[i])) {
        best_v[i] = v;
        best_i[i] = vi;
      }
    }
  }
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = r0 + ty * 4 + i;
      if (r < n) {
        labels[r] = best_i[i];
        own[r] = best_v[i];
        if (counts) atomicAdd(counts + best_i[i], 1);
      }
    }
  }
}

// argmax with first-index ties over a[0..n) by one block (result in thread 0)
__device__ void block_argmax(const double *a, int64_t n, double &bv, int64_t &bi) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  double v = -INFINITY;
  int64_t idx = INT64_MAX;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = a[i];
    if (x > v) {  // strided scan visits indices in increasing order per thread
      v = x;
      idx = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sv[wid] = v;
    si[wid] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w)
      if (sv[w] > v || (sv[w] == v && si[w] < idx)) {
        v = sv[w];
        idx = si[w];
      }
    bv = v;
    bi = idx;
  }
  __syncthreads();
}

__global__ void repair_kernel(int32_t *__restrict__ labels, double *__restrict__ own,
                              const int32_t *__restrict__ counts, int64_t n, int64_t k) {
  __shared__ int64_t chosen;
  for (int64_t j = 0; j < k; ++j) {
    if (counts[j] != 0) continue;  // uniform across the block
    double bv;
    int64_t bi = 0;
    block_argmax(own, n, bv, bi);
    if (threadIdx.x == 0) {
      chosen = bi;
      labels[bi] = (int32_t)j;
      own[bi] = -1.0;
    }
    __syncthreads();
    (void)chosen;
  }
}

// partial sums: block (b, y) owns rows [b*chunk, ...) and columns
// [y*cw, y*cw+cw); smem holds k x cw sums.
__global__ void update_partial_kernel(const double *__restrict__ f,
                                      const int32_t *__restrict__ labels, int64_t n, int64_t d,
                                      int64_t ld, int64_t k, int64_t chunk, int cw,
                                      double *__restrict__ psum, int32_t *__restrict__ pcnt) {
  extern __shared__ double sm[];
  int32_t *scnt = reinterpret_cast<int32_t *>(sm + (size_t)k * cw);
  const int64_t b = blockIdx.x;
  const int64_t col0 = (int64_t)blockIdx.y * cw;
  for (int64_t i = threadIdx.x; i < k * cw; i += blockDim.x) sm[i] = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) scnt[i] = 0;
  __syncthreads();
  const int64_t rbeg = b * chunk, rend = min(n, rbeg + chunk);
  const int c = threadIdx.x;
  const bool active = c < cw && col0 + c < d;
  if (active) {
    for (int64_t r = rbeg; r < rend; ++r) {
      const int32_t l = labels[r];
      sm[(size_t)l * cw + c] += f[r * ld + col0 + c];
    }
  }
  if (blockIdx.y == 0)
    for (int64_t r = rbeg + threadIdx.x; r < rend; r += blockDim.x) atomicAdd(scnt + labels[r], 1);
  __syncthreads();
  const int64_t nb = gridDim.x;
  for (int64_t i = threadIdx.x; i < k * cw; i += blockDim.x) {
    const int64_t j = i / cw, cc = i % cw;
    if (col0 + cc < d) psum[(b * k + j) * d + col0 + cc] = sm[i];
  }
  if (blockIdx.y == 0)
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) pcnt[b * k + j] = scnt[j];
  (void)nb;
}

__global__ void update_finish_kernel(const double *__restrict__ psum,
                                     const int32_t *__restrict__ pcnt, int64_t nb, int64_t d,
                                     int64_t k, double *__restrict__ cent, int64_t ldc,
                                     double *__restrict__ cnorm, int32_t *__restrict__ counts) {
  __shared__ double red[32];
  __shared__ int32_t s_cnt;
  const int64_t j = blockIdx.x;
  if (threadIdx.x == 0) {
    int32_t cnt = 0;
    for (int64_t b = 0; b < nb; ++b) cnt += pcnt[b * k + j];
    s_cnt = cnt;
    counts[j] = cnt;
  }
  __syncthreads();
  const double denom = (double)(s_cnt > 1 ? s_cnt : 1);
  double nrm = 0.0;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < nb; ++b) s += psum[(b * k + j) * d + c];
    const double mean = __ddiv_rn(s, denom);
    cent[j * ldc + c] = mean;
    nrm = fma(mean, mean, nrm);
  }
  nrm = block_sum<128>(nrm, red);
  if (threadIdx.x == 0) cnorm[j] = nrm;
}

__global__ void cost_kernel(const double *__restrict__ f, const int32_t *__restrict__ labels,
                            const double *__restrict__ cent, int64_t ldc, int64_t n, int64_t d,
                            int64_t ld, double *__restrict__ partials) {
  __shared__ double red[8];
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  double s = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < n;
       r += warps) {
    const double *row = f + r * ld;
    const double *c = cent + (int64_t)labels[r] * ldc;
    for (int64_t col = lane; col < d; col += 32) {
      const double t = row[col] - c[col];
      s = fma(t, t, s);
    }
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// k-means++ distances over contiguous row chunks (chunk sums kept for the draw)
__global__ void kpp_dist_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                                const double *__restrict__ crow, double *__restrict__ closest,
                                int first, int64_t chunk, double *__restrict__ chunk_sums) {
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t rbeg = blockIdx.x * chunk, rend = min(n, rbeg + chunk);
  double s = 0.0;
  for (int64_t r = rbeg + wid; r < rend; r += blockDim.x / 32) {
    const double *row = f + r * ld;
    double acc = 0.0;
    for (int64_t c = lane; c < d; c += 32) {
      const double t = row[c] - crow[c];
      acc = fma(t, t, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    double v = acc;
    if (!first) v = fmin(closest[r], acc);
    if (lane == 0) {
      closest[r] = v;
      s += v;
    }
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) chunk_sums[blockIdx.x] = s;
}

// Single-block D^2 draw. target = u * total (total = chunk sums in order);
// walk the chunk sums, then scan the chosen chunk tile by tile with a
// block-wide inclusive scan; the first positive entry whose running prefix
// exceeds the target is drawn (searchsorted(cdf, u, 'right') semantics).
__global__ void __launch_bounds__(1024)
    kpp_pick_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                    const double *__restrict__ closest, const double *__restrict__ chunk_sums,
                    int64_t nchunks, int64_t chunk, double u, int64_t fixed_idx,
                    double *__restrict__ crow, int64_t *__restrict__ idx_out) {
  typedef cub::BlockScan<double, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long s_idx;
  __shared__ double s_base, s_target;
  __shared__ int64_t s_chunk;
  if (threadIdx.x == 0) {
    s_idx = (unsigned long long)(fixed_idx >= 0 ? fixed_idx : -1);
    if (fixed_idx < 0) {
      double total = 0.0;
      for (int64_t b = 0; b < nchunks; ++b) total += chunk_sums[b];
      const double target = u * total;
      double base = 0.0;
      int64_t b = 0;
      for (; b < nchunks - 1; ++b) {
        if (base + chunk_sums[b] > target) break;
        base += chunk_sums[b];
      }
      s_base = base;
      s_target = target;
      s_chunk = b;
    }
  }
  __syncthreads();
  if (fixed_idx < 0) {
    const double target = s_target;
    double running = s_base;
    bool found = false;
    for (int64_t t0 = s_chunk * chunk; t0 < n && !found; t0 += 1024) {
      const int64_t i = t0 + threadIdx.x;
      const double v = i < n ? closest[i] : 0.0;
      double incl, agg;
      Scan(tmp).InclusiveSum(v, incl, agg);
      const bool hit = i < n && v > 0.0 && running + incl > target;
      if (__syncthreads_or(hit)) {
        if (threadIdx.x == 0) s_idx = ~0ull;
        __syncthreads();
        if (hit) atomicMin(&s_idx, (unsigned long long)i);
        __syncthreads();
        found = true;
      }
      running += agg;
    }
    if (!found) {  // rounding fell off the end: last positive entry
      if (threadIdx.x == 0) {
        int64_t last = n - 1;
        while (last > 0 && !(closest[last] > 0.0)) --last;
        s_idx = (unsigned long long)last;
      }
    }
  }
  __syncthreads();
  const int64_t idx = (int64_t)s_idx;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) crow[c] = f[idx * ld + c];
  if (threadIdx.x == 0) idx_out[0] = idx;
}

__global__ void gather_cols_kernel(const double *__restrict__ src, int64_t n, int64_t lds,
                                   const int64_t *__restrict__ cols, int64_t ncols,
                                   double *__restrict__ dst, int64_t ldd, int64_t col0) {
  const int64_t total = n * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncols, j = t - (t / ncols) * ncols;
    dst[i * ldd + col0 + j] = src[i * lds + cols[j]];
  }
}

int grid_cap(int64_t want, int per_sm = 8) {
  return (int)std::min<int64_t>((int64_t)csc::device_info().sm_count * per_sm,
                                std::max<int64_t>(1, want));
}

}  // namespace

extern "C" {

int csc_kmeans_rownorms(const double *f, int64_t n, int64_t d, int64_t ld, double *out,
                        void *stream) {
  CSC_REQUIRE(n >= 0 && d >= 1 && ld >= d, "csc_kmeans_rownorms: bad shape");
  if (n == 0) return CSC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rownorm_kernel<<<grid_cap(csc::ceil_div(n, 8)), 256, 0, st>>>(f, n, d, ld, out);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeans_assign(const double *f, const double *fnorm, int64_t n, int64_t d, int64_t ld,
                      const double *c, int64_t ldc, const double *cnorm, int64_t k,
                      int32_t *labels, double *own, int32_t *counts, void *stream) {
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && k >= 1 && ldc >= d, "csc_kmeans_assign: bad shape");
  CSC_REQUIRE(k < INT32_MAX, "csc_kmeans_assign: k too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (counts) CSC_TRY_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * k, st));
  assign_kernel<<<(unsigned)csc::ceil_div(n, kBM), kAssignThreads, 0, st>>>(
      f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeans_repair(int32_t *labels, double *own, int32_t *counts, int64_t n, int64_t k,
                      void *stream) {
  CSC_REQUIRE(n >= 1 && k >= 1, "csc_kmeans_repair: bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  repair_kernel<<<1, 1024, 0, st>>>(labels, own, counts, n, k);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeans_update(const double *f, const int32_t *labels, int64_t n, int64_t d, int64_t ld,
                      int64_t k, double *c, int64_t ldc, double *cnorm, int32_t *counts,
                      void *stream) {
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && k >= 1 && ldc >= d, "csc_kmeans_update: bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const csc::DeviceInfo &info = csc::device_info();
  // columns per block so that k*cw doubles (+ k counts) fit in shared memory
  const int64_t budget = std::max<int64_t>(48 * 1024, (int64_t)info.max_smem_optin) - 1024;
  const int64_t cnt_bytes = sizeof(int32_t) * k;
  int64_t cw = (budget - cnt_bytes) / (int64_t)(sizeof(double) * k);
  CSC_REQUIRE(cw >= 1, "csc_kmeans_update: k=%lld too large for shared-memory partials",
              (long long)k);
  cw = std::min<int64_t>(std::min<int64_t>(cw, 256), d);
  const int64_t ny = csc::ceil_div(d, cw);
  // rows per block: enough blocks to fill the GPU, at least 32 rows each
  const int64_t nb = std::max<int64_t>(
      1, std::min<int64_t>((int64_t)info.sm_count * 2, csc::ceil_div(n, 32)));
  const int64_t chunk = csc::ceil_div(n, nb);
  const size_t smem = sizeof(double) * k * cw + cnt_bytes;
  CSC_TRY_CUDA(cudaFuncSetAttribute(update_partial_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  csc::Scratch psum, pcnt;
  CSC_TRY_CUDA(psum.alloc(sizeof(double) * nb * k * d, st));
  CSC_TRY_CUDA(pcnt.alloc(sizeof(int32_t) * nb * k, st));
  const int threads = (int)std::max<int64_t>(32, csc::ceil_div(cw, 32) * 32);
  update_partial_kernel<<<dim3((unsigned)nb, (unsigned)ny), threads, smem, st>>>(
      f, labels, n, d, ld, k, chunk, (int)cw, psum.as<double>(), pcnt.as<int32_t>());
  CSC_CHECK_LAUNCH();
  update_finish_kernel<<<(unsigned)k, 128, 0, st>>>(psum.as<double>(), pcnt.as<int32_t>(), nb, d,
                                                    k, c, ldc, cnorm, counts);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeans_cost(const double *f, const int32_t *labels, const double *c, int64_t ldc,
                    int64_t n, int64_t d, int64_t ld, double *cost2, void *stream) {
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && ldc >= d, "csc_kmeans_cost: bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_cap(csc::ceil_div(n, 8));
  csc::Scratch parts;
  CSC_TRY_CUDA(parts.alloc(sizeof(double) * grid, st));
  cost_kernel<<<grid, 256, 0, st>>>(f, labels, c, ldc, n, d, ld, parts.as<double>());
  CSC_CHECK_LAUNCH();
  reduce_partials_kernel<<<1, 1024, 0, st>>>(parts.as<double>(), grid, cost2);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeanspp_nchunks(int64_t n) {
  const int64_t want = csc::ceil_div(std::max<int64_t>(n, 1), 256);
  return (int)std::min<int64_t>((int64_t)csc::device_info().sm_count * 4, want);
}

int csc_kmeanspp_dist(const double *f, int64_t n, int64_t d, int64_t ld, const double *crow,
                      double *closest, int first, double *chunk_sums, int64_t nchunks,
                      double *total, void *stream) {
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && nchunks >= 1, "csc_kmeanspp_dist: bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunk = csc::ceil_div(n, nchunks);
  kpp_dist_kernel<<<(unsigned)nchunks, 256, 0, st>>>(f, n, d, ld, crow, closest, first, chunk,
                                                     chunk_sums);
  CSC_CHECK_LAUNCH();
  if (total) {
    reduce_partials_kernel<<<1, 1024, 0, st>>>(chunk_sums, nchunks, total);
    CSC_CHECK_LAUNCH();
  }
  return CSC_OK;
}

int csc_kmeanspp_pick(const double *f, int64_t n, int64_t d, int64_t ld, const double *closest,
                      const double *chunk_sums, int64_t nchunks, double u, int64_t fixed_idx,
                      double *crow, int64_t *idx_dev, void *stream) {
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && nchunks >= 1, "csc_kmeanspp_pick: bad shape");
  CSC_REQUIRE(fixed_idx < n, "csc_kmeanspp_pick: index out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunk = csc::ceil_div(n, nchunks);
  kpp_pick_kernel<<<1, 1024, 0, st>>>(f, n, d, ld, closest, chunk_sums, nchunks, chunk, u,
                                      fixed_idx, crow, idx_dev);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_gather_columns(const double *src, int64_t n, int64_t lds, const int64_t *cols,
                       int64_t ncols, double *dst, int64_t ldd, int64_t col0, void *stream) {
  CSC_REQUIRE(n >= 0 && ncols >= 0 && col0 >= 0 && col0 + ncols <= ldd,
              "csc_gather_columns: bad shape");
  if (n == 0 || ncols == 0) return CSC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  gather_cols_kernel<<<grid_cap(csc::ceil_div(n * ncols, 256), 16), 256, 0, st>>>(
      src, n, lds, cols, ncols, dst, ldd, col0);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

}  // extern "C"
