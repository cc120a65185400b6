// On-device Laplacian construction and edge-set deltas (bit-exact with
// cscluster.graphs, graphs.py:29-76 and 339-362).
//
// Input is the Graph's canonical edge list (lo < hi, sorted by code lo*n+hi).
// Row i of the symmetric CSR is
//     [lower neighbours j < i | diagonal | upper neighbours j > i]
// The upper neighbours of i are the contiguous edge range with lo == i (already
// ascending in hi). The lower neighbours are the edges with hi == i; a stable
// radix sort of the hi keys groups them while keeping canonical (ascending lo)
// order inside each group. Hence every row comes out sorted without a
// per-row sort, and the two degree partial sums are formed in exactly the
// order numpy's bincount uses (edge order), then added as deg1 + deg2.
//
// Values: inv = 1/sqrt(deg) with IEEE-rounded sqrt and division
// (__dsqrt_rn/__ddiv_rn), off-diagonal -((inv_i*w)*inv_j) with rounded
// multiplies (__dmul_rn; no contraction), normalized diagonal 1.0 on
// non-isolated rows, combinatorial diagonal deg (zeros not stored, as SciPy's
// csr subtraction drops them).
#include <cub/cub.cuh>

#include "common.cuh"

namespace {

__global__ void degree_hist_kernel(const int64_t *__restrict__ lo, const int64_t *__restrict__ hi,
                                   int64_t m, int32_t *__restrict__ cnt_lo,
                                   int32_t *__restrict__ cnt_hi, int32_t *__restrict__ hi32) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = lo[e], b = hi[e];
    atomicAdd(cnt_lo + a, 1);
    atomicAdd(cnt_hi + b, 1);
    hi32[e] = (int32_t)b;
  }
}

__global__ void degree_kernel(int64_t n, const int32_t *__restrict__ lo_ptr,
                              const int32_t *__restrict__ hi_ptr,
                              const int32_t *__restrict__ perm, const double *__restrict__ w,
                              int variant, double *__restrict__ deg, double *__restrict__ inv,
                              int32_t *__restrict__ row_cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d1 = 0.0, d2 = 0.0;
    if (w) {
      for (int32_t e = lo_ptr[i]; e < lo_ptr[i + 1]; ++e) d1 = __dadd_rn(d1, w[e]);
      for (int32_t t = hi_ptr[i]; t < hi_ptr[i + 1]; ++t) d2 = __dadd_rn(d2, w[perm[t]]);
    } else {
      d1 = (double)(lo_ptr[i + 1] - lo_ptr[i]);
      d2 = (double)(hi_ptr[i + 1] - hi_ptr[i]);
    }
    const double dg = __dadd_rn(d1, d2);
    deg[i] = dg;
    bool diag;
    if (variant == CSC_LAP_NORMALIZED) {
      diag = dg > 0.0;
      inv[i] = diag ? __ddiv_rn(1.0, __dsqrt_rn(dg)) : 0.0;
    } else {
      diag = dg != 0.0;
      inv[i] = 0.0;
    }
    row_cnt[i] = (lo_ptr[i + 1] - lo_ptr[i]) + (hi_ptr[i + 1] - hi_ptr[i]) + (diag ? 1 : 0);
  }
}

__device__ __forceinline__ double off_value(int variant, double inv_i, double w, double inv_j) {
  if (variant == CSC_LAP_NORMALIZED) return -__dmul_rn(__dmul_rn(inv_i, w), inv_j);
  return -w;
}

// Entry-parallel fill (same values and positions as fill_kernel): the row of
// an entry and its slot are known without walking the row, so hub rows of
// skewed graphs do not serialise.
__global__ void fill_upper_kernel(int64_t m, const int64_t *__restrict__ lo,
                                  const int64_t *__restrict__ hi, const double *__restrict__ w,
                                  const int32_t *__restrict__ lo_ptr,
                                  const int32_t *__restrict__ hi_ptr,
                                  const double *__restrict__ deg, const double *__restrict__ inv,
                                  int variant, const int32_t *__restrict__ indptr,
                                  int32_t *__restrict__ indices, double *__restrict__ vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = lo[e], j = hi[e];
    const double dg = deg[i];
    const int diag = (variant == CSC_LAP_NORMALIZED ? dg > 0.0 : dg != 0.0) ? 1 : 0;
    const int64_t pos = indptr[i] + (hi_ptr[i + 1] - hi_ptr[i]) + diag + (e - lo_ptr[i]);
    indices[pos] = (int32_t)j;
    vals[pos] = off_value(variant, inv[i], w ? w[e] : 1.0, inv[j]);
  }
}

__global__ void fill_lower_kernel(int64_t m, const int64_t *__restrict__ lo,
                                  const int64_t *__restrict__ hi, const double *__restrict__ w,
                                  const int32_t *__restrict__ hi_ptr,
                                  const int32_t *__restrict__ perm,
                                  const double *__restrict__ inv, int variant,
                                  const int32_t *__restrict__ indptr,
                                  int32_t *__restrict__ indices, double *__restrict__ vals) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = perm[t];
    const int64_t i = hi[e], j = lo[e];
    const int64_t pos = indptr[i] + (t - hi_ptr[i]);
    indices[pos] = (int32_t)j;
    vals[pos] = off_value(variant, inv[i], w ? w[e] : 1.0, inv[j]);
  }
}

__global__ void fill_diag_kernel(int64_t n, const int32_t *__restrict__ hi_ptr,
                                 const double *__restrict__ deg, int variant,
                                 const int32_t *__restrict__ indptr, int32_t *__restrict__ indices,
                                 double *__restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dg = deg[i];
    if (variant == CSC_LAP_NORMALIZED ? dg > 0.0 : dg != 0.0) {
      const int64_t pos = indptr[i] + (hi_ptr[i + 1] - hi_ptr[i]);
      indices[pos] = (int32_t)i;
      vals[pos] = variant == CSC_LAP_NORMALIZED ? 1.0 : dg;
    }
  }
}

// --- edge delta --------------------------------------------------------------

__device__ __forceinline__ int64_t lower_bound(const int64_t *a, int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void mark_deleted_kernel(const int64_t *__restrict__ prev, int64_t m,
                                    const int64_t *__restrict__ del, int64_t n_del,
                                    int8_t *__restrict__ keep, unsigned long long *found) {
  unsigned long long f = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = prev[e];
    const int64_t p = lower_bound(del, n_del, c);
    const bool hit = p < n_del && del[p] == c;
    keep[e] = hit ? 0 : 1;
    f += hit;
  }
  if (f) atomicAdd(found, f);
}

// out[i + #{b < a_i}] = a_i for a sorted, b sorted, a and b disjoint
__global__ void merge_scatter_kernel(const int64_t *__restrict__ a, int64_t na,
                                     const int64_t *__restrict__ b, int64_t nb,
                                     int64_t *__restrict__ out, unsigned long long *collisions) {
  unsigned long long col = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = a[i];
    const int64_t p = lower_bound(b, nb, key);
    if (p < nb && b[p] == key) ++col;
    out[i + p] = key;
  }
  if (collisions && col) atomicAdd(collisions, col);
}

__global__ void split_kernel(int64_t n, const int64_t *__restrict__ codes, int64_t m,
                             int64_t *__restrict__ lo, int64_t *__restrict__ hi) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = codes[e];
    lo[e] = c / n;
    hi[e] = c - (c / n) * n;
  }
}

__global__ void iota_kernel(int32_t *__restrict__ a, int64_t m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    a[e] = (int32_t)e;
}

// --- Graph canonicalisation (graphs.py:29-54) -------------------------------
// flags: [0] endpoint out of range, [1] self-loop, [2] weight <= 0, [3] duplicate
__global__ void canon_codes_kernel(int64_t n, int64_t m, const int64_t *__restrict__ ei,
                                   const int64_t *__restrict__ ej, const double *__restrict__ w,
                                   int64_t *__restrict__ codes, int64_t *__restrict__ iota,
                                   unsigned int *__restrict__ flags) {
  unsigned int f0 = 0, f1 = 0, f2 = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ei[e], b = ej[e];
    f0 |= (a < 0 || b < 0 || a >= n || b >= n);
    f1 |= (a == b);
    f2 |= !(w[e] > 0.0);
    const int64_t lo = a < b ? a : b, hi = a < b ? b : a;
    codes[e] = lo * n + hi;
    iota[e] = e;
  }
  if (f0) atomicOr(flags + 0, 1u);
  if (f1) atomicOr(flags + 1, 1u);
  if (f2) atomicOr(flags + 2, 1u);
}

__global__ void canon_finish_kernel(int64_t m, const int64_t *__restrict__ sorted,
                                    const int64_t *__restrict__ perm, const double *__restrict__ w,
                                    double *__restrict__ w_out, unsigned int *__restrict__ flags) {
  unsigned int dup = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e > 0 && sorted[e] == sorted[e - 1]) dup = 1;
    w_out[e] = w[perm[e]];
  }
  if (dup) atomicOr(flags + 3, 1u);
}

int grid_for(int64_t work, int threads = 256) {
  return (int)std::min<int64_t>(csc::device_info().sm_count * 16,
                                std::max<int64_t>(1, csc::ceil_div(work, threads)));
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 31 && (int64_t(1) << b) < n) ++b;
  return b;
}

}  // namespace

extern "C" {

int csc_laplacian_build(int64_t n, int64_t m, const int64_t *lo, const int64_t *hi,
                        const double *w, int variant, int32_t *indptr, int32_t *indices,
                        double *vals, int64_t capacity, double *deg_out, int64_t *nnz_out,
                        double *bound_out, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 0 && m >= 0, "csc_laplacian_build: negative size");
  CSC_REQUIRE(variant == CSC_LAP_NORMALIZED || variant == CSC_LAP_COMBINATORIAL,
              "unknown Laplacian variant %d", variant);
  CSC_REQUIRE(2 * m + n < (int64_t)INT32_MAX, "csc_laplacian_build: nnz exceeds int32 indexing");
  CSC_REQUIRE(capacity >= 2 * m + n, "csc_laplacian_build: capacity %lld < 2m+n = %lld",
              (long long)capacity, (long long)(2 * m + n));
  CSC_REQUIRE(nnz_out && bound_out, "csc_laplacian_build: NULL host outputs");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  csc::device_info();
  csc::Scratch cnt_lo, cnt_hi, lo_ptr, hi_ptr, hi32, hi_sorted, idx, perm, deg, inv, rowcnt,
      tmp, dmax;
  const int64_t n1 = n + 1, mm = std::max<int64_t>(m, 1), nn = std::max<int64_t>(n, 1);
  CSC_TRY_CUDA(cnt_lo.alloc(sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(cnt_hi.alloc(sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(lo_ptr.alloc(sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(hi_ptr.alloc(sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(hi32.alloc(sizeof(int32_t) * mm, st));
  CSC_TRY_CUDA(hi_sorted.alloc(sizeof(int32_t) * mm, st));
  CSC_TRY_CUDA(idx.alloc(sizeof(int32_t) * mm, st));
  CSC_TRY_CUDA(perm.alloc(sizeof(int32_t) * mm, st));
  CSC_TRY_CUDA(deg.alloc(sizeof(double) * nn, st));
  CSC_TRY_CUDA(inv.alloc(sizeof(double) * nn, st));
  CSC_TRY_CUDA(rowcnt.alloc(sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(dmax.alloc(sizeof(double), st));
  CSC_TRY_CUDA(cudaMemsetAsync(cnt_lo.ptr, 0, sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(cudaMemsetAsync(cnt_hi.ptr, 0, sizeof(int32_t) * n1, st));
  CSC_TRY_CUDA(cudaMemsetAsync(rowcnt.ptr, 0, sizeof(int32_t) * n1, st));
  if (m > 0) {
    degree_hist_kernel<<<grid_for(m), 256, 0, st>>>(lo, hi, m, cnt_lo.as<int32_t>(),
                                                    cnt_hi.as<int32_t>(), hi32.as<int32_t>());
    CSC_CHECK_LAUNCH();
    iota_kernel<<<grid_for(m), 256, 0, st>>>(idx.as<int32_t>(), m);
    CSC_CHECK_LAUNCH();
  }
  size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b1, cnt_lo.as<int32_t>(), lo_ptr.as<int32_t>(), n1, st);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, hi32.as<int32_t>(), hi_sorted.as<int32_t>(),
                                  idx.as<int32_t>(), perm.as<int32_t>(), mm, 0, bits_for(n), st);
  cub::DeviceScan::ExclusiveSum(nullptr, b3, rowcnt.as<int32_t>(), indptr, n1, st);
  cub::DeviceReduce::Max(nullptr, b4, deg.as<double>(), dmax.as<double>(), nn, st);
  const size_t tbytes = std::max(std::max(b1, b2), std::max(b3, b4));
  CSC_TRY_CUDA(tmp.alloc(tbytes, st));
  size_t tb = tbytes;
  CSC_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, cnt_lo.as<int32_t>(),
                                             lo_ptr.as<int32_t>(), n1, st));
  tb = tbytes;
  CSC_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, cnt_hi.as<int32_t>(),
                                             hi_ptr.as<int32_t>(), n1, st));
  if (m > 0) {
    tb = tbytes;
    CSC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, hi32.as<int32_t>(),
                                                 hi_sorted.as<int32_t>(), idx.as<int32_t>(),
                                                 perm.as<int32_t>(), m, 0, bits_for(n), st));
  }
  if (n > 0) {
    degree_kernel<<<grid_for(n), 256, 0, st>>>(n, lo_ptr.as<int32_t>(), hi_ptr.as<int32_t>(),
                                               perm.as<int32_t>(), w, variant, deg.as<double>(),
                                               inv.as<double>(), rowcnt.as<int32_t>());
    CSC_CHECK_LAUNCH();
  }
  tb = tbytes;
  CSC_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, rowcnt.as<int32_t>(), indptr, n1, st));
  if (n > 0) {
    if (m > 0) {
      fill_upper_kernel<<<grid_for(m), 256, 0, st>>>(m, lo, hi, w, lo_ptr.as<int32_t>(),
                                                     hi_ptr.as<int32_t>(), deg.as<double>(),
                                                     inv.as<double>(), variant, indptr, indices,
                                                     vals);
      CSC_CHECK_LAUNCH();
      fill_lower_kernel<<<grid_for(m), 256, 0, st>>>(m, lo, hi, w, hi_ptr.as<int32_t>(),
                                                     perm.as<int32_t>(), inv.as<double>(),
                                                     variant, indptr, indices, vals);
      CSC_CHECK_LAUNCH();
    }
    fill_diag_kernel<<<grid_for(n), 256, 0, st>>>(n, hi_ptr.as<int32_t>(), deg.as<double>(),
                                                  variant, indptr, indices, vals);
    CSC_CHECK_LAUNCH();
    tb = tbytes;
    CSC_TRY_CUDA(cub::DeviceReduce::Max(tmp.ptr, tb, deg.as<double>(), dmax.as<double>(), n, st));
    if (deg_out)
      CSC_TRY_CUDA(cudaMemcpyAsync(deg_out, deg.ptr, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                   st));
  }
  int32_t nnz = 0;
  double maxdeg = 0.0;
  CSC_TRY_CUDA(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (n > 0)
    CSC_TRY_CUDA(cudaMemcpyAsync(&maxdeg, dmax.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  *nnz_out = nnz;
  if (variant == CSC_LAP_NORMALIZED)
    *bound_out = 2.0;
  else
    *bound_out = (n > 0 && m > 0) ? 2.0 * maxdeg : 0.0;
  return CSC_OK;
}

int csc_edge_delta(int64_t n, const int64_t *prev, int64_t m_prev, const int64_t *del,
                   int64_t n_del, const int64_t *ins, int64_t n_ins, int64_t *out,
                   int64_t capacity, int64_t *m_new_out, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 0 && m_prev >= 0 && n_del >= 0 && n_ins >= 0, "csc_edge_delta: negative size");
  CSC_REQUIRE(n_del <= m_prev, "csc_edge_delta: more deletions than edges");
  const int64_t m_new = m_prev - n_del + n_ins;
  CSC_REQUIRE(capacity >= m_new, "csc_edge_delta: capacity %lld < %lld", (long long)capacity,
              (long long)m_new);
  CSC_REQUIRE(m_new_out != nullptr, "csc_edge_delta: NULL m_new_out");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  csc::device_info();
  csc::Scratch keep, kept, nkept, counters, tmp;
  const int64_t mm = std::max<int64_t>(m_prev, 1);
  CSC_TRY_CUDA(keep.alloc(mm, st));
  CSC_TRY_CUDA(kept.alloc(sizeof(int64_t) * mm, st));
  CSC_TRY_CUDA(nkept.alloc(sizeof(int64_t), st));
  CSC_TRY_CUDA(counters.alloc(sizeof(unsigned long long) * 2, st));
  CSC_TRY_CUDA(cudaMemsetAsync(counters.ptr, 0, sizeof(unsigned long long) * 2, st));
  CSC_TRY_CUDA(cudaMemsetAsync(nkept.ptr, 0, sizeof(int64_t), st));
  unsigned long long *found = counters.as<unsigned long long>();
  unsigned long long *coll = found + 1;
  if (m_prev > 0) {
    mark_deleted_kernel<<<grid_for(m_prev), 256, 0, st>>>(prev, m_prev, del, n_del,
                                                          keep.as<int8_t>(), found);
    CSC_CHECK_LAUNCH();
    size_t bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, bytes, prev, keep.as<int8_t>(), kept.as<int64_t>(),
                               nkept.as<int64_t>(), m_prev, st);
    CSC_TRY_CUDA(tmp.alloc(bytes, st));
    CSC_TRY_CUDA(cub::DeviceSelect::Flagged(tmp.ptr, bytes, prev, keep.as<int8_t>(),
                                            kept.as<int64_t>(), nkept.as<int64_t>(), m_prev, st));
  }
  const int64_t n_kept = m_prev - n_del;
  if (n_kept > 0) {
    merge_scatter_kernel<<<grid_for(n_kept), 256, 0, st>>>(kept.as<int64_t>(), n_kept, ins, n_ins,
                                                           out, coll);
    CSC_CHECK_LAUNCH();
  }
  if (n_ins > 0) {
    merge_scatter_kernel<<<grid_for(n_ins), 256, 0, st>>>(ins, n_ins, kept.as<int64_t>(), n_kept,
                                                          out, nullptr);
    CSC_CHECK_LAUNCH();
  }
  unsigned long long h[2] = {0, 0};
  CSC_TRY_CUDA(cudaMemcpyAsync(h, counters.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  if ((int64_t)h[0] != n_del) {
    csc::set_error("csc_edge_delta: %lld of %lld deleted codes are not edges of the graph",
                   (long long)(n_del - (int64_t)h[0]), (long long)n_del);
    return CSC_ERR_ARG;
  }
  if (h[1] != 0) {
    csc::set_error("csc_edge_delta: %llu inserted codes duplicate kept edges", h[1]);
    return CSC_ERR_ARG;
  }
  *m_new_out = m_new;
  return CSC_OK;
}

int csc_graph_canonicalize(int64_t n, int64_t m, const int64_t *ei, const int64_t *ej,
                           const double *w, int64_t *codes_out, double *w_out, int32_t *flags_host,
                           void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 0 && m >= 0 && flags_host != nullptr, "csc_graph_canonicalize: bad arguments");
  CSC_REQUIRE(n < (int64_t)3037000499, "csc_graph_canonicalize: n*n overflows int64 codes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  csc::device_info();
  for (int i = 0; i < 4; ++i) flags_host[i] = 0;
  if (m == 0) return CSC_OK;
  csc::Scratch codes, iota, perm, flags, tmp;
  CSC_TRY_CUDA(codes.alloc(sizeof(int64_t) * m, st));
  CSC_TRY_CUDA(iota.alloc(sizeof(int64_t) * m, st));
  CSC_TRY_CUDA(perm.alloc(sizeof(int64_t) * m, st));
  CSC_TRY_CUDA(flags.alloc(sizeof(unsigned int) * 4, st));
  CSC_TRY_CUDA(cudaMemsetAsync(flags.ptr, 0, sizeof(unsigned int) * 4, st));
  canon_codes_kernel<<<grid_for(m), 256, 0, st>>>(n, m, ei, ej, w, codes.as<int64_t>(),
                                                  iota.as<int64_t>(), flags.as<unsigned int>());
  CSC_CHECK_LAUNCH();
  unsigned int h[4];
  CSC_TRY_CUDA(cudaMemcpyAsync(h, flags.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  flags_host[0] = h[0];
  flags_host[1] = h[1];
  flags_host[2] = h[2];
  if (h[0] || h[1] || h[2]) return CSC_OK;  // caller raises in the reference's order
  // stable LSD radix sort of the codes (numpy argsort kind="stable")
  int bits = 1;
  const unsigned long long maxcode = (unsigned long long)n * (unsigned long long)n;
  while (bits < 63 && (1ull << bits) < maxcode) ++bits;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, codes.as<int64_t>(), codes_out, iota.as<int64_t>(),
                                  perm.as<int64_t>(), m, 0, bits, st);
  CSC_TRY_CUDA(tmp.alloc(tb, st));
  CSC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, codes.as<int64_t>(), codes_out,
                                               iota.as<int64_t>(), perm.as<int64_t>(), m, 0, bits,
                                               st));
  canon_finish_kernel<<<grid_for(m), 256, 0, st>>>(m, codes_out, perm.as<int64_t>(), w, w_out,
                                                   flags.as<unsigned int>());
  CSC_CHECK_LAUNCH();
  CSC_TRY_CUDA(cudaMemcpyAsync(h, flags.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  flags_host[3] = h[3];
  return CSC_OK;
}

int csc_codes_split(int64_t n, const int64_t *codes, int64_t m, int64_t *lo, int64_t *hi,
                    void *stream) {
  CSC_REQUIRE(n > 0 || m == 0, "csc_codes_split: n must be positive");
  if (m == 0) return CSC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  split_kernel<<<grid_for(m), 256, 0, st>>>(n, codes, m, lo, hi);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

}  // extern "C"
