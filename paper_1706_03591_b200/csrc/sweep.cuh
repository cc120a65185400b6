// Fused Chebyshev sweep kernels and their launchers (shared by chebyshev.cu,
// index-ordered rows, and chebyshev_perm.cu, length-ordered rows; split so the
// two schedules' instantiations compile in parallel). One launch = one order
// of the recurrence of cscluster.filters.apply_filter (filters.py:172-186):
//     T_1     = M x,                 out  = c_0 x + c_1 T_1
//     T_{j+1} = 2 M T_j - T_{j-1},   out += c_j T_{j+1}
// (or the moment-series epilogues), M = I - s L in CSR.
//
// Layout. Dense blocks are row-major with a 16-byte-multiple row stride, so a
// nonzero gathers one contiguous row of T_j with 128-bit loads. A group of G
// lanes owns one row; lane l loads vectors l, l+G, ... of each gathered row.
// Column indices and values of the row are loaded cooperatively (one per lane)
// and broadcast with width-G shuffles; four gathered rows are in flight per
// lane before their FMAs (memory-level parallelism for the HBM-bound gather).
//
// Skew. Rows with more than kLongThr stored entries are excluded from the
// main sweep and split into kSeg-entry segments, one warp per segment; the
// segment partials are summed in segment order by a finishing kernel, so the
// result is independent of scheduling. For graphs with widely varying row
// lengths the plan also orders the other rows by length (PERM schedule).
//
// Determinism. Every output element is produced by exactly one thread with a
// fixed accumulation order (a row's entries in stored order, whatever the
// schedule); the optional ||out||^2 uses fixed per-block partials reduced in
// block order.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace csc_sweep {

constexpr int kBlock = 256;
constexpr int kLongThr = 1024;  // rows with more entries go to the segment path
constexpr int kSeg = 512;       // entries per segment of a long row

// Row epilogue shared by all sweeps. Modes:
//   kFirst: T_1 = acc;            out = ca*x + cb*T_1     (prev = x)
//   kMid:   T_{j+1} = 2acc - T_{j-1}; out += ca*T_{j+1}
//   kMoment: T_{j+1} = 2acc - T_{j-1} (or acc for the first order);
//            m0 += <T_{j+1},T_{j+1}>, m1 += <T_{j+1}, T_j>   (no out)
enum { kFirst = 0, kMid = 1, kMomFirst = 2, kMomMid = 3 };

struct SweepArgs {
  const int32_t *indptr;
  const int32_t *indices;
  const void *vals;
  int64_t n;
  // length-ordered schedule only: the nrows short rows in perm order (long
  // rows excluded); the index-ordered kernels walk rows 0..n-1
  const int32_t *perm;
  int64_t nrows;
  int nvec;       // 16-byte vectors per row actually used (chunk width)
  int64_t ldv;    // row stride in 16-byte vectors
  const void *gat;   // T_j (gathered)
  const void *prev;  // T_{j-1}, or x for the first order
  const void *own;   // T_j own rows (moments only)
  void *next;        // T_{j+1}
  void *out;
  double ca, cb;
  double *partials;  // per-block partial sums (nullable unless sumsq/moments)
  int sumsq;
  int hint;          // 1: evict_first policy on the row-local streams
  int prefetch;      // 1: L2 prefetch of the next row's CSR and this row's epilogue rows
  // long-row segments handled by the first seg_blocks blocks of the same launch
  int seg_blocks;
  const int32_t *long_rows;
  const int32_t *seg_off;
  int64_t n_long, n_seg;
  void *seg_scratch;
};

// the slice of a csc_chebop the launchers read
struct SweepPlan {
  int64_t n = 0, n_long = 0, n_seg = 0;
  const int32_t *long_rows = nullptr;
  const int32_t *seg_off = nullptr;
  const int32_t *perm = nullptr;  // all rows by length (longest first), or nullptr
};

// defined in chebyshev.cu: per-launch CUDA-event timing hook and tuning knobs
bool sweeptime_begin(cudaStream_t st);
void sweeptime_end(cudaStream_t st);
void sweep_note_launch(int elem_bytes, int G, int VPL, int mode, bool perm, int grid);
int vpl_pref();
int sweep_g();

// one order over the length-ordered schedule (chebyshev_perm.cu)
int run_order_perm_f64(const SweepPlan &op, const SweepArgs &A, int mode, double *partials,
                       int64_t &nparts, cudaStream_t st, void *seg_scratch);
int run_order_perm_f32(const SweepPlan &op, const SweepArgs &A, int mode, double *partials,
                       int64_t &nparts, cudaStream_t st, void *seg_scratch);

}  // namespace csc_sweep

namespace {

using namespace csc_sweep;


template <typename T>
struct V16;
template <>
struct V16<double> {
  using V = double2;
  static constexpr int E = 2;
};
template <>
struct V16<float> {
  using V = float4;
  static constexpr int E = 4;
};

__device__ __forceinline__ double2 vzero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ float4 vzero(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }

__device__ __forceinline__ void vfma(double2 &acc, double a, const double2 &x) {
  acc.x = fma(a, x.x, acc.x);
  acc.y = fma(a, x.y, acc.y);
}
__device__ __forceinline__ void vfma(float4 &acc, float a, const float4 &x) {
  acc.x = fmaf(a, x.x, acc.x);
  acc.y = fmaf(a, x.y, acc.y);
  acc.z = fmaf(a, x.z, acc.z);
  acc.w = fmaf(a, x.w, acc.w);
}
__device__ __forceinline__ void vadd(double2 &acc, const double2 &x) {
  acc.x += x.x;
  acc.y += x.y;
}
__device__ __forceinline__ void vadd(float4 &acc, const float4 &x) {
  acc.x += x.x;
  acc.y += x.y;
  acc.z += x.z;
  acc.w += x.w;
}
__device__ __forceinline__ double vdot(const double2 &a, const double2 &b) {
  return a.x * b.x + a.y * b.y;
}
__device__ __forceinline__ double vdot(const float4 &a, const float4 &b) {
  return (double)a.x * b.x + (double)a.y * b.y + (double)a.z * b.z + (double)a.w * b.w;
}

// L2 cache policies. The row-local streams of a sweep (T_{j-1}, out, T_{j+1},
// CSR) are touched once per order; marking them evict_first keeps the L2 for
// the randomly gathered rows of T_j. (CSC_STREAM_HINT=0 disables, for A/B.)
__device__ __forceinline__ uint64_t make_policy(int hint) {
  uint64_t p;
  if (hint)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ double2 ld_s(const double2 *a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_s(const float4 *a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_s(double2 *a, const double2 &v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
               :: "l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_s(float4 *a, const float4 &v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ int ld_s(const int32_t *a, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_s(const double *a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_s(const float *a, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}


template <int MODE>
__device__ __forceinline__ void epilogue(double2 acc, const double2 *prev, const double2 *own,
                                         double2 *next, double2 *out, size_t off, double ca,
                                         double cb, double &s0, double &s1, bool sumsq,
                                         uint64_t pol) {
  if (MODE == kFirst) {
    const double2 x = ld_s(prev + off, pol);
    st_s(next + off, acc, pol);
    double2 o;
    o.x = fma(cb, acc.x, ca * x.x);
    o.y = fma(cb, acc.y, ca * x.y);
    st_s(out + off, o, pol);
    if (sumsq) s0 += vdot(o, o);
  } else if (MODE == kMid) {
    const double2 p = ld_s(prev + off, pol);
    double2 t;
    t.x = 2.0 * acc.x - p.x;
    t.y = 2.0 * acc.y - p.y;
    st_s(next + off, t, pol);
    double2 o = ld_s(out + off, pol);
    o.x = fma(ca, t.x, o.x);
    o.y = fma(ca, t.y, o.y);
    st_s(out + off, o, pol);
    if (sumsq) s0 += vdot(o, o);
  } else {
    double2 t = acc;
    if (MODE == kMomMid) {
      const double2 p = ld_s(prev + off, pol);
      t.x = 2.0 * acc.x - p.x;
      t.y = 2.0 * acc.y - p.y;
    }
    st_s(next + off, t, pol);
    const double2 c = ld_s(own + off, pol);
    s0 += vdot(t, t);
    s1 += vdot(t, c);
  }
}

template <int MODE>
__device__ __forceinline__ void epilogue(float4 acc, const float4 *prev, const float4 *own,
                                         float4 *next, float4 *out, size_t off, double ca,
                                         double cb, double &s0, double &s1, bool sumsq,
                                         uint64_t pol) {
  const float a = (float)ca, b = (float)cb;
  if (MODE == kFirst) {
    const float4 x = ld_s(prev + off, pol);
    st_s(next + off, acc, pol);
    float4 o;
    o.x = fmaf(b, acc.x, a * x.x);
    o.y = fmaf(b, acc.y, a * x.y);
    o.z = fmaf(b, acc.z, a * x.z);
    o.w = fmaf(b, acc.w, a * x.w);
    st_s(out + off, o, pol);
    if (sumsq) s0 += vdot(o, o);
  } else if (MODE == kMid) {
    const float4 p = ld_s(prev + off, pol);
    float4 t;
    t.x = 2.f * acc.x - p.x;
    t.y = 2.f * acc.y - p.y;
    t.z = 2.f * acc.z - p.z;
    t.w = 2.f * acc.w - p.w;
    st_s(next + off, t, pol);
    float4 o = ld_s(out + off, pol);
    o.x = fmaf(a, t.x, o.x);
    o.y = fmaf(a, t.y, o.y);
    o.z = fmaf(a, t.z, o.z);
    o.w = fmaf(a, t.w, o.w);
    st_s(out + off, o, pol);
    if (sumsq) s0 += vdot(o, o);
  } else {
    float4 t = acc;
    if (MODE == kMomMid) {
      const float4 p = ld_s(prev + off, pol);
      t.x = 2.f * acc.x - p.x;
      t.y = 2.f * acc.y - p.y;
      t.z = 2.f * acc.z - p.z;
      t.w = 2.f * acc.w - p.w;
    }
    st_s(next + off, t, pol);
    const float4 c = ld_s(own + off, pol);
    s0 += vdot(t, t);
    s1 += vdot(t, c);
  }
}


// Entries per gather batch: narrow groups (G < 32) take SWEEP_NARROW_BATCH
// (A/B knob), full-warp groups 4.
#ifndef SWEEP_NARROW_BATCH
#define SWEEP_NARROW_BATCH 4
#endif
// three-vector groups: 5 (B200 A/B at 3 blocks/SM, ms per order at cfg5 d = 48 /
// 72 / 96: batch 3 3.14 / 5.20 / 5.70, 4 3.06 / 4.91 / 5.47, 5 2.96 / 4.80 / 5.41,
// 6 3.01 / 5.01 / 5.63; 6 or 8 at 2 blocks/SM and 3 or 4 at 4 blocks/SM slower)
#ifndef SWEEP_V3_BATCH
#define SWEEP_V3_BATCH 5
#endif
template <int G, int VPL = 1>
struct SweepBatch {
  static constexpr int value = VPL == 3 ? SWEEP_V3_BATCH : (G < 32 ? SWEEP_NARROW_BATCH : 4);
};

// Gather-accumulate of entries [beg, end) of one row into acc[VPL] by a group
// of G lanes (glane = lane within group, gmask = the group's lanes).
template <typename T, int G, int VPL>
__device__ __forceinline__ void gather_row(const int32_t *__restrict__ indices,
                                           const T *__restrict__ vals,
                                           const typename V16<T>::V *__restrict__ gat, int beg,
                                           int end, int glane, unsigned gmask, int nvec,
                                           int64_t ldv, typename V16<T>::V (&acc)[VPL],
                                           uint64_t pol) {
  using VT = typename V16<T>::V;
  for (int base = beg; base < end; base += G) {
    const int nz = base + glane;
    int my_col = 0;
    T my_val = T(0);
    if (nz < end) {
      my_col = ld_s(indices + nz, pol);
      my_val = ld_s(vals + nz, pol);
    }
    const int cnt = min(G, end - base);
    constexpr int B = SweepBatch<G, VPL>::value;  // entries whose gathers are issued together
    int u = 0;
    for (; u + B <= cnt; u += B) {
      int c[B];
      T a[B];
#pragma unroll
      for (int t = 0; t < B; ++t) {
        c[t] = __shfl_sync(gmask, my_col, u + t, G);
        a[t] = __shfl_sync(gmask, my_val, u + t, G);
      }
      VT x[B][VPL];
#pragma unroll
      for (int t = 0; t < B; ++t) {
        const VT *src = gat + (int64_t)c[t] * ldv;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int v = glane + q * G;
          x[t][q] = (v < nvec) ? __ldg(src + v) : vzero(VT());
        }
      }
#pragma unroll
      for (int t = 0; t < B; ++t)
#pragma unroll
        for (int q = 0; q < VPL; ++q) vfma(acc[q], a[t], x[t][q]);
    }
    if (u < cnt) {  // 1..B-1 remaining entries: their gathers issued together
      const int rem = cnt - u;
      int c[B - 1];
      T a[B - 1];
#pragma unroll
      for (int t = 0; t < B - 1; ++t) {
        const int src_lane = min(u + t, cnt - 1);
        c[t] = __shfl_sync(gmask, my_col, src_lane, G);
        a[t] = __shfl_sync(gmask, my_val, src_lane, G);
      }
      VT x[B - 1][VPL];
#pragma unroll
      for (int t = 0; t < B - 1; ++t) {
        const VT *src = gat + (int64_t)c[t] * ldv;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int v = glane + q * G;
          x[t][q] = (t < rem && v < nvec) ? __ldg(src + v) : vzero(VT());
        }
      }
#pragma unroll
      for (int t = 0; t < B - 1; ++t)
        if (t < rem)
#pragma unroll
          for (int q = 0; q < VPL; ++q) vfma(acc[q], a[t], x[t][q]);
    }
  }
}

// One Chebyshev order over all rows with at most kLongThr entries.
template <typename T, int LV>
__device__ __forceinline__ void segment_body(const SweepArgs &A, int64_t first_warp,
                                             int64_t nwarps);

// Narrow row groups (G < 32, <= 2 vectors per lane: d <= 64 fp64) are latency
// bound at 80 registers (3 blocks/SM); capping them at 64 gives 4 blocks/SM:
// cfg4 fp64 d=64 7.30 -> 6.62 ms, cfg5 d=48 3.31 -> 3.00 ms per order (interleaved
// A/B). Wider groups ask for 3 blocks/SM (<= 85 registers): ptxas then issues
// all 4 x VPL gathers of a batch before their FMAs; left to its own register
// heuristic it chose 58 registers and interleaved loads with FMAs (cfg3 fp64
// 4.60 vs 5.96 ms per order, B200 A/B of the same source).
#ifndef SWEEP_NARROW_MIN
#define SWEEP_NARROW_MIN 4
#endif
#ifndef SWEEP_V3_MIN
#define SWEEP_V3_MIN 3
#endif
#ifndef SWEEP_WIDE_MIN
#define SWEEP_WIDE_MIN 3
#endif
template <int G, int VPL>
struct SweepMinBlocks {
  static constexpr int value =
      (G < 32 && VPL <= 2) ? SWEEP_NARROW_MIN : (VPL == 3 ? SWEEP_V3_MIN : (VPL <= 2 ? SWEEP_WIDE_MIN : 0));
};

template <typename T, int G, int VPL, int MODE, bool PERM>
__global__ void __launch_bounds__(kBlock, (SweepMinBlocks<G, VPL>::value)) sweep_kernel(SweepArgs A) {
  using VT = typename V16<T>::V;
  __shared__ double red[kBlock / 32];
  if ((int)blockIdx.x < A.seg_blocks) {  // long-row segments, overlapped with the rows
    constexpr int LV = (VPL * G + 31) / 32;
    segment_body<T, LV>(A, (int64_t)blockIdx.x * (kBlock / 32) + threadIdx.x / 32,
                        (int64_t)A.seg_blocks * (kBlock / 32));
    return;
  }
  const int64_t bid = (int64_t)blockIdx.x - A.seg_blocks;
  const int64_t nblocks = (int64_t)gridDim.x - A.seg_blocks;
  const int lane = threadIdx.x & 31;
  const int glane = lane % G;
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((lane / G) * G));
  const int groups_per_block = kBlock / G;
  const int64_t ngroups = nblocks * groups_per_block;
  const T *vals = static_cast<const T *>(A.vals);
  const VT *gat = static_cast<const VT *>(A.gat);
  const VT *prev = static_cast<const VT *>(A.prev);
  const VT *own = static_cast<const VT *>(A.own);
  VT *next = static_cast<VT *>(A.next);
  VT *out = static_cast<VT *>(A.out);
  double s0 = 0.0, s1 = 0.0;
  const bool sumsq = A.sumsq != 0;
  const uint64_t pol = make_policy(A.hint);

  int64_t i = bid * groups_per_block + threadIdx.x / G;
#define CSC_ROW_BODY                                                                            \
  {                                                                                             \
    VT acc[VPL];                                                                                \
    _Pragma("unroll") for (int q = 0; q < VPL; ++q) acc[q] = vzero(VT());                       \
    gather_row<T, G, VPL>(A.indices, vals, gat, beg, end, glane, gmask, A.nvec, A.ldv, acc, pol); \
    _Pragma("unroll") for (int q = 0; q < VPL; ++q) {                                           \
      const int v = glane + q * G;                                                              \
      if (v < A.nvec)                                                                           \
        epilogue<MODE>(acc[q], prev, own, next, out, (size_t)row * A.ldv + v, A.ca, A.cb, s0,   \
                       s1, sumsq, pol);                                                         \
    }                                                                                           \
  }
  if constexpr (!PERM) {
    // Index order (the graph's own node order keeps community gathers
    // L2-local): the next row's extent one grid stride ahead, rows with more
    // than kLongThr entries left to the segment path.
    int nbeg = 0, nend = 0;
    if (i < A.n) {
      nbeg = __ldg(A.indptr + i);
      nend = __ldg(A.indptr + i + 1);
    }
    for (; i < A.n; i += ngroups) {
      const int64_t row = i;
      const int beg = nbeg, end = nend;
      if (i + ngroups < A.n) {
        nbeg = __ldg(A.indptr + i + ngroups);
        nend = __ldg(A.indptr + i + ngroups + 1);
      }
      if (end - beg > kLongThr) continue;  // segment path
      CSC_ROW_BODY
    }
  } else {
    // Length order (skewed degrees): rows A.perm[0..nrows), longest first, so
    // the row groups of a warp gather rows of similar length. Two grid strides
    // deep: the extent of the next row is already in registers, so its CSR
    // lines are prefetched into L2 while this row gathers (its own index loads
    // then hit L2), together with this row's epilogue rows, and the indptr
    // loads of the row after are in flight. (Measured on configs[3]: -2%; in
    // index order the prefetches cost the L2 more than they save.)
    const int64_t nrows = A.nrows;
    int64_t r1 = 0, r2 = 0;
    int b1 = 0, e1 = 0, b2 = 0, e2 = 0;
    if (i < nrows) {
      r1 = __ldg(A.perm + i);
      b1 = __ldg(A.indptr + r1);
      e1 = __ldg(A.indptr + r1 + 1);
    }
    if (i + ngroups < nrows) {
      r2 = __ldg(A.perm + i + ngroups);
      b2 = __ldg(A.indptr + r2);
      e2 = __ldg(A.indptr + r2 + 1);
    }
    const int row_lines = (A.nvec + 7) / 8;  // 128-byte lines of a row chunk (+1 if unaligned)
    for (; i < nrows; i += ngroups) {
      const int64_t row = r1;
      const int beg = b1, end = e1;
      r1 = r2;
      b1 = b2;
      e1 = e2;
      if (i + 2 * ngroups < nrows) {
        r2 = __ldg(A.perm + i + 2 * ngroups);
        b2 = __ldg(A.indptr + r2);
        e2 = __ldg(A.indptr + r2 + 1);
      }
      if (A.prefetch && glane <= row_lines) {
        const size_t off = (size_t)row * A.ldv + min(glane * 8, A.nvec - 1);
        prefetch_l2(prev + off);
        if (MODE == kMid) prefetch_l2(out + off);
        if (MODE >= kMomFirst) prefetch_l2(own + off);
      }
      if (A.prefetch && i + ngroups < nrows) {
        constexpr int kPerLine = 128 / (int)sizeof(T);
        const int ib = b1 + glane * 32, vb = b1 + glane * kPerLine;
        if (ib < e1) prefetch_l2(A.indices + ib);
        if (vb < e1) prefetch_l2(vals + vb);
      }
      CSC_ROW_BODY
    }
  }
#undef CSC_ROW_BODY
  if (A.partials) {
    const double b0 = block_sum<kBlock>(s0, red);
    if (MODE >= kMomFirst) {
      const double b1 = block_sum<kBlock>(s1, red);
      if (threadIdx.x == 0) {
        A.partials[2 * bid] = b0;
        A.partials[2 * bid + 1] = b1;
      }
    } else if (threadIdx.x == 0) {
      A.partials[bid] = b0;
    }
  }
}

// Long rows, phase 1: one warp per kSeg-entry segment -> scratch[seg].
template <typename T, int VPL>
__device__ __forceinline__ void segment_body(const SweepArgs &A, int64_t first_warp,
                                             int64_t warps) {
  using VT = typename V16<T>::V;
  const int lane = threadIdx.x & 31;
  const T *vals = static_cast<const T *>(A.vals);
  const VT *gat = static_cast<const VT *>(A.gat);
  VT *scratch = static_cast<VT *>(A.seg_scratch);
  const int32_t *long_rows = A.long_rows, *seg_off = A.seg_off;
  const int64_t n_long = A.n_long, n_seg = A.n_seg;
  const uint64_t pol = make_policy(A.hint);
  for (int64_t s = first_warp; s < n_seg; s += warps) {
    // long row owning segment s: last r with seg_off[r] <= s
    int64_t lo = 0, hi = n_long - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (__ldg(seg_off + mid) <= s) lo = mid; else hi = mid - 1;
    }
    const int row = __ldg(long_rows + lo);
    const int rbeg = __ldg(A.indptr + row), rend = __ldg(A.indptr + row + 1);
    const int beg = rbeg + (int)(s - __ldg(seg_off + lo)) * kSeg;
    const int end = min(beg + kSeg, rend);
    VT acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = vzero(VT());
    gather_row<T, 32, VPL>(A.indices, vals, gat, beg, end, lane, 0xffffffffu, A.nvec, A.ldv, acc, pol);
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int v = lane + q * 32;
      if (v < A.nvec) scratch[s * A.nvec + v] = acc[q];
    }
  }
}

// Long rows, phase 2: one warp per long row sums its segments in order and
// applies the epilogue. Partials go after the main sweep's.
template <typename T, int VPL, int MODE>
__global__ void __launch_bounds__(kBlock)
    long_finish_kernel(SweepArgs A, const int32_t *__restrict__ long_rows,
                       const int32_t *__restrict__ seg_off, int64_t n_long,
                       const typename V16<T>::V *__restrict__ scratch, int64_t partial_base) {
  using VT = typename V16<T>::V;
  __shared__ double red[kBlock / 32];
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kBlock / 32);
  const VT *prev = static_cast<const VT *>(A.prev);
  const VT *own = static_cast<const VT *>(A.own);
  VT *next = static_cast<VT *>(A.next);
  VT *out = static_cast<VT *>(A.out);
  double s0 = 0.0, s1 = 0.0;
  const uint64_t pol = make_policy(A.hint);
  for (int64_t r = (int64_t)blockIdx.x * (kBlock / 32) + threadIdx.x / 32; r < n_long;
       r += warps) {
    const int row = long_rows[r];
    VT acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = vzero(VT());
    for (int64_t s = seg_off[r]; s < seg_off[r + 1]; ++s) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int v = lane + q * 32;
        if (v < A.nvec) vadd(acc[q], scratch[s * A.nvec + v]);
      }
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int v = lane + q * 32;
      if (v < A.nvec)
        epilogue<MODE>(acc[q], prev, own, next, out, (size_t)row * A.ldv + v, A.ca, A.cb, s0,
                       s1, A.sumsq != 0, pol);
    }
  }
  if (A.partials) {
    const double b0 = block_sum<kBlock>(s0, red);
    if (MODE >= kMomFirst) {
      const double b1 = block_sum<kBlock>(s1, red);
      if (threadIdx.x == 0) {
        A.partials[2 * (partial_base + blockIdx.x)] = b0;
        A.partials[2 * (partial_base + blockIdx.x) + 1] = b1;
      }
    } else if (threadIdx.x == 0) {
      A.partials[partial_base + blockIdx.x] = b0;
    }
  }
}


template <typename T, int G, int VPL, int MODE, bool PERM>
int launch_sweep(const SweepArgs &A, int grid, cudaStream_t st) {
  const bool timed = sweeptime_begin(st);
  sweep_note_launch((int)sizeof(T), G, VPL, MODE, PERM, grid);
  sweep_kernel<T, G, VPL, MODE, PERM><<<grid, kBlock, 0, st>>>(A);
  CSC_CHECK_LAUNCH();
  if (timed) sweeptime_end(st);
  return CSC_OK;
}

template <typename T, int G, int VPL, bool PERM>
int sweep_grid() {
  static int occ = 0;
  if (occ == 0) {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, sweep_kernel<T, G, VPL, kMid, PERM>, kBlock, 0);
    occ = o > 0 ? o : 1;
  }
  return occ * csc::device_info().sm_count;
}

template <typename T, int G, int VPL, bool PERM>
int run_order_gv(const SweepPlan &op, SweepArgs A, int mode, double *partials,
                 int64_t &nparts, cudaStream_t st, void *seg_scratch) {
  using VT = typename V16<T>::V;
  const int64_t groups_per_block = kBlock / G;
  int grid = (int)std::min<int64_t>(sweep_grid<T, G, VPL, PERM>(),
                                    std::max<int64_t>(1, csc::ceil_div(op.n, groups_per_block)));
  A.partials = partials;
  A.perm = PERM ? op.perm + op.n_long : nullptr;  // the first n_long entries: segment rows
  A.nrows = PERM ? op.n - op.n_long : op.n;
  A.seg_blocks = 0;
  if (op.n_long > 0) {
    A.seg_blocks = (int)std::min<int64_t>(csc::device_info().sm_count * 4,
                                          csc::ceil_div(op.n_seg, kBlock / 32));
    A.long_rows = op.long_rows;
    A.seg_off = op.seg_off;
    A.n_long = op.n_long;
    A.n_seg = op.n_seg;
    A.seg_scratch = seg_scratch;
  }
  const int main_grid = grid;
  grid += A.seg_blocks;
  int rc = CSC_OK;
  switch (mode) {
    case kFirst: rc = launch_sweep<T, G, VPL, kFirst, PERM>(A, grid, st); break;
    case kMid: rc = launch_sweep<T, G, VPL, kMid, PERM>(A, grid, st); break;
    case kMomFirst: rc = launch_sweep<T, G, VPL, kMomFirst, PERM>(A, grid, st); break;
    default: rc = launch_sweep<T, G, VPL, kMomMid, PERM>(A, grid, st); break;
  }
  if (rc != CSC_OK) return rc;
  grid = main_grid;
  nparts = grid;
  if (op.n_long > 0) {
    constexpr int LV = (VPL * G + 31) / 32;  // vectors per lane at G = 32
    const int fgrid = (int)std::min<int64_t>(csc::device_info().sm_count * 4,
                                             csc::ceil_div(op.n_long, kBlock / 32));
    const VT *sc = static_cast<const VT *>(seg_scratch);
    switch (mode) {
      case kFirst:
        long_finish_kernel<T, LV, kFirst><<<fgrid, kBlock, 0, st>>>(A, op.long_rows, op.seg_off,
                                                                    op.n_long, sc, grid);
        break;
      case kMid:
        long_finish_kernel<T, LV, kMid><<<fgrid, kBlock, 0, st>>>(A, op.long_rows, op.seg_off,
                                                                  op.n_long, sc, grid);
        break;
      case kMomFirst:
        long_finish_kernel<T, LV, kMomFirst><<<fgrid, kBlock, 0, st>>>(
            A, op.long_rows, op.seg_off, op.n_long, sc, grid);
        break;
      default:
        long_finish_kernel<T, LV, kMomMid><<<fgrid, kBlock, 0, st>>>(A, op.long_rows, op.seg_off,
                                                                     op.n_long, sc, grid);
        break;
    }
    CSC_CHECK_LAUNCH();
    nparts += fgrid;
  }
  return CSC_OK;
}

template <typename T, int G, bool PERM>
int run_order_g(const SweepPlan &op, const SweepArgs &A, int mode, double *partials,
                int64_t &nparts, cudaStream_t st, void *seg_scratch) {
  const int need = (A.nvec + G - 1) / G;  // vectors per lane at this group width
  if (need <= 1) return run_order_gv<T, G, 1, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  if (need <= 2) return run_order_gv<T, G, 2, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  if constexpr (G == 8 || G == 16) {  // 3 vectors per lane: 24 (d = 48 fp64) / 36-48 vectors without idle lane slots
    if (need == 3) return run_order_gv<T, G, 3, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  }
  if (need <= 4) return run_order_gv<T, G, 4, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  return run_order_gv<T, G, 8, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
}

// Row-group width G: the smallest power of two >= nvec / preferred-VPL
// (4..32); each lane then holds ceil(nvec/G) <= 8 vectors of every gathered row.
template <typename T, bool PERM>
int run_order(const SweepPlan &op, const SweepArgs &A, int mode, double *partials,
              int64_t &nparts, cudaStream_t st, void *seg_scratch) {
  // default (0): 2 vectors per lane for rows up to 512 B, else full-warp groups
  // (A/B on B200: cfg4 fp32 d=64 4.59 vs 4.76 ms/order, cfg5 d=48 3.33 vs 3.40)
  switch (sweep_g()) {
    case 4: return run_order_g<T, 4, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
    case 8: return run_order_g<T, 8, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
    case 16: return run_order_g<T, 16, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
    case 32: return run_order_g<T, 32, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
    default: break;
  }
  const int pref = vpl_pref() ? vpl_pref() : (A.nvec <= 32 ? 2 : 1);
  const int want = (A.nvec + pref - 1) / pref;
  if (!vpl_pref()) {
    // three vectors per lane when that leaves fewer idle lane slots than the
    // power-of-two choice below (B200 A/B, ms per order: cfg5 d = 48 3.20 ->
    // 3.07, d = 72 5.26 -> 4.90, cfg3 d = 40 1.98 -> 1.89)
    const int g0 = want <= 4 ? 4 : want <= 8 ? 8 : want <= 16 ? 16 : 32;
    const int slots0 = g0 * ((A.nvec + g0 - 1) / g0 <= 2 ? (A.nvec + g0 - 1) / g0
                             : (A.nvec + g0 - 1) / g0 <= 4 ? 4 : 8);
    if (A.nvec > 16 && A.nvec <= 24 && 24 < slots0)
      return run_order_g<T, 8, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
    if (A.nvec > 32 && A.nvec <= 48 && 48 < slots0)
      return run_order_g<T, 16, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  }
  if (want <= 4) return run_order_g<T, 4, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  if (want <= 8) return run_order_g<T, 8, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  if (want <= 16) return run_order_g<T, 16, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
  return run_order_g<T, 32, PERM>(op, A, mode, partials, nparts, st, seg_scratch);
}


}  // namespace
