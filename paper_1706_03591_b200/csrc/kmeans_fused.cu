// Fused Lloyd k-means for small feature blocks: every restart of one
// kmeans() call (kmeans.py:120-144) in ONE cooperative persistent launch.
//
// Why: at configs[1] scale (n = 20k, d = 80, k = 20, 10 restarts) one Lloyd
// iteration is ~30 us of arithmetic for all restarts together, but the
// per-restart lane path (csc_kmeans_run) needs ~10 dependent kernel nodes per
// iteration and the restarts contend for the GPU: ~60-85 us per iteration on
// the longest restart's critical path. Here each CTA (one per SM) owns a
// contiguous row range whose features stay resident in shared memory for the
// whole run; restarts advance in lock step (one counter handshake per phase,
// no grid barrier in the steady state):
//
//   phase 1 (per CTA; the active restarts are spread over 1, 2 or 4 thread
//   groups, so a lone long-running restart gets the whole CTA)
//     - the stop rule (prev - cost2 <= tol * prev, or max_iters;
//       kmeans.py:112-116) on the previous iteration's cost by the centroid
//       identity (the lane path's form), decided identically in every block;
//       a stopping restart instead computes its exact difference-form cost
//       sum |f_i - c_{l_i}|^2 (kmeans.py:111, the returned value) and writes
//       its final labels
//     - Hamerly bounds (ub >= |f - c_a|, lb <= min_{j != a} |f - c_j|, moved
//       by the centroid movements): rows whose bounds cannot exclude a label
//       change are recomputed in the reference's GEMM form
//       max(0, (|f|^2 - 2 f.c) + |c|^2), first-index argmin (kmeans.py:54-61,
//       96-97; the per-pair arithmetic of assign_small_kernel, so labels are
//       bit-identical to the lane path's for the same centroids)
//     - per-cluster sums (and |f|^2 sums) of the CTA's rows in row order for
//       the clusters whose membership changed (stable counting sort by label)
//   one arrival per (block, restart)
//   phase 2 ((restart, cluster) items over the blocks, each waiting for its
//   restart's arrivals only)
//     - means = sums / max(count, 1) (kmeans.py:84): block partials added in
//       block order; movement, |c|^2 and the cluster's identity cost term
//     - a stopping restart: the fixed-order sum of the blocks' exact costs
//   every block waits for the k items of every active restart
//   rare path (an empty cluster, kmeans.py:99-108): exact reassignment of every
//   row (own distances), the reference's argmax reseeding in one CTA, updated
//   partials, means again (four grid barriers, only when it happens).
//
// Results: labels / cost of every restart. As in the lane path, the stop rule
// uses the centroid-identity cost and the returned cost the exact difference
// form. All reductions have a fixed order: deterministic.
// No tensor cores (north_star); FP64 SIMT.
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int kFT = 384;          // threads per CTA (one CTA per SM; 168 registers)
constexpr int kFW = kFT / 32;     // warps per CTA
constexpr int kFMaxK = 32;        // one centroid per lane
constexpr int kFMaxD = 128;       // <= 4 columns per lane in the means pass
constexpr int kFMaxR = 32;        // restarts
constexpr int kFMisc = 4 + kFW;   // per-group int scratch

struct FusedArgs {
  const double *F;
  const double *fnorm;
  int64_t n, d, ld, k, R, ldc;
  int max_iters;
  double tol;
  int32_t *labels_out;  // [R][n]
  double *cost_out;     // [R]
  int32_t *iters_out;   // [R]
  double *cent;         // [2][R][k][ldc]   centroids by iteration parity
  double *kvec;         // [2][R][2][k]     |c|^2, movement by iteration parity
  double *psum;         // [R][G][k][d]     block partial sums
  double *cpart;        // [R][G]           block partial exact costs (final iteration)
  double *pq;           // [R][G][k]        block partial sums of |f|^2 per cluster
  double *cterm;        // [2][R][k]        centroid-identity cost terms by iteration parity
  int32_t *stopping;    // [R] iteration whose phase 1 decided the stop (-1 before)
  double *hist;         // [R][max_iters + 1]
  double *own;          // [R][n]           rare path: own distances
  int32_t *pcnt;        // [R][G][k]
  int32_t *done;        // [R]
  int32_t *eflag;       // [R]  = g + 1 when iteration g found an empty cluster
  int32_t *nrep;        // [R]
  int32_t *rep_idx;     // [R][k]
  int32_t *rep_j;       // [R][k]
  unsigned *bar;        // [2] arrival count, generation
  unsigned *arrive;     // [R] blocks' phase-1 arrivals per restart (monotonic: G per iteration)
  unsigned *readycnt;   // [R] finished phase-2 items per restart (monotonic: k per iteration)
  // in-kernel k-means++ (kmeans.py:64-77), when kpp_first != nullptr
  const int64_t *kpp_first;  // [R] the restart's integers(n) draw
  const double *kpp_unif;    // [R][k-1] its random() draws
  double *kpp_part;          // [2][R][G] block sums of the D^2 weights (draw parity)
  double *kpp_w;             // [2][R][G][rows_max] blocks' D^2 weights (draw parity)
  double *kpp_pre;           // [2][R][G][rows_max] their in-block prefix sums
  int32_t *kpp_flag;         // [R] first j whose D^2 mass was 0 (host replays), else -1
  double *seeds_out;         // [R][k][ldc] the seeds (nullable)
  unsigned long long *trace;  // optional: CTA 0's globaltimer at phase boundaries [iter][8]
  int64_t trace_cap;
  int G, rows_max, ldf, lds, ngmax;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire_i(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier (all CTAs co-resident: cooperative launch). Writes before
// it are visible to __ldcg loads after it.
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned G) {
  // one monotonic arrival counter (zeroed per launch): the e-th barrier of
  // every block returns old in [eG, (e+1)G) and releases at (e+1)G -- one
  // atomic per block, no reset round trip
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned target = (atomicAdd(bar, 1u) / G + 1) * G;
    while (ld_acquire(bar) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// sum over the warp, lane 0's association broadcast (all lanes equal)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

// Global row of the block's local row i: start + stride * i. k-means++ uses
// contiguous ranges (its D^2 draw scans rows in order); the Lloyd phases use an
// interleaved map (row = block + G i) so every block holds a sample of every
// community and the blocks' candidate counts (their phase-1 work) balance.
struct RowMap {
  int64_t start, stride;
  __device__ __forceinline__ int64_t operator()(int64_t i) const { return start + stride * i; }
};

// A thread group working on one restart at a time (named barrier id + 1).
struct Grp {
  int id, GT, GW, gt, gw;
  __device__ __forceinline__ void sync() const { named_sync(id + 1, GT); }
};

struct Shared {
  double *Fs, *fns, *fsq, *ubs, *lbs, *p2, *p2q;  // CTA-wide
  int32_t *labs, *act, *p2c, *work;         // CTA-wide
};
struct GShared {
  double *Cs, *cn, *del, *red, *scal;
  int32_t *cand, *perm, *cnt, *runp, *misc;
};

__host__ __device__ inline int64_t gstride_d(int lds) { return 32 * (int64_t)lds + 64 + kFW + 4; }
__host__ __device__ inline int64_t gstride_i(int64_t RM) { return 2 * RM + 64 + kFMisc; }
// double offset of the per-group area: after Fs, |f|^2, sqrt, ub, lb and the
// phase-2 scratch, rounded to 16 bytes (the k-means++ staging reads double2)
__host__ __device__ inline int64_t group_base(int64_t RM, int64_t ldf, int64_t R, int64_t d) {
  return (RM * ldf + 2 * RM + 2 * R * RM + kFW * (d + 1) + 1) & ~int64_t(1);
}

__device__ __forceinline__ Shared carve(unsigned char *raw, const FusedArgs &a) {
  const int64_t RM = a.rows_max, R = a.R;
  Shared s;
  s.Fs = reinterpret_cast<double *>(raw);
  s.fns = s.Fs + RM * a.ldf;
  s.fsq = s.fns + RM;
  s.ubs = s.fsq + RM;
  s.lbs = s.ubs + R * RM;
  s.p2 = s.lbs + R * RM;  // [kFW][d]
  s.p2q = s.p2 + kFW * a.d;  // [kFW]
  int32_t *ib = reinterpret_cast<int32_t *>(reinterpret_cast<double *>(raw) + group_base(RM, a.ldf, R, a.d) +
                                            a.ngmax * gstride_d(a.lds));
  s.labs = ib;
  s.act = ib + R * RM;  // [kFMaxR + 1]
  s.p2c = s.act + kFMaxR + 1;  // [kFW]
  s.work = s.p2c + kFW;        // [1] phase-1 restart counter (groups take the next restart)
  return s;
}

__device__ __forceinline__ GShared gcarve(unsigned char *raw, const FusedArgs &a, int gi) {
  const int64_t RM = a.rows_max, R = a.R;
  GShared g;
  double *gb = reinterpret_cast<double *>(raw) + group_base(RM, a.ldf, R, a.d);
  g.Cs = gb + gi * gstride_d(a.lds);
  g.cn = g.Cs + 32 * a.lds;
  g.del = g.cn + 32;
  g.red = g.del + 32;
  g.scal = g.red + kFW;
  int32_t *ib = reinterpret_cast<int32_t *>(gb + a.ngmax * gstride_d(a.lds)) + R * RM + kFMaxR + 1 +
                kFW + 1;
  int32_t *gi32 = ib + gi * gstride_i(RM);
  g.cand = gi32;
  g.perm = g.cand + RM;
  g.cnt = g.perm + RM;
  g.runp = g.cnt + 32;
  g.misc = g.runp + 32;
  return g;
}

// Centroids of restart r at iteration g into the group's Cs (rows >= k stay
// zero), |c|^2 (computed for the seeds, else from phase 2) and movements.
__device__ void group_load(const FusedArgs &a, const GShared &gs, const Grp &G_, int r, int g) {
  const int64_t k = a.k, d = a.d, R = a.R, kd = k * d;
  const double *Cc = a.cent + ((int64_t)(g & 1) * R + r) * k * a.ldc;
  // element e = gt + u GT of the k x d tile as (row, column), stepped without
  // divisions in the loop (integer division is a long instruction sequence)
  constexpr int U = 8;
  const int di = (int)d, GT = G_.GT;
  const int dj = GT / di, dt = GT - dj * di;
  int j0 = G_.gt / di, t0 = G_.gt - j0 * di;
  for (int64_t e0 = G_.gt; e0 < kd; e0 += (int64_t)U * GT) {
    double v[U];
    int jj[U], tt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      jj[u] = j0;
      tt[u] = t0;
      if (e0 + (int64_t)u * GT < kd) v[u] = __ldcg(Cc + j0 * a.ldc + t0);
      t0 += dt;
      j0 += dj;
      if (t0 >= di) {
        t0 -= di;
        ++j0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + (int64_t)u * GT < kd) gs.Cs[jj[u] * a.lds + tt[u]] = v[u];
  }
  if (g > 0) {
    const double *kv = a.kvec + ((int64_t)(g & 1) * R + r) * 2 * k;
    if (G_.gt < k) {
      gs.cn[G_.gt] = __ldcg(kv + G_.gt);
      gs.del[G_.gt] = __ldcg(kv + k + G_.gt);
    }
  }
  G_.sync();
  if (g == 0) {  // |c|^2 of the seeds, one thread per centroid
    if (G_.gt < k) {
      const double *cr = gs.Cs + (int64_t)G_.gt * a.lds;
      double v = 0.0;
      for (int64_t t = 0; t < d; ++t) v = fma(cr[t], cr[t], v);
      gs.cn[G_.gt] = v;
    }
    G_.sync();
  }
}

// GEMM-form distances of a 32-row tile to all centroids, register-tiled:
// lane = (row group rg = lane/4, centroid group cg = lane%4); the lane owns
// rows p0 + rg + 8q (q < 4) and, per pass of 16 centroids, centroids
// c0 + cg + 4c (c < TC <= 4), so each shared load feeds 4 or TC FMAs and is
// conflict-free (8 consecutive rows / 4 consecutive centroids at odd
// strides). Per pair the arithmetic is assign_small_kernel's: acc =
// fma(f_t, c_t, acc) in ascending t from 0.0, then
// max(0, (|f|^2 - 2 acc) + |c|^2); the (min, argmin, second) merge keeps the
// lowest index on ties. Labels, bounds and own distances are therefore
// bit-identical to the lane path's. cand == nullptr: rows p0.. themselves.
template <int TR, int TC>
__device__ __forceinline__ void assign_pass(const FusedArgs &a, const GShared &gs, int c0,
                                            const double *const (&fp)[TR], const double (&fn)[TR],
                                            double (&v)[TR], double (&v2)[TR], int (&vi)[TR]) {
  const int cg = threadIdx.x & 3;
  const int64_t d = a.d, k = a.k, lds = a.lds;
  const double *cp = gs.Cs + (int64_t)(c0 + cg) * lds;
  double acc[TR][TC];
#pragma unroll
  for (int q = 0; q < TR; ++q)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[q][c] = 0.0;
#pragma unroll (TR == 4 ? 2 : 4)
  for (int64_t t = 0; t < d; ++t) {
    double f[TR], cv[TC];
#pragma unroll
    for (int q = 0; q < TR; ++q) f[q] = fp[q][t];
#pragma unroll
    for (int c = 0; c < TC; ++c) cv[c] = cp[(int64_t)(4 * c) * lds + t];
#pragma unroll
    for (int q = 0; q < TR; ++q)
#pragma unroll
      for (int c = 0; c < TC; ++c) acc[q][c] = fma(f[q], cv[c], acc[q][c]);
  }
#pragma unroll
  for (int c = 0; c < TC; ++c) {
    const int j = c0 + cg + 4 * c;
    if (j < k) {
      const double cnj = gs.cn[j];
#pragma unroll
      for (int q = 0; q < TR; ++q) {
        const double tt = __dsub_rn(fn[q], __dmul_rn(2.0, acc[q][c]));
        const double d2 = fmax(__dadd_rn(tt, cnj), 0.0);
        if (d2 < v[q]) {  // ascending j within the lane: a tie keeps the earlier index
          v2[q] = v[q];
          v[q] = d2;
          vi[q] = j;
        } else {
          v2[q] = fmin(v2[q], d2);
        }
      }
    }
  }
}

// rows p0 + rg + 8q (q < TR) of the candidate list (or of the CTA's rows);
// marks the clusters a changed row left or joined in gs.misc[1] (bit mask)
template <int TR>
__device__ __forceinline__ void assign_rows(const FusedArgs &a, const Shared &s, const GShared &gs,
                                            int r, int p0, int ncand, const int32_t *cand,
                                            bool want_own, RowMap rm, bool fresh) {
  const int lane = threadIdx.x & 31, rg = lane >> 2, cg = lane & 3;
  const int64_t k = a.k, RM = a.rows_max, ldf = a.ldf;
  int row[TR];
  const double *fp[TR];
  double fn[TR], v[TR], v2[TR];
  int vi[TR];
#pragma unroll
  for (int q = 0; q < TR; ++q) {
    const int p = p0 + rg + 8 * q;
    row[q] = p < ncand ? (cand ? cand[p] : p) : -1;
    fp[q] = s.Fs + (int64_t)(row[q] < 0 ? 0 : row[q]) * ldf;
    fn[q] = row[q] >= 0 ? s.fns[row[q]] : 0.0;
    v[q] = INFINITY;
    v2[q] = INFINITY;
    vi[q] = 0x7fffffff;
  }
  // one pass over d when the TR x TC accumulators fit (the chain of d FMAs per
  // pair is the latency of a call), else two passes of <= 16 centroids
  const int tc = (int)((k + 3) / 4);
  if (TR * tc <= 20) {
    switch (tc) {
      case 1: assign_pass<TR, 1>(a, gs, 0, fp, fn, v, v2, vi); break;
      case 2: assign_pass<TR, 2>(a, gs, 0, fp, fn, v, v2, vi); break;
      case 3: assign_pass<TR, 3>(a, gs, 0, fp, fn, v, v2, vi); break;
      case 4: assign_pass<TR, 4>(a, gs, 0, fp, fn, v, v2, vi); break;
      case 5: assign_pass<TR, 5>(a, gs, 0, fp, fn, v, v2, vi); break;
      case 6: assign_pass<TR, (TR <= 2 ? 6 : 1)>(a, gs, 0, fp, fn, v, v2, vi); break;
      case 7: assign_pass<TR, (TR <= 2 ? 7 : 1)>(a, gs, 0, fp, fn, v, v2, vi); break;
      default: assign_pass<TR, (TR <= 2 ? 8 : 1)>(a, gs, 0, fp, fn, v, v2, vi); break;
    }
  } else {
    for (int c0 = 0; c0 < k; c0 += 16) {
      const int64_t tcn = (k - c0 + 3) / 4;
      switch (tcn < 4 ? (int)tcn : 4) {
        case 1: assign_pass<TR, 1>(a, gs, c0, fp, fn, v, v2, vi); break;
        case 2: assign_pass<TR, 2>(a, gs, c0, fp, fn, v, v2, vi); break;
        case 3: assign_pass<TR, 3>(a, gs, c0, fp, fn, v, v2, vi); break;
        default: assign_pass<TR, 4>(a, gs, c0, fp, fn, v, v2, vi); break;
      }
    }
  }
  unsigned moved = 0;
#pragma unroll
  for (int q = 0; q < TR; ++q) {
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v[q], o);
      const double ov2 = __shfl_xor_sync(0xffffffffu, v2[q], o);
      const int oi = __shfl_xor_sync(0xffffffffu, vi[q], o);
      if (ov < v[q] || (ov == v[q] && oi < vi[q])) {
        v2[q] = fmin(ov2, v[q]);
        v[q] = ov;
        vi[q] = oi;
      } else {
        v2[q] = fmin(v2[q], ov);
      }
    }
    if (cg == 0 && row[q] >= 0) {
      const int i = row[q];
      const int old = s.labs[(int64_t)r * RM + i];
      if (!fresh && old != vi[q]) moved |= (1u << old) | (1u << vi[q]);
      s.labs[(int64_t)r * RM + i] = vi[q];
      s.ubs[(int64_t)r * RM + i] = sqrt(v[q]);
      s.lbs[(int64_t)r * RM + i] = sqrt(v2[q]);
      if (want_own) a.own[(int64_t)r * a.n + rm(i)] = v[q];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) moved |= __shfl_xor_sync(0xffffffffu, moved, o);
  if (lane == 0 && moved) atomicOr(reinterpret_cast<unsigned *>(gs.misc + 1), moved);
}

// All rows of the list with the warps of the group: the widest row tile that
// still gives every warp work (latency-bound when few rows are candidates).
__device__ __forceinline__ void assign_list(const FusedArgs &a, const Shared &s, const GShared &gs,
                                            int r, int ncand, const int32_t *cand, bool want_own,
                                            RowMap rm, bool fresh, int gw, int GW) {
  if (ncand >= 32 * GW) {
    for (int p0 = gw * 32; p0 < ncand; p0 += GW * 32)
      assign_rows<4>(a, s, gs, r, p0, ncand, cand, want_own, rm, fresh);
  } else if (ncand >= 16 * GW) {
    for (int p0 = gw * 16; p0 < ncand; p0 += GW * 16)
      assign_rows<2>(a, s, gs, r, p0, ncand, cand, want_own, rm, fresh);
  } else {
    for (int p0 = gw * 8; p0 < ncand; p0 += GW * 8)
      assign_rows<1>(a, s, gs, r, p0, ncand, cand, want_own, rm, fresh);
  }
}

// Counting sort of the CTA's rows of restart r by label (stable), then one
// register run per (cluster, column) in row order -> psum / pcnt.
__device__ void group_partials(const FusedArgs &a, const Shared &s, const GShared &gs,
                               const Grp &G_, int r, int nr, bool counts_only, unsigned dirty) {
  const int lane = threadIdx.x & 31;
  const int64_t k = a.k, d = a.d, RM = a.rows_max, ldf = a.ldf;
  const int cta = blockIdx.x;
  const int32_t *lab = s.labs + (int64_t)r * RM;
  if (dirty == 0) {  // no row of this block changed cluster: its partials stand
    G_.sync();
    return;
  }
  if (G_.gt < 32) gs.cnt[G_.gt] = 0;
  G_.sync();
  for (int i = G_.gt; i < nr; i += G_.GT) atomicAdd(gs.cnt + lab[i], 1);
  G_.sync();
  int32_t *pc = a.pcnt + ((int64_t)r * a.G + cta) * k;
  if (G_.gt < k && ((dirty >> G_.gt) & 1u)) pc[G_.gt] = gs.cnt[G_.gt];
  if (counts_only) {
    G_.sync();
    return;
  }
  if (G_.gw == 0) {
    const int v = gs.cnt[lane];
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    gs.runp[lane] = inc - v;
    __syncwarp();
    for (int g0 = 0; g0 < nr; g0 += 32) {  // stable scatter, 32 rows at a time
      const int p = g0 + lane;
      const int l = p < nr ? lab[p] : -1;
      const unsigned m = __match_any_sync(0xffffffffu, l);
      const int rank = __popc(m & ((1u << lane) - 1u));
      if (p < nr) gs.perm[gs.runp[l] + rank] = p;
      __syncwarp();
      if (p < nr && rank == __popc(m) - 1) gs.runp[l] += __popc(m);
      __syncwarp();
    }
  }
  G_.sync();
  double *ps = a.psum + ((int64_t)r * a.G + cta) * k * d;
  if (G_.gt < k && ((dirty >> G_.gt) & 1u) && gs.cnt[G_.gt] > 0) {  // |f|^2 of the run, row order
    const int j = G_.gt, end = gs.runp[j], beg = end - gs.cnt[j];
    double q = 0.0;
    for (int p = beg; p < end; ++p) q += s.fns[gs.perm[p]];
    a.pq[((int64_t)r * a.G + cta) * k + j] = q;
  }
  {
    const int di = (int)d, GT = G_.GT, dj = GT / di, dt = GT - dj * di;
    int j = G_.gt / di, t = G_.gt - j * di;
    for (int64_t e = G_.gt; e < k * d; e += GT) {  // thread per (cluster, column)
      const int c = gs.cnt[j];
      if (c > 0 && ((dirty >> j) & 1u)) {
        const int end = gs.runp[j], beg = end - c;
        double v = 0.0;
        for (int p = beg; p < end; ++p) v += s.Fs[(int64_t)gs.perm[p] * ldf + t];
        ps[e] = v;
      }
      t += dt;
      j += dj;
      if (t >= di) {
        t -= di;
        ++j;
      }
    }
  }
  G_.sync();
}

__device__ __forceinline__ void submark(const FusedArgs &a, int g, int slot, bool on) {
  if (on && a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && g < a.trace_cap)
    a.trace[(int64_t)g * 16 + slot] = gtimer();
}

__device__ void phase1(const FusedArgs &a, const Shared &s, const GShared &gs, const Grp &G_,
                       int r, int g, int nr, RowMap rm, bool first) {
  const int lane = threadIdx.x & 31;
  const int64_t k = a.k, d = a.d, RM = a.rows_max, ldf = a.ldf;
  const int cta = blockIdx.x;
  if (G_.gt == 0) {
    gs.misc[0] = 0;  // candidate count
    gs.misc[1] = 0;  // clusters whose membership changed in this block
  }
  group_load(a, gs, G_, r, g);
  submark(a, g, 6, first);
  int32_t *lab = s.labs + (int64_t)r * RM;
  double *ub = s.ubs + (int64_t)r * RM, *lb = s.lbs + (int64_t)r * RM;
  if (g > 0) {
    if (G_.gw == 0) {  // largest / second largest movement (first index wins), max |c|
      const double dj = lane < k ? gs.del[lane] : 0.0;
      const double cj = lane < k ? gs.cn[lane] : 0.0;
      double m1 = dj, cm = cj;
      int i1 = lane;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, m1, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i1, o);
        if (om > m1 || (om == m1 && oi < i1)) {
          m1 = om;
          i1 = oi;
        }
        cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
      }
      double m2 = lane == i1 ? 0.0 : dj;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
      // stop rule (kmeans.py:112-116) on the centroid-identity cost of
      // iteration g-1 (sum of its k cluster terms in order) and of g-2
      const double term = lane < k ? __ldcg(a.cterm + ((int64_t)((g - 1) & 1) * a.R + r) * k + lane) : 0.0;
      double cost = term;
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, cost, o);
        if (lane >= o) cost += y;  // inclusive prefix in lane order: the total is lane 31's
      }
      cost = __shfl_sync(0xffffffffu, cost, 31);
      cost = cost > 0.0 ? cost : 0.0;
      const int64_t hs = a.max_iters + 1;
      const double prev = g >= 2 ? __ldcg(a.hist + r * hs + g - 2) : INFINITY;
      const bool stop = (g >= 2 && prev - cost <= a.tol * prev) || g >= a.max_iters;
      if (lane == 0) {
        gs.scal[0] = fmax(m1, 0.0);
        gs.scal[1] = fmax(m2, 0.0);
        gs.scal[2] = m1 > 0.0 ? (double)i1 : 0.0;
        gs.scal[3] = sqrt(cm);
        gs.misc[3] = stop ? 1 : 0;
        if (cta == 0) {
          a.hist[r * hs + g - 1] = cost;
          if (stop) a.stopping[r] = g;
        }
      }
    }
    G_.sync();
  }
  if (g > 0 && gs.misc[3]) {
    // the restart stops after iteration g-1: the returned cost2 in the
    // reference's difference form (kmeans.py:111) and the final labels
    // exact cost of iteration g-1 (labels of g-1, means of g-1): SP adjacent
    // threads per row (columns split in SP contiguous parts, added by a fixed
    // xor tree), rows in rounds of GT / SP
    int SP = 1;
    while (SP < 8 && nr * SP * 2 <= G_.GT) SP *= 2;
    const int part = G_.gt % SP;
    const int t0 = part * (int)d / SP, t1 = (part + 1) * (int)d / SP;
    double acc = 0.0;
    for (int i0 = 0; i0 < nr; i0 += G_.GT / SP) {
      const int i = i0 + G_.gt / SP;
      double v = 0.0;
      if (i < nr && G_.gt < (G_.GT / SP) * SP) {
        const double *fr = s.Fs + (int64_t)i * ldf;
        const int l = lab[i];
        const double *cr = gs.Cs + (int64_t)l * a.lds;
        for (int64_t t = t0; t < t1; ++t) {
          const double df = fr[t] - cr[t];
          v = fma(df, df, v);
        }
        if (part == 0) a.labels_out[(int64_t)r * a.n + rm(i)] = l;
      }
      for (int o = 1; o < SP; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (part == 0) acc += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) gs.red[G_.gw] = acc;
    G_.sync();
    if (G_.gt == 0) {
      double c = 0.0;
      for (int w = 0; w < G_.GW; ++w) c += gs.red[w];
      a.cpart[(int64_t)r * a.G + cta] = c;
    }
    G_.sync();
    return;
  }
  submark(a, g, 7, first);
  // rows that need a distance computation
  int ncand = nr;
  if (g > 0) {
    const double d1 = gs.scal[0], d2 = gs.scal[1], cmax = gs.scal[3];
    const int j1 = (int)gs.scal[2];
    for (int c0 = 0; c0 < nr; c0 += G_.GT) {
      const int i = c0 + G_.gt;
      bool need = false;
      if (i < nr) {
        const int l = lab[i];
        const double u = ub[i] + gs.del[l];
        const double lw = lb[i] - (l == j1 ? d2 : d1);
        const double eta = 1e-7 * (s.fsq[i] + cmax);
        need = !(u + eta <= lw);
        ub[i] = u;
        lb[i] = lw;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, need);
      if (lane == 0) gs.misc[4 + G_.gw] = __popc(bal);
      G_.sync();
      int off = gs.misc[0], tot = 0;
      for (int w = 0; w < G_.GW; ++w) {
        const int cw = gs.misc[4 + w];
        if (w < G_.gw) off += cw;
        tot += cw;
      }
      if (need) gs.cand[off + __popc(bal & ((1u << lane) - 1u))] = i;
      G_.sync();
      if (G_.gt == 0) gs.misc[0] += tot;
      G_.sync();
    }
    ncand = gs.misc[0];
  }
  submark(a, g, 8, first);
  if (first && a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && g < a.trace_cap)
    a.trace[(int64_t)g * 16 + 11] = (unsigned long long)ncand;
  assign_list(a, s, gs, r, ncand, g == 0 ? nullptr : gs.cand, false, rm, g == 0, G_.gw, G_.GW);
  G_.sync();
  submark(a, g, 9, first);
  group_partials(a, s, gs, G_, r, nr, false, g == 0 ? ~0u : (unsigned)gs.misc[1]);
  submark(a, g, 10, first);
}

// Sum of the cost partials of restart r (identical in every warp that asks).
__device__ __forceinline__ double cost_sum(const FusedArgs &a, int r) {
  const int lane = threadIdx.x & 31;
  const int G = a.G;
  double v[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const int b = lane + 32 * u;
    v[u] = b < G ? __ldcg(a.cpart + (int64_t)r * G + b) : 0.0;
  }
  double c = 0.0;
#pragma unroll
  for (int u = 0; u < 5; ++u)
    if (lane + 32 * u < G) c += v[u];
  for (int b = lane + 160; b < G; b += 32) c += __ldcg(a.cpart + (int64_t)r * G + b);
  return warp_sum(c);
}

// Means of (restart r, cluster j) from the block partials, by a whole CTA:
// warp w adds the partials of blocks [w G / kFW, (w+1) G / kFW) in block order
// (loads issued in batches of 4 ahead of the adds), warp 0 adds the kFW range
// sums in order. Movement and |c|^2 for the next bounds. Called uniformly by
// every thread of the CTA.
__device__ void means_item(const FusedArgs &a, const Shared &s, int r, int j, int g,
                           bool flag_empty) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t k = a.k, d = a.d, R = a.R, G = a.G;
  const int b_lo = (int)((int64_t)wid * G / kFW), b_hi = (int)((int64_t)(wid + 1) * G / kFW);
  const double *cold = a.cent + ((int64_t)(g & 1) * R + r) * k * a.ldc + j * a.ldc;
  double old[4];
  if (wid == 0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = lane + 32 * u;
      old[u] = t < d ? __ldcg(cold + t) : 0.0;
    }
  }
  const int b = b_lo + lane;  // kFW >= 12 warps: a range has <= 13 blocks
  const int pc = b < b_hi ? __ldcg(a.pcnt + ((int64_t)r * G + b) * k + j) : 0;
  int cnt = pc;
  double sv[4] = {0.0, 0.0, 0.0, 0.0};
  double qv = 0.0;  // sum of the blocks' |f|^2 partials (same value in every lane)
  const double *pbase = a.psum + ((int64_t)r * G * k + j) * d;
  unsigned m = __ballot_sync(0xffffffffu, pc > 0);
  constexpr int NB = 3;  // nonzero blocks whose loads are in flight together
  while (m) {
    int bb[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      bb[q] = m ? b_lo + __ffs(m) - 1 : -1;
      m &= m ? m - 1 : 0u;
    }
    double v[NB][4], vq[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = lane + 32 * u;
        v[q][u] = (bb[q] >= 0 && t < d) ? __ldcg(pbase + (int64_t)bb[q] * k * d + t) : 0.0;
      }
      vq[q] = bb[q] >= 0 ? __ldcg(a.pq + ((int64_t)r * G + bb[q]) * k + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NB; ++q)
      if (bb[q] >= 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) sv[u] += v[q][u];
        qv += vq[q];
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  double *mine = s.p2 + (int64_t)wid * d;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t t = lane + 32 * u;
    if (t < d) mine[t] = sv[u];
  }
  if (lane == 0) {
    s.p2c[wid] = cnt;
    s.p2q[wid] = qv;
  }
  __syncthreads();
  if (wid == 0) {
    int tot = 0;
    for (int w = 0; w < kFW; ++w) tot += s.p2c[w];
    const double denom = (double)(tot > 1 ? tot : 1);
    double *cnew = a.cent + ((int64_t)((g + 1) & 1) * R + r) * k * a.ldc + j * a.ldc;
    double mv = 0.0, nrm = 0.0, dot = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = lane + 32 * u;
      if (t < d) {
        double sum = 0.0;
        for (int w = 0; w < kFW; ++w) sum += s.p2[(int64_t)w * d + t];
        const double mean = __ddiv_rn(sum, denom);
        cnew[t] = mean;
        const double df = mean - old[u];
        mv = fma(df, df, mv);
        nrm = fma(mean, mean, nrm);
        dot = fma(mean, sum, dot);
      }
    }
    mv = warp_sum(mv);
    nrm = warp_sum(nrm);
    dot = warp_sum(dot);
    if (lane == 0) {
      double *kv = a.kvec + ((int64_t)((g + 1) & 1) * R + r) * 2 * k;
      kv[j] = nrm;
      kv[k + j] = sqrt(mv);
      // this cluster's cost term by the centroid identity (as the lane path):
      // sum |f - m|^2 = Q - 2 m.S + n |m|^2 with the rounded mean m
      double q = 0.0;
      for (int w = 0; w < kFW; ++w) q += s.p2q[w];
      a.cterm[((int64_t)(g & 1) * R + r) * k + j] = tot > 0 ? (q - 2.0 * dot) + (double)tot * nrm : 0.0;
      if (flag_empty && tot == 0) a.eflag[r] = g + 1;
    }
  }
  __syncthreads();  // p2 reuse
}

// k-means++ D^2 update for (row, Q restarts) items: difference form in
// ascending columns per (row, restart) chain, closest = min over the draws
template <int Q>
__device__ __forceinline__ void kpp_dist_items(const Shared &s, const GShared &g0, double *cl,
                                               int nr, int RP, int R, int di, int64_t ldf,
                                               int64_t RM, int j) {
  for (int e = threadIdx.x; e < nr * (RP / Q); e += kFT) {
    const int i = e / (RP / Q), c0 = (e - i * (RP / Q)) * Q;
    const double *fr = s.Fs + (int64_t)i * ldf;
    const double2 *cr = reinterpret_cast<const double2 *>(g0.Cs + c0);
    double acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = 0.0;
#pragma unroll 2
    for (int t = 0; t < di; ++t) {
      const double f = fr[t];
#pragma unroll
      for (int h = 0; h < Q / 2; ++h) {
        const double2 c = cr[((t * RP) >> 1) + h];
        const double x0 = f - c.x, x1 = f - c.y;
        acc[2 * h] = fma(x0, x0, acc[2 * h]);
        acc[2 * h + 1] = fma(x1, x1, acc[2 * h + 1]);
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (c0 + q >= R) break;
      double *c = cl + (int64_t)(c0 + q) * RM + i;
      *c = j == 0 ? acc[q] : fmin(*c, acc[q]);
    }
  }
}

__device__ __forceinline__ void kmark(const FusedArgs &a, int j, int slot) {
  if (a.trace && a.trace_cap >= 128 && blockIdx.x == 0 && threadIdx.x == 0)
    a.trace[(int64_t)(96 + j) * 16 + slot] = gtimer();
}

// k-means++ seeds of every restart (kmeans.py:64-77) before the Lloyd loop:
// per draw j, the D^2 weights closest_i = min over chosen centroids of
// |f_i - c|^2 (difference form, ascending column order, as kppb_dist_kernel)
// stay in shared memory; each block's inclusive prefix of its weights (warp
// scan, fixed order) gives a block sum; after a grid barrier every block forms
// the same prefix over the block sums, the draw u * total
// (Generator.choice(n, p) == searchsorted(cumsum(p), u, 'right')) selects the
// block whose prefix first exceeds it, and that block selects the first row
// with a positive weight whose prefix exceeds it. A zero D^2 mass (the
// reference then draws integers(n)) is flagged for the host to replay.
// Closest weights live in s.ubs, prefixes in s.lbs (free before Lloyd).
__device__ void kmeanspp_phase(const FusedArgs &a, const Shared &s, const GShared &g0, int nr,
                               int64_t rb) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int cta = blockIdx.x, G = a.G;
  const int64_t k = a.k, d = a.d, R = a.R, RM = a.rows_max, ldf = a.ldf, lds = a.lds;
  const int di = (int)d, ki = (int)k;
  double *cl = s.ubs, *pre = s.lbs;
  // centroid j of every restart, transposed into g0.Cs as [t][RP], RP = R
  // rounded up to Q, the restarts one (row, Q restarts) distance item covers:
  // the smallest even Q >= 4 whose items fit one round of the block's threads
  // (and RP <= 32: g0.Cs holds 32 x lds doubles)
  int Q = 4;
  while (Q < 8 && nr * (((int)R + Q - 1) / Q) > kFT) Q += 2;
  if (((int)R + Q - 1) / Q * Q > 32) Q = 4;
  const int RP = ((int)R + Q - 1) / Q * Q;
  auto stage = [&](int j) {
    for (int e = tid; e < (int)R * di; e += kFT) {
      const int r = e / di, t = e - r * di;
      const int64_t idx = j == 0 ? a.kpp_first[r] : (int64_t)s.act[r];
      const double v = __ldg(a.F + idx * a.ld + t);
      g0.Cs[(int64_t)t * RP + r] = v;
      if (cta == 0) {
        a.cent[((int64_t)r * k + j) * a.ldc + t] = v;  // buffer 0: the Lloyd seeds
        if (a.seeds_out) a.seeds_out[((int64_t)r * k + j) * a.ldc + t] = v;
      }
    }
    __syncthreads();
  };
  stage(0);
  for (int j = 0; j + 1 < ki; ++j) {
    kmark(a, j, 0);
    if (Q == 8)
      kpp_dist_items<8>(s, g0, cl, nr, RP, (int)R, di, ldf, RM, j);
    else if (Q == 6)
      kpp_dist_items<6>(s, g0, cl, nr, RP, (int)R, di, ldf, RM, j);
    else
      kpp_dist_items<4>(s, g0, cl, nr, RP, (int)R, di, ldf, RM, j);
    __syncthreads();
    // the weights and their in-block prefix to global memory as well: after
    // the barrier every block finds every restart's pick itself
    const int64_t GRM = (int64_t)G * RM;
    double *gw = a.kpp_w + (int64_t)(j & 1) * R * GRM, *gp = a.kpp_pre + (int64_t)(j & 1) * R * GRM;
    for (int r = wid; r < R; r += kFW) {
      double carry = 0.0;
      double *wr = gw + r * GRM + (int64_t)cta * RM, *pr = gp + r * GRM + (int64_t)cta * RM;
      for (int i0 = 0; i0 < nr; i0 += 32) {
        const int i = i0 + lane;
        double x = i < nr ? cl[(int64_t)r * RM + i] : 0.0;
        if (i < nr) wr[i] = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        x += carry;
        if (i < nr) pr[i] = x;
        carry = __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) a.kpp_part[((int64_t)(j & 1) * R + r) * G + cta] = carry;
    }
    kmark(a, j, 1);
    grid_sync(a.bar, G);
    for (int r = wid; r < R; r += kFW) {
      double p[5], loc[5], sl = 0.0;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int c = 5 * lane + q;
        p[q] = c < G ? __ldcg(a.kpp_part + ((int64_t)(j & 1) * R + r) * G + c) : 0.0;
        sl += p[q];
        loc[q] = sl;
      }
      double incl = sl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      double excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = 0.0;
      const double total = __shfl_sync(0xffffffffu, incl, 31);
      if (!(total > 0.0)) {
        if (cta == 0 && lane == 0 && __ldcg(a.kpp_flag + r) < 0) a.kpp_flag[r] = j + 1;
        if (lane == 0) s.act[r] = 0;
        continue;
      }
      const double target = a.kpp_unif[(int64_t)r * (k - 1) + j] * total;
      int qf = -1;
#pragma unroll
      for (int q = 4; q >= 0; --q)
        if (5 * lane + q < G && excl + loc[q] > target) qf = q;
      const unsigned hit = __ballot_sync(0xffffffffu, qf >= 0);
      // the last block always reaches the total (its prefix is the total)
      const int lf = hit ? __ffs(hit) - 1 : (G - 1) / 5;
      const int qsel = __shfl_sync(0xffffffffu, hit ? qf : (G - 1) % 5, lf);
      const int cstar = 5 * lf + qsel;
      double base = excl;
      if (qsel > 0) base = excl + loc[qsel - 1];
      base = __shfl_sync(0xffffffffu, base, lf);
      // block cstar's rows (a contiguous range), 256 per batch of loads
      const int64_t cb = (int64_t)cstar * a.n / G;
      const int ncs = (int)((int64_t)(cstar + 1) * a.n / G - cb);
      const double *wc = gw + r * GRM + (int64_t)cstar * RM, *pc = gp + r * GRM + (int64_t)cstar * RM;
      int found = -1, lastpos = -1;
      for (int i0 = 0; i0 < ncs && found < 0; i0 += 256) {
        double w[8], pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + 32 * u + lane;
          w[u] = i < ncs ? __ldcg(wc + i) : 0.0;
          pv[u] = i < ncs ? __ldcg(pc + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + 32 * u + lane;
          const bool pos = i < ncs && w[u] > 0.0;
          const bool ok = pos && base + pv[u] > target;
          const unsigned hb = __ballot_sync(0xffffffffu, ok);
          const unsigned pb = __ballot_sync(0xffffffffu, pos);
          if (pb) lastpos = i0 + 32 * u + 31 - __clz(pb);
          if (hb) {
            found = i0 + 32 * u + __ffs(hb) - 1;
            break;
          }
        }
      }
      if (found < 0) found = lastpos >= 0 ? lastpos : 0;  // rounding fallback
      if (lane == 0) s.act[r] = (int32_t)(cb + found);
    }
    kmark(a, j, 2);
    __syncthreads();
    kmark(a, j, 3);
    stage(j + 1);
    kmark(a, j, 4);
  }
  grid_sync(a.bar, G);  // buffer 0 (written by block 0) before the first Lloyd phase
}

__global__ void __launch_bounds__(kFT, 1) lloyd_fused_kernel(const FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int cta = blockIdx.x, G = a.G;
  const int64_t n = a.n, d = a.d, k = a.k, R = a.R, RM = a.rows_max, ldf = a.ldf;
  const Shared s = carve(smem_raw, a);
  // the block's rows into shared memory: features, |f|^2, |f|
  auto load_rows = [&](RowMap m, int cnt) {
    __syncthreads();
    for (int64_t i = tid / 32; i < cnt; i += kFT / 32) {  // warp per row
      const int64_t src = m(i) * a.ld;
      for (int64_t t = tid % 32; t < d; t += 32) s.Fs[i * ldf + t] = a.F[src + t];
    }
    if (a.fnorm) {
      for (int i = tid; i < cnt; i += kFT) s.fns[i] = a.fnorm[m(i)];
    } else {  // |f|^2 with csc_kmeans_rownorms' association (lane-strided, xor tree)
      __syncthreads();
      for (int i = wid; i < cnt; i += kFW) {
        const double *fr = s.Fs + (int64_t)i * ldf;
        double v = 0.0;
        for (int64_t t = lane; t < d; t += 32) v = fma(fr[t], fr[t], v);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s.fns[i] = v;
      }
    }
    __syncthreads();
    for (int i = tid; i < cnt; i += kFT) s.fsq[i] = sqrt(s.fns[i]);
    __syncthreads();
  };
  if (a.kpp_first) {  // k-means++ over contiguous row ranges (draws scan rows in order)
    const int64_t rb = (int64_t)cta * n / G, re = (int64_t)(cta + 1) * n / G;
    load_rows(RowMap{rb, 1}, (int)(re - rb));
    kmeanspp_phase(a, s, gcarve(smem_raw, a, 0), (int)(re - rb), rb);
  }
  const RowMap rm{cta, G};
  const int nr = (int)((n - cta + G - 1) / G);
  load_rows(rm, nr);
  for (int gi = 0; gi < a.ngmax; ++gi) {  // centroid rows >= k read as zero
    const GShared gs = gcarve(smem_raw, a, gi);
    for (int64_t e = tid; e < (32 - k) * a.lds; e += kFT) gs.Cs[k * a.lds + e] = 0.0;
  }
  if (tid == 0) {
    for (int r = 0; r < R; ++r) s.act[r] = r;
    s.act[kFMaxR] = (int)R;
    *s.work = 0;
  }
  __syncthreads();

  const bool tr = a.trace != nullptr && cta == 0 && tid == 0;
  auto mark = [&](int g, int slot) {
    if (tr && g < a.trace_cap) a.trace[(int64_t)g * 16 + slot] = gtimer();
  };
  for (int g = 0;; ++g) {
    const int A = s.act[kFMaxR];
    mark(g, 0);
    // ---- phase 1: cost of g-1, assignment of g, block partials -------------
    {
      const int ng = (A >= 4 && a.ngmax >= 4) ? 4 : (A >= 2 && a.ngmax >= 2) ? 2 : 1;
      Grp G_;
      G_.GT = kFT / ng;
      G_.GW = G_.GT / 32;
      G_.id = tid / G_.GT;
      G_.gt = tid % G_.GT;
      G_.gw = G_.gt >> 5;
      const GShared gs = gcarve(smem_raw, a, G_.id);
      // groups take the next active restart from a block counter (restarts'
      // costs differ with their candidate counts)
      for (;;) {
        if (G_.gt == 0) gs.misc[2] = atomicAdd(s.work, 1);
        G_.sync();
        const int ai = gs.misc[2];
        G_.sync();
        if (ai >= A) break;
        phase1(a, s, gs, G_, s.act[ai], g, nr, rm, ai == 0);
        // this block's partials of the restart are written (phase1 ends on a
        // group barrier): release them with one arrival on the restart's count
        if (G_.gt == 0) {
          __threadfence();
          atomicAdd(a.arrive + s.act[ai], 1u);
        }
      }
    }
    __syncthreads();
    mark(g, 1);
    // ---- phase 2: stop rule, means; (restart, cluster) items spread over the
    // blocks, each waiting only for the arrivals of its restart; no grid barrier
    for (int q = cta; q < A * (int)k; q += G) {
      const int r = s.act[q / (int)k], j = q % (int)k;
      if (tid == 0) {
        const unsigned want = (unsigned)G * (unsigned)(g + 1);
        while (ld_acquire(a.arrive + r) < want) __nanosleep(20);
      }
      __syncthreads();
      // phase 1 of this iteration decided (identically in every block) whether
      // the restart stopped after iteration g-1; then its blocks computed the
      // exact cost instead of assigning
      const bool stop = g > 0 && __ldcg(a.stopping + r) == g;
      if (stop) {
        if (j == 0) {
          const double c = cost_sum(a, r);  // identical in every warp
          if (tid == 0) {
            a.cost_out[r] = c;
            a.iters_out[r] = g;
            a.done[r] = 1;
          }
        }
      } else {
        means_item(a, s, r, j, g, true);
      }
      __syncthreads();
      if (tid == 0) {  // the mean (or the stop decision) of (r, j) is published
        __threadfence();
        atomicAdd(a.readycnt + r, 1u);
      }
    }
    __syncthreads();
    mark(g, 2);
    mark(g, 3);
    // every active restart's k items of this iteration are done
    if (tid < A) {
      const unsigned want = (unsigned)k * (unsigned)(g + 1);
      while (ld_acquire(a.readycnt + s.act[tid]) < want) __nanosleep(20);
    }
    __syncthreads();
    mark(g, 4);
    // ---- rare path: empty cluster -> exact reassignment + reseeding --------
    const bool flagged = __syncthreads_or(tid < R && __ldcg(a.eflag + tid) == g + 1);
    if (flagged) {
      Grp W;  // the whole CTA as one group
      W.id = 0;
      W.GT = kFT;
      W.GW = kFW;
      W.gt = tid;
      W.gw = wid;
      const GShared gs = gcarve(smem_raw, a, 0);
      for (int r = 0; r < R; ++r) {
        if (__ldcg(a.eflag + r) != g + 1) continue;
        group_load(a, gs, W, r, g);
        assign_list(a, s, gs, r, nr, nullptr, true, rm, true, wid, kFW);
        W.sync();
        group_partials(a, s, gs, W, r, nr, true, ~0u);
      }
      grid_sync(a.bar, G);
      // reseeding (kmeans.py:101-108), one CTA per flagged restart
      for (int r = cta; r < R; r += G) {
        if (__ldcg(a.eflag + r) != g + 1) continue;
        __shared__ int s_cnt[kFMaxK];
        __shared__ double s_bv[kFW];
        __shared__ int64_t s_bi[kFW];
        if (tid < k) {
          int c = 0;
          for (int b = 0; b < G; ++b) c += __ldcg(a.pcnt + ((int64_t)r * G + b) * k + tid);
          s_cnt[tid] = c;
        }
        __syncthreads();
        int nrep = 0;
        double *own = a.own + (int64_t)r * n;
        for (int64_t j = 0; j < k; ++j) {
          if (s_cnt[j] != 0) continue;
          double bv = -INFINITY;
          int64_t bi = 0;
          for (int64_t i = tid; i < n; i += kFT) {
            const double v = __ldcg(own + i);
            if (v > bv) {
              bv = v;
              bi = i;
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
              bv = ov;
              bi = oi;
            }
          }
          if (lane == 0) {
            s_bv[wid] = bv;
            s_bi[wid] = bi;
          }
          __syncthreads();
          if (tid == 0) {
            for (int w = 1; w < kFW; ++w)
              if (s_bv[w] > bv || (s_bv[w] == bv && s_bi[w] < bi)) {
                bv = s_bv[w];
                bi = s_bi[w];
              }
            a.rep_idx[(int64_t)r * k + nrep] = (int32_t)bi;
            a.rep_j[(int64_t)r * k + nrep] = (int32_t)j;
            __stcg(own + bi, -1.0);
            __threadfence();
          }
          ++nrep;
          __syncthreads();
        }
        if (tid == 0) a.nrep[r] = nrep;
        __syncthreads();
      }
      grid_sync(a.bar, G);
      for (int r = 0; r < R; ++r) {
        if (__ldcg(a.eflag + r) != g + 1) continue;
        if (tid == 0) {
          const int m = __ldcg(a.nrep + r);
          for (int q = 0; q < m; ++q) {
            const int64_t i = __ldcg(a.rep_idx + (int64_t)r * k + q);
            if (i % G == cta) {  // this block's row (interleaved map)
              const int64_t li = i / G;
              s.labs[(int64_t)r * RM + li] = __ldcg(a.rep_j + (int64_t)r * k + q);
              s.ubs[(int64_t)r * RM + li] = INFINITY;  // recomputed next iteration
              s.lbs[(int64_t)r * RM + li] = 0.0;
            }
          }
        }
        W.sync();
        group_partials(a, s, gs, W, r, nr, false, ~0u);
      }
      grid_sync(a.bar, G);
      for (int q = cta; q < (int)(R * k); q += G) {
        const int r = q / (int)k, j = q % (int)k;
        if (__ldcg(a.eflag + r) == g + 1) means_item(a, s, r, j, g, false);
      }
      grid_sync(a.bar, G);
    }
    mark(g, 5);
    if (tid == 0) {  // restarts still running (identical list on every CTA)
      *s.work = 0;
      int m = 0;
      for (int r = 0; r < R; ++r)
        if (!__ldcg(a.done + r)) s.act[m++] = r;
      s.act[kFMaxR] = m;
    }
    __syncthreads();
    if (s.act[kFMaxR] == 0) break;
  }
}

struct FusedGeom {
  int G = 0, RM = 0, ngmax = 0, ldf = 0, lds = 0;
  size_t smem = 0;
};

size_t fused_smem(int64_t RM, int64_t d, int64_t R, int ngmax, int ldf, int lds) {
  const int64_t dbl = group_base(RM, ldf, R, d) + ngmax * gstride_d(lds);
  const int64_t ints = R * RM + kFMaxR + 1 + kFW + 1 + ngmax * gstride_i(RM);
  return (size_t)(dbl * 8 + ints * 4);
}

bool fused_geometry(int64_t n, int64_t d, int64_t k, int64_t R, int max_iters, FusedGeom &g) {
  if (n < 1 || d < 1 || d > kFMaxD || k < 1 || k > kFMaxK || k > n || R < 1 || R > kFMaxR ||
      max_iters < 1)
    return false;
  const csc::DeviceInfo &info = csc::device_info();
  const int64_t smem_cap = info.max_smem_optin > 0 ? info.max_smem_optin : 232448;
  // the k-means++ pick reads the block sums as 5 per lane of one warp: G <= 160
  g.G = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(info.sm_count, 5 * 32), n / 16));
  g.RM = (int)csc::ceil_div(n, g.G);
  g.ldf = (int)(d | 1);
  g.lds = (int)(d | 1);
  for (int ng : {4, 2, 1}) {
    const size_t sm = fused_smem(g.RM, d, R, ng, g.ldf, g.lds);
    if ((int64_t)sm <= smem_cap - 1024) {  // static shared arrays of the rare path
      g.ngmax = ng;
      g.smem = sm;
      return true;
    }
  }
  return false;
}

unsigned long long *g_trace = nullptr;
int64_t g_trace_cap = 0;

}  // namespace

// diagnostics (tools/): the next fused runs record CTA 0's globaltimer at the
// phase boundaries of every iteration into trace_dev[iter * 16 + slot]
extern "C" int csc_kmeans_fused_trace(unsigned long long *trace_dev, int64_t iters_cap) {
  g_trace = trace_dev;
  g_trace_cap = trace_dev ? iters_cap : 0;
  return CSC_OK;
}

extern "C" int csc_kmeans_fused_supported(int64_t n, int64_t d, int64_t k, int64_t R,
                                          int max_iters) {
  FusedGeom g;
  return fused_geometry(n, d, k, R, max_iters, g) ? 1 : 0;
}

namespace {

// Shared launcher: seeds (device, R x k x ldc) or the k-means++ draws (host).
int fused_launch(const char *who, const double *f, const double *fnorm, int64_t n, int64_t d,
                 int64_t ld, int64_t k, int64_t R, const double *seeds,
                 const int64_t *first_host, const double *unif_host, double *seeds_out,
                 int32_t *flags, int64_t ldc, int max_iters, double tol, int32_t *labels,
                 double *cost2, int32_t *iters, cudaStream_t st) {
  CSC_REQUIRE(ld >= d && ldc >= d, "%s: ld/ldc < d", who);
  FusedGeom g;
  CSC_REQUIRE(fused_geometry(n, d, k, R, max_iters, g),
              "%s: shape outside the fused kernel (n=%lld d=%lld k=%lld R=%lld)", who,
              (long long)n, (long long)d, (long long)k, (long long)R);
  const int64_t G = g.G;
  const bool kpp = first_host != nullptr;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b_cent = al(sizeof(double) * 2 * R * k * ldc);
  const size_t b_kvec = al(sizeof(double) * 2 * R * 2 * k);
  const size_t b_psum = al(sizeof(double) * R * G * k * d);
  const size_t b_cpart = al(sizeof(double) * R * G);
  const size_t b_pq = al(sizeof(double) * R * G * k);
  const size_t b_cterm = al(sizeof(double) * 2 * R * k);
  const size_t b_stop = al(sizeof(int32_t) * R);
  const size_t b_hist = al(sizeof(double) * R * (max_iters + 1));
  const size_t b_own = al(sizeof(double) * R * n);
  const size_t b_pcnt = al(sizeof(int32_t) * R * G * k);
  const size_t b_ints = al(sizeof(int32_t) * (3 * R + 2 * R * k) + (2 + 2 * R) * sizeof(unsigned));
  const size_t b_kfirst = kpp ? al(sizeof(int64_t) * R) : 0;
  const size_t b_kunif = kpp ? al(sizeof(double) * R * std::max<int64_t>(1, k - 1)) : 0;
  // double-buffered by draw parity: a block that leaves barrier j early writes
  // draw j+1's sums while slower blocks still read draw j's
  const size_t b_kpart = kpp ? al(sizeof(double) * 2 * R * G) : 0;
  const size_t b_kpick = kpp ? al(sizeof(double) * 4 * R * G * g.RM) : 0;
  csc::Scratch ws;
  CSC_TRY_CUDA(ws.alloc(b_cent + b_kvec + b_psum + b_cpart + b_pq + b_cterm + b_stop + b_hist + b_own +
                            b_pcnt + b_ints + b_kfirst + b_kunif + b_kpart + b_kpick,
                        st));
  unsigned char *p = ws.as<unsigned char>();
  FusedArgs a;
  a.F = f;
  a.fnorm = fnorm;
  a.n = n;
  a.d = d;
  a.ld = ld;
  a.k = k;
  a.R = R;
  a.ldc = ldc;
  a.max_iters = max_iters;
  a.tol = tol;
  a.labels_out = labels;
  a.cost_out = cost2;
  a.iters_out = iters;
  a.cent = reinterpret_cast<double *>(p);
  p += b_cent;
  a.kvec = reinterpret_cast<double *>(p);
  p += b_kvec;
  a.psum = reinterpret_cast<double *>(p);
  p += b_psum;
  a.cpart = reinterpret_cast<double *>(p);
  p += b_cpart;
  a.pq = reinterpret_cast<double *>(p);
  p += b_pq;
  a.cterm = reinterpret_cast<double *>(p);
  p += b_cterm;
  a.stopping = reinterpret_cast<int32_t *>(p);
  p += b_stop;
  CSC_TRY_CUDA(cudaMemsetAsync(a.stopping, 0xff, sizeof(int32_t) * R, st));
  a.hist = reinterpret_cast<double *>(p);
  p += b_hist;
  a.own = reinterpret_cast<double *>(p);
  p += b_own;
  a.pcnt = reinterpret_cast<int32_t *>(p);
  p += b_pcnt;
  int32_t *ints = reinterpret_cast<int32_t *>(p);
  p += b_ints;
  a.done = ints;
  a.eflag = ints + R;
  a.nrep = ints + 2 * R;
  a.rep_idx = ints + 3 * R;
  a.rep_j = ints + 3 * R + R * k;
  a.bar = reinterpret_cast<unsigned *>(ints + 3 * R + 2 * R * k);
  a.arrive = a.bar + 2;
  a.readycnt = a.arrive + R;
  a.kpp_first = nullptr;
  a.kpp_unif = nullptr;
  a.kpp_part = nullptr;
  a.kpp_w = nullptr;
  a.kpp_pre = nullptr;
  a.kpp_flag = flags;
  a.seeds_out = seeds_out;
  if (kpp) {
    int64_t *kf = reinterpret_cast<int64_t *>(p);
    p += b_kfirst;
    double *ku = reinterpret_cast<double *>(p);
    p += b_kunif;
    a.kpp_part = reinterpret_cast<double *>(p);
    p += b_kpart;
    a.kpp_w = reinterpret_cast<double *>(p);
    a.kpp_pre = a.kpp_w + 2 * R * G * g.RM;
    CSC_TRY_CUDA(cudaMemcpyAsync(kf, first_host, sizeof(int64_t) * R, cudaMemcpyHostToDevice, st));
    if (k > 1)
      CSC_TRY_CUDA(cudaMemcpyAsync(ku, unif_host, sizeof(double) * R * (k - 1),
                                   cudaMemcpyHostToDevice, st));
    CSC_TRY_CUDA(cudaMemsetAsync(flags, 0xff, sizeof(int32_t) * R, st));
    a.kpp_first = kf;
    a.kpp_unif = ku;
  } else {
    CSC_TRY_CUDA(cudaMemcpyAsync(a.cent, seeds, sizeof(double) * R * k * ldc,
                                 cudaMemcpyDeviceToDevice, st));
  }
  a.trace = g_trace;
  a.trace_cap = g_trace_cap;
  a.G = (int)G;
  a.rows_max = g.RM;
  a.ldf = g.ldf;
  a.lds = g.lds;
  a.ngmax = g.ngmax;
  if (const char *e = getenv("CSC_FUSED_GROUPS")) {  // A/B knob: cap the thread groups
    const int cap = atoi(e);
    if (cap == 1 || cap == 2) a.ngmax = std::min(a.ngmax, cap);
  }
  CSC_TRY_CUDA(cudaMemsetAsync(ints, 0, b_ints, st));
  CSC_TRY_CUDA(cudaFuncSetAttribute(lloyd_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)g.smem));
  void *args[] = {&a};
  CSC_TRY_CUDA(cudaLaunchCooperativeKernel((const void *)lloyd_fused_kernel, dim3(g.G), dim3(kFT),
                                           args, g.smem, st));
  return CSC_OK;
}

}  // namespace

extern "C" int csc_kmeans_fused_run(const double *f, const double *fnorm, int64_t n, int64_t d,
                                    int64_t ld, int64_t k, int64_t R, const double *seeds,
                                    int64_t ldc, int max_iters, double tol, int32_t *labels,
                                    double *cost2, int32_t *iters, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(f && fnorm && seeds && labels && cost2 && iters, "csc_kmeans_fused_run: NULL pointer");
  return fused_launch("csc_kmeans_fused_run", f, fnorm, n, d, ld, k, R, seeds, nullptr, nullptr,
                      nullptr, nullptr, ldc, max_iters, tol, labels, cost2, iters,
                      static_cast<cudaStream_t>(stream));
}

extern "C" int csc_kmeans_fused_kpp_run(const double *f, int64_t n, int64_t d, int64_t ld,
                                        int64_t k, int64_t R, const int64_t *first_idx_host,
                                        const double *uniforms_host, int64_t ldc, int max_iters,
                                        double tol, int32_t *labels, double *cost2,
                                        int32_t *iters, double *seeds_out, int32_t *flags,
                                        void *stream) {
  csc::clear_error();
  CSC_REQUIRE(f && first_idx_host && labels && cost2 && iters && flags &&
                  (k < 2 || uniforms_host),
              "csc_kmeans_fused_kpp_run: NULL pointer");
  for (int64_t r = 0; r < R; ++r)
    CSC_REQUIRE(first_idx_host[r] >= 0 && first_idx_host[r] < n,
                "csc_kmeans_fused_kpp_run: first index out of range");
  return fused_launch("csc_kmeans_fused_kpp_run", f, nullptr, n, d, ld, k, R, nullptr,
                      first_idx_host, uniforms_host, seeds_out, flags, ldc, max_iters, tol, labels,
                      cost2, iters, static_cast<cudaStream_t>(stream));
}
