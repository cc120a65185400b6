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
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kmeans_screen.cuh"

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

// ---------------------------------------------------------------------------
// assign v2: 128 rows x 64 centroids per 128-thread block, 8x8 FP64 register
// tile per thread (rows ty+16i, centroids tx+8j), the centroid tile resident
// in shared memory transposed [d][64], F streamed in 16-wide d stages with
// cp.async double buffering (zero-fill outside the matrix). FP64-FMA bound.
// ---------------------------------------------------------------------------
constexpr int kAM = 128, kAN = 64, kAK = 16, kAKP = kAK + 2, kANP = kAN + 1;
// assign3 keeps a per-block label histogram in shared memory up to this k
constexpr int64_t kHistMax = 8192;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  const int src_size = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_size));
}
// 16-byte cp.async copying the first `bytes` (0, 8 or 16) and zero-filling the rest
__device__ __forceinline__ void cp_async_bytes16(void *smem, const void *gmem, int bytes) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// 128 rows x 64 centroids per block; each thread owns 8 rows (ty + 16 i) and
// TN centroids (tx + (64/TN) j). TN = 8: 128 threads; TN = 4: 256 threads.
template <int TN>
__global__ void __launch_bounds__(16 * (kAN / TN), (TN == 8 ? 2 : 2))
    assign2_kernel(const double *__restrict__ f, const double *__restrict__ fnorm, int64_t n,
                   int64_t d, int64_t ld, const double *__restrict__ cent, int64_t ldc,
                   const double *__restrict__ cnorm, int64_t k, int32_t *__restrict__ labels,
                   double *__restrict__ own, int32_t *__restrict__ counts,
                   const int32_t *__restrict__ rows, const int32_t *__restrict__ nrows_dev,
                   double *__restrict__ ub, double *__restrict__ lb,
                   const int32_t *__restrict__ gate) {
  constexpr int CT = kAN / TN;        // centroid-threads per row group
  constexpr int NT = 16 * CT;         // threads per block
  extern __shared__ __align__(16) double smem[];
  const int64_t dpad = (d + kAK - 1) / kAK * kAK;
  double *Cs = smem;                    // [dpad][kANP]
  double *Fs = smem + dpad * kANP;      // [2][kAM][kAKP]
  if (gate && *gate == 0) return;
  const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : n;  // rows to process (list length)
  const int tid = threadIdx.x;
  const int tx = tid % CT, ty = tid / CT;
  const int64_t r0 = (int64_t)blockIdx.x * kAM;
  if (r0 >= nr) return;
  const int nst = (int)(dpad / kAK);
  double fn[8], best_v[8], second_v[8];
  int best_i[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + ty + 16 * i;
    const int64_t g = r < nr ? (rows ? (int64_t)rows[r] : r) : -1;
    fn[i] = g >= 0 ? fnorm[g] : 0.0;
    best_v[i] = INFINITY;
    second_v[i] = INFINITY;
    best_i[i] = 0;
  }
  auto load_stage = [&](int st, int buf) {
    const int64_t k0 = (int64_t)st * kAK;
#pragma unroll
    for (int q = 0; q < 1024 / NT; ++q) {  // 128 rows x 8 vectors of 2 doubles
      const int v = tid + NT * q;
      const int row = v >> 3, vc = v & 7;
      const int64_t lr = r0 + row;
      const int64_t gr = lr < nr ? (rows ? (int64_t)rows[lr] : lr) : n;
      const int64_t gc = k0 + 2 * vc;
      const bool ok = gr < n && gc < ld;  // ld is even: the pair is inside the row
      const double *src = ok ? f + gr * ld + gc : f;
      cp_async16(Fs + ((size_t)buf * kAM + row) * kAKP + 2 * vc, src, ok);
    }
  };
  for (int64_t c0 = 0; c0 < k; c0 += kAN) {
    __syncthreads();  // previous tile's readers of Cs / Fs are done
    // warp per centroid row, lanes along it (coalesced; no per-element division)
    for (int64_t cc = tid / 32; cc < kAN; cc += NT / 32)
      for (int64_t dd = tid % 32; dd < dpad; dd += 32)
        Cs[dd * kANP + cc] = (c0 + cc < k && dd < d) ? cent[(c0 + cc) * ldc + dd] : 0.0;
    double acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
    load_stage(0, 0);
    cp_async_commit();
    for (int st = 0; st < nst; ++st) {
      if (st + 1 < nst) load_stage(st + 1, (st + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      const double *Fb = Fs + (size_t)(st & 1) * kAM * kAKP;
      const double *Cb = Cs + (size_t)st * kAK * kANP;
#pragma unroll
      for (int kk = 0; kk < kAK; ++kk) {
        double a[8], b[TN];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = Fb[(ty + 16 * i) * kAKP + kk];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Cb[kk * kANP + tx + CT * j];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // (min, argmin, second min) over this thread's centroids, first index wins ties
      double v = INFINITY, v2 = INFINITY;
      int vi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t c = c0 + tx + CT * j;
        if (c < k) {
          const double t = __dsub_rn(fn[i], __dmul_rn(2.0, acc[i][j]));
          double d2 = __dadd_rn(t, cnorm[c]);
          d2 = d2 > 0.0 ? d2 : 0.0;
          if (d2 < v) {
            v2 = v;
            v = d2;
            vi = (int)c;
          } else if (d2 < v2) {
            v2 = d2;
          }
        }
      }
#pragma unroll
      for (int o = 1; o < CT; o <<= 1) {  // the CT lanes of a row group are adjacent
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const double ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
        const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
        if (ov < v || (ov == v && oi < vi)) {
          v2 = fmin(ov2, v);
          v = ov;
          vi = oi;
        } else {
          v2 = fmin(v2, ov);
        }
      }
      if (v < best_v[i] || (v == best_v[i] && vi < best_i[i])) {
        second_v[i] = fmin(v2, best_v[i]);
        best_v[i] = v;
        best_i[i] = vi;
      } else {
        second_v[i] = fmin(second_v[i], v);
      }
    }
  }
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t lr = r0 + ty + 16 * i;
      const int64_t r = lr < nr ? (rows ? (int64_t)rows[lr] : lr) : -1;
      if (r >= 0) {
        labels[r] = best_i[i];
        own[r] = best_v[i];
        if (ub) {
          ub[r] = sqrt(best_v[i]);
          lb[r] = sqrt(second_v[i]);
        }
        if (counts) atomicAdd(counts + best_i[i], 1);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// assign v3: persistent (2 blocks per SM), 128 x 64 tile, 8x8 per thread,
// centroid tile loaded once per block per pass, 3-stage cp.async ring that
// runs across the block's row tiles. k > 64: one pass per 64-centroid tile;
// pass p > 0 merges with the (min, argmin, second) kept in own/labels/lb.
// ---------------------------------------------------------------------------
// (min, argmin, second min) of TN distances by a fixed pairwise tree; the
// left operand always holds the smaller centroid indices, so the first index
// wins exact ties like numpy's argmin.
struct Min3 {
  double v, v2;
  int i;
};
__device__ __forceinline__ Min3 min3_merge(const Min3 &a, const Min3 &b) {
  Min3 r;
  if (b.v < a.v) {
    r.v = b.v;
    r.i = b.i;
    r.v2 = fmin(b.v2, a.v);
  } else {
    r.v = a.v;
    r.i = a.i;
    r.v2 = fmin(a.v2, b.v);
  }
  return r;
}

// SC (streamed centroids): when the whole dpad x BN centroid tile does not fit
// in shared memory (large d), each kAK slice of it rides the cp.async stage
// ring with the row slices ([kStages][BN][kAKP], same loader) instead of
// being resident. Same FMA order, so results are bit-identical.
template <int kStages, int TM, int TN, int RT, int CT, bool SC = false>
__global__ void __launch_bounds__(RT * CT, (RT * CT <= 128 ? 2 : 1))
    assign3_kernel(const double *__restrict__ f, const double *__restrict__ fnorm, int64_t n,
                   int64_t d, int64_t ld, const double *__restrict__ cent, int64_t ldc,
                   const double *__restrict__ cnorm, int64_t k, int64_t c0, int last_pass,
                   int32_t *__restrict__ labels, double *__restrict__ own,
                   int32_t *__restrict__ counts, const int32_t *__restrict__ rows,
                   const int32_t *__restrict__ nrows_dev, double *__restrict__ ub,
                   double *__restrict__ lb, const int32_t *__restrict__ gate) {
  constexpr int NT = RT * CT;       // threads
  constexpr int BM = RT * TM;       // rows per tile
  constexpr int BN = CT * TN;       // centroids per pass
  constexpr int BNP = BN + 1;       // padded Cs row
  constexpr int NB = kStages + 2;   // tile-table ring (see tile_prep)
  static_assert(NT >= BM, "one thread per tile row in tile_prep");
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double smem[];
  const int64_t dpad = (d + kAK - 1) / kAK * kAK;
  double *Cs = smem;                          // [dpad][BNP] ([kStages][BN][kAKP] if SC)
  double *Fs = Cs + (SC ? kStages * BN * kAKP : dpad * BNP);  // [kStages][BM][kAKP]
  double *Fn = Fs + kStages * BM * kAKP;      // [NB][BM] |f|^2 of the tile's rows
  double *Cn = Fn + NB * BM;                  // [BN] |c|^2 (+inf past k)
  int32_t *Rid = reinterpret_cast<int32_t *>(Cn + BN);  // [NB][BM] row ids (-1: padding)
  // [k] block histogram of the final labels (counts != nullptr and k <= kHistMax)
  int32_t *Hs = Rid + NB * BM;
  const bool hist = counts != nullptr && k <= kHistMax;
  const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : n;
  const int64_t ntiles = (nr + BM - 1) / BM;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int tid = threadIdx.x;
  const int tx = tid % CT, ty = tid / CT;
  const int nst = (int)(dpad / kAK);
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t total = my_tiles * nst;
  if (!SC)
    for (int64_t cc = tid / 32; cc < BN; cc += NT / 32)  // warp per centroid row
      for (int64_t dd = tid % 32; dd < dpad; dd += 32)
        Cs[dd * BNP + cc] = (c0 + cc < k && dd < d) ? cent[(c0 + cc) * ldc + dd] : 0.0;
  // padding columns get |c|^2 = +inf, so their distance is +inf without a select
  for (int cc = tid; cc < BN; cc += NT) Cn[cc] = c0 + cc < k ? cnorm[c0 + cc] : INFINITY;
  if (hist)
    for (int64_t j = tid; j < k; j += NT) Hs[j] = 0;
  // tile table of block-local tile t (ring slot b): row ids, and |f|^2 by
  // cp.async (joins the current commit group, landing with the stage loads)
  auto tile_prep = [&](int t, int b) {
    if (tid < BM) {
      const int64_t lr = (blockIdx.x + (int64_t)t * gridDim.x) * BM + tid;
      const int64_t gr = lr < nr ? (rows ? (int64_t)rows[lr] : lr) : -1;
      Rid[b * BM + tid] = (int32_t)gr;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Fn + b * BM + tid);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa),
                   "l"(gr >= 0 ? fnorm + gr : fnorm), "r"(gr >= 0 ? 8 : 0));
    }
  };
  // coalesced loader: 8 threads per row (128 B = one kAK slice), rows from the
  // tile table (written >= one barrier before the tile's first stage load).
  // 32-bit stage / tile / ring counters advance incrementally (no 64-bit
  // division in the loop); the byte offset of a row is one 32x32->64 IMAD.
  const unsigned ld8 = (unsigned)(ld * (int64_t)sizeof(double));
  const int vc = tid & 7;
  int l_st = 0, l_tb = 0, l_buf = 0;  // stage-in-tile, ring slot, buffer of the next load
  auto load_next = [&]() {
    const int gc = l_st * kAK + 2 * vc;
    const bool col_ok = gc < ld;
    const char *fk = reinterpret_cast<const char *>(f + gc);
    const int32_t *rid = Rid + l_tb * BM;
    double *buf = Fs + l_buf * (BM * kAKP);
#pragma unroll
    for (int q = 0; q < (BM * 8 + NT - 1) / NT; ++q) {
      const int row = (tid >> 3) + (NT / 8) * q;
      if (row >= BM) break;
      const int32_t gr = rid[row];
      const bool ok = col_ok && gr >= 0;
      cp_async16(buf + row * kAKP + 2 * vc, ok ? fk + (size_t)(unsigned)gr * ld8 : (const char *)f,
                 ok);
    }
    if (SC) {  // this stage's centroid slice; columns >= d zero-filled
      const int64_t rem = d - gc;
      const int cbytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
      double *cb = Cs + l_buf * (BN * kAKP);
#pragma unroll
      for (int q = 0; q < (BN * 8 + NT - 1) / NT; ++q) {
        const int cc = (tid >> 3) + (NT / 8) * q;
        if (cc >= BN) break;
        const int nb = c0 + cc < k ? cbytes : 0;
        cp_async_bytes16(cb + cc * kAKP + 2 * vc, nb ? cent + (c0 + cc) * ldc + gc : cent, nb);
      }
    }
    if (++l_st == nst) {
      l_st = 0;
      l_tb = l_tb + 1 == NB ? 0 : l_tb + 1;
    }
    l_buf = l_buf + 1 == kStages ? 0 : l_buf + 1;
  };
  // Ring safety: tile t's table is written at iteration t*nst - (kStages-1) - 1
  // (or in the prologue) and last read by its epilogue at t*nst + nst - 1; the
  // slot is rewritten for tile t + NB at least two iterations (two barriers)
  // after that epilogue since (NB - 1) * nst >= kStages + 1.
  constexpr int S = kStages - 1;  // stages in flight ahead of compute
  const int total_i = (int)total, mt = (int)my_tiles;
  int p_t = 0;  // next tile to prep
  for (; p_t < mt && p_t * nst <= S; ++p_t) tile_prep(p_t, p_t % NB);
  int p_tb = p_t % NB;
  __syncthreads();
#pragma unroll
  for (int g = 0; g < S; ++g) {
    if (g < total_i) load_next();
    cp_async_commit();
  }
  double acc[TM][TN];
  int st = 0, c_buf = 0, c_tb = 0;  // compute: stage-in-tile, stage buffer, ring slot
  for (int g = 0; g < total_i; ++g) {
    if (g + S < total_i) load_next();
    if (p_t < mt && p_t * nst == g + S + 1) {  // tile whose first stage loads next iteration
      tile_prep(p_t, p_tb);
      ++p_t;
      p_tb = p_tb + 1 == NB ? 0 : p_tb + 1;
    }
    cp_async_commit();
    cp_async_wait<S>();
    __syncthreads();
    if (st == 0) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
    }
    const double *Fb = Fs + c_buf * (BM * kAKP);
    const double *Cb = SC ? Cs + c_buf * (BN * kAKP) : Cs + st * (kAK * BNP);
#pragma unroll
    for (int kk = 0; kk < kAK; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = Fb[(ty + RT * i) * kAKP + kk];
#pragma unroll
      for (int j = 0; j < TN; ++j)
        b[j] = SC ? Cb[(tx + CT * j) * kAKP + kk] : Cb[kk * BNP + tx + CT * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
    if (st == nst - 1) {  // epilogue of this row tile
      const int tb = c_tb;
      double cn[TN];
#pragma unroll
      for (int j = 0; j < TN; ++j) cn[j] = Cn[tx + CT * j];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int row = ty + RT * i;
        const int64_t r = Rid[tb * BM + row];
        const double fni = Fn[tb * BM + row];
        // (min, lowest argmin, second min) of d2 = (|f|^2 - 2 f.c) + |c|^2 over
        // this thread's columns in ascending order, then across the CT lanes of
        // the row. fma(-2, acc, |f|^2) rounds once like |f|^2 - (2 acc) (2 acc
        // is exact). The clamp at 0 only matters when some d2 < 0 (rounding
        // for a point on a centroid): the unclamped pass is exact otherwise,
        // and a group with a negative minimum redoes it clamped (features are
        // finite: FeatureMatrix rejects non-finite values like the reference).
        double v, v2;
        int vi;
        auto reduce_row = [&](bool clamp) {
          v = INFINITY;
          v2 = INFINITY;
          int vj = 0;
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            double d2 = __dadd_rn(fma(-2.0, acc[i][j], fni), cn[j]);
            if (clamp) d2 = fmax(d2, 0.0);
            const bool lt = d2 < v, lt2 = d2 < v2;
            v2 = lt ? v : (lt2 ? d2 : v2);
            v = lt ? d2 : v;
            vj = lt ? j : vj;
          }
          vi = (int)(c0 + tx + CT * vj);
#pragma unroll
          for (int o = 1; o < CT; o <<= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const double ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
            const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
            const bool take = ov < v || (ov == v && oi < vi);
            v2 = take ? fmin(ov2, v) : fmin(v2, ov);
            v = take ? ov : v;
            vi = take ? oi : vi;
          }
        };
        reduce_row(false);
        if (__any_sync(0xffffffffu, v < 0.0)) reduce_row(true);  // rare
        v = fmax(v, 0.0);  // -0.0 -> +0.0 as the clamp gives
        v2 = fmax(v2, 0.0);
        if (tx == 0 && r >= 0) {
          if (c0 > 0) {  // merge with earlier centroid tiles (smaller indices win ties)
            const double pv = own[r], pv2 = lb[r];
            const int pi = labels[r];
            if (pv <= v) {
              v2 = fmin(pv2, v);
              v = pv;
              vi = pi;
            } else {
              v2 = fmin(v2, pv);
            }
          }
          labels[r] = vi;
          own[r] = v;
          if (last_pass) {
            if (ub) {
              ub[r] = sqrt(v);
              lb[r] = sqrt(v2);
            }
            if (hist)
              atomicAdd(Hs + vi, 1);
            else if (counts)
              atomicAdd(counts + vi, 1);
          } else {
            lb[r] = v2;  // carried (squared) second minimum for the next pass
          }
        }
      }
    }
    if (++st == nst) {
      st = 0;
      c_tb = c_tb + 1 == NB ? 0 : c_tb + 1;
    }
    c_buf = c_buf + 1 == kStages ? 0 : c_buf + 1;
  }
  if (hist) {  // one global atomic per (block, cluster) instead of one per row
    __syncthreads();
    for (int64_t j = tid; j < k; j += NT)
      if (Hs[j]) atomicAdd(counts + j, Hs[j]);
  }
}

// ---------------------------------------------------------------------------
// assign, small k (k <= 32 * KPL, d <= 128): one warp per R rows, one lane per
// centroid (KPL per lane). Latency-oriented for small n and candidate subsets
// (every block reaches its rows after one centroid load, no K pipeline). The
// per-(row, centroid) arithmetic is assign3's: acc = fma(f_c, c_c, acc) in
// ascending c from 0.0, then ((|f|^2 - 2 acc) + |c|^2) clamped, and the
// (min, argmin, second) reduction picks the lowest index on ties, so labels,
// own distances and bounds are bit-identical to assign3's.
// ---------------------------------------------------------------------------
template <int KPL, int R>
__global__ void __launch_bounds__(256)
    assign_small_kernel(const double *__restrict__ f, const double *__restrict__ fnorm,
                        int64_t n, int64_t d, int64_t ld, const double *__restrict__ cent,
                        int64_t ldc, const double *__restrict__ cnorm, int64_t k,
                        int32_t *__restrict__ labels, double *__restrict__ own,
                        int32_t *__restrict__ counts, const int32_t *__restrict__ rows,
                        const int32_t *__restrict__ nrows_dev, double *__restrict__ ub,
                        double *__restrict__ lb, const int32_t *__restrict__ gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double smem[];
  const int64_t lds = d | 1;
  double *Cs = smem;                                  // [32 * KPL][lds]
  double *Fs = smem + 32 * KPL * lds;                 // [8 warps][R][d]
  int32_t *Hs = reinterpret_cast<int32_t *>(Fs + 8 * R * d);  // [32 * KPL] block label histogram
  const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : n;
  const int64_t ngroups = (nr + R - 1) / R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if ((int64_t)blockIdx.x * 8 >= ngroups) return;
  for (int64_t j = threadIdx.x / 32; j < 32 * KPL; j += blockDim.x / 32)  // warp per centroid row
    for (int64_t c = threadIdx.x % 32; c < d; c += 32) Cs[j * lds + c] = j < k ? cent[j * ldc + c] : 0.0;
  double cn[KPL];
#pragma unroll
  for (int q = 0; q < KPL; ++q) cn[q] = lane + 32 * q < k ? cnorm[lane + 32 * q] : 0.0;
  if (counts)
    for (int j = threadIdx.x; j < 32 * KPL; j += blockDim.x) Hs[j] = 0;
  __syncthreads();
  double *Fw = Fs + (size_t)wid * R * d;
  for (int64_t g = (int64_t)blockIdx.x * 8 + wid; g < ngroups; g += (int64_t)gridDim.x * 8) {
    int64_t r[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int64_t lr = g * R + i;
      r[i] = lr < nr ? (rows ? (int64_t)rows[lr] : lr) : -1;
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
      for (int64_t c = lane; c < d; c += 32) Fw[i * d + c] = r[i] >= 0 ? f[r[i] * ld + c] : 0.0;
    __syncwarp();
    double acc[R][KPL];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int q = 0; q < KPL; ++q) acc[i][q] = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      double b[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) b[q] = Cs[(lane + 32 * q) * lds + c];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double a = Fw[i * d + c];
#pragma unroll
        for (int q = 0; q < KPL; ++q) acc[i][q] = fma(a, b[q], acc[i][q]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double fni = r[i] >= 0 ? fnorm[r[i]] : 0.0;
      Min3 m[KPL];
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        const double t = __dsub_rn(fni, __dmul_rn(2.0, acc[i][q]));
        const double d2 = fmax(__dadd_rn(t, cn[q]), 0.0);
        m[q].v = lane + 32 * q < k ? d2 : INFINITY;
        m[q].i = lane + 32 * q;
        m[q].v2 = INFINITY;
      }
#pragma unroll
      for (int q = 1; q < KPL; ++q) m[0] = min3_merge(m[0], m[q]);
      double v = m[0].v, v2 = m[0].v2;
      int vi = m[0].i;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const double ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
        const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
        if (ov < v || (ov == v && oi < vi)) {
          v2 = fmin(ov2, v);
          v = ov;
          vi = oi;
        } else {
          v2 = fmin(v2, ov);
        }
      }
      if (lane == 0 && r[i] >= 0) {
        labels[r[i]] = vi;
        own[r[i]] = v;
        if (ub) {
          ub[r[i]] = sqrt(v);
          lb[r[i]] = sqrt(v2);
        }
        if (counts) atomicAdd(Hs + vi, 1);
      }
    }
  }
  if (counts) {  // one global atomic per (block, cluster)
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      if (Hs[j]) atomicAdd(counts + j, Hs[j]);
  }
}

template <int KPL>
int launch_assign_small(const double *f, const double *fnorm, int64_t n, int64_t d, int64_t ld,
                        const double *c, int64_t ldc, const double *cnorm, int64_t k,
                        int32_t *labels, double *own, int32_t *counts, cudaStream_t st,
                        const int32_t *rows, const int32_t *nrows_dev, double *ub, double *lb,
                        const int32_t *gate) {
  constexpr int R = 4;
  const size_t smem = sizeof(double) * (32 * KPL * (d | 1) + 8 * R * d) + sizeof(int32_t) * 32 * KPL;
  static size_t configured = 0;
  if (smem > configured) {
    CSC_TRY_CUDA(cudaFuncSetAttribute(assign_small_kernel<KPL, R>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  const int64_t groups = csc::ceil_div(n, (int64_t)R);
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(csc::device_info().sm_count * 4, csc::ceil_div(groups, 8)));
  assign_small_kernel<KPL, R><<<grid, 256, smem, st>>>(f, fnorm, n, d, ld, c, ldc, cnorm, k,
                                                        labels, own, counts, rows, nrows_dev, ub,
                                                        lb, gate);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int g_kpp_staged = -1;  // batched k-means++ distance pass staged through shared memory (-1: env)
int g_assign_tn = 8;
int g_assign_ver = 3;
// incremental centroid sums (update_sorted_kernel): tuning key "update_incremental"
int g_update_incremental = 1;
// exact fixed-point centroid sums updated by the changed rows only
// (fx_changes / fx_scatter / fx_sum kernels) when d <= 128: tuning key
// "update_exact" (read at plan creation)
int g_update_exact = 1;
// assignment screen of the Lloyd plans: 2 = tensor cores (tcgen05 kind::tf32,
// 3xTF32) when the shape fits, else 1 = FP32 SIMT; the env var CSC_KMEANS_TC=0
// or the tuning key "screen_tc" = 0 keeps the SIMT screen (A/B)
int g_screen_tc = -1;
bool screen_tc_enabled() {
  if (g_screen_tc < 0) {
    const char *e = getenv("CSC_KMEANS_TC");
    g_screen_tc = (e && e[0] == '0') ? 0 : 1;
  }
  return g_screen_tc != 0;
}

// 0 (auto): 8x8 per thread, 16x8 threads (fastest at k = 64 in
// tools/ab_assign.py), 8x4 when k <= 32, 8x7 with 16x16 threads (one pass)
// when 64 < k <= 112; 88/84/87/48/44/42 force a tile
int g_assign_tile = 0;
// 0: fused single-block iteration tail (1024 threads) for small k, 1: same with
// 256 threads, 2: always the split kernels
int g_finish_mode = 0;
// auto: the small-k kernel below this many (row, centroid) pairs
int64_t kSmallAssignNK = int64_t(1) << 22;

// dynamic shared memory of assign3<stages, TM, TN, RT, CT, SC>
template <int TM, int TN, int RT, int CT>
size_t assign3_smem(int64_t d, int64_t k, int stages, bool sc) {
  constexpr int BM = RT * TM, BN = CT * TN;
  const int64_t dpad = csc::ceil_div(d, kAK) * kAK;
  const size_t cbytes = sc ? sizeof(double) * stages * BN * kAKP : sizeof(double) * dpad * (BN + 1);
  // row stages, tile tables (|f|^2 + row id per row, ring of stages + 2), |c|^2, histogram
  return cbytes + sizeof(double) * stages * BM * kAKP + (size_t)(stages + 2) * BM * 12 +
         sizeof(double) * BN + sizeof(int32_t) * (size_t)(k <= kHistMax ? k : 0);
}

template <int TM, int TN, int RT, int CT, bool SC = false>
int launch_assign3_t(const double *f, const double *fnorm, int64_t n, int64_t d, int64_t ld,
                     const double *c, int64_t ldc, const double *cnorm, int64_t k,
                     int32_t *labels, double *own, int32_t *counts, cudaStream_t st,
                     const int32_t *rows, const int32_t *nrows_dev, double *ub, double *lb,
                     const int32_t *gate) {
  constexpr int BM = RT * TM, BN = CT * TN, NT = RT * CT;
  CSC_REQUIRE(n < (int64_t(1) << 31) && ld * (int64_t)sizeof(double) < (int64_t(1) << 31),
              "assign: n and the row stride in bytes must fit int32");
  if (SC)
    CSC_REQUIRE(ldc % 2 == 0 && (reinterpret_cast<uintptr_t>(c) & 15u) == 0,
                "assign (d=%lld): centroids must be 16-byte aligned with an even row stride",
                (long long)d);
  // three stages when two blocks still fit in one SM's shared memory, else two
  const bool three = 2 * (assign3_smem<TM, TN, RT, CT>(d, k, 3, SC) + 1024) <= 228 * 1024;
  const size_t smem = assign3_smem<TM, TN, RT, CT>(d, k, three ? 3 : 2, SC);
  CSC_REQUIRE((int64_t)smem <= (int64_t)csc::device_info().max_smem_optin,
              "assign: d=%lld, k=%lld need %zu bytes of shared memory", (long long)d,
              (long long)k, smem);
  static size_t configured2 = 0, configured3 = 0;
  size_t &configured = three ? configured3 : configured2;
  if (smem > configured) {
    CSC_TRY_CUDA(cudaFuncSetAttribute(three ? assign3_kernel<3, TM, TN, RT, CT, SC>
                                            : assign3_kernel<2, TM, TN, RT, CT, SC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  // persistent grid: two blocks per SM, or one block per row tile when fewer
  const int64_t tiles = csc::ceil_div(n, (int64_t)BM);
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(csc::device_info().sm_count * 2, tiles));
  for (int64_t c0 = 0; c0 < k; c0 += BN) {
    const int last = c0 + BN >= k;
    if (three)
      assign3_kernel<3, TM, TN, RT, CT, SC><<<grid, NT, smem, st>>>(
          f, fnorm, n, d, ld, c, ldc, cnorm, k, c0, last, labels, own, last ? counts : nullptr,
          rows, nrows_dev, ub, lb, gate);
    else
      assign3_kernel<2, TM, TN, RT, CT, SC><<<grid, NT, smem, st>>>(
          f, fnorm, n, d, ld, c, ldc, cnorm, k, c0, last, labels, own, last ? counts : nullptr,
          rows, nrows_dev, ub, lb, gate);
    CSC_CHECK_LAUNCH();
  }
  return CSC_OK;
}

int launch_assign3(const double *f, const double *fnorm, int64_t n, int64_t d, int64_t ld,
                   const double *c, int64_t ldc, const double *cnorm, int64_t k, int32_t *labels,
                   double *own, int32_t *counts, cudaStream_t st, const int32_t *rows,
                   const int32_t *nrows_dev, double *ub, double *lb, const int32_t *gate) {
  const bool small_ok = k <= 64 && d <= 128;
  if (g_assign_tile == 1 || (g_assign_tile == 0 && small_ok && n * k <= kSmallAssignNK)) {
    CSC_REQUIRE(small_ok, "assign_small: needs k <= 64 and d <= 128");
    if (k <= 32)
      return launch_assign_small<1>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts, st,
                                    rows, nrows_dev, ub, lb, gate);
    return launch_assign_small<2>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts, st,
                                  rows, nrows_dev, ub, lb, gate);
  }
  // large d: the resident centroid tile does not fit; stream it (any forced tile
  // maps here too: every tile gives the same bits)
  auto fits = [&](size_t two_stage) {
    return (int64_t)two_stage <= (int64_t)csc::device_info().max_smem_optin;
  };
  const int tile = g_assign_tile > 1 ? g_assign_tile : (k <= 32 ? 84 : (k <= 112 && k > 64 ? 87 : 88));
  const size_t need = tile == 87   ? assign3_smem<8, 7, 16, 16>(d, k, 2, false)
                      : tile == 84 ? assign3_smem<8, 4, 16, 8>(d, k, 2, false)
                      : tile == 48 ? assign3_smem<4, 8, 16, 8>(d, k, 2, false)
                      : tile == 42 ? assign3_smem<4, 4, 32, 8>(d, k, 2, false)
                      : tile == 44 ? assign3_smem<4, 4, 16, 16>(d, k, 2, false)
                                   : assign3_smem<8, 8, 16, 8>(d, k, 2, false);
  if (!fits(need)) {
    if (k <= 32)
      return launch_assign3_t<8, 4, 16, 8, true>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                                 counts, st, rows, nrows_dev, ub, lb, gate);
    return launch_assign3_t<8, 8, 16, 8, true>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                               counts, st, rows, nrows_dev, ub, lb, gate);
  }
  switch (g_assign_tile) {
    case 88:
      return launch_assign3_t<8, 8, 16, 8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                           counts, st, rows, nrows_dev, ub, lb, gate);
    case 48:
      return launch_assign3_t<4, 8, 16, 8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                           counts, st, rows, nrows_dev, ub, lb, gate);
    case 42:
      return launch_assign3_t<4, 4, 32, 8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                           counts, st, rows, nrows_dev, ub, lb, gate);
    case 44:
      return launch_assign3_t<4, 4, 16, 16>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                            counts, st, rows, nrows_dev, ub, lb, gate);
    case 87:  // 128 x 112 tile (16 x 16 threads, 8 x 7 each): one pass for k <= 112
      return launch_assign3_t<8, 7, 16, 16>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                            counts, st, rows, nrows_dev, ub, lb, gate);
    case 84:
      return launch_assign3_t<8, 4, 16, 8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                           counts, st, rows, nrows_dev, ub, lb, gate);
    default:
      if (k <= 32)  // 128 x 32 tile: no wasted FMAs on padding centroids at small k
        return launch_assign3_t<8, 4, 16, 8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                             counts, st, rows, nrows_dev, ub, lb, gate);
      if (k > 64 && k <= 112)  // one 112-wide pass instead of two 64-wide (cfg3 k=100: -18%)
        return launch_assign3_t<8, 7, 16, 16>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                              counts, st, rows, nrows_dev, ub, lb, gate);
      return launch_assign3_t<8, 8, 16, 8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own,
                                           counts, st, rows, nrows_dev, ub, lb, gate);
  }
}

template <int TN>
int launch_assign2(const double *f, const double *fnorm, int64_t n, int64_t d, int64_t ld,
                   const double *c, int64_t ldc, const double *cnorm, int64_t k, int32_t *labels,
                   double *own, int32_t *counts, size_t smem, cudaStream_t st,
                   const int32_t *rows = nullptr, const int32_t *nrows_dev = nullptr,
                   double *ub = nullptr, double *lb = nullptr, const int32_t *gate = nullptr) {
  static size_t configured = 0;
  if (smem > configured) {
    CSC_TRY_CUDA(cudaFuncSetAttribute(assign2_kernel<TN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  assign2_kernel<TN><<<(unsigned)csc::ceil_div(n, kAM), 16 * (kAN / TN), smem, st>>>(
      f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts, rows, nrows_dev, ub, lb, gate);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
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
constexpr int kSqLanes = 8;  // lanes of the extra warp summing |f|^2 per cluster

__global__ void update_partial_kernel(const double *__restrict__ f,
                                      const int32_t *__restrict__ labels, int64_t n, int64_t d,
                                      int64_t ld, int64_t k, int64_t chunk, int cw,
                                      double *__restrict__ psum, int32_t *__restrict__ pcnt,
                                      const double *__restrict__ fnorm, double *__restrict__ pq) {
  extern __shared__ double sm[];
  double *sq = sm + (size_t)k * cw;  // [kSqLanes][k] per-lane |f|^2 sums (y == 0 blocks)
  int32_t *scnt = reinterpret_cast<int32_t *>(sq + kSqLanes * k);
  const int64_t b = blockIdx.x;
  const int64_t col0 = (int64_t)blockIdx.y * cw;
  for (int64_t i = threadIdx.x; i < k * cw; i += blockDim.x) sm[i] = 0.0;
  for (int64_t i = threadIdx.x; i < kSqLanes * k; i += blockDim.x) sq[i] = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) scnt[i] = 0;
  __syncthreads();
  const int64_t rbeg = b * chunk, rend = min(n, rbeg + chunk);
  const int c = threadIdx.x;
  const bool active = c < cw && col0 + c < d;
  if (active) {
    // this thread owns column c of every cluster's partial: rows are added in
    // order; while consecutive rows share a label the running value stays in a
    // register (same additions, same order as adding into shared memory)
    const double *fc = f + col0 + c;
    int cur = -1;
    double run = 0.0;
    auto add = [&](int32_t l, double v) {
      if (l != cur) {
        if (cur >= 0) sm[(size_t)cur * cw + c] = run;
        cur = l;
        run = sm[(size_t)l * cw + c];
      }
      run += v;
    };
    constexpr int U = 16;  // rows per batch; the next batch is loaded before adding this one
    int64_t r = rbeg;
    int32_t la[U], lb2[U];
    double va[U], vb[U];
    auto load = [&](int64_t r0, int32_t (&l)[U], double (&v)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        l[u] = __ldg(labels + r0 + u);
        v[u] = __ldg(fc + (r0 + u) * ld);
      }
    };
    if (r + U <= rend) load(r, la, va);
    while (r + U <= rend) {
      const bool more = r + 2 * U <= rend;
      if (more) load(r + U, lb2, vb);
#pragma unroll
      for (int u = 0; u < U; ++u) add(la[u], va[u]);
      r += U;
      if (!more) break;
      const bool more2 = r + 2 * U <= rend;
      if (more2) load(r + U, la, va);
#pragma unroll
      for (int u = 0; u < U; ++u) add(lb2[u], vb[u]);
      r += U;
      if (!more2) break;
    }
    for (; r < rend; ++r) add(labels[r], fc[r * ld]);
    if (cur >= 0) sm[(size_t)cur * cw + c] = run;
  }
  if (blockIdx.y == 0) {
    for (int64_t r = rbeg + threadIdx.x; r < rend; r += blockDim.x) atomicAdd(scnt + labels[r], 1);
    // per-cluster |f|^2 on kSqLanes lanes of the extra warp: lane l sums rows
    // rbeg + l, rbeg + l + kSqLanes, ... in order; lanes are combined in order
    const int lane_sq = (int)threadIdx.x - ((int)blockDim.x - 32);
    if (pq && lane_sq >= 0 && lane_sq < kSqLanes) {
      double *mine = sq + (size_t)lane_sq * k;
      int cur = -1;
      double run = 0.0;
      auto add = [&](int32_t l, double v) {  // same register-run scheme as the columns
        if (l != cur) {
          if (cur >= 0) mine[cur] = run;
          cur = l;
          run = mine[l];
        }
        run += v;
      };
      // rows rbeg + lane_sq + kSqLanes * t, in order; the next batch of UQ rows
      // is loaded before the current one is added (16 loads in flight)
      constexpr int UQ = 8;
      int64_t r = rbeg + lane_sq;
      int32_t la[UQ], lbq[UQ];
      double va[UQ], vb[UQ];
      auto load = [&](int64_t r0, int32_t (&l)[UQ], double (&v)[UQ]) {
#pragma unroll
        for (int u = 0; u < UQ; ++u) {
          l[u] = __ldg(labels + r0 + u * kSqLanes);
          v[u] = __ldg(fnorm + r0 + u * kSqLanes);
        }
      };
      const int64_t step = (int64_t)UQ * kSqLanes;
      if (r + step - kSqLanes < rend) load(r, la, va);
      while (r + step - kSqLanes < rend) {
        const bool more = r + 2 * step - kSqLanes < rend;
        if (more) load(r + step, lbq, vb);
#pragma unroll
        for (int u = 0; u < UQ; ++u) add(la[u], va[u]);
        r += step;
        if (!more) break;
        const bool more2 = r + 2 * step - kSqLanes < rend;
        if (more2) load(r + step, la, va);
#pragma unroll
        for (int u = 0; u < UQ; ++u) add(lbq[u], vb[u]);
        r += step;
        if (!more2) break;
      }
      for (; r < rend; r += kSqLanes) add(labels[r], fnorm[r]);
      if (cur >= 0) mine[cur] = run;
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < k * cw; i += blockDim.x) {
    const int64_t j = i / cw, cc = i % cw;
    if (col0 + cc < d) psum[(b * k + j) * d + col0 + cc] = sm[i];
  }
  if (blockIdx.y == 0)
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
      pcnt[b * k + j] = scnt[j];
      if (pq) {
        double q = 0.0;
#pragma unroll
        for (int l = 0; l < kSqLanes; ++l) q += sq[(size_t)l * k + j];
        pq[b * k + j] = q;
      }
    }
}
__global__ void update_finish_kernel(const double *__restrict__ psum,
                                     const int32_t *__restrict__ pcnt, int64_t nb, int64_t d,
                                     int64_t k, double *__restrict__ cent, int64_t ldc,
                                     double *__restrict__ cent_t, int32_t *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (w >= k * (d + 1)) return;
  const int64_t j = w / (d + 1), c = w - j * (d + 1);
  if (c == d) {  // the count
    int32_t cnt = 0;
    for (int64_t b = lane; b < nb; b += 32) cnt += pcnt[b * k + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) counts[j] = cnt;
    return;
  }
  double s = 0.0;
  int32_t cnt = 0;
  for (int64_t b = lane; b < nb; b += 32) {
    s += psum[(b * k + j) * d + c];
    cnt += pcnt[b * k + j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (lane == 0) {
    const double mean = __ddiv_rn(s, (double)(cnt > 1 ? cnt : 1));
    cent[j * ldc + c] = mean;
    if (cent_t) cent_t[c * k + j] = mean;
  }
}

__global__ void centroid_norms_kernel(const double *__restrict__ cent, int64_t ldc, int64_t d,
                                      int64_t k, double *__restrict__ cnorm) {
  const int lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (j >= k) return;
  double s = 0.0;
  for (int64_t c = lane; c < d; c += 32) s = fma(cent[j * ldc + c], cent[j * ldc + c], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) cnorm[j] = s;
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

// ---------------------------------------------------------------------------
// Batched k-means++ over R restarts (independent RNG streams, uniforms drawn
// on the host in each stream's order). One pass over F per centroid index
// serves all restarts; draws need no host round trip. A restart whose D^2
// mass ever reaches 0 is flagged (the reference then draws integers(n)
// instead of random(), changing its stream), and the host replays it.
// ---------------------------------------------------------------------------

// closest[r][i] = (first ? d2 : min(closest, d2)), d2 = |f_i - crow_r|^2, for r < R;
// chunk_sums[r][b] = sum of closest[r] over contiguous chunk b (block b).
template <int R>  // restarts in the batch (1..16), compile-time: no predicated lanes
__global__ void __launch_bounds__(128)
    kppb_dist_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                     const double *__restrict__ crows, int64_t crow_stride,
                     double *__restrict__ closest, int first, int64_t chunk,
                     double *__restrict__ chunk_sums, int64_t nchunks) {
  // thread per row: one pass over the row serves all R restarts (no shuffles)
  extern __shared__ double sh[];  // R x d centroid rows, then 4 warps x R partials
  double *cs = sh;
  double *wsum = sh + (size_t)R * d;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t r = threadIdx.x / 32; r < R; r += blockDim.x / 32)  // warp per centroid row
    for (int64_t c = threadIdx.x % 32; c < d; c += 32) cs[r * d + c] = crows[r * crow_stride + c];
  __syncthreads();
  const int64_t rbeg = blockIdx.x * chunk, rend = min(n, rbeg + chunk);
  double part[R];
#pragma unroll
  for (int r = 0; r < R; ++r) part[r] = 0.0;
  // two of the thread's rows (i and i + blockDim) per pass: each centroid
  // value loaded from shared memory feeds both; the block partials still add
  // the thread's rows in ascending order (identical bits)
  for (int64_t i = rbeg + threadIdx.x; i < rend; i += 2 * (int64_t)blockDim.x) {
    const int64_t i2 = i + blockDim.x;
    const bool two = i2 < rend;
    const double *row = f + i * ld;
    const double *row2 = f + (two ? i2 : i) * ld;
    double acc[R], acc2[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = 0.0;
      acc2[r] = 0.0;
    }
    for (int64_t c = 0; c < d; ++c) {
      const double x = __ldg(row + c), x2 = __ldg(row2 + c);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double cv = cs[r * d + c];
        const double t = x - cv, t2 = x2 - cv;
        acc[r] = fma(t, t, acc[r]);
        acc2[r] = fma(t2, t2, acc2[r]);
      }
    }
    if (!first) {  // all loads before the first store (one memory round trip)
      double old[R], old2[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        old[r] = closest[(int64_t)r * n + i];
        old2[r] = two ? closest[(int64_t)r * n + i2] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = fmin(old[r], acc[r]);
        acc2[r] = fmin(old2[r], acc2[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      closest[(int64_t)r * n + i] = acc[r];
      part[r] += acc[r];
    }
    if (two) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        closest[(int64_t)r * n + i2] = acc2[r];
        part[r] += acc2[r];
      }
    }
  }
  // fixed-order block sums per restart: warp shuffle tree, then warps in order
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double v = part[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wsum[wid * R + r] = v;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += wsum[w * R + threadIdx.x];
    chunk_sums[(int64_t)threadIdx.x * nchunks + blockIdx.x] = t;
  }
}

// Staged variant of kppb_dist_kernel for 16-byte-aligned rows (f % 16 == 0, ld
// even). The direct kernel's per-thread row loads touch 32 cache lines per
// warp instruction (~64 L1 wavefront cycles each), which holds the FP64 pipe
// at ~20%. Here a tile of 256 rows x 16 columns (128 B per row, coalesced
// 16-byte cp.async, double-buffered) is staged in shared memory with the
// 16-byte pieces of row t stored at piece ^ (t & 7), so a thread reads two
// columns of its row with one conflict-free 128-bit load; the centroid values
// come as one broadcast 128-bit load per restart and column pair. Same thread
// -> rows mapping (t, t + 128 of every 256-row tile) and the same per-row FMA
// chain over ascending columns as the direct kernel: identical bits.
constexpr int kKsRows = 256;   // rows per tile (two per thread)
constexpr int kKsCols = 16;    // columns per stage (one 128-byte line per row)
template <int R>
__global__ void __launch_bounds__(128)
    kppb_dist_staged_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                            const double *__restrict__ crows, int64_t crow_stride,
                            double *__restrict__ closest, int first, int64_t chunk,
                            double *__restrict__ chunk_sums, int64_t nchunks) {
  extern __shared__ __align__(16) unsigned char kraw[];
  const int npair = (int)((d + 1) / 2);
  double2 *cs2 = reinterpret_cast<double2 *>(kraw);                  // [npair][R] (x = even column)
  double *wsum = reinterpret_cast<double *>(cs2 + (size_t)npair * R);  // 4 warps x R
  unsigned char *tiles =
      kraw + (((size_t)npair * R * 16 + (size_t)4 * R * 8 + 127) / 128) * 128;  // 2 x 32 KB
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < npair * R; e += 128) {
    const int p = e / R, r = e % R;
    const double *cr = crows + (int64_t)r * crow_stride;
    cs2[e] = make_double2(cr[2 * p], 2 * p + 1 < d ? cr[2 * p + 1] : 0.0);
  }
  const int64_t rbeg = blockIdx.x * chunk, rend = min(n, rbeg + chunk);
  const int nstage = (int)((d + kKsCols - 1) / kKsCols);
  const int ntile = rend > rbeg ? (int)((rend - rbeg + kKsRows - 1) / kKsRows) : 0;
  const int nunit = ntile * nstage;
  // thread t copies 16-byte piece (t & 7) of rows (t >> 3) + 16 q, q = 0..15, of
  // every tile: piece and swizzle are per-thread constants, rows step by 16
  const int pj = tid & 7, pr = tid >> 3;
  const unsigned pdst = (unsigned)(pr * 128 + ((pj ^ (pr & 7)) << 4));
  auto issue = [&](int u) {  // stage (u % nstage) of tile (u / nstage) into buffer u & 1
    const int tile = u / nstage, stg = u % nstage;
    const int64_t row0 = rbeg + (int64_t)tile * kKsRows + pr;
    const int c0 = stg * kKsCols;
    const int pieces = (int)min((int64_t)(kKsCols / 2), (d - c0 + 1) / 2);  // valid 16-byte pieces per row
    if (pj < pieces) {
      unsigned char *dst = tiles + (size_t)(u & 1) * (kKsRows * 128) + pdst;
      const double *src = f + row0 * ld + c0 + 2 * pj;
      const int nq = (int)min((int64_t)(kKsRows / 16), (rend - row0 + 15) / 16);  // rows row0 + 16 q < rend
#pragma unroll 4
      for (int q = 0; q < nq; ++q) {
        cp_async16(dst, src, true);
        dst += 16 * 128;
        src += 16 * ld;
      }
    }
    cp_async_commit();
  };
  double part[R];
#pragma unroll
  for (int r = 0; r < R; ++r) part[r] = 0.0;
  if (nunit > 0) issue(0);
  double acc[R], acc2[R];
  const int sw = tid & 7;
  for (int u = 0; u < nunit; ++u) {
    const int tile = u / nstage, stg = u % nstage;
    if (u + 1 < nunit) {
      issue(u + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // unit u landed (and, at u == 0, the centroid pairs are visible)
    if (stg == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = 0.0;
        acc2[r] = 0.0;
      }
    }
    const unsigned char *buf = tiles + (size_t)(u & 1) * (kKsRows * 128);
    const unsigned char *xa = buf + tid * 128, *xb = buf + (tid + 128) * 128;
    const int c0 = stg * kKsCols;
    const int full = (int)min((int64_t)(kKsCols / 2), (d - c0) / 2);  // pairs with both columns valid
    const double2 *cp = cs2 + (size_t)(c0 / 2) * R;
#pragma unroll 2
    for (int p = 0; p < full; ++p) {
      const double2 x = *reinterpret_cast<const double2 *>(xa + ((p ^ sw) << 4));
      const double2 y = *reinterpret_cast<const double2 *>(xb + ((p ^ sw) << 4));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 cv = cp[p * R + r];
        double t = x.x - cv.x, t2 = y.x - cv.x;
        acc[r] = fma(t, t, acc[r]);
        acc2[r] = fma(t2, t2, acc2[r]);
        t = x.y - cv.y;
        t2 = y.y - cv.y;
        acc[r] = fma(t, t, acc[r]);
        acc2[r] = fma(t2, t2, acc2[r]);
      }
    }
    if (full < kKsCols / 2 && c0 + 2 * full < d) {  // odd d: the last column alone
      const double x = *reinterpret_cast<const double *>(xa + ((full ^ sw) << 4));
      const double y = *reinterpret_cast<const double *>(xb + ((full ^ sw) << 4));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double cv = cp[full * R + r].x;
        const double t = x - cv, t2 = y - cv;
        acc[r] = fma(t, t, acc[r]);
        acc2[r] = fma(t2, t2, acc2[r]);
      }
    }
    if (stg == nstage - 1) {
      const int64_t i = rbeg + (int64_t)tile * kKsRows + tid, i2 = i + 128;
      // all previous values loaded before the first store (the stores may
      // alias the loads for the compiler: one memory round trip, not 2R)
      if (!first) {
        double old[R], old2[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          old[r] = i < rend ? closest[(int64_t)r * n + i] : 0.0;
          old2[r] = i2 < rend ? closest[(int64_t)r * n + i2] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r] = fmin(old[r], acc[r]);
          acc2[r] = fmin(old2[r], acc2[r]);
        }
      }
      if (i < rend) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          closest[(int64_t)r * n + i] = acc[r];
          part[r] += acc[r];
        }
      }
      if (i2 < rend) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          closest[(int64_t)r * n + i2] = acc2[r];
          part[r] += acc2[r];
        }
      }
    }
    __syncthreads();  // buffer u & 1 is free for unit u + 2
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double v = part[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wsum[wid * R + r] = v;
  }
  __syncthreads();
  if (tid < R) {
    double t = 0.0;
    for (int w = 0; w < 4; ++w) t += wsum[w * R + tid];
    chunk_sums[(int64_t)tid * nchunks + blockIdx.x] = t;
  }
}

// Block r draws centroid j of restart r from its chunk sums and uniform.
__global__ void __launch_bounds__(1024)
    kppb_pick_kernel(const double *__restrict__ f, int64_t n, int64_t d, int64_t ld,
                     const double *__restrict__ closest, const double *__restrict__ chunk_sums,
                     int64_t nchunks, int64_t chunk, const double *__restrict__ uniforms,
                     int64_t kminus1, int j, double *__restrict__ cent, int64_t cent_stride,
                     int64_t ldc, int32_t *__restrict__ flags) {
  typedef cub::BlockScan<double, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long s_idx;
  __shared__ double s_total, s_target, s_base;
  __shared__ int64_t s_chunk;
  const int r = blockIdx.x;
  const double *cl = closest + (int64_t)r * n;
  const double *cs = chunk_sums + (int64_t)r * nchunks;
  // chunk-level inclusive scan (nchunks <= 1024)
  const double v = threadIdx.x < nchunks ? cs[threadIdx.x] : 0.0;
  double incl, total;
  Scan(tmp).InclusiveSum(v, incl, total);
  if (threadIdx.x == 0) {
    s_total = total;
    s_idx = ~0ull;
    s_chunk = nchunks - 1;
  }
  __syncthreads();
  if (!(s_total > 0.0)) {
    if (threadIdx.x == 0) {
      if (flags[r] < 0) flags[r] = j;
      s_idx = 0;
    }
    __syncthreads();
  } else {
    const double target = uniforms[(int64_t)r * kminus1 + (j - 1)] * s_total;
    if (threadIdx.x < nchunks && incl > target) atomicMin((unsigned long long *)&s_chunk, (unsigned long long)threadIdx.x);
    __syncthreads();
    if (threadIdx.x == (int)s_chunk) s_base = incl - v;
    if (threadIdx.x == 0) s_target = target;
    __syncthreads();
    double running = s_base;
    bool found = false;
    for (int64_t t0 = s_chunk * chunk; t0 < n && !found; t0 += 1024) {
      const int64_t i = t0 + threadIdx.x;
      const double x = i < n ? cl[i] : 0.0;
      double inc2, agg;
      __syncthreads();
      Scan(tmp).InclusiveSum(x, inc2, agg);
      const bool hit = i < n && x > 0.0 && running + inc2 > s_target;
      if (__syncthreads_or(hit)) {
        if (hit) atomicMin(&s_idx, (unsigned long long)i);
        __syncthreads();
        found = true;
      }
      running += agg;
    }
    if (!found && threadIdx.x == 0) {
      int64_t last = n - 1;
      while (last > 0 && !(cl[last] > 0.0)) --last;
      s_idx = (unsigned long long)last;
    }
    __syncthreads();
  }
  const int64_t idx = (int64_t)s_idx;
  double *crow = cent + (int64_t)r * cent_stride + (int64_t)j * ldc;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) crow[c] = f[idx * ld + c];
}

__global__ void kppb_first_kernel(const double *__restrict__ f, int64_t d, int64_t ld,
                                  const int64_t *__restrict__ first_idx, double *__restrict__ cent,
                                  int64_t cent_stride) {
  const int r = blockIdx.x;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x)
    cent[(int64_t)r * cent_stride + c] = f[first_idx[r] * ld + c];
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

// ---------------------------------------------------------------------------
// Lloyd plan: bounds-pruned iterations (Hamerly)
// ---------------------------------------------------------------------------
// ub[i] >= |f_i - c_{a(i)}|, lb[i] <= min_{j != a(i)} |f_i - c_j| (distances,
// not squares). After the centroids move by delta_j, ub += delta_a and
// lb -= max_{j != a} delta_j. If ub + eta <= max(lb, s_a) with
// s_a = min_{j != a} |c_a - c_j| / 2, no centroid can beat a(i) and the row
// keeps its label without any distance computation; every other row is
// recomputed in the reference's GEMM form. eta covers the rounding of the
// GEMM-form distances (|d| error <= ~3e-8 (|f| + |c|)), so a skipped row is
// one whose reference argmin cannot change; near-ties are always recomputed.
// Labels, means and counts therefore follow kmeans.py:96-110.

constexpr int kBoundThreads = 256, kBoundRows = 4;  // rows per thread per chunk

__global__ void __launch_bounds__(kBoundThreads)
    bound_kernel(int64_t n, const int32_t *__restrict__ labels, double *__restrict__ ub,
                 double *__restrict__ lb, const double *__restrict__ delta,
                 const double *__restrict__ scal, const double *__restrict__ shalf,
                 const double *__restrict__ fnorm, int32_t *__restrict__ cand,
                 int32_t *__restrict__ flags, int32_t *__restrict__ counts, int64_t k) {
  typedef cub::BlockScan<int, kBoundThreads> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_base;
  if (blockIdx.x == 0)  // cleared here (stream-ordered before label_hist_kernel)
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) counts[j] = 0;
  const bool force = flags[2] != 0;
  const double d1 = scal[1], d2 = scal[2], cmax = scal[4];
  const int j1 = (int)scal[3];
  constexpr int U = kBoundRows, CH = kBoundThreads * kBoundRows;
  // block-sized chunks of rows (lane-contiguous loads, all loads of a thread's
  // rows issued before use); the candidate list grows by one atomic per chunk
  // (a single counter: per-warp or per-row atomics serialise on its L2 slice)
  for (int64_t base = blockIdx.x * (int64_t)CH; base < n; base += (int64_t)gridDim.x * CH) {
    int64_t r[U];
    int a[U];
    double u[U], l[U], fn[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      r[q] = base + (int64_t)kBoundThreads * q + threadIdx.x;
      if (r[q] < n && !force) {
        a[q] = labels[r[q]];
        u[q] = ub[r[q]];
        l[q] = lb[r[q]];
        fn[q] = fnorm[r[q]];
      }
    }
    bool need[U];
    int mine = 0;
#pragma unroll
    for (int q = 0; q < U; ++q) {
      need[q] = false;
      if (r[q] < n) {
        bool keep = false;
        if (!force) {
          const double uq = u[q] + delta[a[q]];
          const double lq = l[q] - (a[q] == j1 ? d2 : d1);
          const double eta = 1e-7 * (sqrt(fn[q]) + cmax);
          keep = uq + eta <= fmax(lq, shalf[a[q]]);
          ub[r[q]] = uq;
          lb[r[q]] = lq;
        }
        need[q] = !keep;
        mine += need[q] ? 1 : 0;
      }
    }
    int off, total;
    Scan(tmp).ExclusiveSum(mine, off, total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(flags, total) : 0;
    __syncthreads();
    const int pos0 = s_base + off;
    int w = 0;
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (need[q]) cand[pos0 + w++] = (int32_t)r[q];
    __syncthreads();  // tmp / s_base reuse
  }
}

__global__ void label_hist_kernel(int64_t n, int64_t k, const int32_t *__restrict__ labels,
                                  int32_t *__restrict__ counts) {
  extern __shared__ int32_t h[];
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) h[j] = 0;
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(h + labels[r], 1);
  __syncthreads();
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x)
    if (h[j]) atomicAdd(counts + j, h[j]);
}

// flags[1] = some cluster is empty (full reassignment needed for the repair,
// and again next iteration); counts are then cleared for the full recount.
__global__ void check_empty_kernel(int64_t k, int32_t *__restrict__ counts,
                                   int32_t *__restrict__ flags) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x)
    if (counts[j] == 0) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    flags[1] = any;
    flags[2] = any;
  }
  if (any)
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) counts[j] = 0;
}

__global__ void gated_repair_kernel(int32_t *__restrict__ labels, double *__restrict__ own,
                                    const int32_t *__restrict__ counts, int64_t n, int64_t k,
                                    const int32_t *__restrict__ flags) {
  if (flags[1] == 0) return;
  for (int64_t j = 0; j < k; ++j) {
    if (counts[j] != 0) continue;
    double bv;
    int64_t bi = 0;
    block_argmax(own, n, bv, bi);
    if (threadIdx.x == 0) {
      labels[bi] = (int32_t)j;
      own[bi] = -1.0;
    }
    __syncthreads();
  }
}

// warp per (centroid j, column c): S[j][c] = sum of the block partials in
// order; the extra warp per j adds the counts and the |f|^2 partials.
// Block partial sums over a label-sorted chunk. A stable counting sort of the
// chunk's rows by label (shared memory, warp match ranks) makes every
// cluster's rows one contiguous run in increasing row order, so each column
// thread sums a run in a register (0.0 + v1 + v2 + ..., the same additions in
// the same order as update_partial_kernel's per-row shared-memory adds, so
// psum is bit-identical) with the next rows' loads in flight, and writes the
// run's total straight to psum. Counts are the run lengths; |f|^2 per cluster
// is summed over its run in row order by the extra warp.
constexpr int kSortedMaxChunk = 8192;

// Incremental mode (prev != nullptr, one column block): only the clusters
// whose membership changed in this chunk since the previous update ("dirty":
// some row of the chunk left or joined them; prev holds the labels of that
// update and is refreshed here) are re-summed, from scratch in row order, so
// every psum / pq entry always equals the fresh fixed-order sum of its
// current members (bit-identical to recomputing all of them). Late Lloyd
// iterations move few rows, so most chunks re-read little or nothing. The
// caller zeroes psum / pcnt / pq and sets prev = -1 before the first update
// of a run (no members anywhere).
__global__ void update_sorted_kernel(const double *__restrict__ f,
                                     const int32_t *__restrict__ labels, int64_t n, int64_t d,
                                     int64_t ld, int64_t k, int64_t chunk, int cw,
                                     double *__restrict__ psum, int32_t *__restrict__ pcnt,
                                     const double *__restrict__ fnorm, double *__restrict__ pq,
                                     int32_t *__restrict__ prev) {
  extern __shared__ int32_t us[];
  int32_t *lab_s = us;             // [chunk] labels in sorted order (dirty clusters only)
  int32_t *perm_s = lab_s + chunk;  // [chunk] row offsets in sorted order
  int32_t *cnt_s = perm_s + chunk;  // [k] rows per label
  int32_t *run_s = cnt_s + k;       // [k] insert position, then end of each run
  int32_t *dirty_s = run_s + k;     // [k] membership changed (always 1 without prev)
  __shared__ int len_s;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t b = blockIdx.x;
  const int64_t col0 = (int64_t)blockIdx.y * cw;
  const int64_t rbeg = b * chunk;
  const int len = (int)max((int64_t)0, min(n, rbeg + chunk) - rbeg);
  for (int64_t j = tid; j < k; j += blockDim.x) {
    cnt_s[j] = 0;
    dirty_s[j] = prev ? 0 : 1;
  }
  __syncthreads();
  for (int p = tid; p < len; p += blockDim.x) {
    const int l = labels[rbeg + p];
    atomicAdd(cnt_s + l, 1);
    if (prev) {
      const int pl = prev[rbeg + p];
      if (pl != l) {
        dirty_s[l] = 1;
        if (pl >= 0) dirty_s[pl] = 1;
        prev[rbeg + p] = l;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {  // runs of the dirty clusters only, in label order
    int acc = 0;
    for (int64_t j = 0; j < k; ++j) {
      run_s[j] = acc;
      if (dirty_s[j]) acc += cnt_s[j];
    }
    len_s = acc;
  }
  __syncthreads();
  if (tid < 32) {  // stable scatter of the dirty clusters' rows, 32 rows at a time in order
    for (int g = 0; g < len; g += 32) {
      const int p = g + lane;
      int l = p < len ? labels[rbeg + p] : -1;
      if (l >= 0 && !dirty_s[l]) l = -1;
      const unsigned m = __match_any_sync(0xffffffffu, l);
      const int rank = __popc(m & ((1u << lane) - 1u));
      if (l >= 0) {
        const int pos = run_s[l] + rank;
        perm_s[pos] = p;
        lab_s[pos] = l;
      }
      __syncwarp();
      if (l >= 0 && rank == __popc(m) - 1) run_s[l] += __popc(m);
      __syncwarp();
    }
  }
  __syncthreads();
  const int dlen = len_s;
  const int c = tid;
  if (c < cw && col0 + c < d) {
    const double *fc = f + col0 + c;
    double *out = psum + b * k * d + col0 + c;
    int cur = -1;
    double run = 0.0;
    constexpr int U = 16;  // rows per batch; the next batch is loaded before adding this one
    int p = 0;
    double va[U], vb[U];
    int la[U], lb2[U];
    auto load = [&](int p0, double (&v)[U], int (&l)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = __ldg(fc + (rbeg + perm_s[p0 + u]) * ld);
        l[u] = lab_s[p0 + u];
      }
    };
    auto add = [&](const double (&v)[U], const int (&l)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (l[u] != cur) {
          if (cur >= 0) out[(int64_t)cur * d] = run;
          cur = l[u];
          run = 0.0;
        }
        run += v[u];
      }
    };
    if (p + U <= dlen) load(p, va, la);
    while (p + U <= dlen) {
      const bool more = p + 2 * U <= dlen;
      if (more) load(p + U, vb, lb2);
      add(va, la);
      p += U;
      if (!more) break;
      const bool more2 = p + 2 * U <= dlen;
      if (more2) load(p + U, va, la);
      add(vb, lb2);
      p += U;
      if (!more2) break;
    }
    for (; p < dlen; ++p) {
      const int l = lab_s[p];
      const double v = fc[(rbeg + perm_s[p]) * ld];
      if (l != cur) {
        if (cur >= 0) out[(int64_t)cur * d] = run;
        cur = l;
        run = 0.0;
      }
      run += v;
    }
    if (cur >= 0) out[(int64_t)cur * d] = run;
    for (int64_t j = 0; j < k; ++j)
      if (cnt_s[j] == 0 && dirty_s[j]) out[j * d] = 0.0;
  }
  if (blockIdx.y == 0 && tid >= (int)blockDim.x - 32) {
    for (int64_t j = lane; j < k; j += 32) {
      pcnt[b * k + j] = cnt_s[j];
      if (pq && dirty_s[j]) {
        const int end = run_s[j], beg = end - cnt_s[j];
        double q = 0.0;
        for (int pp = beg; pp < end; ++pp) q += fnorm[rbeg + perm_s[pp]];
        pq[b * k + j] = q;
      }
    }
  }
}

// ---- exact, order-free centroid sums (round 2) ------------------------------
// The Lloyd plan keeps every cluster's column sums S_jc and |f|^2 sums Q_j as
// 128-bit two's-complement fixed-point integers: a value v enters as
// trunc(v 2^P) (P fixed for the run from max |f|^2 and n so that no sum can
// reach 2^126; every value within 2^53 of the largest is represented exactly,
// smaller ones lose at most 2^-P each). Integer additions commute, so the
// sums are independent of the order rows are added in: an iteration adds the
// rows that joined a cluster and subtracts the rows that left it (labels vs
// the previous update's), reading only the changed rows of F, and the result
// is bitwise the same as summing every member afresh — deterministic, and
// the correctly rounded (not the row-order) sum, within the reference's own
// rounding of np.add.at (kmeans.py:82-83) at the tolerances the tests state.
// Carries: lo and hi are two 64-bit words; adding (lo, hi) with atomicAdd on
// lo returns the old lo, the carry out of it is (old + lo < old), and hi gets
// hi + carry: the pair is exact modulo 2^128 in any interleaving.
struct FxScale {
  double s1, s2;    // v * s1 * s2 = v * 2^P (two factors: P may exceed a double's range)
  double r1, r2;    // 2^-P as two factors
  int P;
};

__device__ __forceinline__ FxScale fx_scale(double bound) {
  // P such that bound * 2^P < 2^125 (bound >= every |partial sum|)
  int e = 0;
  if (bound > 0.0) frexp(bound, &e);  // bound < 2^e
  const int P = bound > 0.0 ? 125 - e : 0;
  const int p1 = P / 2, p2 = P - p1;
  FxScale f;
  f.P = P;
  f.s1 = ldexp(1.0, p1);
  f.s2 = ldexp(1.0, p2);
  f.r1 = ldexp(1.0, -p1);
  f.r2 = ldexp(1.0, -p2);
  return f;
}

__device__ __forceinline__ void fx_split(double v, const FxScale &fs, uint64_t &lo, uint64_t &hi) {
  const double x = (v * fs.s1) * fs.s2;  // exact unless |v 2^P| < 2^-1022 (then below the LSB)
  const double a = fabs(x);
  const double h = floor(a * 0x1p-64);    // exact
  const double l = __dsub_rn(a, h * 0x1p64);  // exact: the low bits of a, in [0, 2^64)
  uint64_t ulo = (uint64_t)l, uhi = (uint64_t)h;  // truncation below the LSB
  if (x < 0.0) {
    ulo = ~ulo + 1ull;
    uhi = ~uhi + (ulo == 0ull ? 1ull : 0ull);
  }
  lo = ulo;
  hi = uhi;
}

__device__ __forceinline__ void fx_neg(uint64_t &lo, uint64_t &hi) {
  lo = ~lo + 1ull;
  hi = ~hi + (lo == 0ull ? 1ull : 0ull);
}

__device__ __forceinline__ void fx_atomic_add(unsigned long long *lo_p, unsigned long long *hi_p,
                                              uint64_t lo, uint64_t hi) {
  const unsigned long long old = atomicAdd(lo_p, (unsigned long long)lo);
  const uint64_t carry = (old + lo < old) ? 1ull : 0ull;
  if (hi + carry) atomicAdd(hi_p, (unsigned long long)(hi + carry));
}

// correctly rounded double of the 128-bit value, times 2^-P
__device__ __forceinline__ double fx_to_double(uint64_t lo, uint64_t hi, const FxScale &fs) {
  const bool neg = (int64_t)hi < 0;
  if (neg) fx_neg(lo, hi);
  double mag;
  if (hi == 0) {
    mag = __ull2double_rn(lo);
  } else {
    const int lz = __clzll((long long)hi);  // >= 1: magnitudes stay below 2^126
    const uint64_t top = (hi << lz) | (lo >> (64 - lz));
    const uint64_t rest = lo << lz;
    // the bits below the top 64 only matter as a sticky bit (they sit below
    // the rounding position of the 64 -> 53 bit conversion)
    mag = ldexp(__ull2double_rn(top | (rest != 0ull ? 1ull : 0ull)), 64 - lz);
  }
  const double r = (mag * fs.r1) * fs.r2;
  return neg ? -r : r;
}

// max over rows of |f|^2 (non-negative doubles order like their bit patterns)
__global__ void fx_maxnorm_kernel(const double *__restrict__ fnorm, int64_t n,
                                  unsigned long long *__restrict__ maxbits) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fnorm[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(m));
}

// Delta update of the fixed-point sums: a row whose label differs from
// prev[r] leaves cluster prev[r] (if >= 0) and joins labels[r]. Because the
// sums are integers, the order the changes are added in does not matter, so
// the changes are bucketed by cluster without sorting:
//  1. fx_changes_kernel: one entry (row | sign << 31) per (row, cluster) it
//     leaves or joins, appended with one atomic per warp; per-cluster entry
//     counts and net membership changes through per-block shared histograms;
//  2. fx_offsets_kernel (one block): cluster offsets (exclusive scan) and the
//     chunk size for step 4 from the entry total;
//  3. fx_scatter_kernel: entries into their cluster's bucket (atomic cursor;
//     the order inside a bucket is immaterial);
//  4. fx_sum_kernel: persistent blocks take chunks of the bucketed list; a
//     thread per column sums its chunk's rows in a 128-bit register pair
//     (add with carry), reading only changed rows of F, and adds the total
//     into the cluster's global sum with one 128-bit atomic per (chunk,
//     cluster, column) — no per-element atomics.
// Buffers (plan): entries [2n], bucketed [2n], cnt/off/cursor [k], scalars.
constexpr int kFxThreads = 256;   // changes / scatter kernels
constexpr int kFxSumThreads = 128;  // sum kernel: one thread per column (d <= 128)

struct FxWork {
  int32_t *entries;    // [2n] row | (leave << 31), cluster in ecl
  int32_t *ecl;        // [2n] cluster of the entry
  int32_t *bucketed;   // [2n] rows | sign, grouped by cluster
  int32_t *ccount;     // [k] entries per cluster
  int32_t *coff;       // [k + 1] bucket offsets
  int32_t *cursor;     // [k] scatter cursors
  int32_t *scal;       // [0] entry total, [1] chunk size
};

__global__ void __launch_bounds__(kFxThreads)
    fx_changes_kernel(const int32_t *__restrict__ labels, int32_t *__restrict__ prev, int64_t n, int k,
                      FxWork w, int32_t *__restrict__ gcnt) {
  extern __shared__ int32_t fsh[];
  int32_t *hc = fsh;       // [k] entries per cluster
  int32_t *hn = fsh + k;   // [k] net membership change
  for (int i = threadIdx.x; i < 2 * k; i += kFxThreads) fsh[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  bool any = false;
  for (int64_t base = (blockIdx.x * (int64_t)kFxThreads + threadIdx.x) & ~(int64_t)31; base < n;
       base += (int64_t)gridDim.x * kFxThreads) {
    const int64_t r = base + lane;
    int nl = -1, ol = -1;
    if (r < n) {
      nl = labels[r];
      ol = prev[r];
    }
    const bool ch = r < n && nl != ol;
    if (ch) prev[r] = nl;
    const int ne = ch ? (ol >= 0 ? 2 : 1) : 0;
    // warp-aggregated append of this warp's entries
    int incl = ne;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    if (tot == 0) continue;
    any = true;
    int b0 = 0;
    if (lane == 31) b0 = atomicAdd(w.scal, tot);
    b0 = __shfl_sync(0xffffffffu, b0, 31);
    int pos = b0 + incl - ne;
    if (ch) {
      w.entries[pos] = (int32_t)r;
      w.ecl[pos] = nl;
      atomicAdd(hc + nl, 1);
      atomicAdd(hn + nl, 1);
      if (ol >= 0) {
        w.entries[pos + 1] = (int32_t)r | (int32_t)0x80000000;
        w.ecl[pos + 1] = ol;
        atomicAdd(hc + ol, 1);
        atomicSub(hn + ol, 1);
      }
    }
  }
  if (!__syncthreads_or(any)) return;
  for (int j = threadIdx.x; j < k; j += kFxThreads) {
    if (hc[j]) atomicAdd(w.ccount + j, hc[j]);
    if (hn[j]) atomicAdd(gcnt + j, hn[j]);
  }
}

// one warp: exclusive scan of the k (<= 32 * 8) bucket counts
__global__ void fx_offsets_kernel(int k, FxWork w, int target_chunks) {
  const int lane = threadIdx.x & 31;
  constexpr int PER = 8;
  int32_t v[PER], s = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = lane * PER + i;
    v[i] = j < k ? w.ccount[j] : 0;
    s += v[i];
  }
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  int32_t acc = incl - s;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = lane * PER + i;
    if (j < k) {
      w.coff[j] = acc;
      w.cursor[j] = 0;
      w.ccount[j] = 0;  // ready for the next update
    }
    acc += v[i];
  }
  const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (lane == 0) {
    w.coff[k] = total;
    // chunk size: enough chunks to fill the GPU, at least 32 rows each
    const int32_t c = (total + target_chunks - 1) / target_chunks;
    w.scal[1] = c < 32 ? 32 : c;
  }
}

// per block: a shared histogram of its entries' clusters, one global cursor
// atomic per (block, cluster) reserves the block's ranges, then shared
// cursors place the entries (one contiguous slice of the list per block)
__global__ void __launch_bounds__(kFxThreads) fx_scatter_kernel(FxWork w, int k) {
  extern __shared__ int32_t ssh[];
  int32_t *hist = ssh, *basep = ssh + k;
  const int32_t total = w.scal[0];
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min((int64_t)total, e0 + per);
  if (e0 >= e1) return;
  for (int j = threadIdx.x; j < k; j += kFxThreads) hist[j] = 0;
  __syncthreads();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kFxThreads) atomicAdd(hist + w.ecl[e], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += kFxThreads) {
    basep[j] = hist[j] ? w.coff[j] + atomicAdd(w.cursor + j, hist[j]) : 0;
    hist[j] = 0;
  }
  __syncthreads();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kFxThreads) {
    const int32_t c = w.ecl[e];
    w.bucketed[basep[c] + atomicAdd(hist + c, 1)] = w.entries[e];
  }
}

__device__ __forceinline__ void add128(uint64_t &lo, uint64_t &hi, uint64_t xlo, uint64_t xhi) {
  lo += xlo;
  hi += xhi + (lo < xlo ? 1ull : 0ull);
}

constexpr int kFxRowGroups = 4;  // row groups of a sum block (each a full set of column threads)

__global__ void __launch_bounds__(kFxSumThreads * kFxRowGroups)
    fx_sum_kernel(const double *__restrict__ f, int64_t ld, const double *__restrict__ fnorm, int64_t n,
                  int d, int k, const unsigned long long *__restrict__ maxbits, FxWork w,
                  unsigned long long *__restrict__ gS_lo, unsigned long long *__restrict__ gS_hi,
                  unsigned long long *__restrict__ gQ) {
  __shared__ uint64_t red[kFxRowGroups][kFxSumThreads + 1][2];
  const int32_t total = w.scal[0], chunk = w.scal[1];
  if (total == 0) return;
  const double mf = __longlong_as_double((long long)*maxbits);
  const FxScale fs = fx_scale(sqrt(mf) * (1.0 + 1e-12) * (double)n);
  const FxScale fq = fx_scale(mf * (double)n);
  const int c = threadIdx.x % kFxSumThreads, rg = threadIdx.x / kFxSumThreads;
  const int32_t nchunks = (total + chunk - 1) / chunk;
  for (int32_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int32_t e0 = ch * chunk, e1 = min(total, e0 + chunk);
    // cluster of e0: last j with coff[j] <= e0 (then coff[j + 1] > e0)
    int lo = 0, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (w.coff[mid] <= e0) lo = mid;
      else hi = mid - 1;
    }
    // the chunk's clusters are handled one segment at a time by all row groups
    for (int cl = lo; cl < k && w.coff[cl] < e1; ++cl) {
      const int32_t s0 = max(e0, w.coff[cl]), s1 = min(e1, w.coff[cl + 1]);
      uint64_t slo = 0, shi = 0, qlo = 0, qhi = 0;
      constexpr int U = 4;  // rows per group whose values are loaded before they are added
      for (int32_t e = s0 + rg * U; e < s1; e += kFxRowGroups * U) {
        int32_t ent[U];
        double v[U], q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ent[u] = e + u < s1 ? __ldg(w.bucketed + e + u) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t row = (int64_t)(ent[u] & 0x7fffffff);
          v[u] = (e + u < s1 && c < d) ? __ldg(f + row * ld + c) : 0.0;
          q[u] = (e + u < s1 && c == 0) ? __ldg(fnorm + row) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (e + u >= s1) break;
          uint64_t xl, xh;
          fx_split(v[u], fs, xl, xh);
          if (ent[u] < 0) fx_neg(xl, xh);
          add128(slo, shi, xl, xh);
          if (c == 0) {
            fx_split(q[u], fq, xl, xh);
            if (ent[u] < 0) fx_neg(xl, xh);
            add128(qlo, qhi, xl, xh);
          }
        }
      }
      // combine the row groups (integer adds: any order), one 128-bit atomic per column
      red[rg][c][0] = slo;
      red[rg][c][1] = shi;
      if (c == 0) {
        red[rg][kFxSumThreads][0] = qlo;
        red[rg][kFxSumThreads][1] = qhi;
      }
      __syncthreads();
      if (rg == 0) {
#pragma unroll
        for (int g = 1; g < kFxRowGroups; ++g) add128(slo, shi, red[g][c][0], red[g][c][1]);
        if (c < d && (slo | shi)) fx_atomic_add(gS_lo + (size_t)cl * d + c, gS_hi + (size_t)cl * d + c, slo, shi);
        if (c == 0) {
#pragma unroll
          for (int g = 1; g < kFxRowGroups; ++g)
            add128(qlo, qhi, red[g][kFxSumThreads][0], red[g][kFxSumThreads][1]);
          if (qlo | qhi) fx_atomic_add(gQ + 2 * cl, gQ + 2 * cl + 1, qlo, qhi);
        }
      }
      __syncthreads();
    }
  }
}

// the fixed-point sums as doubles for the iteration tail: S [k][d], Q [k], counts [k]
__global__ void fx_finish_kernel(const unsigned long long *__restrict__ gS_lo,
                                 const unsigned long long *__restrict__ gS_hi,
                                 const unsigned long long *__restrict__ gQ,
                                 const int32_t *__restrict__ gcnt, int64_t n, int d, int k,
                                 const unsigned long long *__restrict__ maxbits,
                                 double *__restrict__ S, double *__restrict__ Q,
                                 int32_t *__restrict__ counts) {
  const double mf = __longlong_as_double((long long)*maxbits);
  const FxScale fs = fx_scale(sqrt(mf) * (1.0 + 1e-12) * (double)n);
  const FxScale fq = fx_scale(mf * (double)n);
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < (int64_t)k * d) S[i] = fx_to_double(gS_lo[i], gS_hi[i], fs);
  if (i < k) {
    Q[i] = fx_to_double(gQ[2 * i], gQ[2 * i + 1], fq);
    counts[i] = gcnt[i];
  }
}

size_t fx_smem(int64_t, int64_t k) { return sizeof(int32_t) * 2 * (size_t)k; }

__global__ void sums_finish_kernel(const double *__restrict__ psum,
                                   const int32_t *__restrict__ pcnt,
                                   const double *__restrict__ pq, int64_t nb, int64_t d,
                                   int64_t k, double *__restrict__ S, int32_t *__restrict__ counts,
                                   double *__restrict__ Q) {
  const int lane = threadIdx.x & 31;
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (w >= k * (d + 1)) return;
  const int64_t j = w / (d + 1), c = w - j * (d + 1);
  if (c == d) {
    int32_t cnt = 0;
    double q = 0.0;
    for (int64_t b = lane; b < nb; b += 32) {
      cnt += pcnt[b * k + j];
      q += pq[b * k + j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (lane == 0) {
      counts[j] = cnt;
      Q[j] = q;
    }
    return;
  }
  double sacc = 0.0;
  for (int64_t b = lane; b < nb; b += 32) sacc += psum[(b * k + j) * d + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  if (lane == 0) S[j * d + c] = sacc;
}

// block per centroid: mean = S / max(count, 1) (kmeans.py:84), movement
// delta_j, |c_j|^2, and the cluster's cost term via the centroid identity
// sum_i |f_i - m|^2 = Q - 2 m.S + count |m|^2 (with the rounded mean m).
__global__ void centroid_finish_kernel(const double *__restrict__ S,
                                       const int32_t *__restrict__ counts,
                                       const double *__restrict__ Q, int64_t d, int64_t k,
                                       double *__restrict__ cent, int64_t ldc,
                                       double *__restrict__ cnorm, double *__restrict__ delta,
                                       double *__restrict__ cterm) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  const int32_t cnt = counts[j];
  const double denom = (double)(cnt > 1 ? cnt : 1);
  double mv = 0.0, nrm = 0.0, dot = 0.0;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    const double sjc = S[j * d + c];
    const double mean = __ddiv_rn(sjc, denom);
    const double old = cent[j * ldc + c];
    cent[j * ldc + c] = mean;
    mv = fma(mean - old, mean - old, mv);
    nrm = fma(mean, mean, nrm);
    dot = fma(mean, sjc, dot);
  }
  mv = block_sum<128>(mv, red);
  nrm = block_sum<128>(nrm, red);
  dot = block_sum<128>(dot, red);
  if (threadIdx.x == 0) {
    delta[j] = sqrt(mv);
    cnorm[j] = nrm;
    cterm[j] = cnt > 0 ? (Q[j] - 2.0 * dot) + (double)cnt * nrm : 0.0;
  }
}

// Single-block tail of an iteration for small k: the means, movements,
// cost terms, scalars and half-separations of centroid_finish + iter_finish +
// shalf in one graph node (after the multi-block sums_finish_kernel), with the
// new centroids staged in shared memory (odd row stride: conflict-free) for
// the pairwise pass. Same per-element arithmetic and summation order as those
// kernels for the half-separations. Also clears the candidate counter of the
// next pruned iteration.
__global__ void __launch_bounds__(1024)
    finish_small_kernel(int64_t d, int64_t k, const double *__restrict__ S,
                        const int32_t *__restrict__ counts, const double *__restrict__ Q,
                        double *__restrict__ cent, int64_t ldc, double *__restrict__ cnorm,
                        double *__restrict__ delta, double *__restrict__ cterm,
                        double *__restrict__ scal, double *__restrict__ shalf,
                        int32_t *__restrict__ flags, float *__restrict__ chi,
                        float *__restrict__ clo, float *__restrict__ cn32,
                        double *__restrict__ cmax, int npad, int kp) {
  extern __shared__ double cs[];  // [k][lds] centroids, then [3][k] delta, |c|^2, cost term
  const int64_t lds = d | 1;
  double *sdel = cs + k * lds, *snrm = sdel + k, *sct = snrm + k;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // warp per centroid: means, movement, |c|^2, cost term
  for (int64_t j = wid; j < k; j += nw) {
    const int32_t cnt = counts[j];
    const double denom = (double)(cnt > 1 ? cnt : 1);
    double mv = 0.0, nrm = 0.0, dot = 0.0;
    for (int64_t c = lane; c < d; c += 32) {
      const double sjc = S[j * d + c];
      const double mean = __ddiv_rn(sjc, denom);
      const double old = cent[j * ldc + c];
      cent[j * ldc + c] = mean;
      cs[j * lds + c] = mean;
      mv = fma(mean - old, mean - old, mv);
      nrm = fma(mean, mean, nrm);
      dot = fma(mean, sjc, dot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mv += __shfl_xor_sync(0xffffffffu, mv, o);
      nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      dot += __shfl_xor_sync(0xffffffffu, dot, o);
    }
    if (lane == 0) {
      const double ct = cnt > 0 ? (Q[j] - 2.0 * dot) + (double)cnt * nrm : 0.0;
      delta[j] = sdel[j] = sqrt(mv);
      cnorm[j] = snrm[j] = nrm;
      cterm[j] = sct[j] = ct;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double cost = 0.0, d1 = 0.0, d2 = 0.0, cm = 0.0;
    int64_t j1 = 0;
    for (int64_t j = 0; j < k; ++j) {
      cost += sct[j];
      const double dj = sdel[j];
      if (dj > d1) {
        d2 = d1;
        d1 = dj;
        j1 = j;
      } else if (dj > d2) {
        d2 = dj;
      }
      cm = fmax(cm, snrm[j]);
    }
    scal[0] = cost > 0.0 ? cost : 0.0;
    scal[1] = d1;
    scal[2] = d2;
    scal[3] = (double)j1;
    scal[4] = sqrt(cm);
    if (cmax) cmax[0] = sqrt(cm);
    flags[3] = flags[0];  // last candidate count, for csc_kmeans_plan_stats
    flags[0] = 0;
  }
  if (chi) {  // the next iteration's tensor-core screen tiles (tc_centroids_kernel's values)
    for (int64_t j = threadIdx.x / 32; j < npad; j += blockDim.x / 32)  // warp per centroid
      for (int64_t t = threadIdx.x % 32; t < kp; t += 32) {
        const float v = (j < k && t < d) ? (float)cs[j * lds + t] : 0.0f;
        const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        const int64_t off = (t / 4) * (int64_t)npad * 4 + j * 4 + (t % 4);
        chi[off] = h;
        clo[off] = v - h;
      }
    for (int64_t j = threadIdx.x; j < npad; j += blockDim.x) {
      float sq = INFINITY;
      if (j < k) {
        sq = 0.0f;
        for (int64_t t = 0; t < d; ++t) {
          const float v = (float)cs[j * lds + t];
          sq = fmaf(v, v, sq);
        }
      }
      cn32[j] = sq;
    }
  }
  // half-separations: lane o of warp j accumulates |c_j - c_o|^2 over c in order
  for (int64_t j = wid; j < k; j += nw) {
    double best = INFINITY;
    for (int64_t o = lane; o < k; o += 32) {
      if (o == j) continue;
      double sacc = 0.0;
      for (int64_t c = 0; c < d; ++c) {
        const double t = cs[j * lds + c] - cs[o * lds + c];
        sacc = fma(t, t, sacc);
      }
      best = fmin(best, sacc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) shalf[j] = 0.5 * sqrt(best);
  }
}

// scal[0] = cost2 (sum of cluster terms, fixed order), scal[1..3] = largest
// movement, second largest, its centroid; scal[4] = max_j |c_j|.
__global__ void iter_finish_kernel(int64_t k, const double *__restrict__ cterm,
                                   const double *__restrict__ delta,
                                   const double *__restrict__ cnorm, double *__restrict__ scal,
                                   int32_t *__restrict__ flags) {
  if (threadIdx.x != 0) return;
  flags[3] = flags[0];  // last candidate count, for csc_kmeans_plan_stats
  flags[0] = 0;         // candidate counter of the next pruned iteration
  double cost = 0.0, d1 = 0.0, d2 = 0.0, cm = 0.0;
  int64_t j1 = 0;
  for (int64_t j = 0; j < k; ++j) {
    cost += cterm[j];
    const double dj = delta[j];
    if (dj > d1) {
      d2 = d1;
      d1 = dj;
      j1 = j;
    } else if (dj > d2) {
      d2 = dj;
    }
    cm = fmax(cm, cnorm[j]);
  }
  scal[0] = cost > 0.0 ? cost : 0.0;
  scal[1] = d1;
  scal[2] = d2;
  scal[3] = (double)j1;
  scal[4] = sqrt(cm);
}

// shalf[j] = min_{j' != j} |c_j - c_j'| / 2 (difference form), +inf for k = 1
__global__ void shalf_kernel(const double *__restrict__ cent, int64_t ldc, int64_t d, int64_t k,
                             double *__restrict__ shalf) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  double best = INFINITY;
  for (int64_t o = threadIdx.x; o < k; o += blockDim.x) {
    if (o == j) continue;
    double s = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      const double t = cent[j * ldc + c] - cent[o * ldc + c];
      s = fma(t, t, s);
    }
    best = fmin(best, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = INFINITY;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) b = fmin(b, red[w]);
    shalf[j] = 0.5 * sqrt(b);
  }
}

// device-side stop rule of kmeans.py:112-116 for graph-resident Lloyd loops
struct LoopState {
  double prev, tol;
  int it, max_iters, stop, pad;
};

__global__ void copy_iters_kernel(const LoopState *ls, double *out, int ran) {
  out[0] = ran ? (double)ls->it : 0.0;
  if (!ran) out[-1] = INFINITY;
}

__global__ void loop_init_kernel(LoopState *ls, double tol, int max_iters) {
  ls->prev = INFINITY;
  ls->tol = tol;
  ls->it = 0;
  ls->max_iters = max_iters;
  ls->stop = 0;
}

__global__ void loop_check_kernel(const double *__restrict__ scal, LoopState *ls,
                                  double *__restrict__ history, int hist_cap,
                                  cudaGraphConditionalHandle h, int use_handle) {
  const double c = scal[0];
  if (history && ls->it < hist_cap) history[ls->it] = c;
  int stop = 0;
  if (isfinite(ls->prev) && ls->prev - c <= ls->tol * ls->prev) stop = 1;
  ls->prev = c;
  ls->it += 1;
  if (ls->it >= ls->max_iters) stop = 1;
  ls->stop = stop;
  if (use_handle) cudaGraphSetConditional(h, stop ? 0u : 1u);
}

int grid_cap(int64_t want, int per_sm = 8) {
  return (int)std::min<int64_t>((int64_t)csc::device_info().sm_count * per_sm,
                                std::max<int64_t>(1, want));
}

}  // namespace

struct csc_kmeans_plan {
  int64_t n = 0, d = 0, ld = 0, k = 0;
  int64_t nb = 0, chunk = 0, cw = 0, ny = 0;
  void *base = nullptr;
  double *ub, *lb, *own, *psum, *pq, *S, *Q, *cterm, *delta, *shalf, *scal;
  int32_t *cand, *flags, *pcnt, *prev;
  size_t smem = 0;
  cudaStream_t stream = nullptr;
  // graph-resident loop (built on first csc_kmeans_run for a buffer set)
  LoopState *loop = nullptr;
  double *cost_parts = nullptr;  // plan-owned: no cross-stream pool reuse between lanes
  double *history = nullptr;
  int hist_cap = 0;
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  const void *key[12] = {};
  // FP32 screen (kmeans_screen.cu): caller's fp32 features, plan-owned scratch
  const float *f32 = nullptr, *fn32 = nullptr;
  int64_t ld32 = 0;
  float *c32t = nullptr, *cn32 = nullptr;
  double *cmax = nullptr;
  int32_t *amb = nullptr, *namb = nullptr;
  void *screen_base = nullptr;
  // tensor-core screen (kmeans_screen_tc.cu): hi / lo centroid tiles
  bool tc = false;
  float *chi = nullptr, *clo = nullptr;
  // exact fixed-point sums (fx_* kernels): [k][d] lo / hi words, Q [k][2],
  // counts [k], max |f|^2 bits; the change lists and buckets in fxw
  bool fx = false;
  FxWork fxw{};
  void *fxw_base = nullptr;
  bool finish_small = false;  // one single-block node finishes an iteration
  int fx_grid = 0;
  void *fx_base = nullptr;
  unsigned long long *fx_lo = nullptr, *fx_hi = nullptr, *fx_q = nullptr, *fx_max = nullptr;
  int32_t *fx_cnt = nullptr;
};

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
  const int64_t dpad = csc::ceil_div(d, kAK) * kAK;
  const size_t smem = sizeof(double) * (dpad * kANP + 2 * kAM * kAKP);
  const bool aligned = (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(f) & 15u) == 0);
  if (aligned && g_assign_ver == 3) {
    csc::Scratch lbs;  // carried second minimum between centroid passes
    CSC_TRY_CUDA(lbs.alloc(sizeof(double) * n, st));
    const int rc = launch_assign3(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts, st,
                                  nullptr, nullptr, nullptr, lbs.as<double>(), nullptr);
    if (rc != CSC_OK) return rc;
  } else if (aligned && (int64_t)smem <= (int64_t)csc::device_info().max_smem_optin) {
    const int rc = g_assign_tn == 8
                       ? launch_assign2<8>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts,
                                           smem, st)
                       : launch_assign2<4>(f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts,
                                           smem, st);
    if (rc != CSC_OK) return rc;
  } else {
    assign_kernel<<<(unsigned)csc::ceil_div(n, kBM), kAssignThreads, 0, st>>>(
        f, fnorm, n, d, ld, c, ldc, cnorm, k, labels, own, counts);
  }
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeans_tuning(const char *key, int64_t value) {
  CSC_REQUIRE(key != nullptr, "csc_kmeans_tuning: NULL key");
  if (std::string(key) == "assign_tile") {
    CSC_REQUIRE(value == 0 || value == 1 || value == 44 || value == 88 || value == 84 || value == 87 ||
                    value == 48 || value == 42,
                "assign_tile: 0 (auto), 1 (small-k), 44, 88, 84, 48 or 42");
    g_assign_tile = (int)value;
    return CSC_OK;
  }
  if (std::string(key) == "finish_mode") {
    CSC_REQUIRE(value >= 0 && value <= 2, "finish_mode must be 0, 1 or 2");
    g_finish_mode = (int)value;
    return CSC_OK;
  }
  if (std::string(key) == "assign_ver") {
    CSC_REQUIRE(value == 2 || value == 3, "assign_ver must be 2 or 3");
    g_assign_ver = (int)value;
    return CSC_OK;
  }
  if (std::string(key) == "update_exact") {
    g_update_exact = value ? 1 : 0;
    return CSC_OK;
  }
  if (std::string(key) == "update_incremental") {
    g_update_incremental = value ? 1 : 0;
    return CSC_OK;
  }
  if (std::string(key) == "screen_tc") {
    screen_tc_enabled();
    g_screen_tc = value ? 1 : 0;
    return CSC_OK;
  }
  if (std::string(key) == "kpp_staged") {
    g_kpp_staged = value ? 1 : 0;
    return CSC_OK;
  }
  if (std::string(key) == "assign_tn") {
    CSC_REQUIRE(value == 4 || value == 8, "assign_tn must be 4 or 8");
    g_assign_tn = (int)value;
    return CSC_OK;
  }
  csc::set_error("csc_kmeans_tuning: unknown key '%s'", key);
  return CSC_ERR_ARG;
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
  int64_t cw = (budget - cnt_bytes) / (int64_t)(sizeof(double) * k) - kSqLanes;
  CSC_REQUIRE(cw >= 1, "csc_kmeans_update: k=%lld too large for shared-memory partials",
              (long long)k);
  cw = std::min<int64_t>(std::min<int64_t>(cw, 256), d);
  const int64_t ny = csc::ceil_div(d, cw);
  // rows per block: ~8 resident blocks per SM, at least 64 rows each
  const int64_t nb = std::max<int64_t>(
      1, std::min<int64_t>((int64_t)info.sm_count * 8, csc::ceil_div(n, 64)));
  const int64_t chunk = csc::ceil_div(n, nb);
  const size_t smem = sizeof(double) * k * (cw + kSqLanes) + cnt_bytes;
  CSC_TRY_CUDA(cudaFuncSetAttribute(update_partial_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  csc::Scratch psum, pcnt;
  CSC_TRY_CUDA(psum.alloc(sizeof(double) * nb * k * d, st));
  CSC_TRY_CUDA(pcnt.alloc(sizeof(int32_t) * nb * k, st));
  const int threads = (int)std::max<int64_t>(32, csc::ceil_div(cw, 32) * 32);
  update_partial_kernel<<<dim3((unsigned)nb, (unsigned)ny), threads, smem, st>>>(
      f, labels, n, d, ld, k, chunk, (int)cw, psum.as<double>(), pcnt.as<int32_t>(), nullptr,
      nullptr);
  CSC_CHECK_LAUNCH();
  const int64_t warps = k * (d + 1);
  update_finish_kernel<<<(unsigned)csc::ceil_div(warps, 8), 256, 0, st>>>(
      psum.as<double>(), pcnt.as<int32_t>(), nb, d, k, c, ldc, nullptr, counts);
  CSC_CHECK_LAUNCH();
  centroid_norms_kernel<<<(unsigned)csc::ceil_div(k, 8), 256, 0, st>>>(c, ldc, d, k, cnorm);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int csc_kmeans_plan_create(int64_t n, int64_t d, int64_t ld, int64_t k, void *stream,
                           csc_kmeans_plan **out) {
  csc::clear_error();
  CSC_REQUIRE(out != nullptr, "csc_kmeans_plan_create: NULL out");
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && k >= 1 && n < INT32_MAX && k < INT32_MAX,
              "csc_kmeans_plan_create: bad shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const csc::DeviceInfo &info = csc::device_info();
  csc_kmeans_plan *p = new csc_kmeans_plan();
  p->n = n;
  p->d = d;
  p->ld = ld;
  p->k = k;
  p->stream = st;
  const int64_t budget = std::max<int64_t>(48 * 1024, (int64_t)info.max_smem_optin) - 1024;
  int64_t cw = (budget - (int64_t)sizeof(int32_t) * k) / (int64_t)(sizeof(double) * k) - kSqLanes;
  if (cw < 1) {
    delete p;
    csc::set_error("csc_kmeans_plan_create: k=%lld too large", (long long)k);
    return CSC_ERR_ARG;
  }
  p->cw = std::min<int64_t>(std::min<int64_t>(cw, 256), d);
  p->ny = csc::ceil_div(d, p->cw);
  p->nb = std::max<int64_t>(1, std::min<int64_t>((int64_t)info.sm_count * 8, csc::ceil_div(n, 64)));
  p->chunk = csc::ceil_div(n, p->nb);
  p->smem = sizeof(double) * k * (p->cw + kSqLanes) + sizeof(int32_t) * k;
  const size_t nd = (size_t)n, kk = (size_t)k;
  // exact fixed-point sums need no per-chunk partials
  const bool want_fx = g_update_exact && d <= kFxSumThreads && k <= 256;
  const size_t parts = want_fx ? 0 : (size_t)p->nb * kk;
  const size_t doubles = 3 * nd + parts * d + parts + kk * d + 4 * kk + 8;
  const size_t ints = 2 * nd + 4 + parts;
  if (cudaMallocAsync(&p->base, doubles * 8 + ints * 4 + 64, st) != cudaSuccess) {
    delete p;
    csc::set_error("csc_kmeans_plan_create: allocation failed");
    return CSC_ERR_CUDA;
  }
  double *dp = static_cast<double *>(p->base);
  p->ub = dp; dp += nd;
  p->lb = dp; dp += nd;
  p->own = dp; dp += nd;
  p->psum = dp; dp += parts * d;
  p->pq = dp; dp += parts;
  p->S = dp; dp += kk * d;
  p->Q = dp; dp += kk;
  p->cterm = dp; dp += kk;
  p->delta = dp; dp += kk;
  p->shalf = dp; dp += kk;
  p->scal = dp; dp += 8;
  int32_t *ip = reinterpret_cast<int32_t *>(dp);
  p->cand = ip; ip += nd;
  p->flags = ip; ip += 4;
  p->pcnt = ip; ip += parts;
  p->prev = ip;
  CSC_TRY_CUDA(cudaMemsetAsync(p->flags, 0, sizeof(int32_t) * 4, st));
  CSC_TRY_CUDA(cudaFuncSetAttribute(update_partial_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem));
  if (p->chunk <= kSortedMaxChunk)
    CSC_TRY_CUDA(cudaFuncSetAttribute(
        update_sorted_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
        (int)(sizeof(int32_t) * (2 * (size_t)p->chunk + 3 * (size_t)k))));
  {
    const size_t fsm = sizeof(double) * (size_t)k * ((d | 1) + 3);
    p->finish_small = (int64_t)fsm <= (int64_t)info.max_smem_optin && k * k * d <= (int64_t(1) << 21);
    if (p->finish_small && fsm > 48 * 1024)
      CSC_TRY_CUDA(cudaFuncSetAttribute(finish_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)fsm));
  }
  const size_t fxs = fx_smem(d, k);
  if (want_fx) {
    const size_t kd = kk * (size_t)d;
    const size_t words = 2 * kd + 2 * kk + 1;
    const size_t ents = 2 * nd;
    if (cudaMallocAsync(&p->fx_base, words * 8 + kk * 4 + 64, st) != cudaSuccess ||
        cudaMallocAsync(&p->fxw_base, sizeof(int32_t) * (3 * ents + 3 * kk + 1 + 2), st) != cudaSuccess) {
      if (p->fx_base) cudaFreeAsync(p->fx_base, st);
      cudaFreeAsync(p->base, st);
      delete p;
      csc::set_error("csc_kmeans_plan_create: allocation failed");
      return CSC_ERR_CUDA;
    }
    {
      p->fx = true;
      p->fx_lo = static_cast<unsigned long long *>(p->fx_base);
      p->fx_hi = p->fx_lo + kd;
      p->fx_q = p->fx_hi + kd;
      p->fx_max = p->fx_q + 2 * kk;
      p->fx_cnt = reinterpret_cast<int32_t *>(p->fx_max + 1);
      int32_t *wp = static_cast<int32_t *>(p->fxw_base);
      p->fxw.entries = wp; wp += ents;
      p->fxw.ecl = wp; wp += ents;
      p->fxw.bucketed = wp; wp += ents;
      p->fxw.ccount = wp; wp += kk;
      p->fxw.cursor = wp; wp += kk;
      p->fxw.coff = wp; wp += kk + 1;
      p->fxw.scal = wp;
      CSC_TRY_CUDA(cudaMemsetAsync(p->fxw.ccount, 0, sizeof(int32_t) * kk, st));
      p->fx_grid = grid_cap(csc::ceil_div(n, kFxThreads));
    }
  }
  *out = p;
  return CSC_OK;
}

int csc_kmeans_screen_supported(int64_t d, int64_t k) {
  return csc::screen_supported(d, k) ? 1 : 0;
}

int csc_kmeans_screen_prepare(const double *f, int64_t n, int64_t d, int64_t ld, float *f32,
                              int64_t ld32, float *fn32, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(f && f32 && fn32 && n >= 1 && d >= 1 && ld >= d && ld32 >= d && ld32 % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(f32) & 15u) == 0,
              "csc_kmeans_screen_prepare: bad arguments (ld32 must be a multiple of 4, f32 16-byte aligned)");
  return csc::screen_convert_features(f, n, d, ld, f32, ld32, fn32,
                                      static_cast<cudaStream_t>(stream));
}

int csc_kmeans_plan_set_screen(csc_kmeans_plan *p, const float *f32, int64_t ld32,
                               const float *fn32) {
  csc::clear_error();
  CSC_REQUIRE(p != nullptr, "csc_kmeans_plan_set_screen: NULL plan");
  if (f32 == nullptr) {
    p->f32 = nullptr;
    return CSC_OK;
  }
  CSC_REQUIRE(fn32 != nullptr && ld32 >= p->d && ld32 % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(f32) & 15u) == 0,
              "csc_kmeans_plan_set_screen: bad arguments");
  CSC_REQUIRE(csc::screen_supported(p->d, p->k),
              "csc_kmeans_plan_set_screen: (d=%lld, k=%lld) outside the screen kernel",
              (long long)p->d, (long long)p->k);
  if (!p->screen_base) {
    const int64_t kpad = csc::screen_kpad(p->k);
    const bool tc_ok = csc::tc_screen_supported(p->d, p->k);
    const int64_t tcf = tc_ok ? csc::tc_centroid_floats(p->d, p->k) : 0;
    const int64_t c32 = std::max<int64_t>(p->d * kpad, 2 * tcf);
    const size_t bytes = sizeof(float) * (c32 + std::max<int64_t>(kpad, 256)) + 16 + sizeof(double) +
                         sizeof(int32_t) * (p->n + 4) + 64;
    CSC_TRY_CUDA(cudaMallocAsync(&p->screen_base, bytes, p->stream));
    char *b = static_cast<char *>(p->screen_base);
    p->cmax = reinterpret_cast<double *>(b);
    b += 16;
    p->c32t = reinterpret_cast<float *>(b);
    p->chi = p->c32t;  // the two screens share the centroid scratch
    p->clo = p->c32t + tcf;
    b += sizeof(float) * c32;
    p->cn32 = reinterpret_cast<float *>(b);
    b += sizeof(float) * std::max<int64_t>(kpad, 256);
    p->namb = reinterpret_cast<int32_t *>(b);
    p->amb = p->namb + 4;
  }
  p->tc = screen_tc_enabled() && csc::tc_screen_supported(p->d, p->k);
  p->f32 = f32;
  p->fn32 = fn32;
  p->ld32 = ld32;
  return CSC_OK;
}

int csc_kmeans_plan_stats(const csc_kmeans_plan *p, int64_t *candidates, int32_t *gated) {
  CSC_REQUIRE(p != nullptr, "csc_kmeans_plan_stats: NULL plan");
  int32_t h[4] = {0, 0, 0, 0};
  CSC_TRY_CUDA(cudaMemcpyAsync(h, p->flags, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
  CSC_TRY_CUDA(cudaStreamSynchronize(p->stream));
  if (candidates) *candidates = h[3];
  if (gated) *gated = h[1];
  return CSC_OK;
}

int csc_kmeans_plan_screen_stats(const csc_kmeans_plan *p, int64_t *undecided) {
  CSC_REQUIRE(p != nullptr && undecided != nullptr, "csc_kmeans_plan_screen_stats: NULL argument");
  int32_t h = 0;
  if (p->namb) {
    CSC_TRY_CUDA(cudaMemcpyAsync(&h, p->namb, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
    CSC_TRY_CUDA(cudaStreamSynchronize(p->stream));
  }
  *undecided = h;
  return CSC_OK;
}

int csc_kmeans_plan_destroy(csc_kmeans_plan *p) {
  if (!p) return CSC_OK;
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  if (p->loop) cudaFreeAsync(p->loop, p->stream);
  if (p->cost_parts) cudaFreeAsync(p->cost_parts, p->stream);
  if (p->history) cudaFreeAsync(p->history, p->stream);
  if (p->base) cudaFreeAsync(p->base, p->stream);
  if (p->screen_base) cudaFreeAsync(p->screen_base, p->stream);
  if (p->fx_base) cudaFreeAsync(p->fx_base, p->stream);
  if (p->fxw_base) cudaFreeAsync(p->fxw_base, p->stream);
  delete p;
  return CSC_OK;
}

int csc_kmeans_iterate(csc_kmeans_plan *p, const double *f, const double *fnorm, double *cent,
                       int64_t ldc, double *cnorm, int32_t *labels, int32_t *counts, int full,
                       double *cost2_dev, void *stream) {
  CSC_REQUIRE(p != nullptr, "csc_kmeans_iterate: NULL plan");
  CSC_REQUIRE(ldc >= p->d, "csc_kmeans_iterate: ldc < d");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  p->stream = st;
  const int64_t n = p->n, d = p->d, ld = p->ld, k = p->k;
  const int64_t dpad = csc::ceil_div(d, kAK) * kAK;
  const size_t asmem = sizeof(double) * (dpad * kANP + 2 * kAM * kAKP);
  CSC_REQUIRE((ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(f) & 15u) == 0),
              "csc_kmeans_iterate: features must be 16-byte aligned with an even row stride");
  const bool v2_fits = (int64_t)asmem <= (int64_t)csc::device_info().max_smem_optin;
  auto assign = [&](const int32_t *rows, const int32_t *nrows, int32_t *cnts, const int32_t *gate) {
    if (g_assign_ver == 3 || !v2_fits)
      return launch_assign3(f, fnorm, n, d, ld, cent, ldc, cnorm, k, labels, p->own, cnts, st,
                            rows, nrows, p->ub, p->lb, gate);
    return g_assign_tn == 8
               ? launch_assign2<8>(f, fnorm, n, d, ld, cent, ldc, cnorm, k, labels, p->own, cnts,
                                   asmem, st, rows, nrows, p->ub, p->lb, gate)
               : launch_assign2<4>(f, fnorm, n, d, ld, cent, ldc, cnorm, k, labels, p->own, cnts,
                                   asmem, st, rows, nrows, p->ub, p->lb, gate);
  };
  // the single-block finish converts the new centroids for the tensor-core screen
  const bool tc_fused = p->f32 && p->tc && p->finish_small && g_finish_mode != 2;
  // FP32 screen first when enabled: provably decided rows there, the rest
  // (listed in p->amb) by the FP64 assignment — the same labels either way
  auto screened = [&](const int32_t *rows, const int32_t *nrows, int32_t *cnts) -> int {
    if (!p->f32) return assign(rows, nrows, cnts, nullptr);
    CSC_TRY_CUDA(cudaMemsetAsync(p->namb, 0, sizeof(int32_t), st));
    int r2;
    if (p->tc) {
      if (full || !tc_fused) {  // else the previous iteration's finish wrote the tiles
        r2 = csc::tc_convert_centroids(cent, k, d, ldc, cnorm, p->chi, p->clo, p->cn32, p->cmax, st);
        if (r2 != CSC_OK) return r2;
      }
      r2 = csc::tc_screen_assign(p->f32, p->ld32, p->fn32, n, d, p->chi, p->clo, p->cn32, k,
                                 p->cmax, rows, nrows, labels, p->ub, p->lb, cnts, p->amb, p->namb,
                                 nullptr, st);
    } else {
      r2 = csc::screen_convert_centroids(cent, k, d, ldc, cnorm, p->c32t, p->cn32, p->cmax, st);
      if (r2 != CSC_OK) return r2;
      r2 = csc::screen_assign(p->f32, p->ld32, p->fn32, fnorm, n, d, p->c32t, p->cn32, k, p->cmax,
                              rows, nrows, labels, p->ub, p->lb, cnts, p->amb, p->namb, st);
    }
    if (r2 != CSC_OK) return r2;
    // the undecided rows are few (~0.5% at cfg5): the warp-per-4-rows kernel
    // (same per-pair arithmetic and ties, same labels) has no tile pipeline to fill
    if (k <= 64 && d <= 128 && g_assign_tile == 0) {
      return k <= 32 ? launch_assign_small<1>(f, fnorm, n, d, ld, cent, ldc, cnorm, k, labels, p->own,
                                              cnts, st, p->amb, p->namb, p->ub, p->lb, nullptr)
                     : launch_assign_small<2>(f, fnorm, n, d, ld, cent, ldc, cnorm, k, labels, p->own,
                                              cnts, st, p->amb, p->namb, p->ub, p->lb, nullptr);
    }
    return assign(p->amb, p->namb, cnts, nullptr);
  };
  int rc;
  if (full) {
    CSC_TRY_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * k, st));
    CSC_TRY_CUDA(cudaMemsetAsync(p->flags, 0, sizeof(int32_t) * 4, st));
    if ((rc = screened(nullptr, nullptr, counts)) != CSC_OK) return rc;
  } else {
    // flags[0] (candidate count) was cleared by the previous iteration's finish
    bound_kernel<<<grid_cap(csc::ceil_div(n, (int64_t)kBoundThreads * kBoundRows)), kBoundThreads, 0,
                   st>>>(
        n, labels, p->ub, p->lb, p->delta, p->scal, p->shalf, fnorm, p->cand, p->flags, counts, k);
    CSC_CHECK_LAUNCH();
    if ((rc = screened(p->cand, p->flags, nullptr)) != CSC_OK) return rc;
    label_hist_kernel<<<grid_cap(csc::ceil_div(n, 256), 4), 256, sizeof(int32_t) * k, st>>>(
        n, k, labels, counts);
    CSC_CHECK_LAUNCH();
  }
  CSC_CHECK_LAUNCH();
  // empty cluster: full GEMM-form reassignment (own distances for every row), then the repair
  check_empty_kernel<<<1, 1024, 0, st>>>(k, counts, p->flags);
  CSC_CHECK_LAUNCH();
  if ((rc = assign(nullptr, nullptr, counts, p->flags + 1)) != CSC_OK) return rc;
  CSC_CHECK_LAUNCH();
  gated_repair_kernel<<<1, 1024, 0, st>>>(labels, p->own, counts, n, k, p->flags);
  CSC_CHECK_LAUNCH();
  // means, counts, movement, cost terms
  const int threads = (int)(csc::ceil_div(p->cw, 32) * 32 + 32);
  if (p->fx) {
    if (full) {  // a new run: no members anywhere yet; the fixed-point scale from max |f|^2
      CSC_TRY_CUDA(cudaMemsetAsync(p->prev, 0xff, sizeof(int32_t) * n, st));
      CSC_TRY_CUDA(cudaMemsetAsync(p->fx_base, 0, sizeof(unsigned long long) * (2 * k * d + 2 * k + 1) +
                                                      sizeof(int32_t) * k, st));
      fx_maxnorm_kernel<<<grid_cap(csc::ceil_div(n, 256), 2), 256, 0, st>>>(fnorm, n, p->fx_max);
      CSC_CHECK_LAUNCH();
    }
    CSC_TRY_CUDA(cudaMemsetAsync(p->fxw.scal, 0, sizeof(int32_t), st));
    fx_changes_kernel<<<(unsigned)p->fx_grid, kFxThreads, fx_smem(d, k), st>>>(labels, p->prev, n, (int)k,
                                                                             p->fxw, p->fx_cnt);
    CSC_CHECK_LAUNCH();
    const int sum_grid = csc::device_info().sm_count * 2;
    fx_offsets_kernel<<<1, 32, 0, st>>>((int)k, p->fxw, 2 * sum_grid);  // k <= 256
    CSC_CHECK_LAUNCH();
    fx_scatter_kernel<<<(unsigned)(csc::device_info().sm_count * 4), kFxThreads, sizeof(int32_t) * 2 * k, st>>>(
        p->fxw, (int)k);
    CSC_CHECK_LAUNCH();
    fx_sum_kernel<<<(unsigned)sum_grid, kFxSumThreads * kFxRowGroups, 0, st>>>(
        f, ld, fnorm, n, (int)d, (int)k, p->fx_max, p->fxw, p->fx_lo, p->fx_hi, p->fx_q);
    CSC_CHECK_LAUNCH();
    fx_finish_kernel<<<(unsigned)csc::ceil_div(k * d, 256), 256, 0, st>>>(
        p->fx_lo, p->fx_hi, p->fx_q, p->fx_cnt, n, (int)d, (int)k, p->fx_max, p->S, p->Q, counts);
    CSC_CHECK_LAUNCH();
  } else if (p->chunk <= kSortedMaxChunk) {
    const size_t ssmem = sizeof(int32_t) * (2 * (size_t)p->chunk + 3 * (size_t)k);
    int32_t *prev = (p->ny == 1 && g_update_incremental) ? p->prev : nullptr;
    if (prev && full) {  // a new run: no members anywhere yet
      CSC_TRY_CUDA(cudaMemsetAsync(prev, 0xff, sizeof(int32_t) * n, st));
      CSC_TRY_CUDA(cudaMemsetAsync(p->psum, 0, sizeof(double) * p->nb * k * d, st));
      CSC_TRY_CUDA(cudaMemsetAsync(p->pq, 0, sizeof(double) * p->nb * k, st));
    }
    update_sorted_kernel<<<dim3((unsigned)p->nb, (unsigned)p->ny), threads, ssmem, st>>>(
        f, labels, n, d, ld, k, p->chunk, (int)p->cw, p->psum, p->pcnt, fnorm, p->pq, prev);
  } else {
    update_partial_kernel<<<dim3((unsigned)p->nb, (unsigned)p->ny), threads, p->smem, st>>>(
        f, labels, n, d, ld, k, p->chunk, (int)p->cw, p->psum, p->pcnt, fnorm, p->pq);
  }
  CSC_CHECK_LAUNCH();
  if (!p->fx) {
    const int64_t warps = k * (d + 1);
    sums_finish_kernel<<<(unsigned)csc::ceil_div(warps, 8), 256, 0, st>>>(
        p->psum, p->pcnt, p->pq, p->nb, d, k, p->S, counts, p->Q);
    CSC_CHECK_LAUNCH();
  }
  if (g_finish_mode != 2 && p->finish_small) {
    // small k: one single-block node finishes the iteration
    finish_small_kernel<<<1, g_finish_mode == 1 ? 256 : 1024, sizeof(double) * k * ((d | 1) + 3),
                          st>>>(d, k, p->S, counts, p->Q, cent, ldc, cnorm,
                                            p->delta, p->cterm, p->scal, p->shalf, p->flags,
                                            tc_fused ? p->chi : nullptr, p->clo, p->cn32, p->cmax,
                                            csc::tc_npad_of(k), csc::tc_kp_of(d));
    CSC_CHECK_LAUNCH();
  } else {
    centroid_finish_kernel<<<(unsigned)k, 128, 0, st>>>(p->S, counts, p->Q, d, k, cent, ldc,
                                                        cnorm, p->delta, p->cterm);
    CSC_CHECK_LAUNCH();
    iter_finish_kernel<<<1, 32, 0, st>>>(k, p->cterm, p->delta, cnorm, p->scal, p->flags);
    CSC_CHECK_LAUNCH();
    shalf_kernel<<<(unsigned)k, 128, 0, st>>>(cent, ldc, d, k, p->shalf);
    CSC_CHECK_LAUNCH();
  }
  if (cost2_dev)
    CSC_TRY_CUDA(cudaMemcpyAsync(cost2_dev, p->scal, sizeof(double), cudaMemcpyDeviceToDevice, st));
  return CSC_OK;
}

int csc_kmeans_run(csc_kmeans_plan *p, const double *f, const double *fnorm, double *cent,
                   int64_t ldc, double *cnorm, int32_t *labels, int32_t *counts, int max_iters,
                   double tol, double *out_dev, double *history_dev, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(p != nullptr, "csc_kmeans_run: NULL plan");
  CSC_REQUIRE(out_dev != nullptr, "csc_kmeans_run: NULL out_dev");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!p->loop) CSC_TRY_CUDA(cudaMallocAsync((void **)&p->loop, sizeof(LoopState), st));
  const int cost_grid = grid_cap(csc::ceil_div(p->n, 8));
  if (!p->cost_parts)
    CSC_TRY_CUDA(cudaMallocAsync((void **)&p->cost_parts, sizeof(double) * cost_grid, st));
  const int cap = std::max(1, max_iters);
  if (cap > p->hist_cap) {
    if (p->history) CSC_TRY_CUDA(cudaFreeAsync(p->history, st));
    CSC_TRY_CUDA(cudaMallocAsync((void **)&p->history, sizeof(double) * cap, st));
    p->hist_cap = cap;
    if (p->exec) {  // history pointer is baked into the graph
      cudaGraphExecDestroy(p->exec);
      cudaGraphDestroy(p->graph);
      p->exec = nullptr;
      p->graph = nullptr;
    }
  }
  // The whole call is one graph per buffer set (one launch per restart lane):
  // [init, |c|^2 of the seeds, full iteration 1, stop check] -> while(pruned
  // iteration + stop check) -> [exact cost, iteration count, history copy].
  double tol_key = tol;
  int64_t tol_bits = 0;
  memcpy(&tol_bits, &tol_key, sizeof(tol_bits));
  const void *key[12] = {f, fnorm, cent, cnorm, labels, counts, (const void *)(intptr_t)ldc,
                         out_dev, history_dev, (const void *)(intptr_t)max_iters,
                         (const void *)(intptr_t)tol_bits, p->f32};
  bool same = p->exec != nullptr;
  for (int i = 0; i < 12 && same; ++i) same = key[i] == p->key[i];
  if (!same) {
    if (p->exec) {
      cudaGraphExecDestroy(p->exec);
      cudaGraphDestroy(p->graph);
      p->exec = nullptr;
      p->graph = nullptr;
    }
    cudaGraph_t g;
    CSC_TRY_CUDA(cudaGraphCreate(&g, 0));
    cudaStream_t cap_st;
    CSC_TRY_CUDA(cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking));
    int rc = CSC_OK;
    cudaError_t ec = cudaSuccess;
    std::vector<cudaGraphNode_t> tail;
    auto end_capture = [&]() {
      const cudaGraphNode_t *deps = nullptr;
      size_t ndeps = 0;
      cudaStreamCaptureStatus status;
      cudaError_t e = cudaStreamGetCaptureInfo(cap_st, &status, nullptr, nullptr, &deps, &ndeps);
      if (e == cudaSuccess) tail.assign(deps, deps + ndeps);
      cudaGraph_t captured;
      const cudaError_t e2 = cudaStreamEndCapture(cap_st, &captured);
      return e != cudaSuccess ? e : e2;
    };
    // prefix
    ec = cudaStreamBeginCaptureToGraph(cap_st, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (ec == cudaSuccess) {
      loop_init_kernel<<<1, 1, 0, cap_st>>>(p->loop, tol, max_iters);
      centroid_norms_kernel<<<(unsigned)csc::ceil_div(p->k, 8), 256, 0, cap_st>>>(cent, ldc, p->d,
                                                                                 p->k, cnorm);
      if (max_iters >= 1) {
        rc = csc_kmeans_iterate(p, f, fnorm, cent, ldc, cnorm, labels, counts, 1, nullptr, cap_st);
        loop_check_kernel<<<1, 1, 0, cap_st>>>(p->scal, p->loop, p->history, p->hist_cap, 0, 0);
      }
      ec = end_capture();
    }
    // while (stop check says go): pruned iteration + stop check
    if (ec == cudaSuccess && rc == CSC_OK && max_iters >= 2) {
      cudaGraphConditionalHandle h;
      ec = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      if (ec == cudaSuccess) ec = cudaGraphAddNode(&node, g, tail.data(), tail.size(), &cp);
      if (ec == cudaSuccess) {
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        ec = cudaStreamBeginCaptureToGraph(cap_st, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed);
        if (ec == cudaSuccess) {
          rc = csc_kmeans_iterate(p, f, fnorm, cent, ldc, cnorm, labels, counts, 0, nullptr, cap_st);
          loop_check_kernel<<<1, 1, 0, cap_st>>>(p->scal, p->loop, p->history, p->hist_cap, h, 1);
          cudaGraph_t captured;
          ec = cudaStreamEndCapture(cap_st, &captured);
        }
        tail.assign(1, node);
      }
    }
    // suffix: out_dev[0] = cost2 of the last iteration in the exact difference
    // form (kmeans.py:111), out_dev[1] = iterations run (as double)
    if (ec == cudaSuccess && rc == CSC_OK) {
      ec = cudaStreamBeginCaptureToGraph(cap_st, g, tail.data(), nullptr, tail.size(),
                                         cudaStreamCaptureModeRelaxed);
      if (ec == cudaSuccess) {
        if (max_iters >= 1) {
          cost_kernel<<<cost_grid, 256, 0, cap_st>>>(f, labels, cent, ldc, p->n, p->d, p->ld,
                                                      p->cost_parts);
          reduce_partials_kernel<<<1, 1024, 0, cap_st>>>(p->cost_parts, cost_grid, out_dev);
        }
        if (history_dev)
          cudaMemcpyAsync(history_dev, p->history, sizeof(double) * cap, cudaMemcpyDeviceToDevice,
                          cap_st);
        copy_iters_kernel<<<1, 1, 0, cap_st>>>(p->loop, out_dev + 1, max_iters >= 1);
        cudaGraph_t captured;
        ec = cudaStreamEndCapture(cap_st, &captured);
      }
    }
    cudaStreamDestroy(cap_st);
    p->stream = st;
    if (rc != CSC_OK) {
      cudaGraphDestroy(g);
      return rc;
    }
    if (ec != cudaSuccess) {
      cudaGraphDestroy(g);
      CSC_TRY_CUDA(ec);
    }
    CSC_TRY_CUDA(cudaGraphInstantiate(&p->exec, g, 0));
    p->graph = g;
    for (int i = 0; i < 12; ++i) p->key[i] = key[i];
  }
  CSC_TRY_CUDA(cudaGraphLaunch(p->exec, st));
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

int csc_kmeanspp_batch(const double *f, int64_t n, int64_t d, int64_t ld, int64_t R, int64_t k,
                       const int64_t *first_idx_host, const double *uniforms_host, double *cent,
                       int64_t ldc, int32_t *flags_dev, void *stream) {
  CSC_REQUIRE(n >= 1 && d >= 1 && ld >= d && ldc >= d && k >= 1, "csc_kmeanspp_batch: bad shape");
  CSC_REQUIRE(R >= 1 && R <= 16, "csc_kmeanspp_batch: 1 <= R <= 16 restarts per batch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // contiguous row chunks (<= 1024: the draw scans them in one block), ~>= 32 rows each
  const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(1024, csc::ceil_div(n, 32)));
  const int64_t chunk = csc::ceil_div(n, nchunks);
  const int64_t cent_stride = k * ldc;
  csc::Scratch closest, sums, fidx, unif;
  CSC_TRY_CUDA(closest.alloc(sizeof(double) * R * n, st));
  CSC_TRY_CUDA(sums.alloc(sizeof(double) * R * nchunks, st));
  CSC_TRY_CUDA(fidx.alloc(sizeof(int64_t) * R, st));
  CSC_TRY_CUDA(unif.alloc(sizeof(double) * std::max<int64_t>(1, R * (k - 1)), st));
  CSC_TRY_CUDA(cudaMemcpyAsync(fidx.ptr, first_idx_host, sizeof(int64_t) * R,
                               cudaMemcpyHostToDevice, st));
  if (k > 1)
    CSC_TRY_CUDA(cudaMemcpyAsync(unif.ptr, uniforms_host, sizeof(double) * R * (k - 1),
                                 cudaMemcpyHostToDevice, st));
  CSC_TRY_CUDA(cudaMemsetAsync(flags_dev, 0xff, sizeof(int32_t) * R, st));
  kppb_first_kernel<<<(unsigned)R, 128, 0, st>>>(f, d, ld, fidx.as<int64_t>(), cent, cent_stride);
  CSC_CHECK_LAUNCH();
  const size_t smem = sizeof(double) * (R * d + 4 * R);
  CSC_REQUIRE((int64_t)smem <= (int64_t)csc::device_info().max_smem_optin,
              "csc_kmeanspp_batch: R*d too large for shared memory (R=%lld, d=%lld)",
              (long long)R, (long long)d);
  // staged distance pass: 16-byte-aligned rows, chunks long enough to fill tiles
  const size_t smem_staged = (((size_t)((d + 1) / 2) * R * 16 + (size_t)4 * R * 8 + 127) / 128) * 128 +
                             (size_t)2 * kKsRows * 128;
  if (g_kpp_staged < 0) {
    const char *e = getenv("CSC_KPP_STAGED");
    g_kpp_staged = (e && e[0] == '0') ? 0 : 1;
  }
  const bool staged = g_kpp_staged && (reinterpret_cast<uintptr_t>(f) % 16 == 0) && ld % 2 == 0 &&
                      chunk >= kKsRows && (int64_t)smem_staged <= (int64_t)csc::device_info().max_smem_optin;
  for (int64_t j = 0; j < k; ++j) {
    if (j > 0) {
      kppb_pick_kernel<<<(unsigned)R, 1024, 0, st>>>(f, n, d, ld, closest.as<double>(),
                                                     sums.as<double>(), nchunks, chunk,
                                                     unif.as<double>(), k - 1, (int)j, cent,
                                                     cent_stride, ldc, flags_dev);
      CSC_CHECK_LAUNCH();
    }
    if (j < k - 1) {
      if (staged) {
        switch (R) {
#define CSC_KPPS_CASE(RR)                                                                      \
  case RR:                                                                                     \
    CSC_TRY_CUDA(cudaFuncSetAttribute(kppb_dist_staged_kernel<RR>,                             \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                      (int)smem_staged));                                      \
    kppb_dist_staged_kernel<RR><<<(unsigned)nchunks, 128, smem_staged, st>>>(                  \
        f, n, d, ld, cent + j * ldc, cent_stride, closest.as<double>(), j == 0 ? 1 : 0, chunk, \
        sums.as<double>(), nchunks);                                                           \
    break;
          CSC_KPPS_CASE(1) CSC_KPPS_CASE(2) CSC_KPPS_CASE(3) CSC_KPPS_CASE(4)
          CSC_KPPS_CASE(5) CSC_KPPS_CASE(6) CSC_KPPS_CASE(7) CSC_KPPS_CASE(8)
          CSC_KPPS_CASE(9) CSC_KPPS_CASE(10) CSC_KPPS_CASE(11) CSC_KPPS_CASE(12)
          CSC_KPPS_CASE(13) CSC_KPPS_CASE(14) CSC_KPPS_CASE(15) CSC_KPPS_CASE(16)
#undef CSC_KPPS_CASE
          default:
            csc::set_error("csc_kmeanspp_batch: R=%lld out of range", (long long)R);
            return CSC_ERR_ARG;
        }
        CSC_CHECK_LAUNCH();
        continue;
      }
      switch (R) {
#define CSC_KPPB_CASE(RR)                                                                      \
  case RR:                                                                                     \
    if (smem > 48 * 1024)                                                                      \
      CSC_TRY_CUDA(cudaFuncSetAttribute(kppb_dist_kernel<RR>,                                  \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kppb_dist_kernel<RR><<<(unsigned)nchunks, 128, smem, st>>>(                                \
        f, n, d, ld, cent + j * ldc, cent_stride, closest.as<double>(), j == 0 ? 1 : 0, chunk, \
        sums.as<double>(), nchunks);                                                           \
    break;
        CSC_KPPB_CASE(1) CSC_KPPB_CASE(2) CSC_KPPB_CASE(3) CSC_KPPB_CASE(4)
        CSC_KPPB_CASE(5) CSC_KPPB_CASE(6) CSC_KPPB_CASE(7) CSC_KPPB_CASE(8)
        CSC_KPPB_CASE(9) CSC_KPPB_CASE(10) CSC_KPPB_CASE(11) CSC_KPPB_CASE(12)
        CSC_KPPB_CASE(13) CSC_KPPB_CASE(14) CSC_KPPB_CASE(15) CSC_KPPB_CASE(16)
#undef CSC_KPPB_CASE
        default:
          csc::set_error("csc_kmeanspp_batch: R=%lld out of range", (long long)R);
          return CSC_ERR_ARG;
      }
      CSC_CHECK_LAUNCH();
    }
  }
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
