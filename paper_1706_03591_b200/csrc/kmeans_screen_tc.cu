// Tensor-core (tcgen05, kind::tf32) screen of the k-means assignment
// (kmeans.py:54-61, 96-97), with the exact FP64 fallback of kmeans_screen.cu:
// labels stay bit-identical to the pure FP64 path.
//
// The inner products f.c_j of a 128-row tile against all centroids are one
// UMMA D[128 x N] (fp32 accumulators in tensor memory) per 8-column K step,
// in the 3xTF32 split: with f = f_hi + f_lo and c = c_hi + c_lo (hi = the
// fp32 value with its 13 low mantissa bits cleared, exactly a tf32; lo = the
// exact fp32 remainder, rounded to tf32 by the tensor core),
//     f.c ~ f_hi.c_hi + f_lo.c_hi + f_hi.c_lo,
// three MMAs per K step accumulating in the same TMEM columns. Error bound
// (per row, all j), conservative for an accumulator that truncates:
//   split:  |f.c - (three products)| <= (2^-20 + 2 * 2^-21) |f| |c|
//   sum:    3d products of tf32 operands are exact in fp32; each of the 3d
//           accumulations loses < 2^-23 of the running |sum| <= sum |f_t c_t|
//   norms / inputs: as the FP32 screen ((d + 5) 2^-24 (|f| + |c|)^2)
// so |E_ij - T_ij| <= delta_i = (3d + 8) 2^-23 (|f_i| + max_j |c_j|)^2, and a
// row whose best/second gap exceeds 2 delta_i is decided exactly as in the
// FP32 screen (same Hamerly widening); the others go to the FP64 list.
//
// Layout. Operands are K-major, no swizzle: element (r, c) of a ROWS x K tile
// sits at byte (c / 4) * ROWS * 16 + r * 16 + (c % 4) * 4 (16-byte K chunks,
// the ROWS rows of a chunk contiguous), i.e. core matrices of 8 rows x 16 B
// at SBO = 128 B along rows and LBO = ROWS * 16 B along K; one MMA (K = 8)
// reads chunks 2s, 2s+1.
//
// Pipeline (warp-specialised, persistent, one CTA per SM): two producer warps
// gather the candidate rows' fp32 features by index with cp.async into a raw
// ring of shared-memory units (a unit = 128 rows x 32 columns; each producer
// warp copies 64 of the rows); two splitter warps write the units' low parts
// into a two-unit lo ring; one elected thread issues the 3 x 4 MMAs of a unit
// (high parts read straight from the raw unit) into one of two TMEM
// accumulators and commits them to both rings' "empty" mbarriers (and, after
// a tile's last unit, to the accumulator's "full" one); four epilogue warps
// read their 32 TMEM lanes (rows) with tcgen05.ld, settle the rows and
// release the accumulator. Every role walks the units in order, so each
// mbarrier wait is at most one phase ahead of the barrier (a parity wait
// cannot tell phase p from phase p + 2).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "kmeans_screen.cuh"

namespace {

constexpr int kTM = 128;       // rows per tile = UMMA M


__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0, SWIZZLE_NONE
  return d;
}

// K-major, 128-byte swizzle (rows of 128 B = 32 fp32 in 1024-byte atoms of 8
// rows, the 16-byte chunk index XORed with the row within the atom: the
// layout TMA writes with CU_TENSOR_MAP_SWIZZLE_128B); SBO = 1024 B between
// 8-row groups, LBO unused; a K step of 8 tf32 advances the start by 32 B
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                  // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO
  d |= (uint64_t)1 << 46;                  // version 1 (sm_100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_tile2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                           uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *map, int c0, int r0,
                                            int r1, int r2, int r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

// kind::tf32 instruction descriptor: D fp32, A/B tf32, both K-major, M = 128
__host__ __device__ constexpr uint32_t tf32_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// issued by the whole warp with warp-uniform operands; one elected lane (the
// same one every time: elect.sync picks the lowest active lane) executes it
__device__ __forceinline__ void mma_tf32_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 16 : 0));
}

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// centroids -> hi / lo K-major canonical tiles [Q][N][4] (zero past k / d),
// cn (+inf past k), cmax = max_j |c_j| (from the fp64 norms)
__global__ void tc_centroids_kernel(const double *__restrict__ c, int64_t k, int64_t d,
                                    int64_t ldc, const double *__restrict__ cnorm, int n_pad,
                                    int kp, float *__restrict__ chi, float *__restrict__ clo,
                                    float *__restrict__ cn32, double *__restrict__ cmax) {
  __shared__ double red[32];
  for (int64_t j = threadIdx.x / 32; j < n_pad; j += blockDim.x / 32)  // warp per centroid
    for (int64_t t = threadIdx.x % 32; t < kp; t += 32) {
      const float v = (j < k && t < d) ? (float)c[j * ldc + t] : 0.0f;
      const float h = tf32_hi(v);
      const int64_t off = (t / 4) * (int64_t)n_pad * 4 + j * 4 + (t % 4);
      chi[off] = h;
      clo[off] = v - h;
    }
  double m = 0.0;
  for (int j = threadIdx.x; j < n_pad; j += blockDim.x) {
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

struct TcArgs {
  const float *f32;  // fp32 features (ld32, zero padding); split into hi / lo per unit
  int64_t ld32;
  const float *fn32;
  int64_t n;
  int d, kp, k, n_pad;
  const float *chi, *clo, *cn32;
  const double *cmax;
  const int32_t *rows;
  const int32_t *nrows;
  int32_t *labels;
  double *ub, *lb;
  int32_t *counts;
  int32_t *amb, *namb;
  float *raw_out;  // test hook: E (n x n_pad fp32) instead of the decision
};

// Warp roles: 0-3 epilogue (warp w reads TMEM lanes 32w..32w+31 = tile rows),
// 4 MMA issue (one elected lane), 5-6 row producers (warp 5 + h copies rows
// 64h..64h+63 of every unit: cp.async gathers of the candidate rows' fp32
// features into the "raw" ring, from 16 row pointers per lane formed once per
// tile, the next tile's row ids prefetched; never blocking on their own copies: each unit's
// completion arrives on its raw "full" mbarrier via
// cp.async.mbarrier.arrive.noinc), 7-8 splitters (each writes half of every
// unit's low parts lo = f - tf32(f) into the small "lo" ring, fences to the
// async proxy and arrives on its "full" barrier). A unit = 128 rows x kKU
// columns of one tile. The tensor core reads a raw unit directly as the high
// parts: kind::tf32 takes the top 19 bits of each fp32 operand (truncation),
// exactly tf32_hi(f) — so a raw slot is never rewritten and is free again as
// soon as its MMAs ran, and the raw ring (as deep as shared memory allows: 9
// units at cfg5) carries the gathers in flight. Two TMEM accumulators
// (2 x NP columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
constexpr int kKU = 32;                // columns per unit (4 MMA K steps)
constexpr int kMaxRaw = 12;            // raw ring units (as many as fit, >= 2)
#ifndef TC_LO_STAGES
#define TC_LO_STAGES 2
#endif
constexpr int kLoStages = TC_LO_STAGES;  // lo ring units
constexpr int kEpiWarps = 4, kMmaWarp = 4, kProdWarp0 = 5, kProdWarps = 2, kSplitWarp0 = 7,
              kSplitWarps = 4;
// Warps issue on sub-partition warp % 4. With 11 consecutive warps the MMA warp
// (4) shares sub-partition 0 with an epilogue warp (0) and a splitter (8): ~2,000
// warp instructions per tile there, the kernel's critical path. TC_IDLE_WARP
// leaves warp 8 idle and moves its splitter to warp 11, so sub-partition 0
// carries the MMA and one epilogue warp only.
#ifndef TC_IDLE_WARP
#define TC_IDLE_WARP 1
#endif
// TC_EPI_SETS = 2 (A/B knob, off): a second set of four epilogue warps (12-15;
// warp % 4 selects the TMEM lane quarter) settles the odd tiles (accumulator 1)
// while warps 0-3 settle the even ones. Measured on cfg5 features (60 host-
// driven iterations, us per screen launch, full / late): one set 228 / 126, two
// sets 228 / 126; lo ring of 3 or 4 units instead of 2: 229 / 124; the idle warp
// above: 228 vs 233 without. None of the consumer roles is the limit: the MMA
// warp itself is (36 UTCHMMA per tile, each behind an ELECT and ~6 R2UR
// broadcasts of its descriptors: ~950 dependent warp instructions per tile).
// TC_CAT = 1: the centroid tiles' high and low parts form one N = 2 NP operand
// per K quad ([Q][2 NP][4]: rows 0..NP-1 high, NP..2NP-1 low), so a K step is
// two MMAs — A_hi x [B_hi | B_lo] (N = 2 NP) and A_lo x B_hi (N = NP, the first
// rows of the same tiles) — instead of three: A_hi is read from shared memory
// once per K step instead of twice (14 instead of 18 KB per K step). The
// accumulator holds f_hi.c_hi + f_lo.c_hi in columns 0..NP-1 and f_hi.c_lo in
// NP..2NP-1; the epilogue adds them (one more fp32 rounding: inside the bound's
// +8 slack).
#ifndef TC_CAT
#define TC_CAT 1
#endif
constexpr int kAccW = TC_CAT ? 2 : 1;  // accumulator columns per centroid
// TC_MMA_WARPS = 2 (A/B knob, off; needs TC_IDLE_WARP): the idle warp issues the
// odd tiles' MMAs. Correct (tests pass) and no faster (227 / 127 us, also with a
// lo ring of 4 or 6 units): the MMA warp is not the limit either. The final ncu
// capture shows no unit above half of its peak (DRAM 42%, tensor-core shared-
// memory wavefronts 46%, LSU 37%): the splitters wait on the raw units' arrival
// (profiles/r02_tc_screen_cfg5.md).
#ifndef TC_MMA_WARPS
#define TC_MMA_WARPS 1
#endif
#ifndef TC_EPI_SETS
#define TC_EPI_SETS 1
#endif
constexpr int kEpi2Warp0 = kEpiWarps + 1 + kProdWarps + kSplitWarps + (TC_IDLE_WARP ? 1 : 0);  // 12
static_assert(TC_EPI_SETS == 1 || kEpi2Warp0 % 4 == 0, "second epilogue set must start a warp quad");
constexpr int kTcThreads = 32 * (kEpi2Warp0 + (TC_EPI_SETS == 2 ? kEpiWarps : 0));  // 512
constexpr uint32_t kUnitBytes = kTM * kKU * 4;

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
               : "memory");
}

// NP: padded centroid count = UMMA N (multiple of 16, <= 128); RAW: the test
// hook (E to raw_out instead of decisions) — a separate instantiation, so the
// production epilogue carries no per-element store code
template <int NP, bool RAW>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_screen_kernel(TcArgs a, int stages, const __grid_constant__ CUtensorMap tile_map,
                     const __grid_constant__ CUtensorMap row_map) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  const int kp = a.kp;
  const int units = kp / kKU;  // per tile
  uint8_t *raw = tsm;                                          // [stages][kUnitBytes]
  uint8_t *lor = raw + (size_t)stages * kUnitBytes;            // [kLoStages][kUnitBytes]
  float *Bhi = reinterpret_cast<float *>(lor + (size_t)kLoStages * kUnitBytes);
  float *Blo = Bhi + (size_t)NP * kp;
  float *Cn = Blo + (size_t)NP * kp;
  int32_t *Hs = reinterpret_cast<int32_t *>(Cn + NP);
  int32_t *Rs = Hs + NP;                                  // [kTM] row ids (half per producer)
  uint64_t *rfull = reinterpret_cast<uint64_t *>(Rs + kTM);  // 8-byte aligned
  uint64_t *rempty = rfull + kMaxRaw;
  uint64_t *lfull = rempty + kMaxRaw;
  uint64_t *lempty = lfull + kLoStages;
  uint64_t *tfull = lempty + kLoStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_hold = reinterpret_cast<uint32_t *>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nr = a.nrows ? (int64_t)*a.nrows : a.n;
  const int64_t ntiles = (nr + kTM - 1) / kTM;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  constexpr int kAccCols = 2 * kAccW * NP;  // two accumulators
  constexpr uint32_t kCols = kAccCols <= 32 ? 32 : kAccCols <= 64 ? 64 : kAccCols <= 128 ? 128 : kAccCols <= 256 ? 256 : 512;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_hold)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < stages; ++s) {
      // TMA: the producer's expect_tx (the bytes complete it); gathers: the
      // cp.async arrivals (noinc) of every producer lane
      mbar_init(smem_u32(rfull + s), a.rows ? 32 * kProdWarps : 1);
      mbar_init(smem_u32(rempty + s), 1);               // MMA commit
    }
    for (int s = 0; s < kLoStages; ++s) {
      mbar_init(smem_u32(lfull + s), 32 * kSplitWarps);  // both splitters
      mbar_init(smem_u32(lempty + s), TC_MMA_WARPS);     // MMA commit (+ the other MMA warp's pass)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(tfull + s), 1);          // MMA commit
      mbar_init(smem_u32(tempty + s), kEpiWarps);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {  // centroid tiles (already in the canonical layout) and norms
    const float4 *sh = reinterpret_cast<const float4 *>(a.chi);
    const float4 *sl = reinterpret_cast<const float4 *>(a.clo);
    float4 *dh = reinterpret_cast<float4 *>(Bhi);
    float4 *dl = reinterpret_cast<float4 *>(Blo);
    for (int e = tid; e < NP * kp / 4; e += kTcThreads) {
      if (TC_CAT) {  // [Q][2 NP][4]: quad q's high rows, then its low rows
        const int q = e / NP, j = e - q * NP;
        dh[q * 2 * NP + j] = sh[e];
        dh[q * 2 * NP + NP + j] = sl[e];
      } else {
        dh[e] = sh[e];
        dl[e] = sl[e];
      }
    }
    for (int j = tid; j < NP; j += kTcThreads) {
      Cn[j] = a.cn32[j];
      Hs[j] = 0;
    }
  }
  fence_async_smem();  // B tiles written by the generic proxy, read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_hold;
  const int64_t nunits = my_tiles * units;

  if (warp >= kProdWarp0 && warp < kProdWarp0 + kProdWarps) {
    // ===== producers, in unit order; every unit lands in the 128-byte-swizzled
    // K-major layout (row r at r * 128 B, its 16-byte chunk q at (q ^ (r % 8)) * 16).
    if (!a.rows) {
      // full pass: each unit is one 128-row x 32-column TMA tile (warp 5, lane 0),
      // armed with the unit's bytes
      if (warp == kProdWarp0 && lane == 0) {
        for (int64_t i = 0; i < my_tiles; ++i) {
          const int64_t tile = blockIdx.x + i * gridDim.x;
          for (int h = 0; h < units; ++h) {
            const int64_t u = i * units + h;
            const int s = (int)(u % stages);
            if (u >= stages) mbar_wait(smem_u32(rempty + s), (uint32_t)((u / stages - 1) & 1));
            const uint32_t bar = smem_u32(rfull + s);
            mbar_expect_tx(bar, kUnitBytes);
            tma_tile2d(smem_u32(raw + (size_t)s * kUnitBytes), &tile_map, h * kKU, (int)(tile * kTM), bar);
          }
        }
      }
    } else {
      // candidate rows: warp 5 + h gathers rows 64h..64h+63 of every unit with
      // cp.async (TMA gather4 moves 512 B per instruction: too few for one warp
      // to keep the memory busy). Lane l copies chunk q = l % 8 of the rows
      // 64h + l / 8 + 4t (t = 0..15) from 16 row pointers formed once per tile;
      // completion arrives on the unit's raw full barrier (noinc).
      constexpr int kHalf = kTM / kProdWarps;       // 64 rows per producer
      constexpr int kPer = kHalf * (kKU / 4) / 32;  // 16 chunks per lane per unit
      const int pw = warp - kProdWarp0;
      const int q = lane & 7, r0 = lane >> 3;
      int32_t rn[kHalf / 32];
      auto load_ids = [&](int64_t i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
#pragma unroll
        for (int j = 0; j < kHalf / 32; ++j) {
          const int64_t lr = tile * kTM + pw * kHalf + lane + 32 * j;
          rn[j] = lr < nr ? __ldg(a.rows + lr) : -1;
        }
      };
      load_ids(0);
      for (int64_t i = 0; i < my_tiles; ++i) {
        const float *src[kPer];
        uint32_t valid = 0;
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
          const int32_t gr = __shfl_sync(0xffffffffu, rn[t >> 3], r0 + 4 * (t & 7));
          src[t] = a.f32 + (int64_t)(gr < 0 ? 0 : gr) * a.ld32 + 4 * q;
          valid |= (gr >= 0 ? 1u : 0u) << t;
        }
        if (i + 1 < my_tiles) load_ids(i + 1);
        for (int h = 0; h < units; ++h) {
          const int64_t u = i * units + h;
          const int s = (int)(u % stages);
          if (u >= stages) mbar_wait(smem_u32(rempty + s), (uint32_t)((u / stages - 1) & 1));
          const uint32_t base = smem_u32(raw + (size_t)s * kUnitBytes);
          const uint32_t vmask = (h * kKU + 4 * q < a.d) ? valid : 0u;
#pragma unroll
          for (int t = 0; t < kPer; ++t) {
            const int r = pw * kHalf + r0 + 4 * t;
            cp_async16(base + (uint32_t)r * 128 + (uint32_t)((q ^ (r & 7)) << 4), src[t] + h * kKU,
                       (vmask >> t) & 1u);
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(rfull + s))
                       : "memory");
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
  } else if (TC_IDLE_WARP && TC_MMA_WARPS == 1 && warp == kSplitWarp0 + 1) {
    // idle: keeps the MMA warp's sub-partition free of a third role
  } else if (warp >= kSplitWarp0 && warp < kEpi2Warp0 && !(TC_IDLE_WARP && warp == kSplitWarp0 + 1)) {
    // ===== splitters (warps 7, 9, 10, 11; 8 is idle or the second MMA warp): each writes the low parts of one quarter of every unit, in unit order
    const int sw = (TC_IDLE_WARP && warp > kSplitWarp0) ? warp - kSplitWarp0 - 1 : warp - kSplitWarp0;
    constexpr int kQuads = (int)(kUnitBytes / 16) / kSplitWarps;
    for (int64_t u = 0; u < nunits; ++u) {
      const int s = (int)(u % stages);
      const int t = (int)(u % kLoStages);
      mbar_wait(smem_u32(rfull + s), (uint32_t)((u / stages) & 1));
      if (u >= kLoStages) mbar_wait(smem_u32(lempty + t), (uint32_t)((u / kLoStages - 1) & 1));
      const float4 *pr = reinterpret_cast<const float4 *>(raw + (size_t)s * kUnitBytes) + sw * kQuads;
      float4 *pl = reinterpret_cast<float4 *>(lor + (size_t)t * kUnitBytes) + sw * kQuads;
      constexpr int kPerLane = kQuads / 32;  // every load issued before the first store
      float4 v[kPerLane];
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) v[j] = pr[lane + 32 * j];
#pragma unroll
      for (int j = 0; j < kPerLane; ++j)
        pl[lane + 32 * j] = make_float4(v[j].x - tf32_hi(v[j].x), v[j].y - tf32_hi(v[j].y),
                                        v[j].z - tf32_hi(v[j].z), v[j].w - tf32_hi(v[j].w));
      fence_async_smem();  // this thread's smem writes -> visible to the tensor core
      mbar_arrive(smem_u32(lfull + t));
    }
  } else if (warp == kMmaWarp || (TC_MMA_WARPS == 2 && TC_IDLE_WARP && warp == kSplitWarp0 + 1)) {
    // ===== MMA issue: A_hi = the raw unit (read as tf32 = its top 19 bits), A_lo
    // from the lo ring; the lo full barrier implies the raw unit's arrival.
    // TC_MMA_WARPS = 2: warp 4 issues the even tiles (accumulator 0), warp 8 the
    // odd ones (accumulator 1); each accumulator's MMAs stay in one thread's order.
    const uint32_t idesc = tf32_idesc(NP), idesc2 = tf32_idesc(2 * NP);
    const uint32_t sB = smem_u32(Bhi), sBl = smem_u32(Blo);
    const uint32_t lboB = (TC_CAT ? 2 : 1) * NP * 16, sbo = 128;
    const int mw = (TC_MMA_WARPS == 2 && warp != kMmaWarp) ? 1 : 0;
    int64_t u = 0;
    for (int64_t i = 0; i < my_tiles; ++i) {
      if (TC_MMA_WARPS == 2 && (int)(i & 1) != mw) {
        // the other warp's tile: follow its units' lo barriers in order (a
        // parity wait is only valid one phase away) and release them for this
        // warp (lempty counts both MMA warps), without touching the data
        for (int h = 0; h < units; ++h, ++u) {
          const int t = (int)(u % kLoStages);
          mbar_wait(smem_u32(lfull + t), (uint32_t)((u / kLoStages) & 1));
          if (lane == 0) mbar_arrive(smem_u32(lempty + t));
        }
        continue;
      }
      const int slot = (int)(i & 1);
      if (i >= 2) mbar_wait(smem_u32(tempty + slot), (uint32_t)((i / 2 - 1) & 1));
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(slot * kAccW * NP);
      for (int h = 0; h < units; ++h, ++u) {
        const int s = (int)(u % stages);
        const int t = (int)(u % kLoStages);
        mbar_wait(smem_u32(lfull + t), (uint32_t)((u / kLoStages) & 1));
        tc_fence_after();
        // warp-uniform descriptors (the address field is the low 14 bits of
        // addr >> 4: offsets add without carries below 256 KB)
        const uint64_t dhi = umma_desc_sw128(smem_u32(raw + (size_t)s * kUnitBytes));
        const uint64_t dlo = umma_desc_sw128(smem_u32(lor + (size_t)t * kUnitBytes));
#pragma unroll
        for (int ks = 0; ks < kKU / 8; ++ks) {
          const uint64_t ahi = dhi + (uint64_t)(ks * 2), alo = dlo + (uint64_t)(ks * 2);  // + 32 B
          const uint32_t ob = (uint32_t)(h * (kKU / 8) + ks) * 2 * lboB;
          const uint64_t bhi = umma_desc(sB + ob, lboB, sbo);
          if (TC_CAT) {
            mma_tf32_elect(acc, ahi, bhi, idesc2, (h > 0 || ks > 0) ? 1u : 0u);  // [hi.hi | hi.lo]
            mma_tf32_elect(acc, alo, bhi, idesc, 1u);                             // lo.hi into the first half
          } else {
            const uint64_t blo = umma_desc(sBl + ob, lboB, sbo);
            mma_tf32_elect(acc, ahi, bhi, idesc, (h > 0 || ks > 0) ? 1u : 0u);
            mma_tf32_elect(acc, alo, bhi, idesc, 1u);
            mma_tf32_elect(acc, ahi, blo, idesc, 1u);
          }
        }
        mma_commit_elect(smem_u32(rempty + s));  // the raw slot and the lo slot are free once these MMAs ran
        mma_commit_elect(smem_u32(lempty + t));
        if (h == units - 1) mma_commit_elect(smem_u32(tfull + slot));
      }
    }
  } else {
    // ===== epilogue: thread (warp w, lane l) settles row 32 w + l of each tile
    const double cmax = *a.cmax;
    const double dscale = (double)(3 * a.d + 8) * 1.1920928955078125e-7;  // (3d + 8) 2^-23
    const int eset = (TC_EPI_SETS == 2 && warp >= kEpi2Warp0) ? 1 : 0;
    const int qw = warp & 3;  // TMEM lane quarter = tile rows 32 qw .. 32 qw + 31
    for (int64_t i = (TC_EPI_SETS == 2 ? eset : 0); i < my_tiles; i += TC_EPI_SETS) {
      const int slot = (int)(i & 1);
      const int64_t tile = blockIdx.x + i * gridDim.x;
      const int64_t lr = tile * kTM + qw * 32 + lane;
      const int64_t gr = lr < nr ? (a.rows ? (int64_t)__ldg(a.rows + lr) : lr) : -1;
      const float fni = gr >= 0 ? __ldg(a.fn32 + gr) : 0.0f;
      mbar_wait(smem_u32(tfull + slot), (uint32_t)((i / 2) & 1));
      tc_fence_after();
      // the row's norm is common to its k distances: rank g_j = |c_j|^2 - 2 f.c_j
      // (one fp32 rounding per entry, as many as E had) and add |f|^2 to the best two
      float bv = INFINITY, bv2 = INFINITY;
      int bi = 0x7fffffff;
      const uint32_t taddr = tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)(slot * kAccW * NP);
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + (uint32_t)c0, v);
        if (TC_CAT) {
          float w[16];
          tmem_ld16(taddr + (uint32_t)(NP + c0), w);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += w[j];
        }
        float cn[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 t4 = reinterpret_cast<const float4 *>(Cn + c0)[q];
          cn[4 * q] = t4.x;
          cn[4 * q + 1] = t4.y;
          cn[4 * q + 2] = t4.z;
          cn[4 * q + 3] = t4.w;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int cj = c0 + j;
          const float g = fmaf(-2.0f, v[j], cn[j]);
          if (RAW) {
            if (gr >= 0) a.raw_out[gr * NP + cj] = fni + g;
          }
          if (g < bv) {
            bv2 = bv;
            bv = g;
            bi = cj;
          } else {
            bv2 = fminf(bv2, g);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(tempty + slot));
      if (!RAW && gr >= 0) {
        const double fr = sqrt((double)fni * (1.0 + 2e-5)) + cmax;
        const double delta = dscale * fr * fr * (1.0 + 1e-6);
        const double e1 = (double)fni + (double)bv, e2 = (double)fni + (double)bv2;  // exact in double
        if (e2 - e1 > 2.0 * delta) {
          a.labels[gr] = bi;
          a.ub[gr] = sqrt(fmax(e1 + delta, 0.0));
          a.lb[gr] = sqrt(fmax(e2 - delta, 0.0));
          if (a.counts) atomicAdd(Hs + bi, 1);
        } else {
          a.amb[atomicAdd(a.namb, 1)] = (int32_t)gr;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (a.counts)
    for (int j = tid; j < a.k; j += kTcThreads)
      if (Hs[j]) atomicAdd(a.counts + j, Hs[j]);
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

int tc_npad(int64_t k) { return (int)((k + 15) / 16 * 16); }
int tc_kp(int64_t d) { return (int)((d + kKU - 1) / kKU * kKU); }

size_t tc_smem_fixed(int64_t d, int64_t k) {
  const int64_t kp = tc_kp(d), np = tc_npad(k);
  return sizeof(float) * (2 * np * kp + np) + sizeof(int32_t) * (np + kTM) +
         sizeof(uint64_t) * (2 * kMaxRaw + 2 * kLoStages + 4) + 16 + 1024 +
         (size_t)kLoStages * kUnitBytes;
}

// raw ring units that fit next to the centroid tiles and the lo ring (>= 2 required)
int tc_stages(int64_t d, int64_t k) {
  const int64_t cap = (int64_t)csc::device_info().max_smem_optin;
  const int64_t left = cap - (int64_t)tc_smem_fixed(d, k);
  return (int)std::min<int64_t>(kMaxRaw, std::max<int64_t>(0, left / kUnitBytes));
}

size_t tc_smem(int64_t d, int64_t k) {
  return (size_t)std::max(tc_stages(d, k), 2) * kUnitBytes + tc_smem_fixed(d, k);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp32 map over the n x ld32 features, box = 32 columns x box_rows rows,
// 128-byte swizzle (the UMMA K-major SW128 layout), zero fill out of bounds
int feature_map(CUtensorMap *m, const float *f32, int64_t n, int64_t ld32, uint32_t box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) {
    csc::set_error("tc screen: cuTensorMapEncodeTiled unavailable");
    return CSC_ERR_CUDA;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)ld32, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)ld32 * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)kKU, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(f32), dims, strides,
                         box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    csc::set_error("tc screen: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return CSC_ERR_CUDA;
  }
  return CSC_OK;
}

template <int NP, bool RAW>
int tc_launch_t(const TcArgs &a, cudaStream_t st) {
  const size_t smem = tc_smem(a.d, a.k);
  CUtensorMap tile_map, row_map;
  int rc = feature_map(&tile_map, a.f32, a.n, a.ld32, kTM);
  if (rc == CSC_OK) rc = feature_map(&row_map, a.f32, a.n, a.ld32, 1);
  if (rc != CSC_OK) return rc;
  static std::mutex mu;
  static size_t configured = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > configured) {
      CSC_TRY_CUDA(cudaFuncSetAttribute(tc_screen_kernel<NP, RAW>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      configured = smem;
    }
  }
  const int64_t tiles = csc::ceil_div(a.n, kTM);
  // CSC_TC_GRID (A/B knob): fewer CTAs than SMs leaves SMs to the other
  // restarts' lanes while this screen runs
  static const int env_grid = [] {
    const char *e = getenv("CSC_TC_GRID");
    return e ? atoi(e) : 0;
  }();
  const int64_t cap = env_grid > 0 ? env_grid : csc::device_info().sm_count;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(cap, tiles));
  tc_screen_kernel<NP, RAW><<<(unsigned)grid, kTcThreads, smem, st>>>(a, tc_stages(a.d, a.k), tile_map, row_map);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

template <int NP>
int tc_launch(const TcArgs &a, cudaStream_t st) {
  return a.raw_out ? tc_launch_t<NP, true>(a, st) : tc_launch_t<NP, false>(a, st);
}

int tc_dispatch(const TcArgs &a, cudaStream_t st) {
  switch (a.n_pad) {
    case 16: return tc_launch<16>(a, st);
    case 32: return tc_launch<32>(a, st);
    case 48: return tc_launch<48>(a, st);
    case 64: return tc_launch<64>(a, st);
    case 80: return tc_launch<80>(a, st);
    case 96: return tc_launch<96>(a, st);
    case 112: return tc_launch<112>(a, st);
    case 128: return tc_launch<128>(a, st);
    default: break;
  }
  csc::set_error("tc screen: unsupported centroid count (padded %d)", a.n_pad);
  return CSC_ERR_ARG;
}

}  // namespace

namespace csc {

bool tc_screen_supported(int64_t d, int64_t k) {
  const csc::DeviceInfo &info = csc::device_info();
  return info.cc_major == 10 && d >= 1 && d <= 256 && k >= 2 && tc_npad(k) <= 128 &&
         tc_stages(d, k) >= 2;
}

int64_t tc_centroid_floats(int64_t d, int64_t k) { return (int64_t)tc_npad(k) * tc_kp(d); }

int tc_convert_centroids(const double *c, int64_t k, int64_t d, int64_t ldc, const double *cnorm,
                         float *chi, float *clo, float *cn32, double *cmax, cudaStream_t st) {
  tc_centroids_kernel<<<1, 256, 0, st>>>(c, k, d, ldc, cnorm, tc_npad(k), tc_kp(d), chi, clo, cn32,
                                          cmax);
  CSC_CHECK_LAUNCH();
  return CSC_OK;
}

int tc_screen_assign(const float *f32, int64_t ld32, const float *fn32, int64_t n, int64_t d,
                     const float *chi, const float *clo, const float *cn32, int64_t k,
                     const double *cmax, const int32_t *rows, const int32_t *nrows_dev,
                     int32_t *labels, double *ub, double *lb, int32_t *counts, int32_t *amb,
                     int32_t *namb, float *raw_out, cudaStream_t st) {
  TcArgs a{};
  a.f32 = f32;
  a.ld32 = ld32;
  a.fn32 = fn32;
  a.n = n;
  a.d = (int)d;
  a.kp = tc_kp(d);
  a.k = (int)k;
  a.n_pad = tc_npad(k);
  a.chi = chi;
  a.clo = clo;
  a.cn32 = cn32;
  a.cmax = cmax;
  a.rows = rows;
  a.nrows = nrows_dev;
  a.labels = labels;
  a.ub = ub;
  a.lb = lb;
  a.counts = counts;
  a.amb = amb;
  a.namb = namb;
  a.raw_out = raw_out;
  return tc_dispatch(a, st);
}

}  // namespace csc

extern "C" int csc_kmeans_tc_supported(int64_t d, int64_t k) {
  return csc::tc_screen_supported(d, k) ? 1 : 0;
}

extern "C" int csc_kmeans_tc_distances(const void *f32, int64_t n, int64_t d, int64_t ld32,
                                       const float *fn32, const double *c, int64_t k, int64_t ldc,
                                       const double *cnorm, float *e_out, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(csc::tc_screen_supported(d, k), "csc_kmeans_tc_distances: shape (d=%lld, k=%lld) "
              "outside the tensor-core screen", (long long)d, (long long)k);
  CSC_REQUIRE(ld32 % 4 == 0 && ld32 >= d, "csc_kmeans_tc_distances: ld32 must be a multiple of 4 >= d");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  csc::Scratch chi, clo, cn, cm;
  const int64_t cf = csc::tc_centroid_floats(d, k);
  CSC_TRY_CUDA(chi.alloc(sizeof(float) * cf, st));
  CSC_TRY_CUDA(clo.alloc(sizeof(float) * cf, st));
  CSC_TRY_CUDA(cn.alloc(sizeof(float) * tc_npad(k), st));
  CSC_TRY_CUDA(cm.alloc(sizeof(double), st));
  int rc = csc::tc_convert_centroids(c, k, d, ldc, cnorm, chi.as<float>(), clo.as<float>(),
                                     cn.as<float>(), cm.as<double>(), st);
  if (rc != CSC_OK) return rc;
  return csc::tc_screen_assign(static_cast<const float *>(f32), ld32, fn32, n, d, chi.as<float>(),
                               clo.as<float>(), cn.as<float>(), k, cm.as<double>(), nullptr,
                               nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, e_out,
                               st);
}
