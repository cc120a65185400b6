// Device generation of the reference's random probe block (signals.py:16-37):
// column c = sigma * standard_normal(n) of numpy's Generator(PCG64(child_c)),
// reproduced on the GPU from each column's initial PCG64 state.
//
// PCG64 (numpy): 128-bit LCG s <- s*MULT + inc, output XSL-RR of the new
// state. standard_normal: numpy's 256-layer ziggurat (tables probed from the
// library by tools/derive_ziggurat.py): one 64-bit draw r, idx = r & 0xff,
// sign = bit 8, rabs = bits 9..60; accept if rabs < k[idx]; else the wedge
// (one extra uniform) or, for idx 0, the tail loop (pairs of uniforms).
//
// Parallel parse. A column's draw stream is cut into chunks of B draws; the
// chunk thread jumps ahead (O(log) LCG power) to lookback W before its chunk
// and runs the sampler speculatively: the parse synchronises with the true
// one at the first output boundary they share, well inside W. It counts the
// outputs that start inside its chunk; an exclusive scan gives their indices
// and a second pass writes them. Each chunk also reports its first output
// start at/after its own start and at/after its end; neighbouring chunks
// must agree (checked on device), otherwise the column is flagged and the
// caller regenerates it on the host.
//
// Bit-exactness of the tail and wedge. numpy calls the C library's log1p
// (npy_log1p) in the tail loop; on x86-64 with FMA, glibc 2.39 dispatches to
// its FMA build of the fdlibm log1p. glibc_log1p below restates that
// published algorithm (argument reduction 1+x = 2^k (1+f), s = f/(2+f),
// log(1+f) = 2s + s R(s^2) with the fdlibm Lp1..Lp7 minimax coefficients,
// R evaluated in the split form z*Lp1 + z^2 (Lp2 + z Lp3) + z^4 (...) + z^6
// (...)) with every fused multiply-add placed where that build has one and
// all other operations in non-contractible _rn intrinsics; it equals the
// host log1p bit for bit (1e8 inputs over (-1, 0] and arbitrary doubles,
// tools/log1p_check.c). The wedge test and the tail arithmetic use _rn
// intrinsics too (numpy's build has no FMA there). exp() in the wedge test
// only decides a comparison, whose outcome could differ only for a left side
// within one ulp of exp (probability ~1e-16 per wedge draw).
#include <cub/cub.cuh>
#include <math_constants.h>

#include <vector>

#include "common.cuh"

namespace {

#include "ziggurat_tables.inc"

struct U128 {
  uint64_t lo, hi;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

__constant__ U128 kMult = {0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};

// state after k steps: s_k = A^k s + c (A^k - 1)/(A - 1), by squaring
__device__ U128 pcg_advance(U128 s, U128 inc, uint64_t k) {
  U128 am = {1, 0}, ap = {0, 0}, cm = kMult, cp = inc;
  while (k) {
    if (k & 1) {
      am = mul128(am, cm);
      ap = add128(mul128(ap, cm), cp);
    }
    cp = mul128(add128(cm, U128{1, 0}), cp);
    cm = mul128(cm, cm);
    k >>= 1;
  }
  return add128(mul128(am, s), ap);
}

struct Pcg {
  U128 s, inc;
  __device__ __forceinline__ uint64_t next64() {
    s = add128(mul128(s, kMult), inc);
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    return rot ? (x >> rot) | (x << (64 - rot)) : x;
  }
  __device__ __forceinline__ double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
};

// glibc's log1p (fdlibm algorithm, FMA build) restated; see the header.
__device__ __forceinline__ int32_t hi_word(double x) {
  return (int32_t)(__double_as_longlong(x) >> 32);
}
__device__ __forceinline__ double with_hi_word(double x, int32_t h) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return __longlong_as_double((long long)((u & 0xffffffffull) | ((unsigned long long)(uint32_t)h << 32)));
}

__device__ __noinline__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double f = 0.0, c = 0.0, u;
  int32_t k = 1, hu = 0;
  const int32_t hx = hi_word(x), ax = hx & 0x7fffffff;
  if (hx < 0x3FDA827A) {  // 1 + x < sqrt(2)
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (__dadd_rn(two54, x) > 0.0 && ax < 0x3c900000) return x;
      return fma(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return __dadd_rn(x, x);
  if (k != 0) {
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = with_hi_word(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double dk = (double)k;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma(dk, ln2_lo, c);
      return fma(dk, ln2_hi, c);
    }
    const double R = __dmul_rn(fma(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return fma(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, fma(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double R2 = fma(Lp3, z, Lp2), R3 = fma(Lp5, z, Lp4), R4 = fma(Lp7, z, Lp6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  double R = fma(z, Lp1, __dmul_rn(z2, R2));
  R = fma(z4, R3, R);
  R = fma(z6, R4, R);
  const double t = __dmul_rn(s, __dadd_rn(R, hfsq));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  return fma(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(fma(dk, ln2_lo, c), t)), f));
}

// one standard normal; `pos` counts consumed draws
__device__ __forceinline__ double zig_normal(Pcg &g, int64_t &pos, const double *W,
                                             const unsigned long long *K, const double *F) {
  for (;;) {
    uint64_t r = g.next64();
    ++pos;
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * W[idx];
    if (sign) x = -x;
    if (rabs < K[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-ZIG_INV_R, glibc_log1p(-g.next_double()));
        const double yy = -glibc_log1p(-g.next_double());
        pos += 2;
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 1) ? -__dadd_rn(ZIG_R, xx) : __dadd_rn(ZIG_R, xx);
      }
    }
    const double u = g.next_double();
    ++pos;
    if (__dadd_rn(__dmul_rn(__dsub_rn(F[idx - 1], F[idx]), u), F[idx]) <
        exp(__dmul_rn(__dmul_rn(-0.5, x), x)))
      return x;
  }
}

struct ChunkPlan {
  int64_t n, ncols, nch, B, W;
};

// pass 1 (write == 0): count outputs starting in [c0, c1), boundary checks.
// pass 2 (write == 1): write them (index = scanned offset + local index).
__global__ void __launch_bounds__(128)
    zig_chunk_kernel(ChunkPlan P, const uint64_t *__restrict__ states, int write,
                     int32_t *__restrict__ counts, int64_t *__restrict__ first_ge_start,
                     int64_t *__restrict__ first_ge_end, const int32_t *__restrict__ offsets,
                     double sigma, double *__restrict__ out, int64_t ld, int64_t col0) {
  __shared__ double W[256], F[256];
  __shared__ unsigned long long K[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    W[i] = kZigW[i];
    F[i] = kZigF[i];
    K[i] = kZigK[i];
  }
  __syncthreads();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= P.ncols * P.nch) return;
  const int64_t col = tid % P.ncols, ch = tid / P.ncols;
  const int64_t c0 = ch * P.B, c1 = c0 + P.B;
  const int64_t start = ch == 0 ? 0 : c0 - P.W;
  Pcg g;
  g.s = U128{states[4 * col], states[4 * col + 1]};
  g.inc = U128{states[4 * col + 2], states[4 * col + 3]};
  if (start > 0) g.s = pcg_advance(g.s, g.inc, (uint64_t)start);
  int64_t pos = start;
  int64_t fstart = -1, cnt = 0;
  int64_t index = 0;
  if (write) {
    const int32_t *co = offsets + col * P.nch;
    index = co[ch] - co[0];  // offsets are a flattened exclusive scan
  }
  for (;;) {
    const int64_t s0 = pos;
    if (s0 >= c1) break;
    const double z = zig_normal(g, pos, W, K, F);
    if (s0 >= c0) {
      if (fstart < 0) fstart = s0;
      if (write) {
        if (index < P.n) out[index * ld + col0 + col] = 0.0 + sigma * z;
        ++index;
      }
      ++cnt;
    }
  }
  if (!write) {
    counts[tid] = (int32_t)cnt;
    first_ge_start[tid] = fstart < 0 ? pos : fstart;  // no start inside: the next one
    first_ge_end[tid] = pos;                          // first output start >= c1
  }
}

__global__ void zig_check_kernel(ChunkPlan P, const int32_t *__restrict__ counts,
                                 const int64_t *__restrict__ first_ge_start,
                                 const int64_t *__restrict__ first_ge_end,
                                 const int32_t *__restrict__ offsets, int32_t *__restrict__ bad) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= P.ncols * P.nch) return;
  const int64_t col = tid % P.ncols, ch = tid / P.ncols;
  // neighbouring chunks must agree on the output boundary between them
  if (ch + 1 < P.nch) {
    const int64_t nb = tid + P.ncols;
    if (first_ge_end[tid] != first_ge_start[nb]) atomicExch(bad + col, 1);
  } else {
    // enough draws for n outputs? (offsets are in [col][ch] order)
    const int64_t total = (int64_t)offsets[col * P.nch + ch] + counts[tid] - offsets[col * P.nch];
    if (total < P.n) atomicExch(bad + col, 1);
  }
}

__global__ void transpose_counts_kernel(const int32_t *__restrict__ in, int64_t ncols, int64_t nch,
                                        int32_t *__restrict__ out) {
  // in: [ch][col] (thread order) -> out: [col][ch] (scan order)
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ncols * nch) return;
  const int64_t col = t % ncols, ch = t / ncols;
  out[col * nch + ch] = in[t];
}

}  // namespace

// ---------------------------------------------------------------------------
// numpy's SeedSequence -> PCG64 seeding, restated on the host (published
// algorithm: numpy/random/bit_generator.pyx SeedSequence.mix_entropy /
// generate_state / get_assembled_entropy, _pcg64.pyx + pcg64.h
// pcg64_set_seed): the per-column (state, inc) of default_rng(child) for the
// children first..first+d-1 of a SeedSequence, without building the d
// SeedSequence / PCG64 objects in Python (signals.py:34-37 draws one child per
// column).
// ---------------------------------------------------------------------------
namespace seedseq {
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16;

inline uint32_t hashmix(uint32_t value, uint32_t &hc) {
  value ^= hc;
  hc *= kMultA;
  value *= hc;
  value ^= value >> kXShift;
  return value;
}
inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kXShift;
  return r;
}
void mix_entropy(uint32_t *pool, int ps, const uint32_t *ent, int64_t n) {
  uint32_t hc = kInitA;
  for (int i = 0; i < ps; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u, hc);
  for (int src = 0; src < ps; ++src)
    for (int dst = 0; dst < ps; ++dst)
      if (src != dst) pool[dst] = mix(pool[dst], hashmix(pool[src], hc));
  for (int64_t src = ps; src < n; ++src)
    for (int dst = 0; dst < ps; ++dst) pool[dst] = mix(pool[dst], hashmix(ent[src], hc));
}
}  // namespace seedseq

extern "C" {

int csc_seed_states(const uint32_t *run_entropy, int64_t n_run, const uint32_t *key_prefix,
                    int64_t n_key, int64_t first_child, int64_t d, int32_t pool_size,
                    uint64_t *states_out) {
  csc::clear_error();
  CSC_REQUIRE(n_run >= 1 && n_key >= 0 && first_child >= 0 && d >= 0 && states_out != nullptr,
              "csc_seed_states: bad arguments");
  CSC_REQUIRE(pool_size >= 1 && pool_size <= 1024, "csc_seed_states: pool_size out of range");
  // assembled entropy of a child: run entropy (zero-padded to the pool size,
  // since a spawned child always has a spawn key), then the spawn key words:
  // key_prefix, then the child index as little-endian 32-bit words
  std::vector<uint32_t> ent;
  ent.reserve((size_t)std::max<int64_t>(n_run, pool_size) + n_key + 2);
  std::vector<uint32_t> pool(pool_size);
  for (int64_t c = 0; c < d; ++c) {
    ent.assign(run_entropy, run_entropy + n_run);
    if ((int64_t)ent.size() < pool_size) ent.resize(pool_size, 0u);
    ent.insert(ent.end(), key_prefix, key_prefix + n_key);
    uint64_t idx = (uint64_t)(first_child + c);
    if (idx == 0) ent.push_back(0u);
    while (idx > 0) {
      ent.push_back((uint32_t)(idx & 0xffffffffu));
      idx >>= 32;
    }
    seedseq::mix_entropy(pool.data(), pool_size, ent.data(), (int64_t)ent.size());
    // generate_state(4, uint64): 8 words cycling over the pool
    uint32_t w[8];
    uint32_t hc = seedseq::kInitB;
    for (int i = 0; i < 8; ++i) {
      uint32_t v = pool[i % pool_size];
      v ^= hc;
      hc *= seedseq::kMultB;
      v *= hc;
      v ^= v >> seedseq::kXShift;
      w[i] = v;
    }
    const uint64_t val[4] = {w[0] | (uint64_t)w[1] << 32, w[2] | (uint64_t)w[3] << 32,
                             w[4] | (uint64_t)w[5] << 32, w[6] | (uint64_t)w[7] << 32};
    // pcg64_set_seed: state0 = (val0 << 64) | val1, seq = (val2 << 64) | val3;
    // srandom_r: state = 0, inc = seq * 2 + 1, step, state += state0, step
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ed051fc65da4ull << 64) | 0x4385df649fccf645ull;
    const unsigned __int128 s0 = ((unsigned __int128)val[0] << 64) | val[1];
    const unsigned __int128 seq = ((unsigned __int128)val[2] << 64) | val[3];
    const unsigned __int128 inc = (seq << 1) | 1u;
    unsigned __int128 st = 0;
    st = st * mult + inc;
    st += s0;
    st = st * mult + inc;
    states_out[4 * c + 0] = (uint64_t)st;
    states_out[4 * c + 1] = (uint64_t)(st >> 64);
    states_out[4 * c + 2] = (uint64_t)inc;
    states_out[4 * c + 3] = (uint64_t)(inc >> 64);
  }
  return CSC_OK;
}

}  // extern "C"

namespace {

// bad_host != nullptr: flags copied back and the stream synchronised;
// otherwise they stay in bad_dev (ncols int32) and nothing synchronises.
int normal_columns(const uint64_t *states_host, int64_t ncols, int64_t n, double sigma,
                   double *out, int64_t ld, int64_t col0, int32_t *bad_host, int32_t *bad_dev,
                   cudaStream_t st) {
  CSC_REQUIRE(ncols >= 1 && n >= 1 && col0 >= 0 && col0 + ncols <= ld,
              "csc_normal_columns: bad shape");
  csc::device_info();
  ChunkPlan P;
  P.n = n;
  P.ncols = ncols;
  // ~1.02 draws per output; chunks of B draws with a W-draw lookback. Every
  // draw of a chunk thread is a dependent LCG + ziggurat step, so the chunk
  // length is the latency: B is chosen for ~19k chunk threads (148 SMs x 4
  // warps) over all columns, between 64 and 4096 draws. A misaligned parse
  // resynchronises at the first one-draw output (~98% of outputs), so short
  // chunks use a 32-draw lookback (boundaries are still checked below).
  const int64_t est = n + n / 16;
  P.B = std::max<int64_t>(64, std::min<int64_t>(4096, csc::ceil_div(est * ncols, 148 * 128)));
  P.W = P.B < 512 ? 32 : 128;
  const int64_t draws = est + 4 * P.B;
  P.nch = csc::ceil_div(draws, P.B);
  const int64_t T = ncols * P.nch;
  csc::Scratch st_dev, counts, fgs, fge, cnt_t, offs, bad, tmp;
  CSC_TRY_CUDA(st_dev.alloc(sizeof(uint64_t) * 4 * ncols, st));
  CSC_TRY_CUDA(counts.alloc(sizeof(int32_t) * T, st));
  CSC_TRY_CUDA(cnt_t.alloc(sizeof(int32_t) * T, st));
  CSC_TRY_CUDA(offs.alloc(sizeof(int32_t) * T, st));
  CSC_TRY_CUDA(fgs.alloc(sizeof(int64_t) * T, st));
  CSC_TRY_CUDA(fge.alloc(sizeof(int64_t) * T, st));
  int32_t *badp = nullptr;
  if (bad_dev) {
    badp = bad_dev;  // caller-owned
  } else {
    CSC_TRY_CUDA(bad.alloc(sizeof(int32_t) * ncols, st));
    badp = bad.as<int32_t>();
  }
  CSC_TRY_CUDA(cudaMemsetAsync(badp, 0, sizeof(int32_t) * ncols, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(st_dev.ptr, states_host, sizeof(uint64_t) * 4 * ncols,
                               cudaMemcpyHostToDevice, st));
  const int threads = 128;
  const unsigned blocks = (unsigned)csc::ceil_div(T, threads);
  zig_chunk_kernel<<<blocks, threads, 0, st>>>(P, st_dev.as<uint64_t>(), 0, counts.as<int32_t>(),
                                              fgs.as<int64_t>(), fge.as<int64_t>(), nullptr, sigma,
                                              out, ld, col0);
  CSC_CHECK_LAUNCH();
  transpose_counts_kernel<<<blocks, threads, 0, st>>>(counts.as<int32_t>(), ncols, P.nch,
                                                      cnt_t.as<int32_t>());
  CSC_CHECK_LAUNCH();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt_t.as<int32_t>(), offs.as<int32_t>(), T, st);
  CSC_TRY_CUDA(tmp.alloc(tb, st));
  CSC_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tb, cnt_t.as<int32_t>(), offs.as<int32_t>(),
                                             T, st));
  // offsets in [col][ch] order; the kernels index them as col * nch + ch
  zig_check_kernel<<<blocks, threads, 0, st>>>(P, counts.as<int32_t>(), fgs.as<int64_t>(),
                                              fge.as<int64_t>(), offs.as<int32_t>(), badp);
  CSC_CHECK_LAUNCH();
  zig_chunk_kernel<<<blocks, threads, 0, st>>>(P, st_dev.as<uint64_t>(), 1, nullptr, nullptr,
                                              nullptr, offs.as<int32_t>(), sigma, out, ld, col0);
  CSC_CHECK_LAUNCH();
  if (bad_dev) return CSC_OK;
  CSC_TRY_CUDA(cudaMemcpyAsync(bad_host, badp, sizeof(int32_t) * ncols, cudaMemcpyDeviceToHost,
                               st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  return CSC_OK;
}

}  // namespace

extern "C" {

int csc_normal_columns(const uint64_t *states_host, int64_t ncols, int64_t n, double sigma,
                       double *out, int64_t ld, int64_t col0, int32_t *bad_host, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(bad_host != nullptr, "csc_normal_columns: NULL bad_host");
  return normal_columns(states_host, ncols, n, sigma, out, ld, col0, bad_host, nullptr,
                        static_cast<cudaStream_t>(stream));
}

int csc_normal_columns_async(const uint64_t *states_host, int64_t ncols, int64_t n, double sigma,
                             double *out, int64_t ld, int64_t col0, int32_t *bad_dev,
                             void *stream) {
  csc::clear_error();
  CSC_REQUIRE(bad_dev != nullptr, "csc_normal_columns_async: NULL bad_dev");
  return normal_columns(states_host, ncols, n, sigma, out, ld, col0, nullptr, bad_dev,
                        static_cast<cudaStream_t>(stream));
}

}  // extern "C"
