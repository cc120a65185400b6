// O(m) synthetic graph generators on the device.
//
// The reference samplers are O(n^2) host loops (sbm_generate, one coin per
// vertex pair, graphs.py:194-221; perturb_edges over the absent pairs,
// graphs.py:228-273; perturb_nodes, graphs.py:276-319) and cannot produce
// configs[2..4] (n = 1M-4M). These produce graphs of the same models in O(m)
// device work, equal in distribution to the reference (not stream-identical):
//
//  * planted partition: per block pair a Binomial edge count (drawn by the
//    caller on the host: O(k^2) numbers), then that many distinct pairs drawn
//    uniformly from the pair's index space: samples with replacement, sort +
//    unique, and redraws of the shortfall until every pair has its count.
//    The process is equivariant under permutations of a pair's index space,
//    so the final set is a uniform subset of the requested size.
//  * Chung-Lu / degree-corrected SBM (configs[3]): a Poisson number of edge
//    draws; each picks a block pair from the caller's cumulative pair
//    weights and its endpoints in proportion to theta within the blocks
//    (inverse CDF by binary search); self-loops and repeats are dropped (the
//    Poissonised model).
//  * edge churn (perturb_edges semantics): `count` distinct present edges
//    deleted uniformly; `count` absent pairs inserted with probability in
//    proportion to q1 (same block) / q2 (different blocks), without
//    replacement; a pair both deleted and inserted is dropped from both.
//  * node switch (perturb_nodes semantics): `count` distinct nodes move to a
//    uniformly drawn other block, every edge at a moved node is deleted and
//    every pair with a moved endpoint is drawn once with the model
//    probability under the new labels (geometric skipping over each block's
//    members); pairs both deleted and inserted are dropped from both.
//
// Randomness: Philox-4x32-10 keyed by the caller's 64-bit seed; every draw is
// a function of (seed, tag, counter), so results are deterministic for a
// seed and independent of the launch geometry. Uniform integers in [0, N)
// use Lemire's multiply with exact rejection.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace {

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = U4{(uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1,
           (uint32_t)p0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 128 random bits for (tag, counter i, attempt a)
__device__ __forceinline__ U4 rand128(uint64_t seed, uint32_t tag, uint64_t i, uint32_t a) {
  return philox(U4{(uint32_t)i, (uint32_t)(i >> 32), tag, a}, (uint32_t)seed, (uint32_t)(seed >> 32));
}

// uniform integer in [0, N), N >= 1 (Lemire, exact rejection)
__device__ __forceinline__ uint64_t uniform_below(uint64_t seed, uint32_t tag, uint64_t i, uint64_t N) {
  const uint64_t thr = (0ull - N) % N;
  for (uint32_t a = 0;; ++a) {
    const U4 r = rand128(seed, tag, i, a);
    uint64_t x = ((uint64_t)r.x << 32) | r.y;
    if (x * N >= thr) return __umul64hi(x, N);
    x = ((uint64_t)r.z << 32) | r.w;
    if (x * N >= thr) return __umul64hi(x, N);
  }
}

__device__ __forceinline__ double u01(uint32_t hi, uint32_t lo) {  // [0, 1), 53 bits
  return (double)((((uint64_t)hi << 32) | lo) >> 11) * 0x1p-53;
}

// ---- block layout: nb near-equal contiguous blocks (sizes[:n % nb] one larger)
struct Blocks {
  int64_t n, q, r;  // q = n / nb, r = n % nb
  int32_t nb;
  __host__ __device__ int64_t off(int64_t b) const { return b * q + (b < r ? b : r); }
  __host__ __device__ int64_t size(int64_t b) const { return q + (b < r ? 1 : 0); }
  __host__ __device__ int64_t of(int64_t i) const {
    const int64_t big = r * (q + 1);
    return i < big ? i / (q + 1) : r + (i - big) / q;
  }
};

// index of block pair (a, b), a <= b, in row-major upper-triangle order
__host__ __device__ __forceinline__ int64_t pair_index(int64_t a, int64_t b, int64_t nb) {
  return a * nb - a * (a - 1) / 2 + (b - a);
}

// strict upper triangle of an s x s block: index -> (i, j), i < j; row i holds s-1-i pairs
__device__ __forceinline__ void tri_unrank(int64_t idx, int64_t s, int64_t &i, int64_t &j) {
  const double t = (double)(2 * s - 1);
  int64_t r = (int64_t)floor((t - sqrt(t * t - 8.0 * (double)idx)) * 0.5);
  r = r < 0 ? 0 : (r > s - 2 ? s - 2 : r);
  auto off = [&](int64_t x) { return x * (2 * s - x - 1) / 2; };
  while (r > 0 && off(r) > idx) --r;
  while (r < s - 2 && off(r + 1) <= idx) ++r;
  i = r;
  j = r + 1 + (idx - off(r));
}

int bits_for(uint64_t v) {  // number of bits to represent v
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return std::max(b, 1);
}

// sorts keys[0..m) (values < 2^end_bit) and removes repeats; returns the
// unique count (synchronises). tmp: m elements of scratch.
int sort_unique(int64_t *keys, int64_t *tmp, int64_t m, int end_bit, int64_t *out_count,
                cudaStream_t st) {
  if (m == 0) {
    *out_count = 0;
    return CSC_OK;
  }
  size_t b1 = 0, b2 = 0;
  CSC_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, tmp, m, 0, end_bit, st));
  CSC_TRY_CUDA(cub::DeviceSelect::Unique(nullptr, b2, tmp, keys, (int64_t *)nullptr, m, st));
  csc::Scratch t, cnt;
  CSC_TRY_CUDA(t.alloc(std::max(b1, b2), st));
  CSC_TRY_CUDA(cnt.alloc(sizeof(int64_t), st));
  CSC_TRY_CUDA(cub::DeviceRadixSort::SortKeys(t.ptr, b1, keys, tmp, m, 0, end_bit, st));
  CSC_TRY_CUDA(cub::DeviceSelect::Unique(t.ptr, b2, tmp, keys, cnt.as<int64_t>(), m, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(out_count, cnt.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  return CSC_OK;
}

// ---- distinct uniform samples per group ------------------------------------
// Group g needs cnt[g] distinct indices of [0, N[g]); Map turns (g, index)
// into a sortable key and a key back into its group. Keys land sorted and
// unique in keys[0..total).
struct PairMap {  // planted partition: key = edge code lo * n + hi
  Blocks bl;
  const int32_t *pa, *pb;  // block pair of group g
  __device__ int64_t key(int64_t g, uint64_t idx) const {
    const int64_t a = pa[g], b = pb[g];
    int64_t i, j;
    if (a == b) {
      tri_unrank((int64_t)idx, bl.size(a), i, j);
      i += bl.off(a);
      j += bl.off(a);
    } else {
      const int64_t sb = bl.size(b);
      i = bl.off(a) + (int64_t)idx / sb;
      j = bl.off(b) + (int64_t)idx % sb;
    }
    return i * bl.n + j;
  }
  __device__ int64_t group(int64_t key) const {
    return pair_index(bl.of(key / bl.n), bl.of(key % bl.n), bl.nb);
  }
};

struct IdMap {  // one group: key = index
  __device__ int64_t key(int64_t, uint64_t idx) const { return (int64_t)idx; }
  __device__ int64_t group(int64_t) const { return 0; }
};

template <class Map>
__global__ void sample_kernel(Map map, const int64_t *__restrict__ need_off, int64_t G,
                              const int64_t *__restrict__ N, int64_t S, uint64_t seed, uint32_t tag,
                              int64_t *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < S;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = G - 1;  // last group with need_off[g] <= t
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (need_off[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    out[t] = map.key(lo, uniform_below(seed, tag, (uint64_t)t, (uint64_t)N[lo]));
  }
}

template <class Map>
__global__ void group_hist_kernel(Map map, const int64_t *__restrict__ keys, int64_t m,
                                  int64_t *__restrict__ have) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long *>(have + map.group(keys[t])), 1ull);
}

int grid_for(int64_t work) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(csc::ceil_div(work, 256),
                                                     (int64_t)csc::device_info().sm_count * 16));
}

template <class Map>
int distinct_sample(const Map &map, int64_t G, const std::vector<int64_t> &N_host,
                    const std::vector<int64_t> &cnt_host, uint64_t seed, uint32_t tag0, int end_bit,
                    int64_t *keys, int64_t capacity, int64_t *m_out, cudaStream_t st) {
  int64_t total = 0;
  for (int64_t g = 0; g < G; ++g) {
    CSC_REQUIRE(cnt_host[g] >= 0 && cnt_host[g] <= N_host[g], "generator: group %lld asks for %lld of %lld",
                (long long)g, (long long)cnt_host[g], (long long)N_host[g]);
    total += cnt_host[g];
  }
  CSC_REQUIRE(capacity >= total, "generator: output capacity %lld < %lld", (long long)capacity,
              (long long)total);
  csc::Scratch tmp, dN, doff, dhave;
  CSC_TRY_CUDA(tmp.alloc(sizeof(int64_t) * std::max<int64_t>(total, 1), st));
  CSC_TRY_CUDA(dN.alloc(sizeof(int64_t) * G, st));
  CSC_TRY_CUDA(doff.alloc(sizeof(int64_t) * G, st));
  CSC_TRY_CUDA(dhave.alloc(sizeof(int64_t) * G, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(dN.ptr, N_host.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, st));
  std::vector<int64_t> need = cnt_host, off(G), have(G);
  int64_t m = 0;
  for (uint32_t round = 0;; ++round) {
    int64_t S = 0;
    for (int64_t g = 0; g < G; ++g) {
      off[g] = S;
      S += need[g];
    }
    if (S == 0) break;
    CSC_REQUIRE(round < 64, "generator: distinct sampling did not converge");
    CSC_TRY_CUDA(cudaMemcpyAsync(doff.ptr, off.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, st));
    sample_kernel<Map><<<grid_for(S), 256, 0, st>>>(map, doff.as<int64_t>(), G, dN.as<int64_t>(), S, seed,
                                                    tag0 + round, keys + m);
    CSC_CHECK_LAUNCH();
    int rc = sort_unique(keys, tmp.as<int64_t>(), m + S, end_bit, &m, st);
    if (rc != CSC_OK) return rc;
    CSC_TRY_CUDA(cudaMemsetAsync(dhave.ptr, 0, sizeof(int64_t) * G, st));
    group_hist_kernel<Map><<<grid_for(m), 256, 0, st>>>(map, keys, m, dhave.as<int64_t>());
    CSC_CHECK_LAUNCH();
    CSC_TRY_CUDA(cudaMemcpyAsync(have.data(), dhave.ptr, sizeof(int64_t) * G, cudaMemcpyDeviceToHost, st));
    CSC_TRY_CUDA(cudaStreamSynchronize(st));
    for (int64_t g = 0; g < G; ++g) need[g] = cnt_host[g] - have[g];
  }
  *m_out = m;
  return CSC_OK;
}

// ---- Chung-Lu ------------------------------------------------------------------
__global__ void chung_lu_kernel(Blocks bl, const double *__restrict__ pair_cum, int64_t npairs,
                                const double *__restrict__ cum_theta, int64_t m_draw, uint64_t seed,
                                int64_t *__restrict__ out, unsigned long long *__restrict__ kept) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m_draw;
       t += (int64_t)gridDim.x * blockDim.x) {
    const U4 r = rand128(seed, 0x43484c55u, (uint64_t)t, 0);
    const U4 r2 = rand128(seed, 0x43484c56u, (uint64_t)t, 0);
    // block pair: first index with pair_cum > u * total
    const double u = u01(r.x, r.y) * pair_cum[npairs - 1];
    int64_t lo = 0, hi = npairs - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (pair_cum[mid] > u) hi = mid;
      else lo = mid + 1;
    }
    const int64_t a = lo / bl.nb, b = lo % bl.nb;
    auto endpoint = [&](int64_t blk, double v) {  // first row with cum_theta > v * block total
      const int64_t o = bl.off(blk), s = bl.size(blk);
      const double x = v * cum_theta[o + s - 1];
      int64_t l = 0, h = s - 1;
      while (l < h) {
        const int64_t mid = (l + h) / 2;
        if (cum_theta[o + mid] > x) h = mid;
        else l = mid + 1;
      }
      return o + l;
    };
    const int64_t ea = endpoint(a, u01(r.z, r.w)), eb = endpoint(b, u01(r2.x, r2.y));
    if (ea != eb) {
      const unsigned long long slot = atomicAdd(kept, 1ull);
      out[slot] = (ea < eb ? ea : eb) * bl.n + (ea < eb ? eb : ea);
    }
  }
}

// ---- churn helpers ---------------------------------------------------------------
__device__ __forceinline__ bool in_sorted(const int64_t *__restrict__ a, int64_t m, int64_t v) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo < m && a[lo] == v;
}

__global__ void gather_codes_kernel(const int64_t *__restrict__ codes, const int64_t *__restrict__ idx,
                                    int64_t c, int64_t *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < c;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = codes[idx[t]];
}

// candidate insertions: inside a block w.p. p_in, else any pair; rejected
// (-1) when the endpoints coincide, the block relation does not match the
// draw, the pair is present after the deletions, or it is already chosen
__global__ void churn_candidates_kernel(int64_t n, const int32_t *__restrict__ labels,
                                        const int32_t *__restrict__ members,
                                        const int64_t *__restrict__ loff, double p_in,
                                        const int64_t *__restrict__ codes, int64_t m,
                                        const int64_t *__restrict__ dels, int64_t nd,
                                        const int64_t *__restrict__ chosen, int64_t nc, int64_t B,
                                        uint64_t seed, uint32_t tag, int64_t *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B;
       t += (int64_t)gridDim.x * blockDim.x) {
    const U4 r = rand128(seed, tag, (uint64_t)t, 0);
    const bool inside = u01(r.x, r.y) < p_in;
    const int64_t a = (int64_t)uniform_below(seed, tag + 0x100u, (uint64_t)t, (uint64_t)n);
    const int32_t la = labels[a];
    int64_t b;
    if (inside) {
      const int64_t s = loff[la + 1] - loff[la];
      b = members[loff[la] + (int64_t)uniform_below(seed, tag + 0x200u, (uint64_t)t, (uint64_t)s)];
    } else {
      b = (int64_t)uniform_below(seed, tag + 0x300u, (uint64_t)t, (uint64_t)n);
    }
    int64_t code = -1;
    if (a != b && ((labels[b] == la) == inside)) {
      const int64_t c = (a < b ? a : b) * n + (a < b ? b : a);
      const bool present = in_sorted(codes, m, c) && !in_sorted(dels, nd, c);
      if (!present && !in_sorted(chosen, nc, c)) code = c;
    }
    out[t] = code;
  }
}

struct NonNeg {
  __device__ bool operator()(const int64_t &v) const { return v >= 0; }
};

__global__ void random_keys_kernel(int64_t c, uint64_t seed, uint32_t tag, uint64_t *__restrict__ keys,
                                   int64_t *__restrict__ vals, const int64_t *__restrict__ src) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < c;
       t += (int64_t)gridDim.x * blockDim.x) {
    const U4 r = rand128(seed, tag, (uint64_t)t, 0);
    keys[t] = ((uint64_t)r.x << 32) | r.y;
    vals[t] = src[t];
  }
}

// drop the codes of a that are in b (both sorted)
__global__ void mark_not_in_kernel(const int64_t *__restrict__ a, int64_t na,
                                   const int64_t *__restrict__ b, int64_t nb,
                                   uint8_t *__restrict__ keep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < na;
       t += (int64_t)gridDim.x * blockDim.x)
    keep[t] = in_sorted(b, nb, a[t]) ? 0 : 1;
}

int select_flagged(const int64_t *in, const uint8_t *flags, int64_t m, int64_t *out, int64_t *count,
                   cudaStream_t st) {
  if (m == 0) {
    *count = 0;
    return CSC_OK;
  }
  size_t b = 0;
  CSC_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, b, in, flags, out, (int64_t *)nullptr, m, st));
  csc::Scratch t, cnt;
  CSC_TRY_CUDA(t.alloc(b, st));
  CSC_TRY_CUDA(cnt.alloc(sizeof(int64_t), st));
  CSC_TRY_CUDA(cub::DeviceSelect::Flagged(t.ptr, b, in, flags, out, cnt.as<int64_t>(), m, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(count, cnt.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  return CSC_OK;
}

// drop pairs both deleted and inserted (the host models' convention)
int drop_common(int64_t *del, int64_t *nd, int64_t *ins, int64_t *ni, cudaStream_t st) {
  if (*nd == 0 || *ni == 0) return CSC_OK;
  csc::Scratch kd, ki, td, ti;
  CSC_TRY_CUDA(kd.alloc(*nd, st));
  CSC_TRY_CUDA(ki.alloc(*ni, st));
  CSC_TRY_CUDA(td.alloc(sizeof(int64_t) * *nd, st));
  CSC_TRY_CUDA(ti.alloc(sizeof(int64_t) * *ni, st));
  mark_not_in_kernel<<<grid_for(*nd), 256, 0, st>>>(del, *nd, ins, *ni, kd.as<uint8_t>());
  CSC_CHECK_LAUNCH();
  mark_not_in_kernel<<<grid_for(*ni), 256, 0, st>>>(ins, *ni, del, *nd, ki.as<uint8_t>());
  CSC_CHECK_LAUNCH();
  CSC_TRY_CUDA(cudaMemcpyAsync(td.ptr, del, sizeof(int64_t) * *nd, cudaMemcpyDeviceToDevice, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(ti.ptr, ins, sizeof(int64_t) * *ni, cudaMemcpyDeviceToDevice, st));
  int64_t a = 0, b = 0;
  int rc = select_flagged(td.as<int64_t>(), kd.as<uint8_t>(), *nd, del, &a, st);
  if (rc == CSC_OK) rc = select_flagged(ti.as<int64_t>(), ki.as<uint8_t>(), *ni, ins, &b, st);
  if (rc != CSC_OK) return rc;
  *nd = a;
  *ni = b;
  return CSC_OK;
}

// members of each label in node order (stable) and label offsets
__global__ void label_hist_kernel(const int32_t *__restrict__ labels, int64_t n, int32_t nb,
                                  int64_t *__restrict__ cnt, int32_t *__restrict__ bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = labels[t];
    if (l < 0 || l >= nb) {
      *bad = 1;
      continue;
    }
    atomicAdd(reinterpret_cast<unsigned long long *>(cnt + l), 1ull);
  }
}

__global__ void iota_kernel(int32_t *__restrict__ v, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    v[t] = (int32_t)t;
}

int build_members(const int32_t *labels, int64_t n, int32_t nb, csc::Scratch &members,
                  csc::Scratch &loff, cudaStream_t st) {
  csc::Scratch keys_out, ids, cnt, bad;
  CSC_TRY_CUDA(members.alloc(sizeof(int32_t) * n, st));
  CSC_TRY_CUDA(loff.alloc(sizeof(int64_t) * (nb + 1), st));
  CSC_TRY_CUDA(keys_out.alloc(sizeof(int32_t) * n, st));
  CSC_TRY_CUDA(ids.alloc(sizeof(int32_t) * n, st));
  CSC_TRY_CUDA(cnt.alloc(sizeof(int64_t) * (nb + 1), st));
  CSC_TRY_CUDA(bad.alloc(sizeof(int32_t), st));
  CSC_TRY_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(int64_t) * (nb + 1), st));
  CSC_TRY_CUDA(cudaMemsetAsync(bad.ptr, 0, sizeof(int32_t), st));
  label_hist_kernel<<<grid_for(n), 256, 0, st>>>(labels, n, nb, cnt.as<int64_t>(), bad.as<int32_t>());
  CSC_CHECK_LAUNCH();
  iota_kernel<<<grid_for(n), 256, 0, st>>>(ids.as<int32_t>(), n);
  CSC_CHECK_LAUNCH();
  size_t b1 = 0, b2 = 0;
  CSC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, labels, keys_out.as<int32_t>(), ids.as<int32_t>(),
                                               members.as<int32_t>(), n, 0, bits_for(nb), st));
  CSC_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, cnt.as<int64_t>(), loff.as<int64_t>(), nb + 1, st));
  csc::Scratch t;
  CSC_TRY_CUDA(t.alloc(std::max(b1, b2), st));
  CSC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(t.ptr, b1, labels, keys_out.as<int32_t>(), ids.as<int32_t>(),
                                               members.as<int32_t>(), n, 0, bits_for(nb), st));
  CSC_TRY_CUDA(cub::DeviceScan::ExclusiveSum(t.ptr, b2, cnt.as<int64_t>(), loff.as<int64_t>(), nb + 1, st));
  int32_t hb = 0;
  CSC_TRY_CUDA(cudaMemcpyAsync(&hb, bad.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  CSC_REQUIRE(hb == 0, "generator: labels must lie in [0, %d)", nb);
  return CSC_OK;
}

// ---- node switch ---------------------------------------------------------------------
__global__ void switch_labels_kernel(const int64_t *__restrict__ sel, int64_t c, int32_t nb,
                                     uint64_t seed, int32_t *__restrict__ labels,
                                     uint8_t *__restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < c;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = sel[t];
    const int64_t step = 1 + (int64_t)uniform_below(seed, 0x53574954u, (uint64_t)u, (uint64_t)(nb - 1));
    labels[u] = (int32_t)((labels[u] + step) % nb);
    flag[u] = 1;
  }
}

__global__ void incident_flags_kernel(int64_t n, const int64_t *__restrict__ codes, int64_t m,
                                      const uint8_t *__restrict__ sel, uint8_t *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = codes[t];
    out[t] = (sel[c / n] | sel[c % n]) ? 1 : 0;
  }
}

// thread per (moved node u, block b): the members of b with probability q
// (q1 if b is u's new block) by geometric skipping; a pair whose other end v
// also moved is drawn by the smaller of the two
__global__ void switch_inserts_kernel(int64_t n, const int64_t *__restrict__ sel, int64_t c, int32_t nb,
                                      const int32_t *__restrict__ labels,
                                      const int32_t *__restrict__ members,
                                      const int64_t *__restrict__ loff,
                                      const uint8_t *__restrict__ flag, double q1, double q2,
                                      uint64_t seed, int64_t *__restrict__ out, int64_t cap,
                                      unsigned long long *__restrict__ count) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < c * nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = sel[t / nb];
    const int32_t b = (int32_t)(t % nb);
    const double q = labels[u] == b ? q1 : q2;
    if (!(q > 0.0)) continue;
    const int64_t o = loff[b], s = loff[b + 1] - o;
    const double lq = q < 1.0 ? log1p(-q) : -INFINITY;
    int64_t pos = -1;
    for (uint32_t a = 0;; ++a) {
      const U4 r = rand128(seed, 0x494e5357u, (uint64_t)t, a);
      const double uu = 1.0 - u01(r.x, r.y);  // (0, 1]
      const double g = q < 1.0 ? floor(log(uu) / lq) : 0.0;
      if (!(g < (double)(s - pos))) break;
      pos += 1 + (int64_t)g;
      if (pos >= s) break;
      const int64_t v = members[o + pos];
      if (v == u || (flag[v] && v < u)) continue;
      const unsigned long long slot = atomicAdd(count, 1ull);
      if ((int64_t)slot < cap) out[slot] = (u < v ? u : v) * n + (u < v ? v : u);
    }
  }
}

}  // namespace

extern "C" {

int csc_gen_planted_partition(int64_t n, int32_t nblocks, const int64_t *pair_counts, uint64_t seed,
                              int64_t *codes_out, int64_t capacity, int64_t *m_out, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 1 && nblocks >= 1 && nblocks <= n && pair_counts && codes_out && m_out,
              "csc_gen_planted_partition: bad arguments");
  CSC_REQUIRE(n < 3037000499LL, "csc_gen_planted_partition: n too large for int64 codes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Blocks bl{n, n / nblocks, n % nblocks, nblocks};
  const int64_t P = (int64_t)nblocks * (nblocks + 1) / 2;
  std::vector<int32_t> pa(P), pb(P);
  std::vector<int64_t> N(P), cnt(P);
  for (int64_t a = 0, g = 0; a < nblocks; ++a)
    for (int64_t b = a; b < nblocks; ++b, ++g) {
      pa[g] = (int32_t)a;
      pb[g] = (int32_t)b;
      const int64_t sa = bl.size(a), sb = bl.size(b);
      N[g] = a == b ? sa * (sa - 1) / 2 : sa * sb;
      cnt[g] = pair_counts[g];
      if (N[g] == 0) N[g] = 1;  // empty index space: count must be 0 (checked)
    }
  csc::Scratch dpa, dpb;
  CSC_TRY_CUDA(dpa.alloc(sizeof(int32_t) * P, st));
  CSC_TRY_CUDA(dpb.alloc(sizeof(int32_t) * P, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(dpa.ptr, pa.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice, st));
  CSC_TRY_CUDA(cudaMemcpyAsync(dpb.ptr, pb.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice, st));
  for (int64_t g = 0; g < P; ++g) {
    const int64_t sa = bl.size(pa[g]), sb = bl.size(pb[g]);
    const int64_t real = pa[g] == pb[g] ? sa * (sa - 1) / 2 : sa * sb;
    CSC_REQUIRE(cnt[g] >= 0 && cnt[g] <= real, "csc_gen_planted_partition: pair %lld count %lld of %lld",
                (long long)g, (long long)cnt[g], (long long)real);
  }
  PairMap map{bl, dpa.as<int32_t>(), dpb.as<int32_t>()};
  return distinct_sample(map, P, N, cnt, seed, 0x50505400u, bits_for((uint64_t)n * (uint64_t)n), codes_out,
                         capacity, m_out, st);
}

int csc_gen_chung_lu(int64_t n, int32_t nblocks, const double *cum_theta_dev, const double *pair_cum_host,
                     int64_t m_draw, uint64_t seed, int64_t *codes_out, int64_t capacity, int64_t *m_out,
                     void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 2 && nblocks >= 1 && nblocks <= n && cum_theta_dev && pair_cum_host && codes_out && m_out &&
                  m_draw >= 0,
              "csc_gen_chung_lu: bad arguments");
  CSC_REQUIRE(capacity >= m_draw, "csc_gen_chung_lu: capacity %lld < draws %lld", (long long)capacity,
              (long long)m_draw);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Blocks bl{n, n / nblocks, n % nblocks, nblocks};
  const int64_t P = (int64_t)nblocks * nblocks;
  csc::Scratch dpc, kept, tmp;
  CSC_TRY_CUDA(dpc.alloc(sizeof(double) * P, st));
  CSC_TRY_CUDA(kept.alloc(sizeof(unsigned long long), st));
  CSC_TRY_CUDA(tmp.alloc(sizeof(int64_t) * std::max<int64_t>(m_draw, 1), st));
  CSC_TRY_CUDA(cudaMemcpyAsync(dpc.ptr, pair_cum_host, sizeof(double) * P, cudaMemcpyHostToDevice, st));
  CSC_TRY_CUDA(cudaMemsetAsync(kept.ptr, 0, sizeof(unsigned long long), st));
  if (m_draw > 0) {
    chung_lu_kernel<<<grid_for(m_draw), 256, 0, st>>>(bl, dpc.as<double>(), P, cum_theta_dev, m_draw, seed,
                                                      codes_out, kept.as<unsigned long long>());
    CSC_CHECK_LAUNCH();
  }
  unsigned long long k = 0;
  CSC_TRY_CUDA(cudaMemcpyAsync(&k, kept.ptr, sizeof(k), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  return sort_unique(codes_out, tmp.as<int64_t>(), (int64_t)k, bits_for((uint64_t)n * (uint64_t)n), m_out, st);
}

int csc_gen_edge_churn(int64_t n, const int64_t *codes, int64_t m, const int32_t *labels, int32_t nblocks,
                       double q1, double q2, int64_t count, uint64_t seed, int64_t *del_out, int64_t *n_del,
                       int64_t *ins_out, int64_t *n_ins, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 2 && nblocks >= 1 && codes && labels && del_out && ins_out && n_del && n_ins && count >= 0 &&
                  count <= m,
              "csc_gen_edge_churn: bad arguments");
  CSC_REQUIRE(q1 >= 0.0 && q2 >= 0.0 && (q1 > 0.0 || q2 > 0.0), "csc_gen_edge_churn: q1, q2 >= 0, not both 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  *n_del = *n_ins = 0;
  if (count == 0) return CSC_OK;
  const int code_bits = bits_for((uint64_t)n * (uint64_t)n);
  // deletions: count distinct positions of the sorted edge list
  csc::Scratch idx;
  CSC_TRY_CUDA(idx.alloc(sizeof(int64_t) * count, st));
  int64_t got = 0;
  int rc = distinct_sample(IdMap{}, 1, std::vector<int64_t>{m}, std::vector<int64_t>{count}, seed, 0x44454c00u,
                           bits_for((uint64_t)m), idx.as<int64_t>(), count, &got, st);
  if (rc != CSC_OK) return rc;
  gather_codes_kernel<<<grid_for(count), 256, 0, st>>>(codes, idx.as<int64_t>(), count, del_out);
  CSC_CHECK_LAUNCH();
  // insertions among the absent pairs, in proportion to the pair probabilities
  csc::Scratch members, loff;
  if ((rc = build_members(labels, n, nblocks, members, loff, st)) != CSC_OK) return rc;
  std::vector<int64_t> off(nblocks + 1);
  CSC_TRY_CUDA(cudaMemcpyAsync(off.data(), loff.ptr, sizeof(int64_t) * (nblocks + 1), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  double n_in = 0.0;
  for (int32_t b = 0; b < nblocks; ++b) {
    const double s = (double)(off[b + 1] - off[b]);
    n_in += s * (s - 1.0) / 2.0;
  }
  const double n_out = (double)n * (double)(n - 1) / 2.0 - n_in;
  const double w_in = q1 * n_in, w_out = q2 * n_out;
  CSC_REQUIRE(w_in + w_out > 0.0, "csc_gen_edge_churn: no pair has positive probability");
  const double p_in = w_in / (w_in + w_out);
  int64_t have = 0;
  for (uint32_t round = 0; have < count; ++round) {
    CSC_REQUIRE(round < 200, "csc_gen_edge_churn: insertion sampling did not converge");
    const int64_t need = count - have;
    const int64_t B = need + need / 5 + 16;
    csc::Scratch cand, sel, tmp, keys, keys2, vals2;
    CSC_TRY_CUDA(cand.alloc(sizeof(int64_t) * B, st));
    CSC_TRY_CUDA(sel.alloc(sizeof(int64_t) * B, st));
    CSC_TRY_CUDA(tmp.alloc(sizeof(int64_t) * B, st));
    churn_candidates_kernel<<<grid_for(B), 256, 0, st>>>(
        n, labels, members.as<int32_t>(), loff.as<int64_t>(), p_in, codes, m, del_out, count, ins_out, have,
        B, seed, 0x494e0000u + round * 0x1000u, cand.as<int64_t>());
    CSC_CHECK_LAUNCH();
    // valid candidates, sorted and unique
    size_t b = 0;
    CSC_TRY_CUDA(cub::DeviceSelect::If(nullptr, b, cand.as<int64_t>(), sel.as<int64_t>(), (int64_t *)nullptr, B,
                                       NonNeg(), st));
    csc::Scratch t, cnt;
    CSC_TRY_CUDA(t.alloc(b, st));
    CSC_TRY_CUDA(cnt.alloc(sizeof(int64_t), st));
    CSC_TRY_CUDA(cub::DeviceSelect::If(t.ptr, b, cand.as<int64_t>(), sel.as<int64_t>(), cnt.as<int64_t>(), B,
                                       NonNeg(), st));
    int64_t nv = 0;
    CSC_TRY_CUDA(cudaMemcpyAsync(&nv, cnt.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CSC_TRY_CUDA(cudaStreamSynchronize(st));
    if ((rc = sort_unique(sel.as<int64_t>(), tmp.as<int64_t>(), nv, code_bits, &nv, st)) != CSC_OK) return rc;
    if (nv == 0) continue;
    int64_t take = std::min(nv, need);
    if (nv > need) {  // a uniform subset of the valid candidates: smallest random keys
      CSC_TRY_CUDA(keys.alloc(sizeof(uint64_t) * nv, st));
      CSC_TRY_CUDA(keys2.alloc(sizeof(uint64_t) * nv, st));
      CSC_TRY_CUDA(vals2.alloc(sizeof(int64_t) * nv, st));
      random_keys_kernel<<<grid_for(nv), 256, 0, st>>>(nv, seed, 0x4b455900u + round, keys.as<uint64_t>(),
                                                      tmp.as<int64_t>(), sel.as<int64_t>());
      CSC_CHECK_LAUNCH();
      size_t bs = 0;
      CSC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bs, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                                   tmp.as<int64_t>(), vals2.as<int64_t>(), nv, 0, 64, st));
      csc::Scratch ts;
      CSC_TRY_CUDA(ts.alloc(bs, st));
      CSC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(ts.ptr, bs, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                                   tmp.as<int64_t>(), vals2.as<int64_t>(), nv, 0, 64, st));
      CSC_TRY_CUDA(cudaMemcpyAsync(sel.ptr, vals2.ptr, sizeof(int64_t) * take, cudaMemcpyDeviceToDevice, st));
    }
    CSC_TRY_CUDA(cudaMemcpyAsync(ins_out + have, sel.ptr, sizeof(int64_t) * take, cudaMemcpyDeviceToDevice, st));
    have += take;
    if ((rc = sort_unique(ins_out, tmp.as<int64_t>(), have, code_bits, &have, st)) != CSC_OK) return rc;
  }
  *n_del = count;
  *n_ins = have;
  return drop_common(del_out, n_del, ins_out, n_ins, st);
}

int csc_gen_node_switch(int64_t n, const int64_t *codes, int64_t m, int32_t *labels, int32_t nblocks, double q1,
                        double q2, int64_t count, uint64_t seed, int64_t *del_out, int64_t *n_del,
                        int64_t *ins_out, int64_t ins_capacity, int64_t *n_ins, void *stream) {
  csc::clear_error();
  CSC_REQUIRE(n >= 2 && nblocks >= 2 && codes && labels && del_out && ins_out && n_del && n_ins && count >= 0 &&
                  count <= n,
              "csc_gen_node_switch: bad arguments (node reassignment needs k >= 2)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  *n_del = *n_ins = 0;
  if (count == 0) return CSC_OK;
  const int code_bits = bits_for((uint64_t)n * (uint64_t)n);
  csc::Scratch sel, flag, eflag;
  CSC_TRY_CUDA(sel.alloc(sizeof(int64_t) * count, st));
  CSC_TRY_CUDA(flag.alloc(n, st));
  CSC_TRY_CUDA(eflag.alloc(std::max<int64_t>(m, 1), st));
  CSC_TRY_CUDA(cudaMemsetAsync(flag.ptr, 0, n, st));
  int64_t got = 0;
  int rc = distinct_sample(IdMap{}, 1, std::vector<int64_t>{n}, std::vector<int64_t>{count}, seed, 0x53454c00u,
                           bits_for((uint64_t)n), sel.as<int64_t>(), count, &got, st);
  if (rc != CSC_OK) return rc;
  switch_labels_kernel<<<grid_for(count), 256, 0, st>>>(sel.as<int64_t>(), count, nblocks, seed, labels,
                                                       flag.as<uint8_t>());
  CSC_CHECK_LAUNCH();
  // deletions: every edge at a moved node (edge order = sorted)
  if (m > 0) {
    incident_flags_kernel<<<grid_for(m), 256, 0, st>>>(n, codes, m, flag.as<uint8_t>(), eflag.as<uint8_t>());
    CSC_CHECK_LAUNCH();
    if ((rc = select_flagged(codes, eflag.as<uint8_t>(), m, del_out, n_del, st)) != CSC_OK) return rc;
  }
  // insertions: every pair with a moved endpoint drawn once under the new labels
  csc::Scratch members, loff, cnt, tmp;
  if ((rc = build_members(labels, n, nblocks, members, loff, st)) != CSC_OK) return rc;
  CSC_TRY_CUDA(cnt.alloc(sizeof(unsigned long long), st));
  CSC_TRY_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(unsigned long long), st));
  switch_inserts_kernel<<<grid_for(count * nblocks), 256, 0, st>>>(
      n, sel.as<int64_t>(), count, nblocks, labels, members.as<int32_t>(), loff.as<int64_t>(), flag.as<uint8_t>(),
      q1, q2, seed, ins_out, ins_capacity, cnt.as<unsigned long long>());
  CSC_CHECK_LAUNCH();
  unsigned long long ni = 0;
  CSC_TRY_CUDA(cudaMemcpyAsync(&ni, cnt.ptr, sizeof(ni), cudaMemcpyDeviceToHost, st));
  CSC_TRY_CUDA(cudaStreamSynchronize(st));
  if ((int64_t)ni > ins_capacity) {
    csc::set_error("csc_gen_node_switch: %llu insertions exceed the capacity %lld", ni, (long long)ins_capacity);
    return CSC_ERR_CAPACITY;
  }
  CSC_TRY_CUDA(tmp.alloc(sizeof(int64_t) * std::max<unsigned long long>(ni, 1ull), st));
  if ((rc = sort_unique(ins_out, tmp.as<int64_t>(), (int64_t)ni, code_bits, n_ins, st)) != CSC_OK) return rc;
  return drop_common(del_out, n_del, ins_out, n_ins, st);
}

}  // extern "C"
