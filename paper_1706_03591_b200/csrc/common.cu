// Library-level entry points and shared helpers.
#include <mutex>
#include <unordered_map>
#include <vector>
#include <string>

#include <cstdlib>

#include "common.cuh"

namespace csc {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }

// Fixed-size table: references handed out stay valid when another thread
// first touches a higher device id (a resized vector would move them).
constexpr int kMaxDevices = 64;

const DeviceInfo &device_info() {
  static std::mutex mu;
  static DeviceInfo cache[kMaxDevices];
  static bool pool_ready[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  std::lock_guard<std::mutex> lock(mu);
  DeviceInfo &info = cache[dev];
  if (info.sm_count == 0) {
    cudaDeviceGetAttribute(&info.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&info.cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&info.cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&info.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (info.sm_count <= 0) info.sm_count = 148;
  }
  if (!pool_ready[dev]) {
    // The stream-ordered pool keeps up to 8 GiB of freed scratch for reuse
    // (per-call partials, sort buffers, segment buffers, k-means lanes) and
    // returns the rest to the driver at synchronisation points, so it does not
    // hold HBM that PyTorch's caching allocator needs. (2 GiB re-mapped the
    // Laplacian build's scratch every configs[4] step: 6.5 vs 3.7 ms.)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 8ull << 30;
      const char *e = getenv("CSC_POOL_KEEP_GB");  // A/B knob: GiB the pool keeps cached
      if (e) thr = (uint64_t)atoll(e) << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    pool_ready[dev] = true;
  }
  return info;
}

// Size classes for pool requests of 1 MiB and more: eight steps per power of
// two (<= 12.5% slack), so that buffers whose size follows nnz (operator plans,
// sort and Laplacian scratch: a fraction of a percent apart between the steps
// of a dynamic sequence) ask for equal sizes.
size_t pool_size_class(size_t bytes) {
  if (bytes < (size_t(1) << 20)) return bytes ? bytes : 16;
  size_t p = size_t(1) << 20;
  while ((p << 1) <= bytes) p <<= 1;
  const size_t step = p >> 3;
  return (bytes + step - 1) / step * step;
}

// Block cache in front of the stream-ordered pool for large blocks on the
// default stream. cudaMallocAsync stalls the host when its free list is
// fragmented: with the pool's reserved size constant (3.5 GiB) the 176 / 352 MB
// plan arrays of a configs[4] step sporadically took 23-2,200 ms to allocate
// (the pool re-maps physical granules into a contiguous range), one step in
// ten. Freed blocks of >= kCacheMin bytes are kept here by size class and
// handed back to the next request of that class on the same stream (work on
// one stream is ordered, so no synchronisation is needed); the oldest blocks
// go back to the pool past kCacheCap.
namespace {
constexpr size_t kCacheMin = size_t(4) << 20;
struct CachedBlock {
  void *ptr;
  size_t bytes;
  int dev;
};
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;                 // free blocks, oldest first
std::unordered_map<void *, size_t> g_block_bytes;  // live large blocks -> class size
size_t g_cache_bytes = 0;
size_t cache_cap() {
  static size_t cap = [] {
    const char *e = getenv("CSC_BLOCK_CACHE_GB");  // 0 turns the cache off
    return (size_t)(e ? atoll(e) : 6) << 30;
  }();
  return cap;
}
}  // namespace

cudaError_t pool_alloc(void **ptr, size_t bytes, cudaStream_t s) {
  const size_t cls = pool_size_class(bytes);
  if (s == nullptr && cls >= kCacheMin && cache_cap() > 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_cache_mu);
    for (size_t i = g_cache.size(); i-- > 0;) {
      if (g_cache[i].bytes == cls && g_cache[i].dev == dev) {
        *ptr = g_cache[i].ptr;
        g_cache.erase(g_cache.begin() + (ptrdiff_t)i);
        g_cache_bytes -= cls;
        g_block_bytes[*ptr] = cls;
        return cudaSuccess;
      }
    }
    const cudaError_t e = cudaMallocAsync(ptr, cls, s);
    if (e == cudaSuccess) g_block_bytes[*ptr] = cls;
    return e;
  }
  return cudaMallocAsync(ptr, cls, s);
}

void pool_free(void *ptr, cudaStream_t s) {
  if (!ptr) return;
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    auto it = g_block_bytes.find(ptr);
    if (it != g_block_bytes.end()) {
      const size_t cls = it->second;
      g_block_bytes.erase(it);  // whatever happens next, the address is no longer tracked
      if (s == nullptr && cache_cap() > 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        g_cache.push_back({ptr, cls, dev});
        g_cache_bytes += cls;
        while (g_cache_bytes > cache_cap()) {  // oldest block of this device back to the pool
          size_t i = 0;
          while (i < g_cache.size() && g_cache[i].dev != dev) ++i;
          if (i == g_cache.size()) break;
          cudaFreeAsync(g_cache[i].ptr, nullptr);
          g_cache_bytes -= g_cache[i].bytes;
          g_cache.erase(g_cache.begin() + (ptrdiff_t)i);
        }
        return;
      }
    }
  }
  cudaFreeAsync(ptr, s);
}

cudaError_t Scratch::alloc(size_t bytes, cudaStream_t s) {
  stream = s;
  return pool_alloc(&ptr, bytes, s);
}

Scratch::~Scratch() {
  if (ptr) pool_free(ptr, stream);
}

}  // namespace csc

__global__ void reduce_partials_kernel(const double *__restrict__ partials, int64_t count,
                                       double *__restrict__ out) {
  __shared__ double smem[32];
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) v += partials[i];
  v = block_sum<1024>(v, smem);
  if (threadIdx.x == 0) out[0] = v;
}

extern "C" {

int csc_version(void) { return 1; }

const char *csc_last_error(void) { return csc::g_last_error.c_str(); }

int csc_device_info(int *sm_count, int *cc_major, int *cc_minor) {
  int ndev = 0;
  CSC_TRY_CUDA(cudaGetDeviceCount(&ndev));
  CSC_REQUIRE(ndev > 0, "no CUDA device visible");
  const csc::DeviceInfo &info = csc::device_info();
  if (sm_count) *sm_count = info.sm_count;
  if (cc_major) *cc_major = info.cc_major;
  if (cc_minor) *cc_minor = info.cc_minor;
  return CSC_OK;
}

int csc_pool_stats(int64_t *out4) {
  CSC_REQUIRE(out4 != nullptr, "csc_pool_stats: NULL output");
  int dev = 0;
  CSC_TRY_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  CSC_TRY_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t v[4] = {0, 0, 0, 0};
  CSC_TRY_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v[0]));
  CSC_TRY_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &v[1]));
  CSC_TRY_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &v[2]));
  CSC_TRY_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &v[3]));
  for (int i = 0; i < 4; ++i) out4[i] = (int64_t)v[i];
  return CSC_OK;
}

int csc_copy2d_async(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width_bytes,
                     int64_t rows, void *stream) {
  CSC_REQUIRE(rows >= 0 && width_bytes >= 0, "csc_copy2d_async: negative extent");
  CSC_REQUIRE(dpitch >= width_bytes && spitch >= width_bytes, "csc_copy2d_async: pitch below width");
  if (rows == 0 || width_bytes == 0) return CSC_OK;
  CSC_TRY_CUDA(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes,
                                 (size_t)rows, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return CSC_OK;
}

}  // extern "C"
