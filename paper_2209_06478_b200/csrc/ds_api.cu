// ds_api.cu -- error state and device queries of the C ABI.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "ds_common.cuh"

namespace ds {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  return DS_ERR_CUDA;
}

// The conversions' multi-GB temporaries come from the stream-ordered
// allocator; by default its pool returns memory to the driver at every
// synchronisation, and re-mapping GBs costs tens of ms per conversion at
// 192^3.  Keep up to 16 GB cached in the device's default pool.
static void keep_pool(int dev) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = 16ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    keep_pool(dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

int max_dynamic_smem() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 227 * 1024;
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
        v <= 0)
      v = 227 * 1024;
    cache[dev] = v;
  }
  return cache[dev];
}

int allow_dynamic_smem(const void* kernel, size_t bytes) {
  cudaFuncAttributes fa;
  DS_CUDA(cudaFuncGetAttributes(&fa, kernel));
  if (fa.maxDynamicSharedSizeBytes >= (int)bytes) return DS_OK;
  const int room = max_dynamic_smem() - (int)fa.sharedSizeBytes;
  if ((int)bytes > room) {
    set_error("kernel needs %zu B of dynamic shared memory, %d available", bytes, room);
    return DS_ERR_NOT_SUPPORTED;
  }
  DS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, room));
  return DS_OK;
}

bool x_window_begin(cudaStream_t st, const void* base, size_t bytes) {
  static int max_persist[64] = {0}, max_window[64] = {0}, done[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  if (!getenv("DS_L2_WINDOW")) return false;   // measured slower (profiles/r01/README.md): opt-in
  if (!done[dev]) {
    cudaDeviceGetAttribute(&max_persist[dev], cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window[dev], cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist[dev] > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, max_persist[dev]);
    done[dev] = 1;
  }
  if (max_persist[dev] <= 0 || max_window[dev] <= 0) return false;
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  a.accessPolicyWindow.num_bytes = bytes < (size_t)max_window[dev] ? bytes : (size_t)max_window[dev];
  const double fit = (double)max_persist[dev] / (double)a.accessPolicyWindow.num_bytes;
  a.accessPolicyWindow.hitRatio = (float)(fit < 1.0 ? fit : 1.0);
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  return cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a) == cudaSuccess;
}

void x_window_end(cudaStream_t st) {
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
  cudaCtxResetPersistingL2Cache();
}

}  // namespace ds

// Persisting-L2 window over [base, base+bytes) for the kernels launched (or
// captured) on `stream` afterwards: the CG vectors stay L2-resident while the
// matrix streams through with evict_first.  The carve-out is sized to the
// window (at most the device's maximum).
extern "C" int ds_l2_persist(const void* base, int64_t bytes, void* stream) {
  int dev = 0, max_persist = 0, max_window = 0;
  DS_CUDA(cudaGetDevice(&dev));
  DS_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  DS_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  // whole windows only: a partial (hitRatio < 1) window over vectors larger
  // than the carve-out measured slower than none (192^3: 385 -> 490 us/step)
  if (max_persist <= 0 || max_window <= 0 || bytes <= 0 || bytes > max_persist ||
      bytes > max_window) {
    ds::set_error("window of %lld B does not fit the persisting L2 (%d B)", (long long)bytes,
                  max_persist);
    return DS_ERR_NOT_SUPPORTED;
  }
  const size_t want = (size_t)bytes < (size_t)max_window ? (size_t)bytes : (size_t)max_window;
  const size_t carve = want < (size_t)max_persist ? want : (size_t)max_persist;
  DS_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  a.accessPolicyWindow.num_bytes = want;
  const double fit = (double)carve / (double)want;
  a.accessPolicyWindow.hitRatio = (float)(fit < 1.0 ? fit : 1.0);
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  DS_CUDA(cudaStreamSetAttribute(ds::as_stream(stream), cudaStreamAttributeAccessPolicyWindow, &a));
  return DS_OK;
}

extern "C" int ds_l2_persist_reset(void* stream) {
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.num_bytes = 0;
  DS_CUDA(cudaStreamSetAttribute(ds::as_stream(stream), cudaStreamAttributeAccessPolicyWindow, &a));
  DS_CUDA(cudaCtxResetPersistingL2Cache());
  DS_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
  return DS_OK;
}

namespace ds {
int aux_stream(cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join) {
  static cudaStream_t s[64] = {};
  static cudaEvent_t f[64] = {}, j[64] = {};
  static std::mutex mu;
  int dev = 0;
  DS_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) {
    set_error("device index %d out of range", dev);
    return DS_ERR_NOT_SUPPORTED;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!s[dev]) {
    DS_CUDA(cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking));
    DS_CUDA(cudaEventCreateWithFlags(&f[dev], cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&j[dev], cudaEventDisableTiming));
  }
  *side = s[dev];
  *fork = f[dev];
  *join = j[dev];
  return DS_OK;
}
}  // namespace ds

extern "C" const char* ds_last_error(void) { return ds::g_err; }
extern "C" int ds_abi_version(void) { return DS_ABI_VERSION; }
extern "C" int ds_device_sm_count(int* out) {
  *out = ds::sm_count();
  return DS_OK;
}
