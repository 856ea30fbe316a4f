// gather_floor.cu -- what bounds the power-law SpMV (BASELINE config 4)?
//
// Standalone microbenchmark (not product code): nnz = 54.55M entries with
// uniformly random columns over n = 4.19M (a 33.5 MB x, the generator of
// BASELINE.md section 2), measured with CUDA events, median of 20 launches:
//   stream   : read col (4 B) + val (8 B) per entry, no gathers
//   gather   : read col, gather x[col] (8 B random, L2-resident x)
//   spmv-ish : read col + val, gather x[col], sum v*x per thread
// each at several CTAs/SM and loads-in-flight per thread.  Gives the LTS
// (L2 slice) sector-throughput floor a CSR / COO SpMV of this matrix can reach.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather_floor tools/gather_floor.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ldf(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldf(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldx(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__global__ void init(int64_t nnz, int n, int* col, double* val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    col[i] = (int)(h % (uint64_t)n);
    val[i] = 1.0 + (double)(h & 1023) * 1e-3;
  }
}

// MODE 0 stream, 1 gather (col + x), 2 col + val + x, 3 = 2 with the x
// gathers through L1 (__ldg) instead of L1::no_allocate
template <int MODE, int U>
__global__ void kern(int64_t nnz, const int* __restrict__ col, const double* __restrict__ val,
                     const double* __restrict__ x, double* out) {
  const uint64_t pol = pol_first();
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); base < nnz;
       base += stride * U) {
    int c[U];
    double v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t k = base + j * stride;
      c[j] = k < nnz ? ldf(col + k, pol) : 0;
      v[j] = (MODE != 1 && k < nnz) ? ldf(val + k, pol) : 1.0;
    }
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < U; ++j) acc += v[j] + (double)c[j];
    } else {
      double g[U];
#pragma unroll
      for (int j = 0; j < U; ++j) g[j] = MODE == 3 ? __ldg(x + c[j]) : ldx(x + c[j]);
#pragma unroll
      for (int j = 0; j < U; ++j) acc += v[j] * g[j];
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int MODE, int U>
float run(int64_t nnz, const int* col, const double* val, const double* x, double* out, int bpsm,
          int threads, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms * bpsm;
  std::vector<float> t;
  for (int r = 0; r < 25; ++r) {
    cudaEventRecord(a);
    kern<MODE, U><<<grid, threads>>>(nnz, col, val, x, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 5) t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2] * 1e3f;
}

int main() {
  const int n = 4194304;
  const int64_t nnz = 54553506;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* col;
  double *val, *x, *out;
  CK(cudaMalloc(&col, nnz * 4));
  CK(cudaMalloc(&val, nnz * 8));
  CK(cudaMalloc(&x, (size_t)n * 8));
  CK(cudaMalloc(&out, 8));
  init<<<sms * 8, 256>>>(nnz, n, col, val);
  CK(cudaMemset(x, 0, (size_t)n * 8));
  CK(cudaDeviceSynchronize());
  const char* names[4] = {"stream(col+val)", "gather(col+x)", "col+val+x", "col+val+x(ldg)"};
  const double bytes[4] = {12.0 * nnz, 4.0 * nnz, 12.0 * nnz, 12.0 * nnz};
  printf("{\"nnz\": %lld, \"n\": %d, \"sms\": %d, \"runs\": [\n", (long long)nnz, n, sms);
  bool first = true;
  const bool quick = getenv("QUICK") != nullptr;
  if (getenv("WINDOW")) {   // persisting L2 window over x, as the SpMV launcher sets it
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)n * 8);
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = x;
    a.accessPolicyWindow.num_bytes = (size_t)n * 8;
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &a);
  }
  for (int threads : {256, 512}) {
    for (int bpsm : {1, 2, 4, 8}) {
      if (quick && !(threads == 256 && bpsm == 4)) continue;
      if (threads * bpsm > 2048) continue;
#define RUN(M, U)                                                                              \
  {                                                                                            \
    float us = run<M, U>(nnz, col, val, x, out, bpsm, threads, sms);                           \
    printf("%s {\"mode\": \"%s\", \"threads\": %d, \"ctas_per_sm\": %d, \"unroll\": %d, "     \
           "\"us\": %.1f, \"stream_GBs\": %.0f, \"gathers_G_per_s\": %.1f}\n",               \
           first ? " " : ",", names[M], threads, bpsm, U, us, bytes[M] / us / 1e3,             \
           M ? nnz / us / 1e3 : 0.0);                                                          \
    first = false;                                                                             \
  }
      RUN(0, 4) RUN(0, 8) RUN(1, 4) RUN(1, 8) RUN(1, 16) RUN(2, 4) RUN(2, 8) RUN(2, 16)
      RUN(3, 4) RUN(3, 8) RUN(3, 16)
    }
  }
  printf("]}\n");
  return 0;
}
