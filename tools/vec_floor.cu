// vec_floor.cu -- what bounds the CG tail (x += a p; r -= a Ap) on B200?
//
// Standalone microbenchmark (not product code).  n = 104^3 doubles per
// vector.  A CUDA graph of 20 iterations of [stream a 243 MB buffer (the DIA
// matrix stand-in) ; update kernel], or of the update kernel alone, timed with
// CUDA events; per-iteration time of the update = difference.  Variants: grid
// (CTAs per SM), elements per thread, 16-B vs 32-B loads.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/vec_floor tools/vec_floor.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void stream_kernel(int64_t n4, const double4* __restrict__ a, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(a + i));
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1.2345) out[0] = s;
}

// the DIA SpMV's traffic without its arithmetic: stream the 243 MB matrix,
// read a 9 MB vector, write a 9 MB vector (one output per 27 matrix values)
__global__ void stream_rw_kernel(int64_t rows, const double* __restrict__ a, const double* __restrict__ xin,
                                 double* yout) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = xin[i];
#pragma unroll
    for (int d = 0; d < 27; ++d) {
      double v;
      asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];"
                   : "=d"(v) : "l"(a + d * rows + i));
      s += v;
    }
    yout[i] = s;
  }
}

// the same traffic with the repo's DIA layout: row-major (nrows, 27), one
// thread per row reading its 27 contiguous values (L1-allocating loads: a
// warp's 27 load instructions cover 54 consecutive 128-B lines)
__global__ void stream_rw_rowmajor(int64_t rows, const double* __restrict__ a,
                                   const double* __restrict__ xin, double* yout) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = xin[i];
    const double* v = a + i * 27;
    double t[27];
#pragma unroll
    for (int d = 0; d < 27; ++d) t[d] = __ldg(v + d);
#pragma unroll
    for (int d = 0; d < 27; ++d) s += t[d];
    yout[i] = s;
  }
}

// U double2 per array per thread, one sweep (grid covers n)
template <int U>
__global__ void update2(int64_t n2, double2* x, double2* r, const double2* __restrict__ p,
                        const double2* __restrict__ ap, double alpha, double* parts) {
  const int64_t base = blockIdx.x * (int64_t)blockDim.x * U + threadIdx.x;
  double2 xv[U], rv[U], pv[U], av[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = min(base + u * (int64_t)blockDim.x, n2 - 1);
    xv[u] = x[i];
    rv[u] = r[i];
    pv[u] = p[i];
    av[u] = ap[i];
  }
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = base + u * (int64_t)blockDim.x;
    if (i < n2) {
      xv[u].x += alpha * pv[u].x;
      xv[u].y += alpha * pv[u].y;
      rv[u].x -= alpha * av[u].x;
      rv[u].y -= alpha * av[u].y;
      x[i] = xv[u];
      r[i] = rv[u];
      v += rv[u].x * rv[u].x + rv[u].y * rv[u].y;
    }
  }
  __shared__ double sh[32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t += sh[w];
    parts[blockIdx.x] = t;
  }
}

// 32-B (double4) version
template <int U>
__global__ void update4(int64_t n4, double4* x, double4* r, const double4* __restrict__ p,
                        const double4* __restrict__ ap, double alpha, double* parts) {
  const int64_t base = blockIdx.x * (int64_t)blockDim.x * U + threadIdx.x;
  double4 xv[U], rv[U], pv[U], av[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = min(base + u * (int64_t)blockDim.x, n4 - 1);
    xv[u] = x[i];
    rv[u] = r[i];
    pv[u] = p[i];
    av[u] = ap[i];
  }
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = base + u * (int64_t)blockDim.x;
    if (i < n4) {
      xv[u].x += alpha * pv[u].x; xv[u].y += alpha * pv[u].y;
      xv[u].z += alpha * pv[u].z; xv[u].w += alpha * pv[u].w;
      rv[u].x -= alpha * av[u].x; rv[u].y -= alpha * av[u].y;
      rv[u].z -= alpha * av[u].z; rv[u].w -= alpha * av[u].w;
      x[i] = xv[u];
      r[i] = rv[u];
      v += rv[u].x * rv[u].x + rv[u].y * rv[u].y + rv[u].z * rv[u].z + rv[u].w * rv[u].w;
    }
  }
  __shared__ double sh[32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t += sh[w];
    parts[blockIdx.x] = t;
  }
}

int main() {
  const int64_t n = 104LL * 104 * 104;
  const int64_t mbytes = 243LL << 20;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *x, *r, *p, *ap, *mat, *parts, *out;
  cudaMalloc(&x, n * 8); cudaMalloc(&r, n * 8); cudaMalloc(&p, n * 8); cudaMalloc(&ap, n * 8);
  cudaMalloc(&mat, mbytes); cudaMalloc(&parts, 1 << 20); cudaMalloc(&out, 8);
  cudaMemset(x, 0, n * 8); cudaMemset(r, 0, n * 8); cudaMemset(p, 0, n * 8);
  cudaMemset(ap, 0, n * 8); cudaMemset(mat, 0, mbytes);
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto time_graph = [&](auto body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) body();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int rep = 0; rep < 30; ++rep) {
      cudaEventRecord(a, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep >= 5) ts.push_back(ms * 1e3f / 20);
    }
    std::sort(ts.begin(), ts.end());
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ts[ts.size() / 2];
  };
  const int64_t m4 = mbytes / 32;
  auto stream = [&] { stream_kernel<<<sms * 4, 512, 0, st>>>(m4, (const double4*)mat, out); };
  const float t_stream = time_graph(stream);
  float t_rw[3];
  for (int k = 0; k < 3; ++k) {
    const int bps = 2 << k;
    t_rw[k] = time_graph([&] { stream_rw_kernel<<<sms * bps, 256, 0, st>>>(n, mat, p, ap); });
  }
  float t_rm[4];
  for (int k = 0; k < 4; ++k) {
    const int bps = 1 << k;
    t_rm[k] = time_graph([&] { stream_rw_rowmajor<<<sms * bps, 256, 0, st>>>(n, mat, p, ap); });
  }
  printf("{\"stream_243MB_us\": %.2f, \"dia_traffic_261MB_us\": [%.2f, %.2f, %.2f], "
         "\"rowmajor_261MB_us_1_2_4_8\": [%.2f, %.2f, %.2f, %.2f], \"runs\": [\n",
         t_stream, t_rw[0], t_rw[1], t_rw[2], t_rm[0], t_rm[1], t_rm[2], t_rm[3]);
  bool first = true;
  auto report = [&](const char* name, int threads, int u, auto launch) {
    const float alone = time_graph(launch);
    const float with = time_graph([&] { stream(); launch(); });
    printf("%s {\"kernel\": \"%s\", \"threads\": %d, \"unroll\": %d, \"alone_us\": %.2f, "
           "\"after_stream_us\": %.2f}\n", first ? " " : ",", name, threads, u, alone,
           with - t_stream);
    first = false;
  };
  const int64_t n2 = n / 2, n4 = n / 4;
  for (int threads : {256, 512}) {
#define R2(U)                                                                              \
  report("update2", threads, U, [&] {                                                      \
    update2<U><<<(unsigned)((n2 + (int64_t)threads * U - 1) / ((int64_t)threads * U)), threads, 0, \
                 st>>>(n2, (double2*)x, (double2*)r, (const double2*)p, (const double2*)ap, \
                       0.5, parts);                                                        \
  });
#define R4(U)                                                                              \
  report("update4", threads, U, [&] {                                                      \
    update4<U><<<(unsigned)((n4 + (int64_t)threads * U - 1) / ((int64_t)threads * U)), threads, 0, \
                 st>>>(n4, (double4*)x, (double4*)r, (const double4*)p, (const double4*)ap, \
                       0.5, parts);                                                        \
  });
    R2(1) R2(2) R2(4) R4(1) R4(2)
  }
  printf("]}\n");
  return 0;
}
