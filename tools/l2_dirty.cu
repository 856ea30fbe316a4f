// l2_dirty.cu -- does a 243 MB evict_first stream slow down when 27 MB of
// DIRTY vector data sits in L2 (the CG tail's x / r / p before the next SpMV),
// and does a persisting-L2 window over the vectors prevent their write-back?
// Standalone microbenchmark (not product code): graphs of 20 x [vector
// kernel ; stream kernel], CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/l2_dirty tools/l2_dirty.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void stream_kernel(long n4, const double4* __restrict__ a, double* out) {
  double s = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(a + i));
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1.2345) out[0] = s;
}
// write (mode 1) or read (mode 0) the vector block
__global__ void vec_kernel(long n, double* v, int write, double* out) {
  double s = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (write) v[i] = v[i] * 0.5 + 1.0;
    else s += v[i];
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  const long nv = 3L * 104 * 104 * 104;   // x, r, p
  const long mbytes = 243L << 20;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *v, *mat, *out;
  cudaMalloc(&v, nv * 8);
  cudaMalloc(&mat, mbytes);
  cudaMalloc(&out, 8);
  cudaMemset(v, 0, nv * 8);
  cudaMemset(mat, 0, mbytes);
  cudaStream_t st;
  cudaStreamCreate(&st);
  auto run = [&](int write, int with_stream, int persist) {
    if (persist) {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, nv * 8);
      cudaStreamAttrValue a = {};
      a.accessPolicyWindow.base_ptr = v;
      a.accessPolicyWindow.num_bytes = nv * 8;
      a.accessPolicyWindow.hitRatio = 1.0f;
      a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
    }
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) {
      vec_kernel<<<sms * 4, 256, 0, st>>>(nv, v, write, out);
      if (with_stream) stream_kernel<<<sms * 4, 512, 0, st>>>(mbytes / 32, (const double4*)mat, out);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int r = 0; r < 15; ++r) {
      cudaEventRecord(a, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 3) ts.push_back(ms * 1e3f / 20);
    }
    std::sort(ts.begin(), ts.end());
    if (persist) {
      cudaStreamAttrValue a0 = {};
      cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a0);
      cudaCtxResetPersistingL2Cache();
    }
    return ts[ts.size() / 2];
  };
  printf("{\"vec_MB\": %.1f", nv * 8 / 1e6);
  for (int persist : {0, 1}) {
    const float rd = run(0, 0, persist), wr = run(1, 0, persist);
    const float rds = run(0, 1, persist), wrs = run(1, 1, persist);
    printf(", \"persist%d\": {\"read_alone\": %.2f, \"write_alone\": %.2f, \"read+stream\": %.2f, "
           "\"write+stream\": %.2f, \"stream_after_read\": %.2f, \"stream_after_write\": %.2f}",
           persist, rd, wr, rds, wrs, rds - rd, wrs - wr);
  }
  printf("}\n");
  return 0;
}
