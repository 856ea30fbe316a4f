// grid_barrier.cu -- cost of one grid-wide barrier (acq_rel arrive + acquire
// spin, as the CG tail's) for co-resident grids of various sizes: a
// cooperative kernel doing 1000 barriers, CUDA events.  Standalone
// microbenchmark (not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/grid_barrier tools/grid_barrier.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, old, cur;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1u) : "memory");
    } else {
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

__global__ void barriers(int n, unsigned* count, unsigned* gen) {
  for (int i = 0; i < n; ++i) grid_barrier(count, gen);
}

// flag-array barrier: every block stores its epoch to its own flag (no
// atomic); block 0's threads poll all flags, then thread 0 releases the epoch
// on one word the other blocks spin on
__device__ __forceinline__ void grid_barrier_flags(unsigned* flags, unsigned* gen, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(epoch) : "memory");
  if (blockIdx.x == 0) {
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
      unsigned f;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flags + b) : "memory");
      } while (f != epoch);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(epoch) : "memory");
  } else if (threadIdx.x == 0) {
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
    } while (cur != epoch);
  }
  __syncthreads();
}

__global__ void barriers_flags(int n, unsigned* flags, unsigned* gen, unsigned base) {
  for (int i = 0; i < n; ++i) grid_barrier_flags(flags, gen, base + i + 1);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* w;
  cudaMalloc(&w, 8);
  cudaMemset(w, 0, 8);
  unsigned* fl;
  cudaMalloc(&fl, 4 * 4096 + 4);
  cudaMemset(fl, 0, 4 * 4096 + 4);
  unsigned base = 0;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{\"sms\": %d", sms);
  for (int per : {1, 2, 4}) {
    for (int threads : {128, 256}) {
      const int grid = sms * per;
      const int n = 1000;
      unsigned *c = w, *g = w + 1;
      void* args[] = {(void*)&n, (void*)&c, (void*)&g};
      cudaLaunchCooperativeKernel((void*)barriers, grid, threads, args, 0, 0);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)barriers, grid, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf(", \"grid%d_x%d_us\": %.3f", grid, threads, ms * 1e3f / n);
      unsigned* gen2 = fl + 4096;
      void* args2[] = {(void*)&n, (void*)&fl, (void*)&gen2, (void*)&base};
      cudaLaunchCooperativeKernel((void*)barriers_flags, grid, threads, args2, 0, 0);
      cudaDeviceSynchronize();
      base += n;
      void* args3[] = {(void*)&n, (void*)&fl, (void*)&gen2, (void*)&base};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)barriers_flags, grid, threads, args3, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      base += n;
      printf(", \"flags_grid%d_x%d_us\": %.3f", grid, threads, ms * 1e3f / n);
    }
  }
  printf("}\n");
  return 0;
}
