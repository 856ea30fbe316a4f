// ds_common.cuh -- shared helpers for the dynsparse sm_100a kernels.
//
// * status/error plumbing for the C ABI (include/dynsparse_b200.h)
// * PTX wrappers: mbarrier + cp.async.bulk (1-D TMA) with L2 cache hints
// * exact-rounding helpers: every product and sum the reference performs in
//   numpy is an individually rounded IEEE op, so kernels use __dmul_rn /
//   __dadd_rn explicitly (and the library is built with -fmad=false).
// * the numpy pairwise-sum emulation that np.add.reduceat uses per CSR row
//   (kernels.py:117):  row = p[first] + pairwise(p[first+1:end]) where
//   pairwise(n < 8)   = ((-0.0 + a0) + a1) + ...   (numpy >= 2 starts small
//                       blocks from -0.0, the sign-preserving identity)
//   pairwise(n <= 128)= 8 strided accumulators r[j] = a[j] + a[j+8] + ...,
//                       ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8
//                       tail added sequentially
//   pairwise(n > 128) = pairwise(a[:n2]) + pairwise(a[n2:]),
//                       n2 = n/2 - (n/2)%8
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/dynsparse_b200.h"

namespace ds {

// ---------------------------------------------------------------- errors ----
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define DS_CUDA(call)                                                   \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) return ::ds::cuda_fail(_e, #call);           \
  } while (0)

#define DS_LAUNCH_CHECK(what)                                           \
  do {                                                                  \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return ::ds::cuda_fail(_e, what);            \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();           // cached per device
// Pin [base, base+bytes) in L2 (persisting access-policy window on the
// stream) for the gathered vector of irregular SpMV; returns false if the
// device offers no persisting L2.  x_window_end() resets the stream.
bool x_window_begin(cudaStream_t st, const void* base, size_t bytes);
void x_window_end(cudaStream_t st);
int max_dynamic_smem();   // opt-in shared memory per block (bytes), cached per device
// raise a kernel's dynamic shared-memory limit to `bytes` (minus its static use)
int allow_dynamic_smem(const void* kernel, size_t bytes);
// stable LSD radix sort (ds_sort.cu): keys (or rows[k]*ncols+cols[k] when
// keys == nullptr) <= max_key -> sorted keys + the stable permutation
int radix_sort_pairs(const unsigned long long* keys, const int* rows, const int* cols,
                     unsigned long long ncols, int64_t n, unsigned long long max_key,
                     unsigned long long* keys_out, int* perm_out, cudaStream_t st);
// row-sorted input: sort inside each row (ds_sort.cu); tiles = a
// tile_plan(off, 128, 128) plan; DS_ERR_NOT_SUPPORTED when a row is longer
// than the shared-memory sort takes (nothing written; fall back to the radix)
int segmented_sort_rows(const int* off, const int* rows, const int* cols,
                        unsigned long long ncols, const int* tiles, int64_t ntiles,
                        unsigned long long* keys_out, int* perm_out, cudaStream_t st);
constexpr int kWarp = 32;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------ exact math ----
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// ---------------------------------------------------------------- loads -----
// read-only streaming loads of the matrix: do not allocate in L1.  Not
// `volatile`: the data is immutable during a kernel, and a volatile asm pins
// the load in program order -- ptxas then interleaves each load with the
// gather and the arithmetic that consume it, serialising the memory round
// trips that batched loads are meant to overlap.
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ld_stream4(const int* p) {
  int4 v;
  asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// gathered vector entries: keep in L1/L2
__device__ __forceinline__ double ld_gather(const double* p) { return __ldg(p); }

// L2 eviction-priority policies: the matrix arrays are streamed once
// (evict_first) so that the gathered vector -- up to tens of MB, e.g. the
// 33.5 MB x of the 4.2M-row power-law matrix -- stays L2-resident
// (evict_last) instead of being re-fetched from HBM one 32-B sector per
// 8-B gather.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int ld_hint(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// ------------------------------------------------------- mbarrier + TMA -----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// L2 policy for data streamed exactly once (matrix arrays): evict first so the
// gathered vector x stays resident in the 126 MB L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk async copy global -> shared (TMA engine), completion signalled on
// the mbarrier's transaction count.  dst/src 16-B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ------------------------------------------------ numpy pairwise emulation --
// Leaf of numpy's pairwise sum (n <= 128) computed by an aligned group of 8
// lanes: lane j owns accumulator r[j].  `elem(i)` returns the i-th addend
// (0 <= i < n) -- it is only called for i < n.  All 8 lanes return the
// same value.  `mask` is the shuffle mask of the participating lanes
// (the 8-lane group must be converged).
template <class Elem>
__device__ __forceinline__ double pairwise_leaf_g8(int n, int lane8, unsigned mask,
                                                   Elem elem) {
  const int full = n & ~7;
  double r = 0.0;
  int i = lane8;
  if (i < full) {            // r[j] = a[j]   (no 0.0 + a: keeps the sign of -0.0)
    r = elem(i);
    i += 8;
  }
  for (; i < full; i += 8) r = add(r, elem(i));
  double tail = (i < n) ? elem(i) : 0.0;     // i == full + lane8 here
  double res;
  if (full > 0) {
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)): the xor-butterfly pairs exactly so
    r = add(r, __shfl_xor_sync(mask, r, 1, 8));
    r = add(r, __shfl_xor_sync(mask, r, 2, 8));
    r = add(r, __shfl_xor_sync(mask, r, 4, 8));
    res = r;
  } else {
    res = -0.0;
  }
  const int ntail = n - full;
  for (int t = 0; t < ntail; ++t) res = add(res, __shfl_sync(mask, tail, t, 8));
  return res;
}

// Sequential single-thread emulation of numpy's pairwise sum for arbitrary n
// (used for duplicate runs during canonicalisation: reduceat on a run is
// first + pairwise(rest)).
template <class Elem>
__device__ double pairwise_serial(int64_t n, Elem elem) {
  // explicit-stack post-order walk of the recursion
  struct Frame {
    int64_t lo, n;
    int expanded;
  };
  Frame st[64];
  double vals[64];
  int ft = 0, vt = 0;
  st[ft++] = {0, n, 0};
  while (ft > 0) {
    Frame f = st[--ft];
    if (f.n <= 128) {
      double res;
      if (f.n < 8) {
        res = -0.0;
        for (int64_t i = 0; i < f.n; ++i) res = add(res, elem(f.lo + i));
      } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = elem(f.lo + j);
        int64_t i = 8;
        const int64_t full = f.n - (f.n % 8);
        for (; i < full; i += 8)
          for (int j = 0; j < 8; ++j) r[j] = add(r[j], elem(f.lo + i + j));
        res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
        for (; i < f.n; ++i) res = add(res, elem(f.lo + i));
      }
      vals[vt++] = res;
    } else if (!f.expanded) {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      st[ft++] = {f.lo, f.n, 1};
      st[ft++] = {f.lo + n2, f.n - n2, 0};
      st[ft++] = {f.lo, n2, 0};
    } else {
      double b = vals[--vt];
      double a = vals[--vt];
      vals[vt++] = add(a, b);
    }
  }
  return vals[0];
}

// ------------------------------------------------ deterministic reductions --
// Block-wide sum with a fixed tree (blockDim.x a power of two <= 1024).
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  // warp butterfly (fixed order), then warp partials in a fixed tree
  for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  // warps actually present (kernels whose tile size sets blockDim may run
  // with fewer than BLOCK threads); same tree when blockDim.x == BLOCK
  const int NW = min(BLOCK, (int)blockDim.x) / 32;
  if (w == 0) {
    double t = (l < NW) ? sh[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t = add(t, __shfl_xor_sync(0xffffffffu, t, o));
    v = t;
  }
  __syncthreads();
  return v;  // valid in thread 0
}

// Last-block-done completion: each block publishes its partial; the block
// that takes the final ticket sums the partials in index order-tree and
// returns true (in every thread of that block) with *total set in thread 0.
template <int BLOCK>
__device__ bool grid_sum_last_block(double block_partial, double* partials, unsigned* ticket,
                                    double* total, double* sh) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = block_partial;
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double v = 0.0;
  const int G = gridDim.x;
  // fixed assignment: thread t sums partials t, t+NT, ... sequentially, NT =
  // the threads present (kernels whose tile size sets blockDim run with fewer
  // than BLOCK: a BLOCK stride would skip partials NT..BLOCK-1 of each round)
  const int NT = min(BLOCK, (int)blockDim.x);
  for (int i = threadIdx.x; i < G; i += NT) v = add(v, *((volatile double*)&partials[i]));
  v = block_sum<BLOCK>(v, sh);
  if (threadIdx.x == 0) {
    *total = v;
    *ticket = 0u;  // re-arm for the next launch (stream-ordered)
  }
  return true;
}

}  // namespace ds
