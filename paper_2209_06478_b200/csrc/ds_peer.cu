// ds_peer.cu -- peer-memory transport for the one-partition-per-process CG:
// the halo exchange and the CG dot-product all-gather done with plain loads
// and stores on CUDA-IPC-mapped peer memory (NVLink 5 / NVSwitch between the
// GPUs of one node), no NCCL on the data path (stencil.py:280-295 exchange,
// solver.py:140-141 global dots).
//
// Every rank exports two of its device allocations with CUDA IPC: the
// iteration's vector block (p with its ghost slots at the front) and a small
// exchange block (the gathered scalars all[stage][rank] and the flag words).
// Each rank maps its peers' blocks once (ds_ipc_import) and then
//   halo push   after its direction update, stores p[send_idx[q]] straight
//               into neighbour q's ghost slots (remote posted writes), then
//               -- after every CTA's writes are fenced at system scope --
//               raises q's halo flag for this rank;
//   halo wait   before the remote spmv_add, waits for the flag of every
//               neighbour it receives from and clears it;
//   all-gather  stores its partition dot into all[stage][rank] of every rank
//               and raises (stage, rank) there; then waits for all of its own
//               (stage, *) flags and clears them.  The next kernel sums
//               all[stage][0..P) in rank order -- every rank the same bits.
// Flags are binary and cleared by their consumer, so a captured CUDA graph
// replays the same values every iteration.  A cleared flag cannot race with
// the producer's next raise: the producer raises the same flag again only
// after the OTHER exchange of the iteration, which needs this rank's
// contribution, which this rank makes after clearing (the stream orders it).
// Exchanges are unconditional (a converged, no-op step still exchanges), so
// every rank raises and clears the same flags the same number of times.
//
// Waits: "spin" = one thread per flag polls with ld.acquire.sys inside a
// kernel (lowest latency; the GPUs of a node run concurrently), "memop" =
// cuStreamWaitValue32 / cuStreamWriteValue32 on the stream (the front end
// blocks, no SM is held -- what several ranks sharing one GPU need, since
// their contexts only time-slice).  A spin wait gives up after
// DS_PEER_SPIN_TIMEOUT_NS and traps, so a broken peer fails the launch
// instead of hanging the GPU.
#include <cuda.h>
#include <string.h>

#include <mutex>

#include "ds_common.cuh"

namespace ds {

constexpr int kPeerMaxRanks = DS_PEER_MAX_RANKS;
constexpr int kPeerMaxNbr = DS_PEER_MAX_NBR;
constexpr unsigned long long kSpinTimeoutNs = 30ull * 1000 * 1000 * 1000;   // 30 s

// ---------------------------------------------------------- driver entry ----
struct DriverApi {
  CUresult (*MemGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  CUresult (*StreamWaitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*StreamWriteValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  bool ok = false;
};
static DriverApi g_drv;
static std::once_flag g_drv_once;

static void load_driver() {
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_drv.MemGetAddressRange = reinterpret_cast<decltype(g_drv.MemGetAddressRange)>(f);
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_drv.StreamWaitValue32 = reinterpret_cast<decltype(g_drv.StreamWaitValue32)>(f);
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_drv.StreamWriteValue32 = reinterpret_cast<decltype(g_drv.StreamWriteValue32)>(f);
  g_drv.ok = g_drv.MemGetAddressRange && g_drv.StreamWaitValue32 && g_drv.StreamWriteValue32;
}

static int driver_ready() {
  std::call_once(g_drv_once, load_driver);
  if (!g_drv.ok) {
    set_error("CUDA driver entry points (cuMemGetAddressRange / cuStreamWaitValue32) unavailable");
    return DS_ERR_NOT_SUPPORTED;
  }
  return DS_OK;
}

#define DS_CU(call)                                                       \
  do {                                                                    \
    CUresult _r = (call);                                                 \
    if (_r != CUDA_SUCCESS) {                                             \
      ::ds::set_error("CUDA driver error %d in %s", (int)_r, #call);      \
      return DS_ERR_CUDA;                                                 \
    }                                                                     \
  } while (0)

// ------------------------------------------------------------- PTX bits ----
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void spin_until_set(const unsigned* flag) {
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(flag) == 0u) {
    if (global_ns() - t0 > kSpinTimeoutNs) __trap();   // a peer never arrived
    __nanosleep(64);
  }
}

// ------------------------------------------------------------ all-gather ----
struct AllGatherArgs {
  double* all[kPeerMaxRanks];        // rank r's all[] base (mapped; this rank's is local)
  unsigned* flag[kPeerMaxRanks];     // rank r's all-gather flag words (mapped)
};

// one block of 32 * ceil(P/32) threads; thread r talks to rank r
__global__ void peer_allgather_kernel(AllGatherArgs a, const double* __restrict__ mine, int stage,
                                      int rank, int nranks, unsigned* my_flags, int spin) {
  const int r = threadIdx.x;
  if (r < nranks) {
    const int slot = stage * nranks + rank;
    a.all[r][slot] = *mine;                // remote posted write (local for r == rank)
    st_release_sys(a.flag[r] + slot, 1u);  // release: the value is visible first
  }
  if (spin && r < nranks) {
    unsigned* f = my_flags + stage * nranks + r;
    spin_until_set(f);
    st_relaxed_sys(f, 0u);
  }
}

// ------------------------------------------------------------------ halo ----
struct HaloPushArgs {
  const int* idx[kPeerMaxNbr];       // this rank's local indices sent to neighbour q
  double* dst[kPeerMaxNbr];          // neighbour q's ghost slots for this rank (mapped)
  unsigned* flag[kPeerMaxNbr];       // neighbour q's halo flag for this rank (mapped)
  long long start[kPeerMaxNbr + 1];  // prefix of the send counts
};

__global__ void peer_halo_push_kernel(HaloPushArgs a, int nnbr, const double* __restrict__ p,
                                      unsigned* ticket) {
  const long long total = a.start[nnbr];
  int q = 0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    while (k >= a.start[q + 1]) ++q;   // k only grows: the neighbour index only advances
    const long long j = k - a.start[q];
    a.dst[q][j] = p[a.idx[q][j]];
  }
  // every CTA's remote stores are fenced at system scope before its ticket;
  // the last CTA then raises the neighbours' flags (threadFenceReduction
  // pattern at .sys scope)
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence_system();
  for (int t = threadIdx.x; t < nnbr; t += blockDim.x) st_release_sys(a.flag[t], 1u);
  if (threadIdx.x == 0) *ticket = 0u;   // re-armed for the next push (stream-ordered)
}

struct HaloWaitArgs {
  unsigned* flag[kPeerMaxNbr];       // this rank's halo flags, one per neighbour it receives from
};

__global__ void peer_wait_kernel(HaloWaitArgs a, int n) {
  const int t = threadIdx.x;
  if (t < n) {
    spin_until_set(a.flag[t]);
    st_relaxed_sys(a.flag[t], 0u);
  }
}

static int memop_wait_clear(unsigned* const* flags, int n, cudaStream_t st) {
  for (int t = 0; t < n; ++t) {
    DS_CU(g_drv.StreamWaitValue32((CUstream)st, (CUdeviceptr)flags[t], 1u, CU_STREAM_WAIT_VALUE_EQ));
    DS_CU(g_drv.StreamWriteValue32((CUstream)st, (CUdeviceptr)flags[t], 0u,
                                   CU_STREAM_WRITE_VALUE_DEFAULT));
  }
  return DS_OK;
}

}  // namespace ds

using namespace ds;

// ------------------------------------------------------------------ IPC ------
extern "C" int ds_ipc_handle_bytes(void) {
  return (int)(sizeof(cudaIpcMemHandle_t) + sizeof(int64_t));
}

extern "C" int ds_ipc_export(const void* ptr, char* out) {
  int rc = driver_ready();
  if (rc) return rc;
  CUdeviceptr base = 0;
  size_t size = 0;
  DS_CU(g_drv.MemGetAddressRange(&base, &size, (CUdeviceptr)ptr));
  cudaIpcMemHandle_t h;
  DS_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  const int64_t off = (int64_t)((CUdeviceptr)ptr - base);
  memcpy(out, &h, sizeof(h));
  memcpy(out + sizeof(h), &off, sizeof(off));
  return DS_OK;
}

extern "C" int ds_ipc_import(const char* in, void** ptr) {
  cudaIpcMemHandle_t h;
  int64_t off = 0;
  memcpy(&h, in, sizeof(h));
  memcpy(&off, in + sizeof(h), sizeof(off));
  void* base = nullptr;
  DS_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = static_cast<char*>(base) + off;
  return DS_OK;
}

extern "C" int ds_ipc_close(void* ptr) {
  int rc = driver_ready();
  if (rc) return rc;
  CUdeviceptr base = 0;
  size_t size = 0;
  DS_CU(g_drv.MemGetAddressRange(&base, &size, (CUdeviceptr)ptr));
  DS_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)));
  return DS_OK;
}

// ------------------------------------------------------------ exchanges ----
extern "C" int ds_peer_allgather_f64(const double* mine, int stage, int rank, int nranks,
                                     double* const* all_ptrs, unsigned* const* flag_ptrs,
                                     unsigned* my_flags, int wait_mode, void* stream) {
  if (nranks < 1 || nranks > kPeerMaxRanks || rank < 0 || rank >= nranks) {
    set_error("peer all-gather: rank %d of %d (at most %d ranks)", rank, nranks, kPeerMaxRanks);
    return DS_ERR_INVALID_ARGUMENT;
  }
  if (wait_mode == DS_PEER_WAIT_MEMOP) {
    int rc = driver_ready();
    if (rc) return rc;
  }
  AllGatherArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < nranks; ++r) {
    a.all[r] = all_ptrs[r];
    a.flag[r] = flag_ptrs[r];
  }
  cudaStream_t st = as_stream(stream);
  const int threads = (nranks + 31) / 32 * 32;
  peer_allgather_kernel<<<1, threads, 0, st>>>(a, mine, stage, rank, nranks, my_flags,
                                               wait_mode == DS_PEER_WAIT_SPIN);
  DS_LAUNCH_CHECK("peer_allgather_kernel");
  if (wait_mode == DS_PEER_WAIT_MEMOP) {
    unsigned* mine_flags[kPeerMaxRanks];
    for (int r = 0; r < nranks; ++r) mine_flags[r] = my_flags + stage * nranks + r;
    return memop_wait_clear(mine_flags, nranks, st);
  }
  return DS_OK;
}

extern "C" int ds_peer_halo_push(int nnbr, const int64_t* counts, const int32_t* const* idx,
                                 const double* p, double* const* dst, unsigned* const* flags,
                                 unsigned* ticket, void* stream) {
  if (nnbr <= 0) return DS_OK;
  if (nnbr > kPeerMaxNbr) {
    set_error("peer halo: %d neighbours (at most %d)", nnbr, kPeerMaxNbr);
    return DS_ERR_INVALID_ARGUMENT;
  }
  HaloPushArgs a;
  memset(&a, 0, sizeof(a));
  a.start[0] = 0;
  for (int q = 0; q < nnbr; ++q) {
    a.idx[q] = idx[q];
    a.dst[q] = dst[q];
    a.flag[q] = flags[q];
    a.start[q + 1] = a.start[q] + counts[q];
  }
  const long long total = a.start[nnbr];
  int64_t g = ceil_div(total > 0 ? total : 1, 256);
  if (g > (int64_t)sm_count() * 2) g = (int64_t)sm_count() * 2;
  peer_halo_push_kernel<<<(unsigned)g, 256, 0, as_stream(stream)>>>(a, nnbr, p, ticket);
  DS_LAUNCH_CHECK("peer_halo_push_kernel");
  return DS_OK;
}

extern "C" int ds_peer_wait_flags(int n, unsigned* const* flags, int wait_mode, void* stream) {
  if (n <= 0) return DS_OK;
  if (n > kPeerMaxNbr) {
    set_error("peer wait: %d flags (at most %d)", n, kPeerMaxNbr);
    return DS_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = as_stream(stream);
  if (wait_mode == DS_PEER_WAIT_MEMOP) {
    int rc = driver_ready();
    if (rc) return rc;
    return memop_wait_clear(flags, n, st);
  }
  HaloWaitArgs a;
  memset(&a, 0, sizeof(a));
  for (int t = 0; t < n; ++t) a.flag[t] = flags[t];
  peer_wait_kernel<<<1, 32, 0, st>>>(a, n);
  DS_LAUNCH_CHECK("peer_wait_kernel");
  return DS_OK;
}
