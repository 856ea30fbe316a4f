// ds_nccl.cu -- one-partition-per-process halo exchange and global dots over
// NCCL (stencil.py:280-295 exchange, solver.py:140-141 global dot).
//
// NCCL is resolved at run time (dlopen/dlsym) from the libnccl.so.2 that the
// process already has loaded (PyTorch's), so the library has no link-time
// NCCL dependency and exactly one NCCL lives in the process.
//
// Halo: each neighbour's send list is packed by a gather kernel into a
// contiguous send buffer, then one ncclGroupStart/End posts every
// ncclSend(pack_q) / ncclRecv(x + recv_start_q) pair -- ghosts of one owner
// are contiguous (stencil.py:198-209), so receives land in place.
// Global dot: ncclAllGather of the partition partials; the finalize kernel
// sums them in rank order like the reference's Python sum.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi g_nccl;
static std::once_flag g_nccl_once;

static void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return;
#define DS_SYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name))
  DS_SYM(GetUniqueId, "ncclGetUniqueId");
  DS_SYM(CommInitRank, "ncclCommInitRank");
  DS_SYM(CommDestroy, "ncclCommDestroy");
  DS_SYM(GroupStart, "ncclGroupStart");
  DS_SYM(GroupEnd, "ncclGroupEnd");
  DS_SYM(Send, "ncclSend");
  DS_SYM(Recv, "ncclRecv");
  DS_SYM(AllGather, "ncclAllGather");
  DS_SYM(GetErrorString, "ncclGetErrorString");
#undef DS_SYM
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy &&
              g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.Send && g_nccl.Recv &&
              g_nccl.AllGather;
}

static int nccl_ready() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.ok) {
    set_error("libnccl.so.2 could not be resolved (import torch first)");
    return DS_ERR_NOT_SUPPORTED;
  }
  return DS_OK;
}

static int nccl_fail(ncclResult_t r, const char* what) {
  set_error("NCCL error %d (%s) in %s", (int)r,
            g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?", what);
  return DS_ERR_CUDA;
}

#define DS_NCCL(call)                                       \
  do {                                                      \
    ncclResult_t _r = (call);                               \
    if (_r != ncclSuccess) return ::ds::nccl_fail(_r, #call); \
  } while (0)

__global__ void pack_kernel(int64_t count, const int* __restrict__ idx,
                            const double* __restrict__ src, double* __restrict__ dst,
                            const ds_cg_scalars* s) {
  if (s && s->done) return;   // converged / stopped: p is final, the buffer already holds it
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[idx[k]];
}

}  // namespace ds

using namespace ds;

extern "C" int ds_nccl_unique_id(char* out, int nbytes) {
  int rc = nccl_ready();
  if (rc) return rc;
  if (nbytes < (int)sizeof(ncclUniqueId)) {
    set_error("unique id buffer too small (%d < %d)", nbytes, (int)sizeof(ncclUniqueId));
    return DS_ERR_INVALID_ARGUMENT;
  }
  ncclUniqueId id;
  DS_NCCL(g_nccl.GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return DS_OK;
}

extern "C" int ds_nccl_unique_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

extern "C" int ds_nccl_comm_init(const char* id_bytes, int nranks, int rank, void** comm) {
  int rc = nccl_ready();
  if (rc) return rc;
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t c = nullptr;
  DS_NCCL(g_nccl.CommInitRank(&c, nranks, id, rank));
  *comm = c;
  return DS_OK;
}

extern "C" int ds_nccl_comm_destroy(void* comm) {
  int rc = nccl_ready();
  if (rc) return rc;
  if (comm) DS_NCCL(g_nccl.CommDestroy(reinterpret_cast<ncclComm_t>(comm)));
  return DS_OK;
}

extern "C" int ds_halo_exchange(int nnbr, const int32_t* peers, const int64_t* send_counts,
                                const int32_t* const* send_idx, double* const* send_bufs,
                                const int64_t* recv_counts, const int64_t* recv_starts,
                                double* x_full, const ds_cg_scalars* s, void* comm,
                                void* stream) {
  int rc = nccl_ready();
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  for (int q = 0; q < nnbr; ++q) {
    if (send_counts[q] <= 0) continue;
    int64_t g = ceil_div(send_counts[q], 256);
    if (g > (int64_t)sm_count() * 4) g = (int64_t)sm_count() * 4;
    pack_kernel<<<(unsigned)g, 256, 0, st>>>(send_counts[q], send_idx[q], x_full, send_bufs[q], s);
  }
  DS_LAUNCH_CHECK("pack_kernel");
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  DS_NCCL(g_nccl.GroupStart());
  for (int q = 0; q < nnbr; ++q) {
    if (send_counts[q] > 0)
      DS_NCCL(g_nccl.Send(send_bufs[q], (size_t)send_counts[q], ncclFloat64, peers[q], c, st));
    if (recv_counts[q] > 0)
      DS_NCCL(g_nccl.Recv(x_full + recv_starts[q], (size_t)recv_counts[q], ncclFloat64, peers[q],
                          c, st));
  }
  DS_NCCL(g_nccl.GroupEnd());
  return DS_OK;
}

extern "C" int ds_allgather_f64(const double* send, double* recv, int64_t count, void* comm,
                                void* stream) {
  int rc = nccl_ready();
  if (rc) return rc;
  DS_NCCL(g_nccl.AllGather(send, recv, (size_t)count, ncclFloat64,
                           reinterpret_cast<ncclComm_t>(comm), as_stream(stream)));
  return DS_OK;
}
