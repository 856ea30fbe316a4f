// ds_kernels.cuh -- cross-file declarations: the fused-dot epilogue shared by
// the SpMV kernels and the CG finalisation hooks.
#pragma once

#include "ds_common.cuh"

namespace ds {

// What the last block does with a completed fused dot product.
enum CgStage : int {
  kStageNone = 0,   // just store the total in *result
  kStagePap = 1,    // total = p.Ap  -> breakdown test, alpha     (solver.py:173-176)
  kStageRr = 2,     // total = r.r   -> history, convergence, beta (solver.py:180-187)
  kStageSetup = 3,  // total = r0.r0 (bb already known) -> history[0], convergence
};

// Device-side CG finalisation.  parts[0..nparts) are the per-partition dots;
// the global dot is their rank-ordered sum starting from int 0, exactly like
// the reference's Python sum (solver.py:140-141).
__device__ __forceinline__ double ordered_sum(const double* parts, int nparts) {
  double g = parts[0];  // 0 + d0 == d0
  for (int k = 1; k < nparts; ++k) g = add(g, parts[k]);
  return g;
}

__device__ __forceinline__ void cg_finalize(int stage, ds_cg_scalars* s, double* history,
                                            const double* parts, int nparts) {
  const double g = ordered_sum(parts, nparts);
  if (stage == kStagePap) {
    if (s->done) return;
    s->pap = g;
    if (g <= 0.0) {  // `pap <= 0.0` (a NaN keeps iterating, as in the reference)
      s->done = 2;
      return;
    }
    s->alpha = s->rr / g;
  } else if (stage == kStageRr) {
    if (s->done) return;
    const int it = s->iter + 1;
    s->iter = it;
    const double h = sqrt(g) / s->scale;
    history[it] = h;
    s->rr_new = g;
    if (h <= s->tol) {
      s->done = 1;
      return;
    }
    if (it >= s->max_iters) {
      s->done = 3;
      return;
    }
    s->beta = g / s->rr;
    s->rr = g;
  } else if (stage == kStageSetup) {
    // bb already reduced into s->bb by the caller
    const double nb = sqrt(s->bb);
    s->scale = nb > 0.0 ? nb : 1.0;
    s->rr = g;
    s->iter = 0;
    const double h = sqrt(g) / s->scale;
    history[0] = h;
    if (h <= s->tol) s->done = 1;
    else if (s->max_iters <= 0) s->done = 3;
    else s->done = 0;
  }
}

// Fused-dot epilogue: blocks publish partial sums; the last block finishes
// the (deterministic, fixed-order) reduction and optionally runs a CG stage.
struct DotOut {
  const int* guard = nullptr;      // if non-null and *guard != 0 the kernel is a no-op
  const double* other = nullptr;   // vector dotted with the kernel's output
  double* partials = nullptr;      // >= max_blocks doubles
  unsigned* ticket = nullptr;
  double* result = nullptr;        // this partition's dot (parts[k])
  int max_blocks = 0;
  int stage = kStageNone;          // CG stage to run when nparts_final > 0
  ds_cg_scalars* s = nullptr;
  double* history = nullptr;
  const double* parts = nullptr;   // all partitions' dots (result is one of them)
  int nparts_final = 0;            // >0: run cg_finalize(parts, nparts_final)
  int partials_only = 0;           // deferred mode: write partials[blockIdx] and the
                                   // grid size (at ticket[2]); the consumer reduces them
  int plus_zero = 0;               // epilogue y = (A x) + 0.0: the exact effect of
                                   // spmv_add with an EMPTY remote part (kernels.py:196-198)

  __host__ __device__ bool fused() const { return partials != nullptr; }
  __device__ __forceinline__ bool skip() const { return guard != nullptr && *guard != 0; }
  __host__ int64_t clamp_grid(int64_t b) const { return b > max_blocks ? max_blocks : b; }

  template <int BLOCK>
  __device__ void finish_block(double v) const {
    __shared__ double sh[32];
    double bsum = block_sum<BLOCK>(v, sh);
    if (partials_only) {
      if (threadIdx.x == 0) {
        partials[blockIdx.x] = bsum;
        if (blockIdx.x == 0) ticket[2] = gridDim.x;   // count word; ticket[0] stays 0
      }
      return;
    }
    double total;
    if (grid_sum_last_block<BLOCK>(bsum, partials, ticket, &total, sh)) {
      if (threadIdx.x == 0) {
        *result = total;
        if (nparts_final > 0) {
          __threadfence();
          cg_finalize(stage, s, history, parts, nparts_final);
        }
      }
    }
  }
};

// Deferred reduction: every block sums the producer's G block partials in
// the same fixed order (thread t: t, t+BLOCK, ... sequentially; then the
// block tree), so all blocks obtain bitwise the same total.
template <int BLOCK>
__device__ double reduce_partials(const double* partials, const unsigned* count, double* sh) {
  const int G = (int)*count;
  const int NT = min(BLOCK, (int)blockDim.x);   // threads present (see grid_sum_last_block)
  double v = 0.0;
  for (int i = threadIdx.x; i < G; i += NT) v = add(v, partials[i]);
  v = block_sum<BLOCK>(v, sh);
  __shared__ double s_tot;
  if (threadIdx.x == 0) s_tot = v;
  __syncthreads();
  return s_tot;
}

// launchers shared between translation units
int launch_csr(int64_t nrows, int64_t nnz, const int* off, const int* col, const double* val,
               const int* long_rows, int64_t n_long, int max_len, const double* x, double* y,
               bool accum,
               const DotOut* dot, cudaStream_t st);
// irregular CSR: entry-parallel tiles (ds_csr_tiles plan) + long rows (bins
// 6 / 7 of the ds_csr_bins plan) concurrently on a side stream
int launch_csr_tiles(int64_t nrows, int64_t ncols, const int* off, const int* col,
                     const double* val, const int* tiles, int64_t ntiles, const int* perm,
                     const int64_t* bins, const double* x, double* y, bool accum,
                     const int* guard, cudaStream_t st);
int launch_csr_binned(int64_t nrows, int64_t ncols, int64_t nnz, const int* off, const int* col,
                      const double* val, const int* perm, const int64_t* bins, const double* x,
                      double* y, bool accum, const DotOut* dot, cudaStream_t st);
int launch_dia(int64_t nrows, int64_t ncols, int ndiags, const int* off, const double* val,
               const double* x, double* y, bool accum, const DotOut* dot, cudaStream_t st);
int launch_coo(int64_t nrows, int64_t nnz, const int* rows, const int* cols, const double* vals,
               bool sorted, int max_len, const double* x, double* y, bool accum, const int* guard,
               cudaStream_t st, bool plus_zero = false, const int* long_runs = nullptr,
               int n_long = 0);
// y = 0 / y = y + 0.0 for a matrix without entries (ds_csr.cu)
int launch_empty_matrix(int64_t nrows, double* y, bool accum, const int* guard, cudaStream_t st);
// per-device auxiliary stream + fork/join events (created once) for kernels
// that run concurrently with the main one
int aux_stream(cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join);
// stand-alone fused dot with the same epilogue (used when a SpMV kernel
// cannot fuse it): result = a[0:n] . b[0:n]
int launch_dot(int64_t n, const double* a, const double* b, const DotOut& d, cudaStream_t st);
constexpr int kMaxPartials = 1 << 16;
// CSR long rows: 130..kCsrWarpRow entries -> warp per row, longer -> CTA per row
constexpr int kCsrWarpRow = 1024;
constexpr int kCsrBinCount = 8;   // ds_csr_bins: 8 bins, 9 offsets
// ds_csr_tiles: a tile boundary where off[r] crosses a multiple of
// kCsrTileTarget and around every row longer than 129 entries, so a tile of
// short rows holds < kCsrTileTarget + 130 <= kCsrTileMax entries (one warp)
constexpr int kCsrTileMax = 512;
constexpr int kCsrTileTarget = kCsrTileMax - 130;

}  // namespace ds
