// ds_hpcg.cu -- HPCG's symmetric Gauss-Seidel smoother and multigrid transfer
// operators (the reference itself has no preconditioner,
// SPEC.md:16, so parity is pinned to the test suite's CPU restatement of HPCG's
// ComputeSYMGS_ref / ComputeMG_ref with an 8-colour ordering).
//
// Colouring: for the 27-point stencil, colour = x%2 + 2(y%2) + 4(z%2) makes
// every pair of coupled rows differ in colour, so all rows of one colour
// relax independently (one thread per row).  Per row the arithmetic is the
// restatement's, operation for operation: s = r[i]; s = s - a_ij*x[j] for j != i
// in stored column order (products rounded, no FMA); x[i] = s / a_ii.
#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

__global__ void symgs_color_kernel(int64_t count, const int* __restrict__ rows,
                                   const int* __restrict__ off, const int* __restrict__ col,
                                   const double* __restrict__ val, const double* __restrict__ r,
                                   double* x) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = rows[k];
    double s = r[i], d = 0.0;
    const int e = off[i + 1];
    for (int q = off[i]; q < e; ++q) {
      const int j = col[q];
      const double a = val[q];
      if (j == i) d = a;
      else s = __dadd_rn(s, -__dmul_rn(a, x[j]));
    }
    x[i] = __ddiv_rn(s, d);
  }
}

// rc[i] = r[f2c[i]] - axf[f2c[i]]   (ComputeRestriction_ref)
__global__ void restrict_kernel(int64_t nc, const int* __restrict__ f2c,
                                const double* __restrict__ r, const double* __restrict__ axf,
                                double* rc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nc;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int f = f2c[i];
    rc[i] = __dadd_rn(r[f], -axf[f]);
  }
}

// x[f2c[i]] += xc[i]   (ComputeProlongation_ref)
__global__ void prolong_kernel(int64_t nc, const int* __restrict__ f2c,
                               const double* __restrict__ xc, double* x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nc;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int f = f2c[i];
    x[f] = __dadd_rn(x[f], xc[i]);
  }
}


// ---- colour-ordered ELL copy of the operator for the sweep -----------------
// Position k (0..n) walks the rows colour by colour (color_rows); slot q of
// position k lives at [q * n + k], so the 32 rows of a warp read each slot
// as one coalesced 256 B (values) / 128 B (columns) segment.  The diagonal is
// held apart (diag[k]); off-diagonals keep their stored order; rows shorter
// than the width are padded with (column i, 0.0) and the padding never enters
// the arithmetic (len[k] predicates it), so the sweep stays bitwise equal to
// the CSR walk.
__global__ void ell_width_kernel(int64_t n, const int* __restrict__ off,
                                 const int* __restrict__ col, int* width) {
  int w = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int q = off[i]; q < off[i + 1]; ++q) c += col[q] != (int)i;
    w = max(w, c);
  }
  for (int o = 16; o; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
  if ((threadIdx.x & 31) == 0) atomicMax(width, w);
}

__global__ void ell_fill_kernel(int64_t n, int width, const int* __restrict__ rows,
                                const int* __restrict__ off, const int* __restrict__ col,
                                const double* __restrict__ val, int* ecol, double* eval,
                                int* elen, double* diag) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = rows[k];
    int q = 0;
    double d = 0.0;
    for (int e = off[i]; e < off[i + 1]; ++e) {
      const int j = col[e];
      if (j == i) { d = val[e]; continue; }
      ecol[(int64_t)q * n + k] = j;
      eval[(int64_t)q * n + k] = val[e];
      ++q;
    }
    elen[k] = q;
    diag[k] = d;
    for (; q < width; ++q) {
      ecol[(int64_t)q * n + k] = i;
      eval[(int64_t)q * n + k] = 0.0;
    }
  }
}

// Slots are processed in chunks of CH: all CH column/value loads, then all CH
// gathers of x, are issued before any arithmetic (compiler barriers keep
// them batched), so each thread has ~2*CH independent loads in flight --
// a colour covers under one wave of the GPU, so the memory-level
// parallelism has to come from inside the thread.
template <int W, int CH>
__device__ __forceinline__ void relax_ell(int64_t n, int64_t k, const int* __restrict__ rows,
                                          const int* __restrict__ ecol,
                                          const double* __restrict__ eval,
                                          const int* __restrict__ elen,
                                          const double* __restrict__ diag,
                                          const double* __restrict__ r, double* x) {
  static_assert(W % CH == 0, "chunk must divide the width");
  const int i = rows[k];
  const int len = elen[k];
  const double dk = diag[k];
  double s = r[i];
#pragma unroll
  for (int c0 = 0; c0 < W; c0 += CH) {
    int j[CH];
    double a[CH], xv[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      j[q] = __ldg(ecol + (int64_t)(c0 + q) * n + k);
      a[q] = __ldg(eval + (int64_t)(c0 + q) * n + k);
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) xv[q] = x[j[q]];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const double t = __dadd_rn(s, -__dmul_rn(a[q], xv[q]));
      s = c0 + q < len ? t : s;
    }
  }
  x[i] = __ddiv_rn(s, dk);
}

// Slots are processed in chunks of CH: the CH column/value loads and then
// the CH gathers of x are independent, so each thread has ~2*CH loads in
// flight -- a colour covers under one wave of the GPU, so the memory-level
// parallelism has to come from inside the thread (MINB steers ptxas towards
// hoisting the loads).
//
// Launched as a programmatic dependent of the previous kernel (the previous
// colour, or the restriction that produced r): a thread first loads what no
// kernel of the sweep writes -- its row index, slot count, diagonal and the
// first chunk of ELL columns / values -- then griddepcontrol.wait()s before
// reading r and x, so the first memory round trip overlaps the previous
// kernel's tail; launch_dependents (after the wait) lets the next colour do
// the same.
template <int W, int CH, int MINB>
__global__ void __launch_bounds__(128, MINB) symgs_ell_kernel(
    int64_t n, int64_t k0, int64_t k1, const int* __restrict__ rows,
    const int* __restrict__ ecol, const double* __restrict__ eval,
    const int* __restrict__ elen, const double* __restrict__ diag,
    const double* __restrict__ r, double* x) {
  static_assert(W % CH == 0, "chunk must divide the width");
  int64_t k = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool first = k < k1;
  int i = 0, len = 0;
  double dk = 1.0;
  int j0[CH];
  double a0[CH];
  if (first) {   // static matrix data only
    i = rows[k];
    len = elen[k];
    dk = diag[k];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      j0[q] = __ldg(ecol + (int64_t)q * n + k);
      a0[q] = __ldg(eval + (int64_t)q * n + k);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // only now let the next colour start its prefetch: triggering at kernel
  // entry lets every colour of the sweep become resident at once, each
  // waiting on the one before (level 1 went 42 -> 69 us)
  asm volatile("griddepcontrol.launch_dependents;");
  if (first) {   // relax_ell with the first chunk already loaded
    double s = r[i];
    double xv[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) xv[q] = x[j0[q]];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      const double t = __dadd_rn(s, -__dmul_rn(a0[q], xv[q]));
      s = q < len ? t : s;
    }
#pragma unroll
    for (int c0 = CH; c0 < W; c0 += CH) {
      int j[CH];
      double a[CH], xw[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        j[q] = __ldg(ecol + (int64_t)(c0 + q) * n + k);
        a[q] = __ldg(eval + (int64_t)(c0 + q) * n + k);
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) xw[q] = x[j[q]];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const double t = __dadd_rn(s, -__dmul_rn(a[q], xw[q]));
        s = c0 + q < len ? t : s;
      }
    }
    x[i] = __ddiv_rn(s, dk);
  }
  for (k += (int64_t)gridDim.x * blockDim.x; k < k1; k += (int64_t)gridDim.x * blockDim.x)
    relax_ell<W, CH>(n, k, rows, ecol, eval, elen, diag, r, x);
}

template <int W, int CH>
static int symgs_ell_launch(unsigned g, int64_t nrows, int64_t k0, int64_t k1,
                            const int32_t* rows, const int32_t* ecol, const double* eval,
                            const int32_t* elen, const double* diag, const double* r, double* x,
                            cudaStream_t st) {
  static int no_pdl = -1;
  if (no_pdl < 0) no_pdl = getenv("DS_NO_PDL") ? 1 : 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(g);
  lc.blockDim = dim3(128);
  lc.dynamicSmemBytes = 0;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&lc, symgs_ell_kernel<W, CH, 8>, nrows, k0, k1, rows, ecol, eval,
                             elen, diag, r, x));
  return DS_OK;
}

// ---- offset ELL: the ELL sweep without column indices --------------------
// For an operator whose off-diagonals fall on at most 32 distinct offsets
// (col - row; the 27-point stencil: 26), slot q of every row is offset q
// (ascending), its value at [q * n + k] (colour-ordered position k, 0.0 where
// the row has no entry there) and a per-position presence mask says which
// slots the row holds.  The column is i + off[q], so the sweep streams 8 B per
// slot instead of the ELL's 12 (level 0 of the 104^3 hierarchy: 243 instead of
// 365 MB per colour pass pair).  Slots are visited in ascending offset = the
// CSR row's stored (ascending column) order and absent ones are selected
// away, so the arithmetic is the ELL / CSR walk's operation for operation.
__global__ void oell_fill_kernel(int64_t n, int W, const int* __restrict__ offs,
                                 const int* __restrict__ rows, const int* __restrict__ off,
                                 const int* __restrict__ col, const double* __restrict__ val,
                                 double* ovals, unsigned* mask, double* diag, int* bad) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = rows[k];
    unsigned m = 0;
    double d = 0.0;
    for (int q = 0; q < W; ++q) ovals[(int64_t)q * n + k] = 0.0;
    int q = 0;
    for (int e = off[i]; e < off[i + 1]; ++e) {
      const int j = col[e];
      if (j == i) {
        d = val[e];
        continue;
      }
      const int o = j - i;
      while (q < W && offs[q] < o) ++q;   // columns ascend, so does the slot
      if (q == W || offs[q] != o || (m >> q) & 1u) {
        *bad = 1;
        break;
      }
      ovals[(int64_t)q * n + k] = val[e];
      m |= 1u << q;
    }
    mask[k] = m;
    diag[k] = d;
  }
}

struct OellOffsets {
  int o[32];
};

template <int W, int CH>
__global__ void __launch_bounds__(128, 8) symgs_oell_kernel(
    int64_t n, int64_t k0, int64_t k1, const OellOffsets offs,
    const int* __restrict__ rows, const double* __restrict__ ovals,
    const unsigned* __restrict__ mask, const double* __restrict__ diag,
    const double* __restrict__ r, double* x) {
  static_assert(W % CH == 0, "chunk must divide the width");
  int64_t k = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t k_first = k;
  int i = 0;
  unsigned m = 0;
  double dk = 1.0;
  double a0[CH];
  if (k < k1) {   // static matrix data only (before the programmatic wait)
    i = rows[k];
    m = mask[k];
    dk = diag[k];
#pragma unroll
    for (int q = 0; q < CH; ++q) a0[q] = __ldg(ovals + (int64_t)q * n + k);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int ni = (int)n;
  for (; k < k1; k += (int64_t)gridDim.x * blockDim.x) {
    if (k != k_first) {
      i = rows[k];
      m = mask[k];
      dk = diag[k];
#pragma unroll
      for (int q = 0; q < CH; ++q) a0[q] = __ldg(ovals + (int64_t)q * n + k);
    }
    double s = r[i];
#pragma unroll
    for (int c0 = 0; c0 < W; c0 += CH) {
      double a[CH], xv[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int c = i + offs.o[c0 + q];   // kernel parameter: constant bank
        xv[q] = x[min(max(c, 0), ni - 1)];
      }
#pragma unroll
      for (int q = 0; q < CH; ++q)
        a[q] = c0 == 0 ? a0[q] : __ldg(ovals + (int64_t)(c0 + q) * n + k);
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const double t = __dadd_rn(s, -__dmul_rn(a[q], xv[q]));
        s = (m >> (c0 + q)) & 1u ? t : s;
      }
    }
    x[i] = __ddiv_rn(s, dk);
  }
}

template <int W, int CH>
static int symgs_oell_launch(unsigned g, int64_t nrows, int64_t k0, int64_t k1,
                             const OellOffsets& offs,
                             const int32_t* rows, const double* ovals, const unsigned* mask,
                             const double* diag, const double* r, double* x, cudaStream_t st) {
  static int no_pdl = -1;
  if (no_pdl < 0) no_pdl = getenv("DS_NO_PDL") ? 1 : 0;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(g);
  lc.blockDim = dim3(128);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  DS_CUDA(cudaLaunchKernelEx(&lc, symgs_oell_kernel<W, CH>, nrows, k0, k1, offs, rows, ovals,
                             mask, diag, r, x));
  return DS_OK;
}

// ---- device-resident PCG scalars (ComputeCG_ref's scalar recurrences) ------
// Tiny single-thread kernels carry the scalar recurrences so an iteration
// never returns to the host and can be captured as a CUDA graph; every
// vector update is guarded by `done`, so replaying past convergence is a
// no-op for x, r and the history.
__global__ void pcg_alpha_kernel(ds_pcg_scalars* s) {
  if (s->done) return;
  if (!(s->pap > 0.0) && s->pap <= 0.0) { s->done = 2; return; }   // p'Ap <= 0
  s->alpha = __ddiv_rn(s->rtz, s->pap);
}

__global__ void pcg_check_kernel(ds_pcg_scalars* s, double* history) {
  if (s->done) return;
  const int it = s->iter + 1;
  s->iter = it;
  const double h = __ddiv_rn(__dsqrt_rn(s->rr), s->scale);
  if (history) history[it] = h;
  if (h <= s->tol) s->done = 1;
  else if (it >= s->max_iters) s->done = 3;
}

__global__ void pcg_beta_kernel(ds_pcg_scalars* s) {
  if (s->done) return;
  s->beta = __ddiv_rn(s->rtz_new, s->rtz);
  s->rtz = s->rtz_new;
}

// w = 1.0*x + c*y with c = +-(*coef)   (waxpby, two rounded products)
__global__ void pcg_axpy_kernel(int64_t n, double* w, const double* x, const double* coef,
                                int negate, const double* y, const int* done) {
  if (*done) return;
  const double c = negate ? -*coef : *coef;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __dadd_rn(__dmul_rn(1.0, x[i]), __dmul_rn(c, y[i]));
}

// The symmetric sweep visits colours 0..C-1 then C-1..0.  The two visits of
// colour C-1 are back to back with no other colour updated in between, and a
// row never reads its own colour, so the second visit recomputes identical
// bits: it is skipped (2C-1 passes, not 2C).
static inline int sweep_color(int q, int ncolors) {
  return q < ncolors ? q : 2 * ncolors - 2 - q;
}

// ---- fused residual + restriction for a DIA level operator -----------------
// rc[i] = r[f] - (A z)[f] with f = f2c[i]: only the coarse points' rows of
// A z are formed (1/8 of the SpMV), each with the DIA SpMV's exact order --
// sequential over the in-range diagonals from +0.0 -- so rc is bitwise the
// SpMV-then-restrict result.
template <int ND>
__global__ void __launch_bounds__(256) dia_restrict_kernel(
    int64_t nc, const int* __restrict__ f2c, int64_t ncols, int ndiags_rt,
    const int* __restrict__ offsets, const double* __restrict__ vals,
    const double* __restrict__ z, const double* __restrict__ r, double* rc) {
  const int nd = ND > 0 ? ND : ndiags_rt;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nc;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = f2c[i];
    const double* v = vals + f * nd;
    double acc = 0.0;
#pragma unroll 9
    for (int j = 0; j < nd; ++j) {
      const int64_t c = f + __ldg(offsets + j);
      const bool in = c >= 0 && c < ncols;
      const double p = __dmul_rn(__ldg(v + j), z[in ? c : f]);
      acc = in ? __dadd_rn(acc, p) : acc;
    }
    rc[i] = __dadd_rn(r[f], -acc);
  }
}

static unsigned grid_n(int64_t n) {
  int64_t g = ceil_div(n, 256);
  const int64_t cap = (int64_t)sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace ds

using namespace ds;

extern "C" int ds_symgs(int64_t nrows, const int32_t* row_offsets, const int32_t* cols,
                        const double* values, const int32_t* color_rows,
                        const int64_t* color_start, int ncolors, const double* r, double* x,
                        void* stream) {
  (void)nrows;
  cudaStream_t st = as_stream(stream);
  for (int q = 0; q < 2 * ncolors - 1; ++q) {
    const int c = sweep_color(q, ncolors);
    const int64_t cnt = color_start[c + 1] - color_start[c];
    if (cnt <= 0) continue;
    symgs_color_kernel<<<grid_n(cnt), 256, 0, st>>>(cnt, color_rows + color_start[c],
                                                    row_offsets, cols, values, r, x);
  }
  DS_LAUNCH_CHECK("symgs_color_kernel");
  return DS_OK;
}


extern "C" int ds_symgs_ell_width(int64_t nrows, const int32_t* row_offsets, const int32_t* cols,
                                  int32_t* width_out, void* stream) {
  if (!width_out) { set_error("ds_symgs_ell_width: width_out is NULL"); return DS_ERR_INVALID_ARGUMENT; }
  *width_out = 0;
  if (nrows <= 0) return DS_OK;
  cudaStream_t st = as_stream(stream);
  int* dw = nullptr;
  DS_CUDA(cudaMallocAsync(&dw, sizeof(int), st));
  DS_CUDA(cudaMemsetAsync(dw, 0, sizeof(int), st));
  ell_width_kernel<<<grid_n(nrows), 256, 0, st>>>(nrows, row_offsets, cols, dw);
  DS_LAUNCH_CHECK("ell_width_kernel");
  int w = 0;
  DS_CUDA(cudaMemcpyAsync(&w, dw, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(dw, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *width_out = w;
  return DS_OK;
}

extern "C" int ds_symgs_ell_fill(int64_t nrows, int32_t width, const int32_t* row_offsets,
                                 const int32_t* cols, const double* values,
                                 const int32_t* color_rows, int32_t* ell_cols, double* ell_vals,
                                 int32_t* ell_len, double* diag, void* stream) {
  if (nrows <= 0) return DS_OK;
  ell_fill_kernel<<<grid_n(nrows), 256, 0, as_stream(stream)>>>(
      nrows, width, color_rows, row_offsets, cols, values, ell_cols, ell_vals, ell_len, diag);
  DS_LAUNCH_CHECK("ell_fill_kernel");
  return DS_OK;
}

extern "C" int ds_symgs_ell(int64_t nrows, int32_t width, const int32_t* color_rows,
                            const int64_t* color_start, int ncolors, const int32_t* ell_cols,
                            const double* ell_vals, const int32_t* ell_len, const double* diag,
                            const double* r, double* x, void* stream) {
  cudaStream_t st = as_stream(stream);
  const int wt = width <= 8 ? 8 : width <= 16 ? 16 : width <= 26 ? 26 : width <= 32 ? 32 : -1;
  if (wt != width) {
    set_error("ds_symgs_ell: width %d must be one of 8, 16, 26, 32 (pad the layout)", width);
    return DS_ERR_NOT_SUPPORTED;
  }
  int rc = DS_OK;
  for (int q = 0; q < 2 * ncolors - 1; ++q) {
    const int c = sweep_color(q, ncolors);
    const int64_t k0 = color_start[c], k1 = color_start[c + 1];
    if (k1 <= k0) continue;
    const unsigned g = (unsigned)min64(ceil_div(k1 - k0, 128), (int64_t)sm_count() * 32);
#define DS_SYMGS_LAUNCH(W_, CH_)                                                           \
  rc = symgs_ell_launch<W_, CH_>(g, nrows, k0, k1, color_rows, ell_cols, ell_vals, ell_len, \
                                 diag, r, x, st)
    switch (width) {
      case 8: DS_SYMGS_LAUNCH(8, 8); break;
      case 16: DS_SYMGS_LAUNCH(16, 8); break;
      case 26: DS_SYMGS_LAUNCH(26, 13); break;
      default: DS_SYMGS_LAUNCH(32, 8); break;
    }
#undef DS_SYMGS_LAUNCH
    if (rc) return rc;
  }
  DS_LAUNCH_CHECK("symgs_ell_kernel");
  return DS_OK;
}

extern "C" int ds_pcg_alpha(ds_pcg_scalars* s, void* stream) {
  pcg_alpha_kernel<<<1, 1, 0, as_stream(stream)>>>(s);
  DS_LAUNCH_CHECK("pcg_alpha_kernel");
  return DS_OK;
}

extern "C" int ds_pcg_check(ds_pcg_scalars* s, double* history, void* stream) {
  pcg_check_kernel<<<1, 1, 0, as_stream(stream)>>>(s, history);
  DS_LAUNCH_CHECK("pcg_check_kernel");
  return DS_OK;
}

extern "C" int ds_pcg_beta(ds_pcg_scalars* s, void* stream) {
  pcg_beta_kernel<<<1, 1, 0, as_stream(stream)>>>(s);
  DS_LAUNCH_CHECK("pcg_beta_kernel");
  return DS_OK;
}

extern "C" int ds_pcg_axpy(int64_t n, double* w, const double* x, const double* coef_dev,
                           int negate, const double* y, const ds_pcg_scalars* s, void* stream) {
  if (n <= 0) return DS_OK;
  pcg_axpy_kernel<<<grid_n(n), 256, 0, as_stream(stream)>>>(n, w, x, coef_dev, negate, y,
                                                            &s->done);
  DS_LAUNCH_CHECK("pcg_axpy_kernel");
  return DS_OK;
}

extern "C" int ds_mg_restrict_residual(const ds_matrix* a, int64_t ncoarse, const int32_t* f2c,
                                       const double* z, const double* r, double* rc,
                                       void* stream) {
  if (!a || a->format != DS_FMT_DIA) {
    set_error("ds_mg_restrict_residual: the level operator must be DIA");
    return DS_ERR_NOT_SUPPORTED;
  }
  if (ncoarse <= 0) return DS_OK;
  cudaStream_t st = as_stream(stream);
  if (a->ndiags == 27)
    dia_restrict_kernel<27><<<grid_n(ncoarse), 256, 0, st>>>(
        ncoarse, f2c, a->ncols, 27, a->idx0, a->values, z, r, rc);
  else
    dia_restrict_kernel<0><<<grid_n(ncoarse), 256, 0, st>>>(
        ncoarse, f2c, a->ncols, a->ndiags, a->idx0, a->values, z, r, rc);
  DS_LAUNCH_CHECK("dia_restrict_kernel");
  return DS_OK;
}

extern "C" int ds_mg_restrict(int64_t ncoarse, const int32_t* f2c, const double* r,
                              const double* axf, double* rc, void* stream) {
  if (ncoarse <= 0) return DS_OK;
  restrict_kernel<<<grid_n(ncoarse), 256, 0, as_stream(stream)>>>(ncoarse, f2c, r, axf, rc);
  DS_LAUNCH_CHECK("restrict_kernel");
  return DS_OK;
}

extern "C" int ds_mg_prolong(int64_t ncoarse, const int32_t* f2c, const double* xc, double* x,
                             void* stream) {
  if (ncoarse <= 0) return DS_OK;
  prolong_kernel<<<grid_n(ncoarse), 256, 0, as_stream(stream)>>>(ncoarse, f2c, xc, x);
  DS_LAUNCH_CHECK("prolong_kernel");
  return DS_OK;
}

extern "C" int ds_symgs_oell_fill(int64_t nrows, int32_t width, const int32_t* offsets,
                                  const int32_t* row_offsets, const int32_t* cols,
                                  const double* values, const int32_t* color_rows,
                                  double* oell_vals, uint32_t* mask, double* diag, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (nrows <= 0) return DS_OK;
  if (width != 26 && width != 32) {
    set_error("ds_symgs_oell_fill: width %d must be 26 or 32", width);
    return DS_ERR_NOT_SUPPORTED;
  }
  int* bad = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), st));
  DS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  oell_fill_kernel<<<grid_n(nrows), 256, 0, st>>>(nrows, width, offsets, color_rows, row_offsets,
                                                   cols, values, oell_vals, mask, diag, bad);
  DS_LAUNCH_CHECK("oell_fill_kernel");
  int h = 0;
  DS_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(bad, st));
  DS_CUDA(cudaStreamSynchronize(st));
  if (h) {
    set_error("ds_symgs_oell_fill: a row holds an offset outside the list (or a duplicate)");
    return DS_ERR_NOT_SUPPORTED;
  }
  return DS_OK;
}

extern "C" int ds_symgs_oell(int64_t nrows, int32_t width, const int32_t* offsets_host,
                             const int32_t* color_rows, const int64_t* color_start, int ncolors,
                             const double* oell_vals, const uint32_t* mask, const double* diag,
                             const double* r, double* x, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (width != 26 && width != 32) {
    set_error("ds_symgs_oell: width %d must be 26 or 32", width);
    return DS_ERR_NOT_SUPPORTED;
  }
  OellOffsets offsets{};
  for (int q = 0; q < width; ++q) offsets.o[q] = offsets_host[q];
  int rc = DS_OK;
  for (int q = 0; q < 2 * ncolors - 1; ++q) {
    const int c = sweep_color(q, ncolors);
    const int64_t k0 = color_start[c], k1 = color_start[c + 1];
    if (k1 <= k0) continue;
    const unsigned g = (unsigned)min64(ceil_div(k1 - k0, 128), (int64_t)sm_count() * 32);
    rc = width == 26 ? symgs_oell_launch<26, 13>(g, nrows, k0, k1, offsets, color_rows, oell_vals,
                                                 mask, diag, r, x, st)
                     : symgs_oell_launch<32, 8>(g, nrows, k0, k1, offsets, color_rows, oell_vals,
                                                mask, diag, r, x, st);
    if (rc) return rc;
  }
  DS_LAUNCH_CHECK("symgs_oell_kernel");
  return DS_OK;
}
