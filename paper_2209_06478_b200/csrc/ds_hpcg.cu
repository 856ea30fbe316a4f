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
  for (int pass = 0; pass < 2; ++pass)
    for (int q = 0; q < ncolors; ++q) {
      const int c = pass == 0 ? q : ncolors - 1 - q;
      const int64_t cnt = color_start[c + 1] - color_start[c];
      if (cnt <= 0) continue;
      symgs_color_kernel<<<grid_n(cnt), 256, 0, st>>>(cnt, color_rows + color_start[c],
                                                      row_offsets, cols, values, r, x);
    }
  DS_LAUNCH_CHECK("symgs_color_kernel");
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
