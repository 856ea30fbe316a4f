// ds_vector.cu -- dense-vector kernels, diagonal helpers, halo gather and the
// CG building blocks (kernels.py:205-337, stencil.py:280-295, solver.py:56-189).
#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

constexpr int kVecBlock = 256;

static unsigned grid_for(int64_t n, int per_thread = 4) {
  int64_t g = ceil_div(n, (int64_t)kVecBlock * per_thread);
  const int64_t cap = (int64_t)sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ------------------------------------------------------------------ dot ----
// Fixed-order reduction: thread t of block b sums i = b*B + t (+ grid stride)
// sequentially, blocks reduce with a fixed tree, the last block sums the
// block partials in a fixed tree.  Same n -> same bits, every run.
__global__ void __launch_bounds__(kVecBlock)
    dot_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b, DotOut d) {
  if (d.skip()) return;
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kVecBlock)
    v = add(v, mul(a[i], b[i]));
  d.finish_block<kVecBlock>(v);
}

int launch_dot(int64_t n, const double* a, const double* b, const DotOut& d, cudaStream_t st) {
  int64_t g = ceil_div(n, (int64_t)kVecBlock * 8);
  if (g < 1) g = 1;
  if (g > 1024) g = 1024;  // a function of n only: reproducible across devices
  g = d.clamp_grid(g);
  dot_kernel<<<(unsigned)g, kVecBlock, 0, st>>>(n, a, b, d);
  DS_LAUNCH_CHECK("dot_kernel");
  return DS_OK;
}

// workspace layout: [ticket (16 B)] [partials kMaxPartials doubles]
struct Workspace {
  unsigned* ticket;
  double* partials;
  explicit Workspace(void* w)
      : ticket(reinterpret_cast<unsigned*>(w)),
        partials(reinterpret_cast<double*>(reinterpret_cast<char*>(w) + 16)) {}
};
constexpr int64_t kWorkspaceBytes = 16 + (int64_t)kMaxPartials * 8;

// --------------------------------------------------------------- waxpby ----
// w = alpha*x + beta*y with both products rounded (numpy evaluates
// alpha * x and beta * y into temporaries, kernels.py:219).  w may alias.
__global__ void __launch_bounds__(kVecBlock)
    waxpby_kernel(int64_t n, double alpha, const double* x, double beta, const double* y,
                  double* w, const int* guard) {
  if (guard && *guard) return;
  for (int64_t i = (int64_t)blockIdx.x * kVecBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kVecBlock)
    w[i] = add(mul(alpha, x[i]), mul(beta, y[i]));
}

// ----------------------------------------------------------------- scan ----
// np.cumsum is strictly sequential; reproduce it exactly: one thread carries
// the running sum while the block stages tiles through shared memory.
constexpr int kScanTile = 4096;
__global__ void __launch_bounds__(kVecBlock)
    scan_seq_kernel(int64_t n, const double* __restrict__ x, double* out, double* total) {
  __shared__ double buf[kScanTile];
  double acc = 0.0;
  for (int64_t t0 = 0; t0 < n; t0 += kScanTile) {
    const int cnt = (int)min64(kScanTile, n - t0);
    for (int k = threadIdx.x; k < cnt; k += kVecBlock) buf[k] = x[t0 + k];
    __syncthreads();
    if (threadIdx.x == 0) {
      int k = 0;
      if (t0 == 0) {
        acc = buf[0];  // out[0] = x[0]
        k = 1;
      }
      for (; k < cnt; ++k) {
        acc = add(acc, buf[k]);
        buf[k] = acc;
      }
    }
    __syncthreads();
    if (out)
      for (int k = threadIdx.x; k < cnt; k += kVecBlock) out[t0 + k] = buf[k];
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = (n > 0) ? acc : 0.0;
}

// --------------------------------------------------------------- gather ----
__global__ void gather_kernel(int64_t count, const int* __restrict__ idx,
                              const double* __restrict__ src, double* __restrict__ dst,
                              const int* guard) {
  if (guard && *guard) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[idx[k]];
}

// ------------------------------------------------------------- diagonal ----
__global__ void extract_diag_csr_kernel(int n, const int* __restrict__ off,
                                        const int* __restrict__ col,
                                        const double* __restrict__ val, double* out) {
  // out[rows[hit]] = values[hit]: with repeated (i,i) the last stored wins
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int k = off[i]; k < off[i + 1]; ++k)
      if (col[k] == i) v = val[k];
    out[i] = v;
  }
}

__global__ void csr_diag_presence(int n, const int* __restrict__ off, const int* __restrict__ col,
                                  long long* first_missing) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    bool hit = false;
    for (int k = off[i]; k < off[i + 1] && !hit; ++k) hit = (col[k] == i);
    if (!hit) atomicMin(first_missing, (long long)i);
  }
}

__global__ void update_diag_csr_kernel(int nrows, int n, const int* __restrict__ off,
                                       const int* __restrict__ col, double* val,
                                       const double* __restrict__ d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows && i < n;
       i += gridDim.x * blockDim.x)
    for (int k = off[i]; k < off[i + 1]; ++k)
      if (col[k] == i) val[k] = d[i];
}

// COO: per-row count of diagonal entries and first occurrence index
__global__ void coo_diag_scan(int64_t nnz, int n, const int* __restrict__ rows,
                              const int* __restrict__ cols, int* count, int* first) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = rows[k];
    if (r == cols[k] && r < n) {
      atomicAdd(count + r, 1);
      atomicMin(first + r, (int)k);
    }
  }
}
__global__ void coo_diag_missing(int n, const int* __restrict__ count, long long* first_missing,
                                 int* maxcount) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = count[i];
    if (c == 0) atomicMin(first_missing, (long long)i);
    atomicMax(maxcount, c);
  }
}
// extract with <= 2 duplicates per row: 0 + a + b is order independent
__global__ void coo_extract_atomic(int64_t nnz, int n, const int* __restrict__ rows,
                                   const int* __restrict__ cols, const double* __restrict__ val,
                                   double* out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = rows[k];
    if (r == cols[k] && r < n) atomicAdd(out + r, val[k]);
  }
}
// general case: sequential in stored order (np.bincount)
__global__ void coo_extract_serial(int64_t nnz, int n, const int* __restrict__ rows,
                                   const int* __restrict__ cols, const double* __restrict__ val,
                                   double* out) {
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int64_t k = 0; k < nnz; ++k) {
      const int r = rows[k];
      if (r == cols[k] && r < n) out[r] = add(out[r], val[k]);
    }
}
__global__ void coo_update_kernel(int64_t nnz, int n, const int* __restrict__ rows,
                                  const int* __restrict__ cols, double* val,
                                  const int* __restrict__ first, const double* __restrict__ d) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = rows[k];
    if (r == cols[k] && r < n) val[k] = (first[r] == (int)k) ? d[r] : 0.0;
  }
}
__global__ void fill_i32(int64_t n, int* p, int v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void fill_f64_plain(int64_t n, double* p, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void dia_diag_column_kernel(int64_t n, int nd, int j0, double* vals, double* vec,
                                       int dir) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (dir == 0) vec[i] = vals[i * nd + j0];
    else vals[i * nd + j0] = vec[i];
  }
}

// nonzero in-range slots: one warp per row, lane j checks slot j (no 64-bit
// divisions; the row's nd values are one coalesced 8*nd-byte segment)
__global__ void dia_nonzero_kernel(int nrows, int ncols, int nd, const int* __restrict__ off,
                                   const double* __restrict__ vals, unsigned long long* count) {
  unsigned long long c = 0;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nrows; i += warps)
    for (int j = lane; j < nd; j += 32) {
      const int64_t c0 = i + off[j];
      if (c0 >= 0 && c0 < ncols && vals[i * nd + j] != 0.0) ++c;
    }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// ------------------------------------------------------------------- CG ----
// setup: r = 1*b + (-1)*ap ; p = 1*r + 0*r ; partial b.b and r.r
__global__ void __launch_bounds__(kVecBlock)
    cg_setup_kernel(int64_t n, const double* __restrict__ b, const double* __restrict__ ap,
                    double* r, double* p, DotOut dbb, DotOut drr) {
  double vb = 0.0, vr = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kVecBlock) {
    const double bi = b[i];
    const double ri = add(mul(1.0, bi), mul(-1.0, ap[i]));
    r[i] = ri;
    p[i] = add(mul(1.0, ri), mul(0.0, ri));
    vb = add(vb, mul(bi, bi));
    vr = add(vr, mul(ri, ri));
  }
  // two reductions share one launch: separate tickets/partials
  dbb.finish_block<kVecBlock>(vb);
  drr.finish_block<kVecBlock>(vr);
}

__global__ void cg_setup_finalize_kernel(ds_cg_scalars* s, const double* bb_parts,
                                         const double* rr_parts, int nparts, double tol,
                                         int max_iters, double* history) {
  s->tol = tol;
  s->max_iters = max_iters;
  s->bb = ordered_sum(bb_parts, nparts);
  s->alpha = s->beta = s->pap = s->rr_new = 0.0;
  cg_finalize(kStageSetup, s, history, rr_parts, nparts);
}

// x = 1*x + alpha*p ; r = 1*r + (-alpha)*ap ; partial r.r   (solver.py:177-180)
// VEC: 16-B aligned operands, element pairs (LDG.128), U pairs per thread and
// iteration with every load issued before any use; the odd tail element is
// folded in by the first thread after its pairs.  Grid = 4 CTAs per SM: few
// partials for the fused reduction, all loads of a sweep in flight.
constexpr int kVecUnroll = 4;

template <bool VEC>
__global__ void __launch_bounds__(kVecBlock)
    cg_update_kernel(int64_t n, double* x, double* r, const double* __restrict__ p,
                     const double* __restrict__ ap, const ds_cg_scalars* s, DotOut d) {
  if (d.skip()) return;
  const double alpha = s->alpha;
  const double nalpha = -alpha;
  double v = 0.0;
  const int64_t gtid = (int64_t)blockIdx.x * kVecBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kVecBlock;
  if (VEC) {
    const int64_t n2 = n >> 1;
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* a2 = reinterpret_cast<const double2*>(ap);
    for (int64_t i0 = gtid; i0 < n2; i0 += stride * kVecUnroll) {
      double2 xv[kVecUnroll], rv[kVecUnroll], pv[kVecUnroll], av[kVecUnroll];
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = min64(i0 + u * stride, n2 - 1);
        xv[u] = x2[i];
        rv[u] = r2[i];
        pv[u] = p2[i];
        av[u] = a2[i];
      }
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < n2) {
          double2 xo, ro;
          xo.x = add(mul(1.0, xv[u].x), mul(alpha, pv[u].x));
          xo.y = add(mul(1.0, xv[u].y), mul(alpha, pv[u].y));
          ro.x = add(mul(1.0, rv[u].x), mul(nalpha, av[u].x));
          ro.y = add(mul(1.0, rv[u].y), mul(nalpha, av[u].y));
          x2[i] = xo;
          r2[i] = ro;
          v = add(v, mul(ro.x, ro.x));
          v = add(v, mul(ro.y, ro.y));
        }
      }
    }
    if ((n & 1) && gtid == 0) {
      const int64_t i = n - 1;
      x[i] = add(mul(1.0, x[i]), mul(alpha, p[i]));
      const double ri = add(mul(1.0, r[i]), mul(nalpha, ap[i]));
      r[i] = ri;
      v = add(v, mul(ri, ri));
    }
  } else {
    for (int64_t i = gtid; i < n; i += stride) {
      x[i] = add(mul(1.0, x[i]), mul(alpha, p[i]));
      const double ri = add(mul(1.0, r[i]), mul(nalpha, ap[i]));
      r[i] = ri;
      v = add(v, mul(ri, ri));
    }
  }
  d.finish_block<kVecBlock>(v);
}

// p = 1*r + beta*p  (solver.py:185-188)
template <bool VEC>
__global__ void __launch_bounds__(kVecBlock)
    cg_direction_kernel(int64_t n, const double* __restrict__ r, double* p,
                        const ds_cg_scalars* s) {
  if (s->done) return;
  const double beta = s->beta;
  const int64_t gtid = (int64_t)blockIdx.x * kVecBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kVecBlock;
  if (VEC) {
    const int64_t n2 = n >> 1;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double2* p2 = reinterpret_cast<double2*>(p);
    for (int64_t i0 = gtid; i0 < n2; i0 += stride * kVecUnroll) {
      double2 rv[kVecUnroll], pv[kVecUnroll];
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = min64(i0 + u * stride, n2 - 1);
        rv[u] = r2[i];
        pv[u] = p2[i];
      }
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < n2) {
          double2 o;
          o.x = add(mul(1.0, rv[u].x), mul(beta, pv[u].x));
          o.y = add(mul(1.0, rv[u].y), mul(beta, pv[u].y));
          p2[i] = o;
        }
      }
    }
    if ((n & 1) && gtid == 0) p[n - 1] = add(mul(1.0, r[n - 1]), mul(beta, p[n - 1]));
  } else {
    for (int64_t i = gtid; i < n; i += stride) p[i] = add(mul(1.0, r[i]), mul(beta, p[i]));
  }
}

static bool aligned16(const void* a, const void* b = nullptr, const void* c = nullptr,
                      const void* d = nullptr) {
  auto ok = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return ok(a) && ok(b) && ok(c) && ok(d);
}

// grid of the streaming vector kernels: 4 resident CTAs per SM (592
// partials for the fused reductions -- thousands of CTAs made the
// same-address completion tickets the bottleneck), kVecUnroll pairs per
// thread in flight
static unsigned vec_grid(int64_t n) {
  int64_t g = ceil_div(n, (int64_t)kVecBlock * 2 * kVecUnroll);
  const int64_t cap = (int64_t)sm_count() * 4;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ---- deferred-reduction single-partition iteration -------------------------
// update: prologue reduces the SpMV's p.Ap partials -> alpha (or breakdown);
// body = cg_update (x, r, partial r.r written without a ticket)
// gathered mode (nparts > 0): the inputs are the P all-gathered partition
// dots, summed sequentially in rank order (solver.py:140-141); the output
// partial goes through the completion-ticket DotOut (one partition total).
__device__ __forceinline__ double gathered_sum(const double* parts, int nparts) {
  __shared__ double s_g;
  if (threadIdx.x == 0) s_g = ordered_sum(parts, nparts);
  __syncthreads();
  return s_g;
}

template <bool VEC>
__global__ void __launch_bounds__(kVecBlock)
    cg_update_deferred_kernel(int64_t n, double* x, double* r, const double* __restrict__ p,
                              const double* __restrict__ ap, ds_cg_scalars* s,
                              const double* pap_parts, const unsigned* pap_count,
                              double* rr_parts, unsigned* rr_count, int nparts, DotOut rr_out) {
  __shared__ double sh[32];
  if (s->done) return;
  const double pap = nparts > 0 ? gathered_sum(pap_parts, nparts)
                                : reduce_partials<kVecBlock>(pap_parts, pap_count, sh);
  if (pap <= 0.0) {  // breakdown: every block sees the same pap
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s->pap = pap;
      s->done = 2;
    }
    return;
  }
  const double rr = s->rr;
  const double alpha = rr / pap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->pap = pap;
    s->alpha = alpha;
    s->rr_used = rr;
    s->iter_next = s->iter + 1;
  }
  const double nalpha = -alpha;
  double v = 0.0;
  const int64_t gtid = (int64_t)blockIdx.x * kVecBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kVecBlock;
  if (VEC) {
    const int64_t n2 = n >> 1;
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* a2 = reinterpret_cast<const double2*>(ap);
    for (int64_t i0 = gtid; i0 < n2; i0 += stride * kVecUnroll) {
      double2 xv[kVecUnroll], rv[kVecUnroll], pv[kVecUnroll], av[kVecUnroll];
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = min64(i0 + u * stride, n2 - 1);
        xv[u] = x2[i];
        rv[u] = r2[i];
        pv[u] = p2[i];
        av[u] = a2[i];
      }
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < n2) {
          double2 xo, ro;
          xo.x = add(mul(1.0, xv[u].x), mul(alpha, pv[u].x));
          xo.y = add(mul(1.0, xv[u].y), mul(alpha, pv[u].y));
          ro.x = add(mul(1.0, rv[u].x), mul(nalpha, av[u].x));
          ro.y = add(mul(1.0, rv[u].y), mul(nalpha, av[u].y));
          x2[i] = xo;
          r2[i] = ro;
          v = add(v, mul(ro.x, ro.x));
          v = add(v, mul(ro.y, ro.y));
        }
      }
    }
    if ((n & 1) && gtid == 0) {
      const int64_t i = n - 1;
      x[i] = add(mul(1.0, x[i]), mul(alpha, p[i]));
      const double ri = add(mul(1.0, r[i]), mul(nalpha, ap[i]));
      r[i] = ri;
      v = add(v, mul(ri, ri));
    }
  } else {
    for (int64_t i = gtid; i < n; i += stride) {
      x[i] = add(mul(1.0, x[i]), mul(alpha, p[i]));
      const double ri = add(mul(1.0, r[i]), mul(nalpha, ap[i]));
      r[i] = ri;
      v = add(v, mul(ri, ri));
    }
  }
  if (nparts > 0) {
    rr_out.finish_block<kVecBlock>(v);   // this partition's r.r -> all-gather
    return;
  }
  v = block_sum<kVecBlock>(v, sh);
  if (threadIdx.x == 0) {
    rr_parts[blockIdx.x] = v;
    if (blockIdx.x == 0) *rr_count = gridDim.x;
  }
}

// direction: prologue reduces the r.r partials -> history, convergence, beta;
// body p = 1*r + beta*p (skipped when converged / at max_iters, like the
// reference's break before the p update, solver.py:182-188)
template <bool VEC>
__global__ void __launch_bounds__(kVecBlock)
    cg_direction_deferred_kernel(int64_t n, const double* __restrict__ r, double* p,
                                 ds_cg_scalars* s, double* history, const double* rr_parts,
                                 const unsigned* rr_count, int nparts) {
  __shared__ double sh[32];
  if (s->done) return;
  const double rr_new = nparts > 0 ? gathered_sum(rr_parts, nparts)
                                   : reduce_partials<kVecBlock>(rr_parts, rr_count, sh);
  const int it = s->iter_next;
  const double h = sqrt(rr_new) / s->scale;
  const bool converged = h <= s->tol;
  const bool last = it >= s->max_iters;
  const double beta = rr_new / s->rr_used;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    history[it] = h;
    s->iter = it;
    s->rr_new = rr_new;
    if (converged) s->done = 1;
    else if (last) s->done = 3;
    else {
      s->beta = beta;
      s->rr = rr_new;
    }
  }
  if (converged || last) return;
  const int64_t gtid = (int64_t)blockIdx.x * kVecBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kVecBlock;
  if (VEC) {
    const int64_t n2 = n >> 1;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double2* p2 = reinterpret_cast<double2*>(p);
    for (int64_t i0 = gtid; i0 < n2; i0 += stride * kVecUnroll) {
      double2 rv[kVecUnroll], pv[kVecUnroll];
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = min64(i0 + u * stride, n2 - 1);
        rv[u] = r2[i];
        pv[u] = p2[i];
      }
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) {
        const int64_t i = i0 + u * stride;
        if (i < n2) {
          double2 o;
          o.x = add(mul(1.0, rv[u].x), mul(beta, pv[u].x));
          o.y = add(mul(1.0, rv[u].y), mul(beta, pv[u].y));
          p2[i] = o;
        }
      }
    }
    if ((n & 1) && gtid == 0) p[n - 1] = add(mul(1.0, r[n - 1]), mul(beta, p[n - 1]));
  } else {
    for (int64_t i = gtid; i < n; i += stride) p[i] = add(mul(1.0, r[i]), mul(beta, p[i]));
  }
}

__global__ void cg_finalize_kernel(int stage, ds_cg_scalars* s, double* history,
                                   const double* parts, int nparts) {
  cg_finalize(stage, s, history, parts, nparts);
}


// ---- fused update + direction (single partition, deferred) ----------------
// One persistent launch per CG iteration tail: the update (x += alpha p,
// r -= alpha Ap, block r.r partials), a grid-wide barrier, then every block
// reduces the r.r partials in the same fixed order (history, convergence,
// beta) and applies p = r + beta p -- r and p are re-read from L2, where the
// update left them.  Saves the direction kernel's launch and its DRAM re-read
// of r and p.  The grid is sized to be co-resident (occupancy query) and is
// launched cooperatively when the driver accepts that, so the barrier cannot
// deadlock.  Same arithmetic per element as the two kernels; the r.r tree
// differs only through the grid size (any fixed tree is within the dot
// tolerance, and it is fixed for a given device).
// Grid barrier: thread 0 of every block arrives with an acq_rel atomic (its
// release covers the block's writes before the preceding __syncthreads, e.g.
// the r.r partial) and spins with acquire loads on the generation word; the
// last arrival resets the count and publishes the next generation with a
// release store.  No full fences (round 1's __threadfence version: +0.3 us per
// CG step, A/B on one box).
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

template <int U, int MINB>
__global__ void __launch_bounds__(kVecBlock, MINB)
    cg_update_direction_fused_kernel(int64_t n, double* x, double* r, double* p,
                                     const double* __restrict__ ap, ds_cg_scalars* s,
                                     double* history, const double* pap_parts,
                                     const unsigned* pap_count, double* rr_parts,
                                     unsigned* bar_count, unsigned* bar_gen) {
  __shared__ double sh[32];
  // Phase 1 (update): r -= alpha Ap and the block r.r partials; phase 2
  // (after the grid barrier): x += alpha p with the OLD p and p = r + beta p,
  // so x and p are read once, in the same sweep (8 vector passes, was 9:
  // phase 1 used to update x too, reading p twice).  Launched as a
  // programmatic dependent of the SpMV: before griddepcontrol.wait it reads
  // only s->done and the first sweep's r, which the SpMV does not write.
  if (s->done) return;
  const int64_t gtid = (int64_t)blockIdx.x * kVecBlock + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kVecBlock;
  const int64_t n2 = n >> 1;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* p2 = reinterpret_cast<double2*>(p);
  const double2* a2 = reinterpret_cast<const double2*>(ap);
  double2 xv[U], rv[U], pv[U], av[U];
#pragma unroll
  for (int u = 0; u < U; ++u) rv[u] = r2[min64(gtid + u * stride, n2 - 1)];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the first sweep's Ap flies during the pAp partials reduction
#pragma unroll
  for (int u = 0; u < U; ++u) av[u] = a2[min64(gtid + u * stride, n2 - 1)];
  const double pap = reduce_partials<kVecBlock>(pap_parts, pap_count, sh);
  if (pap <= 0.0) {  // breakdown: every block sees the same pap
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s->pap = pap;
      s->done = 2;
    }
    return;
  }
  const double rr = s->rr;
  const double alpha = rr / pap, nalpha = -alpha;
  const int it = s->iter + 1;
  double v = 0.0;
  for (int64_t i0 = gtid; i0 < n2; i0 += stride * U) {
    if (i0 != gtid) {   // the first sweep's r and Ap are already loaded
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = min64(i0 + u * stride, n2 - 1);
        rv[u] = r2[i];
        av[u] = a2[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n2) {
        double2 ro;
        ro.x = add(mul(1.0, rv[u].x), mul(nalpha, av[u].x));
        ro.y = add(mul(1.0, rv[u].y), mul(nalpha, av[u].y));
        r2[i] = ro;
        v = add(v, mul(ro.x, ro.x));
        v = add(v, mul(ro.y, ro.y));
      }
    }
  }
  if ((n & 1) && gtid == 0) {
    const int64_t i = n - 1;
    const double ri = add(mul(1.0, r[i]), mul(nalpha, ap[i]));
    r[i] = ri;
    v = add(v, mul(ri, ri));
  }
  v = block_sum<kVecBlock>(v, sh);
  if (threadIdx.x == 0) rr_parts[blockIdx.x] = v;
  // x and p of the first phase-2 sweep fly during the barrier (neither is
  // written before it)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = min64(gtid + u * stride, n2 - 1);
    xv[u] = x2[i];
    pv[u] = p2[i];
  }
  grid_barrier(bar_count, bar_gen);
  // the next SpMV (launched with programmatic stream serialization) may now
  // be scheduled: it prefetches matrix tiles and waits for this grid before
  // reading p
  asm volatile("griddepcontrol.launch_dependents;");
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kVecBlock) t = add(t, __ldcg(rr_parts + i));
  t = block_sum<kVecBlock>(t, sh);
  __shared__ double s_rr;
  if (threadIdx.x == 0) s_rr = t;
  __syncthreads();
  const double rr_new = s_rr;
  const double h = sqrt(rr_new) / s->scale;
  const bool converged = h <= s->tol;
  const bool last = it >= s->max_iters;
  const double beta = rr_new / rr;
  // every block has read s->rr / s->iter above; block 0 publishes after the
  // barrier, so no block can observe a half-updated scalar block
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->pap = pap;
    s->alpha = alpha;
    s->rr_used = rr;
    s->iter_next = it;
    history[it] = h;
    s->iter = it;
    s->rr_new = rr_new;
    if (converged) s->done = 1;
    else if (last) s->done = 3;
    else {
      s->beta = beta;
      s->rr = rr_new;
    }
  }
  const bool stop = converged || last;   // x still takes this step; p stays
  for (int64_t i0 = gtid; i0 < n2; i0 += stride * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = min64(i0 + u * stride, n2 - 1);
      if (i0 != gtid) {
        xv[u] = x2[i];
        pv[u] = p2[i];
      }
      if (!stop) rv[u] = __ldcg(r2 + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n2) {
        double2 xo;
        xo.x = add(mul(1.0, xv[u].x), mul(alpha, pv[u].x));
        xo.y = add(mul(1.0, xv[u].y), mul(alpha, pv[u].y));
        x2[i] = xo;
        if (!stop) {
          double2 po;
          po.x = add(mul(1.0, rv[u].x), mul(beta, pv[u].x));
          po.y = add(mul(1.0, rv[u].y), mul(beta, pv[u].y));
          p2[i] = po;
        }
      }
    }
  }
  if ((n & 1) && gtid == 0) {
    const int64_t i = n - 1;
    const double pi = p[i];
    x[i] = add(mul(1.0, x[i]), mul(alpha, pi));
    if (!stop) p[i] = add(mul(1.0, __ldcg(r + i)), mul(beta, pi));
  }
}

}  // namespace ds

// ============================================================== C ABI ======
using namespace ds;

static DotOut make_dot(void* workspace, int slot, const double* other, double* result) {
  // workspace holds two independent reduction slots (tickets + partials)
  char* base = reinterpret_cast<char*>(workspace) + (int64_t)slot * kWorkspaceBytes;
  Workspace w(base);
  DotOut d;
  d.other = other;
  d.partials = w.partials;
  d.ticket = w.ticket;
  d.result = result;
  d.max_blocks = kMaxPartials;
  return d;
}

extern "C" int64_t ds_dot_workspace_bytes(void) { return 2 * kWorkspaceBytes; }
extern "C" int64_t ds_cg_workspace_bytes(void) { return 2 * kWorkspaceBytes; }

extern "C" int ds_dot(int64_t n, const double* x, const double* y, double* result_dev,
                      void* workspace, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n <= 0) {
    DS_CUDA(cudaMemsetAsync(result_dev, 0, sizeof(double), st));
    return DS_OK;
  }
  DotOut d = make_dot(workspace, 0, nullptr, result_dev);
  return launch_dot(n, x, y, d, st);
}

extern "C" int ds_waxpby(int64_t n, double alpha, const double* x, double beta, const double* y,
                         double* w, void* stream) {
  if (n <= 0) return DS_OK;
  waxpby_kernel<<<grid_for(n), kVecBlock, 0, as_stream(stream)>>>(n, alpha, x, beta, y, w,
                                                                  nullptr);
  DS_LAUNCH_CHECK("waxpby_kernel");
  return DS_OK;
}

extern "C" int ds_scan(int64_t n, const double* x, double* out, double* total_dev,
                       void* stream) {
  scan_seq_kernel<<<1, kVecBlock, 0, as_stream(stream)>>>(n, x, out, total_dev);
  DS_LAUNCH_CHECK("scan_seq_kernel");
  return DS_OK;
}

extern "C" int ds_gather(int64_t count, const int32_t* idx, const double* src, double* dst,
                         void* stream) {
  if (count <= 0) return DS_OK;
  gather_kernel<<<grid_for(count, 2), kVecBlock, 0, as_stream(stream)>>>(count, idx, src, dst,
                                                                         nullptr);
  DS_LAUNCH_CHECK("gather_kernel");
  return DS_OK;
}

extern "C" int ds_cg_gather(int64_t count, const int32_t* idx, const double* src, double* dst,
                            const ds_cg_scalars* s, void* stream) {
  if (count <= 0) return DS_OK;
  gather_kernel<<<grid_for(count, 2), kVecBlock, 0, as_stream(stream)>>>(
      count, idx, src, dst, s ? &s->done : nullptr);
  DS_LAUNCH_CHECK("gather_kernel");
  return DS_OK;
}

extern "C" int ds_extract_diag_csr(int64_t nrows, int64_t ncols, const int32_t* row_offsets,
                                   const int32_t* col_indices, const double* values, double* out,
                                   void* stream) {
  const int64_t n = nrows < ncols ? nrows : ncols;
  if (n <= 0) return DS_OK;
  extract_diag_csr_kernel<<<grid_for(n, 1), kVecBlock, 0, as_stream(stream)>>>(
      (int)n, row_offsets, col_indices, values, out);
  DS_LAUNCH_CHECK("extract_diag_csr_kernel");
  return DS_OK;
}

extern "C" int ds_update_diag_csr(int64_t nrows, int64_t ncols, const int32_t* row_offsets,
                                  const int32_t* col_indices, double* values, const double* d,
                                  int64_t* first_missing, void* stream) {
  cudaStream_t st = as_stream(stream);
  const int64_t n = nrows < ncols ? nrows : ncols;
  *first_missing = -1;
  if (n <= 0) return DS_OK;
  long long* dm = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dm), sizeof(long long), st));
  const long long big = 0x7fffffffffffffffll;
  DS_CUDA(cudaMemcpyAsync(dm, &big, sizeof(big), cudaMemcpyHostToDevice, st));
  csr_diag_presence<<<grid_for(n, 1), kVecBlock, 0, st>>>((int)n, row_offsets, col_indices, dm);
  long long h = big;
  DS_CUDA(cudaMemcpyAsync(&h, dm, sizeof(h), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(dm, st));
  DS_CUDA(cudaStreamSynchronize(st));
  if (h != big) {
    *first_missing = h;
    set_error("diagonal entry (%lld, %lld) is not structurally present", h, h);
    return DS_ERR_STRUCTURALLY_ABSENT_DIAG;
  }
  update_diag_csr_kernel<<<grid_for(n, 1), kVecBlock, 0, st>>>((int)nrows, (int)n, row_offsets,
                                                               col_indices, values, d);
  DS_LAUNCH_CHECK("update_diag_csr_kernel");
  return DS_OK;
}

// shared COO diagonal analysis: count/first per row, first missing, max count
static int coo_diag_analysis(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                             cudaStream_t st, int** count, int** first, long long* missing,
                             int* maxcount) {
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(count), n * sizeof(int), st));
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(first), n * sizeof(int), st));
  long long* dm = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dm), 2 * sizeof(long long), st));
  fill_i32<<<grid_for(n), kVecBlock, 0, st>>>(n, *count, 0);
  fill_i32<<<grid_for(n), kVecBlock, 0, st>>>(n, *first, 0x7fffffff);
  const long long init[2] = {0x7fffffffffffffffll, 0};
  DS_CUDA(cudaMemcpyAsync(dm, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (nnz > 0)
    coo_diag_scan<<<grid_for(nnz), kVecBlock, 0, st>>>(nnz, (int)n, rows, cols, *count, *first);
  coo_diag_missing<<<grid_for(n), kVecBlock, 0, st>>>((int)n, *count, dm,
                                                      reinterpret_cast<int*>(dm + 1));
  DS_LAUNCH_CHECK("coo_diag_analysis");
  long long h[2];
  DS_CUDA(cudaMemcpyAsync(h, dm, sizeof(h), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(dm, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *missing = h[0];
  *maxcount = static_cast<int>(h[1] & 0xffffffff);
  return DS_OK;
}

extern "C" int ds_extract_diag_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                                   const int32_t* cols, const double* values, double* out,
                                   void* stream) {
  cudaStream_t st = as_stream(stream);
  const int64_t n = nrows < ncols ? nrows : ncols;
  if (n <= 0) return DS_OK;
  int *count = nullptr, *first = nullptr;
  long long missing;
  int maxcount;
  int rc = coo_diag_analysis(n, nnz, rows, cols, st, &count, &first, &missing, &maxcount);
  if (rc) return rc;
  fill_f64_plain<<<grid_for(n), kVecBlock, 0, st>>>(n, out, 0.0);
  if (nnz > 0) {
    if (maxcount <= 2)
      coo_extract_atomic<<<grid_for(nnz), kVecBlock, 0, st>>>(nnz, (int)n, rows, cols, values,
                                                              out);
    else
      coo_extract_serial<<<1, 1, 0, st>>>(nnz, (int)n, rows, cols, values, out);
  }
  DS_LAUNCH_CHECK("coo_extract");
  DS_CUDA(cudaFreeAsync(count, st));
  DS_CUDA(cudaFreeAsync(first, st));
  return DS_OK;
}

extern "C" int ds_update_diag_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                                  const int32_t* cols, double* values, const double* d,
                                  int64_t* first_missing, void* stream) {
  cudaStream_t st = as_stream(stream);
  const int64_t n = nrows < ncols ? nrows : ncols;
  *first_missing = -1;
  if (n <= 0) return DS_OK;
  int *count = nullptr, *first = nullptr;
  long long missing;
  int maxcount;
  int rc = coo_diag_analysis(n, nnz, rows, cols, st, &count, &first, &missing, &maxcount);
  if (rc) return rc;
  if (missing != 0x7fffffffffffffffll) {
    DS_CUDA(cudaFreeAsync(count, st));
    DS_CUDA(cudaFreeAsync(first, st));
    *first_missing = missing;
    set_error("diagonal entry (%lld, %lld) is not structurally present", missing, missing);
    return DS_ERR_STRUCTURALLY_ABSENT_DIAG;
  }
  coo_update_kernel<<<grid_for(nnz), kVecBlock, 0, st>>>(nnz, (int)n, rows, cols, values, first,
                                                         d);
  DS_LAUNCH_CHECK("coo_update_kernel");
  DS_CUDA(cudaFreeAsync(count, st));
  DS_CUDA(cudaFreeAsync(first, st));
  return DS_OK;
}

extern "C" int ds_dia_diag_column(int64_t n, int32_t ndiags, int32_t j0, double* values,
                                  double* vec, int direction, void* stream) {
  if (n <= 0) return DS_OK;
  dia_diag_column_kernel<<<grid_for(n), kVecBlock, 0, as_stream(stream)>>>(n, ndiags, j0, values,
                                                                           vec, direction);
  DS_LAUNCH_CHECK("dia_diag_column_kernel");
  return DS_OK;
}

extern "C" int ds_dia_count_nonzero(int64_t nrows, int64_t ncols, int32_t ndiags,
                                    const int32_t* offsets, const double* values, int64_t* count,
                                    void* stream) {
  cudaStream_t st = as_stream(stream);
  *count = 0;
  if (nrows <= 0 || ndiags <= 0) return DS_OK;
  unsigned long long* dc = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dc), sizeof(*dc), st));
  DS_CUDA(cudaMemsetAsync(dc, 0, sizeof(*dc), st));
  dia_nonzero_kernel<<<(unsigned)min64(ceil_div(nrows, 8), (int64_t)sm_count() * 16), kVecBlock,
                       0, st>>>((int)nrows, (int)ncols, ndiags, offsets, values, dc);
  DS_LAUNCH_CHECK("dia_nonzero_kernel");
  unsigned long long h = 0;
  DS_CUDA(cudaMemcpyAsync(&h, dc, sizeof(h), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(dc, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *count = (int64_t)h;
  return DS_OK;
}

// ------------------------------------------------------------------ CG -----
extern "C" int ds_spmv(const ds_matrix* a, const double* x, double* y, int accumulate,
                       void* stream) {
  return ds_cg_spmv_dot(a, x, y, accumulate, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0,
                        nullptr, stream);
}

extern "C" int ds_cg_spmv_dot(const ds_matrix* a, const double* x, double* y, int accumulate,
                              const double* dot_with, double* dot_out, int stage,
                              ds_cg_scalars* s, double* history, const double* parts,
                              int nparts_final, void* workspace, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (a->nrows < 0 || a->nrows >= (1ll << 31) || a->ncols >= (1ll << 31)) {
    set_error("dims out of range");
    return DS_ERR_NOT_SUPPORTED;
  }
  DotOut d;
  d.guard = s ? &s->done : nullptr;
  d.plus_zero = (accumulate == 2);
  const bool want_dot = dot_with != nullptr;
  DotOut fused;
  if (want_dot) {
    fused = make_dot(workspace, 0, dot_with, dot_out);
    fused.guard = d.guard;
    fused.plus_zero = d.plus_zero;
    fused.partials_only = (stage == DS_CG_STAGE_DEFERRED);
    fused.stage = stage;
    fused.s = s;
    fused.history = history;
    fused.parts = parts;
    fused.nparts_final = nparts_final;
  }
  const bool acc = accumulate == 1;
  int rc = DS_OK;
  bool done_dot = false;
  switch (a->format) {
    case DS_FMT_CSR: {
      if (a->row_perm && a->tiles && !want_dot) {   // irregular: entry tiles + long rows
        rc = launch_csr_tiles(a->nrows, a->ncols, a->idx0, a->idx1, a->values, a->tiles,
                              a->ntiles, a->row_perm, a->bins, x, y, acc, d.guard, st);
        break;
      }
      if (a->row_perm) {  // irregular matrix: length-binned kernels
        const bool can_fuse = want_dot && a->bins[8] == a->bins[6];
        rc = launch_csr_binned(a->nrows, a->ncols, a->nnz, a->idx0, a->idx1, a->values, a->row_perm,
                               a->bins, x, y, acc, can_fuse ? &fused : &d, st);
        done_dot = can_fuse;
        break;
      }
      const bool can_fuse = want_dot && (a->long_rows == nullptr || a->n_long == 0);
      rc = launch_csr(a->nrows, a->nnz, a->idx0, a->idx1, a->values, a->long_rows, a->n_long,
                      a->max_row_len, x, y, acc,
                      can_fuse ? &fused : &d, st);
      done_dot = can_fuse;
      break;
    }
    case DS_FMT_DIA: {
      const bool can_fuse =
          want_dot && ceil_div(a->nrows, 256) <= (int64_t)kMaxPartials;
      rc = launch_dia(a->nrows, a->ncols, a->ndiags, a->idx0, a->values, x, y, acc,
                      can_fuse ? &fused : &d, st);
      done_dot = can_fuse;
      break;
    }
    case DS_FMT_COO:
      // COO plans reuse long_rows / n_long: the long-run (start, end) pairs
      rc = launch_coo(a->nrows, a->nnz, a->idx0, a->idx1, a->values, a->rows_sorted != 0,
                      a->max_row_len, x, y, acc, d.guard, st, d.plus_zero != 0,
                      a->rows_sorted ? a->long_rows : nullptr,
                      a->rows_sorted ? (int)a->n_long : 0);
      break;
    default:
      set_error("unknown format %d", a->format);
      return DS_ERR_INVALID_ARGUMENT;
  }
  if (rc) return rc;
  if (want_dot && !done_dot) {
    if (a->nrows == 0) {
      set_error("empty operator in CG");
      return DS_ERR_INVALID_ARGUMENT;
    }
    rc = launch_dot(a->nrows, dot_with, y, fused, st);
  }
  return rc;
}

extern "C" int ds_cg_setup_residual(int64_t n, const double* b, const double* ap, double* r,
                                    double* p, double* bb_out, double* rr_out, void* workspace,
                                    void* stream) {
  cudaStream_t st = as_stream(stream);
  if (n <= 0) {
    DS_CUDA(cudaMemsetAsync(bb_out, 0, sizeof(double), st));
    DS_CUDA(cudaMemsetAsync(rr_out, 0, sizeof(double), st));
    return DS_OK;
  }
  DotOut dbb = make_dot(workspace, 0, nullptr, bb_out);
  DotOut drr = make_dot(workspace, 1, nullptr, rr_out);
  int64_t g = ceil_div(n, (int64_t)kVecBlock * 8);
  if (g > 1024) g = 1024;
  cg_setup_kernel<<<(unsigned)g, kVecBlock, 0, st>>>(n, b, ap, r, p, dbb, drr);
  DS_LAUNCH_CHECK("cg_setup_kernel");
  return DS_OK;
}

extern "C" int ds_cg_setup_finalize(ds_cg_scalars* s, const double* bb_parts,
                                    const double* rr_parts, int nparts, double tol,
                                    int32_t max_iters, double* history, void* stream) {
  cg_setup_finalize_kernel<<<1, 1, 0, as_stream(stream)>>>(s, bb_parts, rr_parts, nparts, tol,
                                                           max_iters, history);
  DS_LAUNCH_CHECK("cg_setup_finalize_kernel");
  return DS_OK;
}

extern "C" int ds_cg_update(int64_t n, double* x, double* r, const double* p, const double* ap,
                            ds_cg_scalars* s, double* rr_out, double* history,
                            const double* parts, int nparts_final, void* workspace,
                            void* stream) {
  cudaStream_t st = as_stream(stream);
  DotOut d = make_dot(workspace, 0, nullptr, rr_out);
  d.guard = &s->done;
  d.stage = kStageRr;
  d.s = s;
  d.history = history;
  d.parts = parts;
  d.nparts_final = nparts_final;
  const unsigned g = vec_grid(n);
  if (aligned16(x, r, p, ap))
    cg_update_kernel<true><<<g, kVecBlock, 0, st>>>(n, x, r, p, ap, s, d);
  else
    cg_update_kernel<false><<<g, kVecBlock, 0, st>>>(n, x, r, p, ap, s, d);
  DS_LAUNCH_CHECK("cg_update_kernel");
  return DS_OK;
}

extern "C" int ds_cg_direction(int64_t n, const double* r, double* p, const ds_cg_scalars* s,
                               void* stream) {
  if (n <= 0) return DS_OK;
  const unsigned g = vec_grid(n);
  if (aligned16(r, p))
    cg_direction_kernel<true><<<g, kVecBlock, 0, as_stream(stream)>>>(n, r, p, s);
  else
    cg_direction_kernel<false><<<g, kVecBlock, 0, as_stream(stream)>>>(n, r, p, s);
  DS_LAUNCH_CHECK("cg_direction_kernel");
  return DS_OK;
}

// Fused update + direction (single partition, deferred): see
// cg_update_direction_fused_kernel.  Returns DS_ERR_NOT_SUPPORTED (nothing
// launched) for misaligned vectors or n < 2: use the two kernels then.
extern "C" int ds_cg_update_direction_deferred(int64_t n, double* x, double* r, double* p,
                                               const double* ap, ds_cg_scalars* s,
                                               double* history, void* workspace, void* stream) {
  if (n < 2 || !aligned16(x, r, p, ap)) return DS_ERR_NOT_SUPPORTED;
  Workspace w0(reinterpret_cast<char*>(workspace));
  Workspace w1(reinterpret_cast<char*>(workspace) + kWorkspaceBytes);
  // 2 CTAs of 256 threads per SM, 4 double2 per thread and sweep (measured
  // against 3-4 CTAs/SM, unroll 1-2, a single-sweep variant holding r and p
  // in registers across the barrier, and 64-register variants at 1-2 CTAs/SM
  // that leave room for the next SpMV's programmatic CTAs: all 0.5-3 us per
  // step slower)
  static int per_sm = -1;
  const void* fn = reinterpret_cast<const void*>(cg_update_direction_fused_kernel<4, 2>);
  if (per_sm < 0) {
    int b = 0;
    DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kVecBlock, 0));
    per_sm = b > 0 ? b : 1;
  }
  int64_t g = vec_grid(n);
  const int64_t cap = (int64_t)sm_count() * per_sm;   // co-resident: the barrier needs it
  if (g > cap) g = cap;
  cudaStream_t st = as_stream(stream);
  const double* pap_parts = w0.partials;
  const unsigned* pap_count = w0.ticket + 2;
  double* rr_parts = w1.partials;
  unsigned* bar_count = w1.ticket + 1;
  unsigned* bar_gen = w1.ticket + 3;
  void* args[] = {&n, &x, &r, &p, const_cast<double**>(&ap), &s, &history,
                  const_cast<double**>(&pap_parts), const_cast<unsigned**>(&pap_count),
                  &rr_parts, &bar_count, &bar_gen};
  // cooperative AND a programmatic dependent of the SpMV before it (its
  // x / r / p loads overlap the SpMV's last wave); without PDL support the
  // plain cooperative launch below
  static int no_pdl = -1;
  if (no_pdl < 0) no_pdl = getenv("DS_NO_PDL") || getenv("DS_NO_TAIL_PDL") ? 1 : 0;
  if (!no_pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(kVecBlock);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelExC(&cfg, fn, args) == cudaSuccess) {
      DS_LAUNCH_CHECK("cg_update_direction_fused_kernel");
      return DS_OK;
    }
    (void)cudaGetLastError();
  }
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)g), dim3(kVecBlock), args, 0, st);
  if (e != cudaSuccess) {
    // not capturable / not supported here: the grid is co-resident by
    // construction, so a plain launch keeps the barrier safe
    (void)cudaGetLastError();
    DS_CUDA(cudaLaunchKernel(fn, dim3((unsigned)g), dim3(kVecBlock), args, 0, st));
  }
  DS_LAUNCH_CHECK("cg_update_direction_fused_kernel");
  return DS_OK;
}

extern "C" int ds_cg_update_deferred(int64_t n, double* x, double* r, const double* p,
                                     const double* ap, ds_cg_scalars* s, void* workspace,
                                     void* stream) {
  return ds_cg_update_gathered(n, x, r, p, ap, s, nullptr, 0, nullptr, workspace, stream);
}

extern "C" int ds_cg_update_gathered(int64_t n, double* x, double* r, const double* p,
                                     const double* ap, ds_cg_scalars* s, const double* pap_all,
                                     int nparts, double* rr_mine, void* workspace,
                                     void* stream) {
  Workspace w0(reinterpret_cast<char*>(workspace));
  Workspace w1(reinterpret_cast<char*>(workspace) + kWorkspaceBytes);
  DotOut d = make_dot(workspace, 1, nullptr, rr_mine);
  const unsigned g = vec_grid(n);
  cudaStream_t st = as_stream(stream);
  const double* in = nparts > 0 ? pap_all : w0.partials;
  if (aligned16(x, r, p, ap))
    cg_update_deferred_kernel<true><<<g, kVecBlock, 0, st>>>(
        n, x, r, p, ap, s, in, w0.ticket + 2, w1.partials, w1.ticket + 2, nparts, d);
  else
    cg_update_deferred_kernel<false><<<g, kVecBlock, 0, st>>>(
        n, x, r, p, ap, s, in, w0.ticket + 2, w1.partials, w1.ticket + 2, nparts, d);
  DS_LAUNCH_CHECK("cg_update_deferred_kernel");
  return DS_OK;
}

extern "C" int ds_cg_direction_deferred(int64_t n, const double* r, double* p, ds_cg_scalars* s,
                                        double* history, void* workspace, void* stream) {
  return ds_cg_direction_gathered(n, r, p, s, history, nullptr, 0, workspace, stream);
}

extern "C" int ds_cg_direction_gathered(int64_t n, const double* r, double* p, ds_cg_scalars* s,
                                        double* history, const double* rr_all, int nparts,
                                        void* workspace, void* stream) {
  Workspace w1(reinterpret_cast<char*>(workspace) + kWorkspaceBytes);
  const unsigned g = vec_grid(n);
  cudaStream_t st = as_stream(stream);
  const double* in = nparts > 0 ? rr_all : w1.partials;
  if (aligned16(r, p))
    cg_direction_deferred_kernel<true><<<g, kVecBlock, 0, st>>>(n, r, p, s, history, in,
                                                                w1.ticket + 2, nparts);
  else
    cg_direction_deferred_kernel<false><<<g, kVecBlock, 0, st>>>(n, r, p, s, history, in,
                                                                 w1.ticket + 2, nparts);
  DS_LAUNCH_CHECK("cg_direction_deferred_kernel");
  return DS_OK;
}

extern "C" int ds_cg_finalize(int stage, ds_cg_scalars* s, double* history, const double* parts,
                              int nparts, void* stream) {
  cg_finalize_kernel<<<1, 1, 0, as_stream(stream)>>>(stage, s, history, parts, nparts);
  DS_LAUNCH_CHECK("cg_finalize_kernel");
  return DS_OK;
}
