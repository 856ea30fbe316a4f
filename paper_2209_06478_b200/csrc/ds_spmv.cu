// ds_spmv.cu -- SpMV over CSR / DIA / COO for sm_100a.
//
// Replaces the reference's format-dispatched kernels (kernels.py:102-198):
//   _csr_spmv  kernels.py:102-119   -> csr_pipe (rows <= 33) / csr_binned / csr_long_rows*
//                                      (csr_rows_g8 without a plan)
//   _dia_spmv  kernels.py:122-140   -> dia_pipe (+ dia_rows_direct)
//   _coo_spmv  kernels.py:143-163   -> coo_pipe / coo_warp_segments (+ coo_long_runs_kernel)
//                                      / coo_atomic
// Results are bitwise equal to the reference (see include/dynsparse_b200.h)
// except for unsorted COO (atomics; within 1e-13 like the reference's
// threaded COO, kernels.py:13-15).
//
// HBM is the roofline for every kernel here (no tensor cores: SpMV is not a
// dense contraction).  The common design: persistent
// CTAs stream their tiles' matrix arrays into a ring of shared-memory stages
// with 1-D TMA bulk copies (cp.async.bulk + mbarrier transaction counts, L2
// evict_first so x stays L2-resident); one thread per row copies its entries
// to registers, issues every gather, and the CTA releases the stage before
// the exact (numpy-order) sums run from registers.
#include <stdlib.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

// ===================================================================== CSR ==

// Sum of one row in np.add.reduceat order, computed by an aligned 8-lane
// group; m = row_len - 1 addends after the first product, m <= 128 handled as
// one pairwise leaf; longer rows walk the recursion (slow path, used only
// when no long-row plan was supplied).
struct CsrElem {
  const int* col;
  const double* val;
  const double* x;
  int64_t base;
  __device__ __forceinline__ double operator()(int64_t i) const {
    return mul(ld_stream(val + base + i), ld_gather(x + ld_stream(col + base + i)));
  }
};

// Leaf (m <= 128) with loads batched 4 rounds at a time so every lane has up
// to 4 independent col->x chains in flight before the dependent adds.
__device__ __forceinline__ double csr_leaf_g8(const int* __restrict__ col,
                                              const double* __restrict__ val,
                                              const double* __restrict__ x, int64_t base, int m,
                                              int lane8, unsigned mask) {
  const int full = m & ~7;
  const int nfull = full >> 3;                 // full rounds of 8
  const int rounds = (m + 7) >> 3;             // rounds incl. the tail round
  double r = 0.0, tail = 0.0;
  for (int k0 = 0; k0 < rounds; k0 += 4) {
    int c[4];
    double v[4], a[4];
    // unpredicated loads of a clamped index (m >= 1 here): every lane keeps
    // 4 col->x chains in flight; products of clamped slots are never used
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int i = min(lane8 + 8 * (k0 + kk), m - 1);
      c[kk] = ld_stream(col + base + i);
      v[kk] = ld_stream(val + base + i);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) a[kk] = mul(v[kk], ld_gather(x + c[kk]));
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k0 + kk;
      if (k < nfull) {
        r = (k == 0) ? a[kk] : add(r, a[kk]);
      } else if (k == nfull) {
        tail = a[kk];  // i == full + lane8 (zero when lane8 >= m - full)
      }
    }
  }
  double res;
  if (full > 0) {
    r = add(r, __shfl_xor_sync(mask, r, 1, 8));
    r = add(r, __shfl_xor_sync(mask, r, 2, 8));
    r = add(r, __shfl_xor_sync(mask, r, 4, 8));
    res = r;
  } else {
    res = -0.0;  // numpy's pairwise_sum identity for n < 8
  }
  const int ntail = m - full;
  for (int t = 0; t < ntail; ++t) res = add(res, __shfl_sync(mask, tail, t, 8));
  return res;
}

// Short-row leaf (m <= 32: one batch of 4 rounds) split into phases so two
// rows can be interleaved: all loads of both rows are issued before either
// row's dependent gathers and adds.
struct ShortLeaf {
  int c[4];
  double v[4];
  double a[4];
  int c0;
  double v0;
};

__device__ __forceinline__ void short_leaf_load(const int* __restrict__ col,
                                                const double* __restrict__ val, int start,
                                                int len, int lane8, ShortLeaf& L) {
  const int m = len - 1;  // addends after p[first]
  // clamped indices keep every load unpredicated; L1-allocating loads make
  // the clamped duplicates (rows shorter than 33) hit L1 instead of L2
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int i = max(min(lane8 + 8 * kk, m - 1), 0);   // clamped: always in the row
    L.c[kk] = __ldg(col + start + 1 + i);
    L.v[kk] = __ldg(val + start + 1 + i);
  }
  L.c0 = ld_stream(col + start);
  L.v0 = ld_stream(val + start);
}

__device__ __forceinline__ void short_leaf_gather(const double* __restrict__ x, ShortLeaf& L) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) L.a[kk] = mul(L.v[kk], ld_gather(x + L.c[kk]));
  L.v0 = mul(L.v0, ld_gather(x + L.c0));   // p[first]
}

// y-value of a row with 1 <= len <= 33 (bitwise np.add.reduceat order)
__device__ __forceinline__ double short_leaf_finish(int len, int lane8, unsigned mask,
                                                    const ShortLeaf& L) {
  const int m = len - 1;
  const int full = m & ~7, nfull = full >> 3;
  double r = 0.0, tail = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < nfull) r = (k == 0) ? L.a[k] : add(r, L.a[k]);
    else if (k == nfull) tail = L.a[k];
  }
  double res;
  if (full > 0) {
    r = add(r, __shfl_xor_sync(mask, r, 1, 8));
    r = add(r, __shfl_xor_sync(mask, r, 2, 8));
    r = add(r, __shfl_xor_sync(mask, r, 4, 8));
    res = r;
  } else {
    res = -0.0;
  }
  const int ntail = m - full;
  for (int t = 0; t < ntail; ++t) res = add(res, __shfl_sync(mask, tail, t, 8));
  return add(L.v0, res);
}

// Leaf (m <= 128) for the long-row kernels, which are latency bound (a few
// rows, each a chain of leaves): every lane issues ALL its column / value
// loads, then all its gathers, before the first add -- one memory round trip
// per leaf instead of one per batch of 4 rounds.
__device__ __forceinline__ double csr_leaf_g8_all(const int* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ x, int64_t base,
                                                  int m, int lane8, unsigned mask) {
  const int full = m & ~7, nfull = full >> 3;
  int c[16];
  double v[16], a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int i = min(lane8 + 8 * k, m - 1);
    c[k] = ld_stream(col + base + i);
    v[k] = ld_stream(val + base + i);
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = mul(v[k], ld_gather(x + c[k]));
  double r = a[0], tail = 0.0;
#pragma unroll
  for (int k = 1; k < 16; ++k) {
    if (k < nfull) r = add(r, a[k]);
  }
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (k == nfull) tail = a[k];
  double res;
  if (full > 0) {
    r = add(r, __shfl_xor_sync(mask, r, 1, 8));
    r = add(r, __shfl_xor_sync(mask, r, 2, 8));
    r = add(r, __shfl_xor_sync(mask, r, 4, 8));
    res = r;
  } else {
    res = -0.0;
  }
  const int ntail = m - full;
  for (int t = 0; t < ntail; ++t) res = add(res, __shfl_sync(mask, tail, t, 8));
  return res;
}

// Recursion for m > 128 by one 8-lane group (no plan): group-uniform DFS.
__device__ double csr_group_pairwise(const int* __restrict__ col, const double* __restrict__ val,
                                     const double* __restrict__ x, int64_t base, int64_t m,
                                     int lane8, unsigned mask) {
  if (m <= 128) return csr_leaf_g8(col, val, x, base, (int)m, lane8, mask);
  struct Frame {
    int64_t lo, n;
    int expanded;
  };
  Frame st[64];
  double vs[64];
  int ft = 0, vt = 0;
  st[ft++] = {0, m, 0};
  while (ft > 0) {
    Frame f = st[--ft];
    if (f.n <= 128) {
      vs[vt++] = csr_leaf_g8(col, val, x, base + f.lo, (int)f.n, lane8, mask);
    } else if (!f.expanded) {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      st[ft++] = {f.lo, f.n, 1};
      st[ft++] = {f.lo + n2, f.n - n2, 0};
      st[ft++] = {f.lo, n2, 0};
    } else {
      double b = vs[--vt];
      double a = vs[--vt];
      vs[vt++] = add(a, b);
    }
  }
  return vs[0];
}

constexpr int kCsrBlock = 256;
constexpr int kLongRow = 129;  // rows longer than this need the recursion
constexpr int kSub = 8192;     // <= 128 leaves per subtree / warp-kernel row limit
constexpr int kMaxLeaves = 160;

// One 8-lane group per PAIR of consecutive rows; grid-stride over pairs.
// Rows of <= 33 entries (the stencil's 8..27, the power-law's typical 6..33)
// take the interleaved fast path; longer ones the general leaf / recursion.
template <bool ACCUM, bool SKIP_LONG, bool FUSE_DOT>
__device__ __forceinline__ void csr_emit(int row, int len, double sres, double* y,
                                         const DotOut& dot, double& dsum) {
  double out = ACCUM ? add(y[row], sres) : sres;
  if (dot.plus_zero) out = add(out, 0.0);
  y[row] = out;
  if (FUSE_DOT) dsum = add(dsum, mul(dot.other[row], out));
}

template <bool ACCUM, bool SKIP_LONG, bool FUSE_DOT>
__device__ __forceinline__ void csr_row_general(int row, int start, int len,
                                                const int* __restrict__ col,
                                                const double* __restrict__ val,
                                                const double* __restrict__ x, double* y,
                                                int lane8, unsigned mask, const DotOut& dot,
                                                double& dsum) {
  if (SKIP_LONG && len > kLongRow) return;  // the long-row kernel owns it
  double res = 0.0, p0 = 0.0;
  if (len > 0) {
    if (lane8 == 0) p0 = mul(ld_stream(val + start), ld_gather(x + ld_stream(col + start)));
    if (len <= kLongRow)
      res = csr_leaf_g8_all(col, val, x, (int64_t)start + 1, len - 1, lane8, mask);
    else
      res = csr_group_pairwise(col, val, x, (int64_t)start + 1, len - 1, lane8, mask);
  }
  if (lane8 == 0) csr_emit<ACCUM, SKIP_LONG, FUSE_DOT>(row, len, len > 0 ? add(p0, res) : 0.0,
                                                      y, dot, dsum);
}

template <bool ACCUM, bool SKIP_LONG, bool FUSE_DOT>
__global__ void __launch_bounds__(kCsrBlock)
    csr_rows_g8(int nrows, const int* __restrict__ off, const int* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ x, double* y,
                DotOut dot) {
  if (dot.skip()) return;
  const int lane8 = threadIdx.x & 7;
  const unsigned mask = 0xffu << (threadIdx.x & 24);
  const int groups_per_grid = (gridDim.x * kCsrBlock) >> 3;
  const int npairs = (nrows + 1) >> 1;
  double dsum = 0.0;
  for (int pr = (blockIdx.x * kCsrBlock + threadIdx.x) >> 3; pr < npairs;
       pr += groups_per_grid) {
    const int ra = 2 * pr, rb = ra + 1;
    const bool has_b = rb < nrows;
    const int sa = __ldg(off + ra), ea = __ldg(off + ra + 1);
    const int eb = has_b ? __ldg(off + rb + 1) : ea;
    const int la = ea - sa, lb = eb - ea;
    if (la >= 1 && la <= 33 && lb >= 1 && lb <= 33) {
      ShortLeaf A, B;
      short_leaf_load(col, val, sa, la, lane8, A);
      short_leaf_load(col, val, ea, lb, lane8, B);
      short_leaf_gather(x, A);
      short_leaf_gather(x, B);
      const double ya = short_leaf_finish(la, lane8, mask, A);
      const double yb = short_leaf_finish(lb, lane8, mask, B);
      if (lane8 == 0) {
        csr_emit<ACCUM, SKIP_LONG, FUSE_DOT>(ra, la, ya, y, dot, dsum);
        csr_emit<ACCUM, SKIP_LONG, FUSE_DOT>(rb, lb, yb, y, dot, dsum);
      }
    } else {
      csr_row_general<ACCUM, SKIP_LONG, FUSE_DOT>(ra, sa, la, col, val, x, y, lane8, mask, dot,
                                                  dsum);
      if (has_b)
        csr_row_general<ACCUM, SKIP_LONG, FUSE_DOT>(rb, ea, lb, col, val, x, y, lane8, mask,
                                                    dot, dsum);
    }
  }
  if (FUSE_DOT) dot.finish_block<kCsrBlock>(dsum);
}

// ---------------------------------------------------------------------------
// Binned CSR (irregular matrices).  Rows are grouped by length bin
// (ds_csr_bins): each bin runs with its exact number of load rounds R
// (bin b in 1..4: rows of <= 8b+1 entries -> R = b), so there is neither
// round padding nor per-lane predication; two rows per 8-lane group keep
// 2R load chains in flight.  Work item = a pair of consecutive rows of the
// permuted list; items of all bins are enumerated in one grid-stride loop.
struct CsrBins {
  int64_t start[8];     // bin b rows = perm[start[b] .. start[b+1])
  int64_t pair_off[8];  // cumulative work items (kBinRows[b] rows each) before bin b
};
// rows per work item (8-lane group) per bin: empty, R=1, R=2, R=3, R=4, general
__constant__ int kBinRows[7] = {4, 4, 4, 2, 2, 2, 1};
static const int kBinRowsHost[7] = {4, 4, 4, 2, 2, 2, 1};

template <int R>
__device__ __forceinline__ void binned_load(const int* __restrict__ col,
                                            const double* __restrict__ val, int start, int len,
                                            int lane8, int (&c)[R], double (&v)[R], int& c0,
                                            double& v0, uint64_t pol) {
  const int m = len - 1;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int i = max(min(lane8 + 8 * k, m - 1), -1);   // -1 -> p[first]: in bounds
    c[k] = ld_hint(col + start + 1 + i, pol);
    v[k] = ld_hint(val + start + 1 + i, pol);
  }
  c0 = ld_hint(col + start, pol);
  v0 = ld_hint(val + start, pol);
}

template <int R>
__device__ __forceinline__ double binned_finish(int len, int lane8, unsigned mask,
                                                const double (&a)[R], double p0) {
  const int m = len - 1;
  const int full = m & ~7, nfull = full >> 3;
  double r = 0.0, tail = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (k < nfull) r = (k == 0) ? a[k] : add(r, a[k]);
    else if (k == nfull) tail = a[k];
  }
  double res;
  if (full > 0) {
    r = add(r, __shfl_xor_sync(mask, r, 1, 8));
    r = add(r, __shfl_xor_sync(mask, r, 2, 8));
    r = add(r, __shfl_xor_sync(mask, r, 4, 8));
    res = r;
  } else {
    res = -0.0;
  }
  const int ntail = m - full;
  for (int t = 0; t < ntail; ++t) res = add(res, __shfl_sync(mask, tail, t, 8));
  return add(p0, res);
}

// U rows per 8-lane group, all U*R loads and gathers issued before any
// reduction (short rows have little work each: more rows = more MLP)
template <int R, int U, bool ACCUM, bool FUSE_DOT>
__device__ __forceinline__ void binned_rows(const int* rws, int nr, const int* __restrict__ off,
                                            const int* __restrict__ col,
                                            const double* __restrict__ val,
                                            const double* __restrict__ x, double* y, int lane8,
                                            unsigned mask, const DotOut& dot, double& dsum,
                                            uint64_t pf, uint64_t pl) {
  int st[U], ln[U], c[U][R], c0[U];
  double v[U][R], v0[U], a[U][R], p0[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int row = rws[min(u, nr - 1)];
    st[u] = __ldg(off + row);
    ln[u] = __ldg(off + row + 1) - st[u];
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    binned_load<R>(col, val, st[u], ln[u], lane8, c[u], v[u], c0[u], v0[u], pf);
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int k = 0; k < R; ++k) a[u][k] = mul(v[u][k], ld_hint(x + c[u][k], pl));
    p0[u] = mul(v0[u], ld_hint(x + c0[u], pl));
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const double yv = binned_finish<R>(ln[u], lane8, mask, a[u], p0[u]);
    if (lane8 == 0 && u < nr) csr_emit<ACCUM, false, FUSE_DOT>(rws[u], ln[u], yv, y, dot, dsum);
  }
}

template <bool ACCUM, bool FUSE_DOT>
__global__ void __launch_bounds__(kCsrBlock, 2)
    csr_binned(const int* __restrict__ off, const int* __restrict__ col,
               const double* __restrict__ val, const double* __restrict__ x, double* y,
               const int* __restrict__ perm, CsrBins bi, DotOut dot) {
  if (dot.skip()) return;
  const int lane8 = threadIdx.x & 7;
  const unsigned mask = 0xffu << (threadIdx.x & 24);
  const int64_t groups = ((int64_t)gridDim.x * kCsrBlock) >> 3;
  const int64_t W = bi.pair_off[6];
  const uint64_t pf = policy_first(), pl = policy_evict_last();
  double dsum = 0.0;
  for (int64_t w = ((int64_t)blockIdx.x * kCsrBlock + threadIdx.x) >> 3; w < W; w += groups) {
    int b = 0;
#pragma unroll
    for (int k = 1; k < 6; ++k) b += (w >= bi.pair_off[k]);
    const int U = kBinRows[b];
    const int64_t q = bi.start[b] + (int64_t)U * (w - bi.pair_off[b]);
    const int nr = (int)min64(U, bi.start[b + 1] - q);
    const int* rws = perm + q;
    switch (b) {
      case 0:
        if (lane8 == 0)
          for (int u = 0; u < nr; ++u) csr_emit<ACCUM, false, FUSE_DOT>(rws[u], 0, 0.0, y, dot, dsum);
        break;
      case 1: binned_rows<1, 4, ACCUM, FUSE_DOT>(rws, nr, off, col, val, x, y, lane8, mask, dot, dsum, pf, pl); break;
      case 2: binned_rows<2, 4, ACCUM, FUSE_DOT>(rws, nr, off, col, val, x, y, lane8, mask, dot, dsum, pf, pl); break;
      case 3: binned_rows<3, 2, ACCUM, FUSE_DOT>(rws, nr, off, col, val, x, y, lane8, mask, dot, dsum, pf, pl); break;
      case 4: binned_rows<4, 2, ACCUM, FUSE_DOT>(rws, nr, off, col, val, x, y, lane8, mask, dot, dsum, pf, pl); break;
      default:
        for (int u = 0; u < nr; ++u) {
          const int row = rws[u];
          const int sr = __ldg(off + row);
          csr_row_general<ACCUM, true, FUSE_DOT>(row, sr, __ldg(off + row + 1) - sr, col, val, x,
                                                 y, lane8, mask, dot, dsum);
        }
    }
  }
  if (FUSE_DOT) dot.finish_block<kCsrBlock>(dsum);
}

// ---------------------------------------------------------------------------
// CSR v3: persistent TMA pipeline, one thread per row (the DIA design).
//
// Regular matrices (every row <= 33 entries: the stencil) are HBM-bound only
// if each SM keeps enough gathers in flight; the 8-lane-group kernels above
// hold ~1.7K per SM.  Here the matrix stream is decoupled from the gathers:
// thread 0 copies each tile's entry range [off[r0], off[r0+T]) -- column
// indices and values, contiguous in CSR -- into a ring of S shared-memory
// stages with two 1-D TMA bulk copies (mbarrier transaction counts, L2
// evict_first so x stays L2-resident), and refills a stage as soon as the
// CTA has consumed it.  Each thread then reads its row from shared memory
// (a row stride of 27 words / doubles is bank-conflict free) and issues all
// LMAX gathers unpredicated (clamped to the row's last entry) before any add,
// so 256 x LMAX gathers per SM are in flight.
//
// Sum order (np.add.reduceat, kernels.py:117): y = p[0] + pw(p[1..m]), m =
// len-1, pw(n < 8) = sequential from -0.0, pw(8 <= n <= 128) = 8 strided
// accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the n%8
// tail.  With every index static (register arrays) this is: r[j] = p[1+j]
// (+ p[1+j+8q] while 8q < full), res = full ? combine(r) : -0.0, then
// res += p[k] for full < k <= m ascending -- exactly the tail of either case.
// Rows longer than LMAX (<= kLongRow) take the serial emulation; a tile whose
// entries do not fit a stage ("fat") is read straight from global memory.
struct CsrPipeCfg {
  int T;            // rows per tile == blockDim.x
  int S;            // stages (<= 8)
  int cap;          // entries per stage (multiple of 4)
  int stage_bytes;  // 4*cap (cols) + 8*cap (vals), 128-B multiple
  int skip_above;   // SKIP_LONG: rows longer than this are left to other kernels
  int hint;         // gather x with L2 evict_last (irregular matrices: x re-used at random)
};

struct CsrPipeHdr {  // per stage, written by thread 0 before its arrive (release)
  int bc, bv;        // first staged col / val entry (aligned down to 16 B)
  int fat;
  int pad;
};

__device__ __forceinline__ void csr_pipe_issue(const int* __restrict__ col,
                                               const double* __restrict__ val, int nnz, int e0,
                                               int e1, const CsrPipeCfg& cfg, unsigned char* st,
                                               CsrPipeHdr* h, uint64_t* bar, uint64_t pol) {
  const int bc = e0 & ~3, bv = e0 & ~1;
  // copy up to the 16-B aligned end: the few entries past e1 belong to the
  // next tile (never read here).  Only where that would leave the arrays
  // (the last tile) is the sub-16-byte tail copied by hand -- a dependent
  // global load on thread 0, so it is kept off every other tile.
  const int cu = (e1 + 3) & ~3, vu = (e1 + 1) & ~1;
  const bool fat = (cu - bc) > cfg.cap;
  h->bc = bc;
  h->bv = bv;
  h->fat = fat;
  uint32_t bytes = 0;
  int* s_col = reinterpret_cast<int*>(st);
  double* s_val = reinterpret_cast<double*>(st + 4 * (size_t)cfg.cap);
  int cb = 0, vb = 0;
  if (!fat) {
    cb = cu <= nnz ? cu : (e1 & ~3);
    vb = vu <= nnz ? vu : (e1 & ~1);
    for (int e = cb; e < e1; ++e) s_col[e - bc] = col[e];
    if (vb < e1) s_val[vb - bv] = val[vb];
    bytes = 4u * (uint32_t)(cb - bc) + 8u * (uint32_t)(vb - bv);
  }
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, bytes);
  if (!fat) {
    if (cb > bc) bulk_g2s(s_col, col + bc, 4u * (uint32_t)(cb - bc), bar, pol);
    if (vb > bv) bulk_g2s(s_val, val + bv, 8u * (uint32_t)(vb - bv), bar, pol);
  }
}

// One row with 1 <= len <= LMAX in two phases around the stage release:
// load() copies the row's columns and values into registers and issues all
// LMAX gathers (unpredicated, clamped to the row's last entry); finish()
// forms the products and the exact np.add.reduceat sum.
template <int LMAX>
struct CsrRowRegs {
  double v[LMAX];
  double p[LMAX];

  template <bool HINT, class IP, class VP>
  __device__ __forceinline__ void load(IP cp, VP vp, int len, const double* __restrict__ x,
                                       uint64_t pl) {
    const int last = len - 1;
    int c[LMAX];
#pragma unroll
    for (int k = 0; k < LMAX; ++k) c[k] = cp[min(k, last)];
    // irregular matrices (HINT): predicated gathers -- clamped duplicates of
    // short rows would multiply the random L2 sector traffic that bounds them
#pragma unroll
    for (int k = 0; k < LMAX; ++k)
      p[k] = HINT ? (k <= last ? ld_hint(x + c[k], pl) : 0.0) : ld_gather(x + c[k]);
#pragma unroll
    for (int k = 0; k < LMAX; ++k) v[k] = vp[min(k, last)];
  }

  __device__ __forceinline__ double finish(int len) {
#pragma unroll
    for (int k = 0; k < LMAX; ++k) p[k] = mul(v[k], p[k]);
    const int m = len - 1, full = m & ~7;
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (1 + j < LMAX) ? p[(1 + j) % LMAX] : 0.0;
#pragma unroll
    for (int q = 1; 1 + 8 * q < LMAX; ++q)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (1 + j + 8 * q < LMAX && 8 * q < full) r[j] = add(r[j], p[(1 + j + 8 * q) % LMAX]);
    double res = -0.0;
    if (full > 0)
      res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
#pragma unroll
    for (int k = 1; k < LMAX; ++k)
      if (k > full && k <= m) res = add(res, p[k]);
    return add(p[0], res);
  }
};

template <class IP, class VP>
__device__ __noinline__ double csr_row_serial(IP cp, VP vp, int len,
                                              const double* __restrict__ x) {
  const double p0 = mul(vp[0], ld_gather(x + cp[0]));
  const double rest =
      pairwise_serial(len - 1, [&](int64_t i) { return mul(vp[1 + i], ld_gather(x + cp[1 + i])); });
  return add(p0, rest);
}

template <int LMAX, bool ACCUM, bool SKIP_LONG, bool FUSE_DOT>
__global__ void __launch_bounds__(256, 1)
    csr_pipe(int nrows, int nnz, const int* __restrict__ off, const int* __restrict__ col,
             const double* __restrict__ val, const double* __restrict__ x, double* y,
             CsrPipeCfg cfg, DotOut dot) {
  if (dot.skip()) return;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);                   // <= 8 barriers
  CsrPipeHdr* hdr = reinterpret_cast<CsrPipeHdr*>(smem + 64);            // <= 8 headers
  unsigned char* stage0 = smem + 256;
  const int tid = threadIdx.x;
  const int T = cfg.T, S = cfg.S;
  const int64_t ntiles = (nrows + T - 1) / T;
  const int64_t G = gridDim.x;
  uint64_t pol = 0;
  const uint64_t pl = policy_evict_last();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    pol = policy_evict_first();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      const int64_t t = blockIdx.x + s * G;
      if (t < ntiles) {
        const int64_t r0 = t * T;
        const int e0 = __ldg(off + r0), e1 = __ldg(off + min64(r0 + T, nrows));
        csr_pipe_issue(col, val, nnz, e0, e1, cfg, stage0 + (size_t)s * cfg.stage_bytes, &hdr[s],
                       &full[s], pol);
      }
    }
  double dsum = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G) {
    const int64_t r0 = t * T;
    const int rows = (int)min64(T, nrows - r0);
    const int i = (int)r0 + tid;
    // this row's bounds and (thread 0) the bounds of the tile issued after
    // this one, loaded before the wait so their latency overlaps it
    int o0 = 0, o1 = 0;
    if (tid < rows) {
      o0 = __ldg(off + i);
      o1 = __ldg(off + i + 1);
    }
    const int64_t tn = t + (int64_t)S * G;
    int n0 = 0, n1 = 0;
    if (tid == 0 && tn < ntiles) {
      n0 = __ldg(off + tn * T);
      n1 = __ldg(off + min64(tn * T + T, nrows));
    }
    unsigned char* st = stage0 + (size_t)s * cfg.stage_bytes;
    mbar_wait(&full[s], ph);
    const int len = o1 - o0;
    const CsrPipeHdr h = hdr[s];
    const int* s_col = reinterpret_cast<const int*>(st) + (o0 - h.bc);
    const double* s_val = reinterpret_cast<const double*>(st + 4 * (size_t)cfg.cap) + (o0 - h.bv);
    CsrRowRegs<LMAX> R;
    const bool fast = tid < rows && len >= 1 && len <= LMAX;
    const bool emit = tid < rows && !(SKIP_LONG && len > cfg.skip_above);  // else: other kernels
    double sres = 0.0;
    // phase 1: everything that reads the stage (rare serial rows entirely)
    if (fast) {
      if (cfg.hint) {
        if (!h.fat) R.template load<true>(s_col, s_val, len, x, pl);
        else R.template load<true>(col + o0, val + o0, len, x, pl);
      } else {
        if (!h.fat) R.template load<false>(s_col, s_val, len, x, pl);
        else R.template load<false>(col + o0, val + o0, len, x, pl);
      }
    } else if (emit && len > LMAX) {
      sres = h.fat ? csr_row_serial(col + o0, val + o0, len, x)
                   : csr_row_serial(s_col, s_val, len, x);
    }
    __syncthreads();  // stage s consumed: refill it while the gathers land
    if (tid == 0 && tn < ntiles)
      csr_pipe_issue(col, val, nnz, n0, n1, cfg, st, &hdr[s], &full[s], pol);
    // phase 2: products and the exact sum from registers
    if (fast) sres = R.finish(len);
    if (emit) {
      double out = ACCUM ? add(y[i], sres) : sres;
      if (dot.plus_zero) out = add(out, 0.0);
      y[i] = out;
      if (FUSE_DOT) dsum = add(dsum, mul(dot.other[i], out));
    }
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
  if (FUSE_DOT) dot.finish_block<256>(dsum);
}

template <int L, bool A, bool K, bool F>
static int csr_pipe_launch1(int64_t nrows, int64_t nnz, const int* off, const int* col, const double* val,
                            const double* x, double* y, DotOut d, CsrPipeCfg cfg, size_t smem,
                            int64_t grid, cudaStream_t st) {
  auto k = csr_pipe<L, A, K, F>;
  int rc = allow_dynamic_smem(reinterpret_cast<const void*>(k), smem);
  if (rc) return rc;
  k<<<(unsigned)grid, cfg.T, smem, st>>>((int)nrows, (int)nnz, off, col, val, x, y, cfg, d);
  DS_LAUNCH_CHECK("csr_pipe");
  return DS_OK;
}

// max_len: longest row if known (<= 27 selects the 27-wide register path),
// else 0.  Returns DS_ERR_NOT_SUPPORTED (nothing launched) when the pipeline
// cannot run (misaligned arrays, shared memory).
static int csr_pipe_launch(int64_t nrows, int64_t nnz, const int* off, const int* col, const double* val,
                           const double* x, double* y, bool accum, bool skip_long, int max_len,
                           DotOut d, bool fuse, cudaStream_t st, int skip_above = kLongRow,
                           bool hint = false) {
  static int eT = -2, eS = -2, eC = -2;
  if (eT == -2) {
    const char* a = getenv("DS_CSR_T");
    const char* b = getenv("DS_CSR_S");
    const char* c = getenv("DS_CSR_CTAS");
    eT = a ? atoi(a) : -1;
    eS = b ? atoi(b) : -1;
    eC = c ? atoi(c) : -1;
  }
  const bool aligned = ((reinterpret_cast<uintptr_t>(col) | reinterpret_cast<uintptr_t>(val)) &
                        15) == 0;
  if (!aligned) return DS_ERR_NOT_SUPPORTED;
  const int L = (max_len > 0 && max_len <= 27) ? 27 : 33;
  CsrPipeCfg cfg;
  // measured at 104^3 (tools/sweep_csr.sh): 128 rows x 2 stages x 2 CTAs/SM
  // 59.9 us, 256 x 2 x 1 61.9 us, 192 x 2 x 1 70.1 us, 128 x 4 x 1 86.5 us
  cfg.T = eT > 0 ? eT : 128;
  cfg.S = eS > 0 ? min(eS, 8) : 2;
  cfg.cap = ((cfg.T * (max_len > 0 ? min(max_len, L) : 27) + 8) + 3) & ~3;
  cfg.stage_bytes = (int)((12 * (int64_t)cfg.cap + 127) & ~127);
  cfg.skip_above = skip_above;
  static int eH = -2;
  if (eH == -2) {
    const char* h = getenv("DS_CSR_HINT");
    eH = h ? atoi(h) : -1;
  }
  cfg.hint = eH >= 0 ? eH : (hint ? 1 : 0);
  const size_t smem = 256 + (size_t)cfg.S * cfg.stage_bytes;
  if (cfg.T > 256 || cfg.T < 32 || smem > (size_t)max_dynamic_smem() - 1024)
    return DS_ERR_NOT_SUPPORTED;
  const int64_t ntiles = ceil_div(nrows, cfg.T);
  int64_t grid = (int64_t)sm_count() * (eC > 0 ? eC : 2);
  if (grid > ntiles) grid = ntiles;
  if (fuse) grid = d.clamp_grid(grid);
#define DS_CSRP(Lv, A, K, F) \
  return csr_pipe_launch1<Lv, A, K, F>(nrows, nnz, off, col, val, x, y, d, cfg, smem, grid, st)
#define DS_CSRP_L(A, K, F)          \
  do {                              \
    if (L == 27) DS_CSRP(27, A, K, F); \
    DS_CSRP(33, A, K, F);           \
  } while (0)
  if (fuse) {
    if (accum) DS_CSRP_L(true, false, true); else DS_CSRP_L(false, false, true);
  } else if (skip_long) {
    if (accum) DS_CSRP_L(true, true, false); else DS_CSRP_L(false, true, false);
  } else {
    if (accum) DS_CSRP_L(true, false, false); else DS_CSRP_L(false, false, false);
  }
#undef DS_CSRP_L
#undef DS_CSRP
}
// One CTA per long row: the pairwise recursion tree is cut into subtrees of
// at most kSub addends; each subtree's leaves (64..128 addends each) are
// summed by the CTA's 32 lane-groups in parallel, then thread 0 replays the
// recursion to combine them in numpy's order.

// Warp per long row (kLongRow < len <= kWarpRow): lane 0 enumerates the pairwise
// recursion's leaves (64..128 addends each) into warp-private shared memory,
// the warp's four 8-lane groups sum leaves in parallel, lane 0 replays the
// recursion to combine them.  No block-wide barriers, 8 rows per CTA.
constexpr int kWarpLeaves = 128;
constexpr int kWarpRow = kCsrWarpRow;   // warp kernel: rows of kLongRow+1 .. kWarpRow entries

template <bool ACCUM>
__global__ void __launch_bounds__(kCsrBlock, 2)
    csr_long_rows_warp(const int* __restrict__ rows, int n, const int* __restrict__ off,
                       const int* __restrict__ col, const double* __restrict__ val,
                       const double* __restrict__ x, double* y, const int* guard) {
  if (guard && *guard) return;
  __shared__ int s_lo[kCsrBlock / 32][kWarpLeaves];
  __shared__ short s_n[kCsrBlock / 32][kWarpLeaves];
  __shared__ double s_v[kCsrBlock / 32][kWarpLeaves];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, lane8 = lane & 7, grp = lane >> 3;
  const unsigned mask = 0xffu << (lane & 24);
  struct Frame {
    int lo, n, expanded;
  };
  const int nw = gridDim.x * (kCsrBlock / 32);
  for (int li = blockIdx.x * (kCsrBlock / 32) + w; li < n; li += nw) {
    const int row = rows[li];
    const int start = off[row];
    const int m = off[row + 1] - start - 1;
    if (m + 1 > kWarpRow) continue;      // the CTA kernel owns it
    int nl = 0;
    if (lane == 0) {                      // leaves left to right
      Frame st[32];
      int ft = 0;
      st[ft++] = {0, m, 0};
      while (ft > 0) {
        Frame f = st[--ft];
        if (f.n <= 128) {
          s_lo[w][nl] = f.lo;
          s_n[w][nl] = (short)f.n;
          ++nl;
        } else {
          int n2 = f.n / 2;
          n2 -= n2 % 8;
          st[ft++] = {f.lo + n2, f.n - n2, 0};
          st[ft++] = {f.lo, n2, 0};
        }
      }
    }
    nl = __shfl_sync(0xffffffffu, nl, 0);
    __syncwarp();
    for (int l = grp; l < nl; l += 4) {
      const double v = csr_leaf_g8_all(col, val, x, (int64_t)start + 1 + s_lo[w][l], s_n[w][l],
                                       lane8, mask);
      if (lane8 == 0) s_v[w][l] = v;
    }
    __syncwarp();
    if (lane == 0) {                      // combine in recursion order
      Frame st[32];
      double vs[32];
      int ft = 0, vt = 0, next = 0;
      st[ft++] = {0, m, 0};
      while (ft > 0) {
        Frame f = st[--ft];
        if (f.n <= 128) {
          vs[vt++] = s_v[w][next++];
        } else if (!f.expanded) {
          int n2 = f.n / 2;
          n2 -= n2 % 8;
          st[ft++] = {f.lo, f.n, 1};
          st[ft++] = {f.lo + n2, f.n - n2, 0};
          st[ft++] = {f.lo, n2, 0};
        } else {
          const double b = vs[--vt];
          const double a = vs[--vt];
          vs[vt++] = add(a, b);
        }
      }
      const double p0 = mul(val[start], __ldg(x + col[start]));
      const double sres = add(p0, vs[0]);
      y[row] = ACCUM ? add(y[row], sres) : sres;
    }
    __syncwarp();
  }
}

template <bool ACCUM>
__global__ void __launch_bounds__(kCsrBlock, 2)
    csr_long_rows(const int* __restrict__ long_rows, int n_long, const int* __restrict__ off,
                  const int* __restrict__ col, const double* __restrict__ val,
                  const double* __restrict__ x, double* y, const int* guard) {
  if (guard && *guard) return;
  __shared__ int64_t s_leaf_lo[kMaxLeaves];
  __shared__ int s_leaf_n[kMaxLeaves];
  __shared__ double s_leaf_v[kMaxLeaves];
  __shared__ int64_t s_lo, s_n;
  __shared__ int s_cmd, s_nleaves;
  const int tid = threadIdx.x, lane8 = tid & 7, grp = tid >> 3;
  const unsigned mask = 0xffu << (tid & 24);
  struct Frame {
    int64_t lo, n;
    int expanded;
  };
  for (int li = blockIdx.x; li < n_long; li += gridDim.x) {
    const int row = long_rows[li];
    const int64_t start = off[row];
    const int64_t m = (int64_t)off[row + 1] - start - 1;
    if (m + 1 <= kWarpRow) continue;   // csr_long_rows_warp owns it
    const int64_t base = start + 1;
    // thread-0 top-level DFS state
    Frame st[48];
    double vs[48];
    int ft = 0, vt = 0;
    if (tid == 0) st[ft++] = {0, m, 0};
    for (;;) {
      if (tid == 0) {
        s_cmd = 0;
        while (ft > 0) {
          Frame f = st[--ft];
          if (f.n <= kSub) {
            s_lo = f.lo;
            s_n = f.n;
            s_cmd = 1;
            break;
          }
          if (!f.expanded) {
            int64_t n2 = f.n / 2;
            n2 -= n2 % 8;
            st[ft++] = {f.lo, f.n, 1};
            st[ft++] = {f.lo + n2, f.n - n2, 0};
            st[ft++] = {f.lo, n2, 0};
          } else {
            double b = vs[--vt];
            double a = vs[--vt];
            vs[vt++] = add(a, b);
          }
        }
        if (s_cmd) {  // enumerate this subtree's leaves left to right
          Frame sst[32];
          int sft = 0, nl = 0;
          sst[sft++] = {s_lo, s_n, 0};
          while (sft > 0) {
            Frame f = sst[--sft];
            if (f.n <= 128) {
              s_leaf_lo[nl] = f.lo;
              s_leaf_n[nl] = (int)f.n;
              ++nl;
            } else {
              int64_t n2 = f.n / 2;
              n2 -= n2 % 8;
              sst[sft++] = {f.lo + n2, f.n - n2, 0};
              sst[sft++] = {f.lo, n2, 0};
            }
          }
          s_nleaves = nl;
        }
      }
      __syncthreads();
      if (!s_cmd) break;
      for (int l = grp; l < s_nleaves; l += kCsrBlock / 8) {
        double v = csr_leaf_g8_all(col, val, x, base + s_leaf_lo[l], s_leaf_n[l], lane8, mask);
        if (lane8 == 0) s_leaf_v[l] = v;
      }
      __syncthreads();
      if (tid == 0) {  // combine the subtree in recursion order
        Frame sst[32];
        double svs[32];
        int sft = 0, svt = 0, next_leaf = 0;
        sst[sft++] = {s_lo, s_n, 0};
        while (sft > 0) {
          Frame f = sst[--sft];
          if (f.n <= 128) {
            svs[svt++] = s_leaf_v[next_leaf++];
          } else if (!f.expanded) {
            int64_t n2 = f.n / 2;
            n2 -= n2 % 8;
            sst[sft++] = {f.lo, f.n, 1};
            sst[sft++] = {f.lo + n2, f.n - n2, 0};
            sst[sft++] = {f.lo, n2, 0};
          } else {
            double b = svs[--svt];
            double a = svs[--svt];
            svs[svt++] = add(a, b);
          }
        }
        vs[vt++] = svs[0];
      }
      __syncthreads();
    }
    if (tid == 0) {
      const double p0 = mul(val[start], __ldg(x + col[start]));
      const double s = add(p0, vs[0]);
      y[row] = ACCUM ? add(y[row], s) : s;
    }
    __syncthreads();
  }
}

__global__ void csr_find_long(int nrows, const int* __restrict__ off, int* long_rows,
                              unsigned* count, int* max_len) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int len = off[r + 1] - off[r];
    if (len > kLongRow) long_rows[atomicAdd(count, 1u)] = r;
    atomicMax(max_len, len);
  }
}

// long-row kernels for the rows > kLongRow listed by ds_csr_analyze
// Each kernel skips the rows of the other one, so an unsorted list
// (ds_csr_analyze) may be passed to both; the bins plan passes exact lists.
static int launch_csr_long2(const int* warp_rows, int64_t n_warp, const int* cta_rows,
                            int64_t n_cta, const int* off, const int* col, const double* val,
                            const double* x, double* y, bool accum, const int* guard,
                            cudaStream_t st) {
  if (n_warp > 0) {
    const int64_t lw = min64(ceil_div(n_warp, kCsrBlock / 32), (int64_t)sm_count() * 8);
    if (accum)
      csr_long_rows_warp<true><<<(unsigned)lw, kCsrBlock, 0, st>>>(warp_rows, (int)n_warp, off,
                                                                  col, val, x, y, guard);
    else
      csr_long_rows_warp<false><<<(unsigned)lw, kCsrBlock, 0, st>>>(warp_rows, (int)n_warp, off,
                                                                   col, val, x, y, guard);
  }
  if (n_cta > 0) {
    const int64_t lb = min64(n_cta, (int64_t)sm_count() * 8);
    if (accum)
      csr_long_rows<true><<<(unsigned)lb, kCsrBlock, 0, st>>>(cta_rows, (int)n_cta, off, col, val,
                                                             x, y, guard);
    else
      csr_long_rows<false><<<(unsigned)lb, kCsrBlock, 0, st>>>(cta_rows, (int)n_cta, off, col,
                                                              val, x, y, guard);
  }
  DS_LAUNCH_CHECK("csr_long_rows");
  return DS_OK;
}

static int launch_csr_long(const int* long_rows, int64_t n_long, const int* off, const int* col,
                           const double* val, const double* x, double* y, bool accum,
                           const int* guard, cudaStream_t st) {
  return launch_csr_long2(long_rows, n_long, long_rows, n_long, off, col, val, x, y, accum, guard,
                          st);
}

int launch_csr_binned(int64_t nrows, int64_t ncols, int64_t nnz, const int* off, const int* col,
                      const double* val, const int* perm, const int64_t* bins, const double* x,
                      double* y, bool accum, const DotOut* dot, cudaStream_t st) {
  if (nrows == 0) return DS_OK;
  DotOut d = dot ? *dot : DotOut{};
  const bool fuse = d.fused();
  static int binned_only = -1;
  if (binned_only < 0) binned_only = getenv("DS_CSR_BINNED_ONLY") ? 1 : 0;
  // Irregular matrix: the TMA pipeline takes every row of <= 33 entries (the
  // bulk of a power-law matrix), the binned kernel only bin 5 (34..129) and
  // the long-row kernels bin 6; x gathers carry L2 evict_last.  (A fused dot
  // needs one kernel to own every row: it keeps the all-binned path.)
  if (!fuse && !binned_only && nnz > 0 && nnz < (1ll << 31)) {
    const int rc = csr_pipe_launch(nrows, nnz, off, col, val, x, y, accum, true, 33, d, false, st,
                                   33, true);
    if (rc == DS_OK) {
      int64_t rest[kCsrBinCount + 1];
      for (int b = 0; b <= kCsrBinCount; ++b) rest[b] = b < 5 ? bins[5] : bins[b];
      if (rest[kCsrBinCount] == rest[5]) return DS_OK;
      return launch_csr_binned(nrows, ncols, 0, off, col, val, perm, rest, x, y, accum, dot, st);
    }
    if (rc != DS_ERR_NOT_SUPPORTED) return rc;
  }
  const int64_t n_long = bins[8] - bins[6];
  if (fuse && n_long > 0) {
    set_error("fused dot with long rows is not supported");
    return DS_ERR_NOT_SUPPORTED;
  }
  CsrBins bi;
  int64_t acc = 0;
  for (int b = 0; b < 8; ++b) bi.start[b] = bins[b];   // bins 0..5 (+ end of 5)
  for (int b = 0; b < 6; ++b) {
    bi.pair_off[b] = acc;
    acc += ceil_div(bins[b + 1] - bins[b], kBinRowsHost[b]);
  }
  bi.pair_off[6] = acc;
  bi.pair_off[7] = acc;
  int64_t blocks = ceil_div(acc * 8, kCsrBlock);
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (fuse) blocks = d.clamp_grid(blocks);
  // the binned path serves irregular matrices whose x is gathered at random:
  // keep x persisting in L2 while the row stream passes through
  const bool win = x_window_begin(st, x, (size_t)ncols * 8);
#define DS_CSRB(A, F) \
  csr_binned<A, F><<<(unsigned)blocks, kCsrBlock, 0, st>>>(off, col, val, x, y, perm, bi, d)
  if (accum) {
    if (fuse) DS_CSRB(true, true); else DS_CSRB(true, false);
  } else {
    if (fuse) DS_CSRB(false, true); else DS_CSRB(false, false);
  }
#undef DS_CSRB
  DS_LAUNCH_CHECK("csr_binned");
  if (n_long > 0) {
    const int rc = launch_csr_long2(perm + bins[6], bins[7] - bins[6], perm + bins[7],
                                    bins[8] - bins[7], off, col, val, x, y, accum, d.guard, st);
    if (rc) return rc;
  }
  if (win) x_window_end(st);
  return DS_OK;
}

// A matrix without entries (e.g. the remote part of a partition without
// ghosts): y = 0 (spmv) or y = y + 0.0 (spmv_add, kernels.py:196-198: the
// +0.0 turns -0.0 into +0.0).  One streaming pass instead of a full SpMV
// kernel walking empty tiles.
__global__ void empty_matrix_kernel(int64_t n, double* y, int accum, const int* guard) {
  if (guard && *guard) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = accum ? add(y[i], 0.0) : 0.0;
}
static int launch_empty_matrix(int64_t nrows, double* y, bool accum, const int* guard,
                               cudaStream_t st) {
  const unsigned g = (unsigned)min64(ceil_div(nrows, 256), (int64_t)sm_count() * 8);
  empty_matrix_kernel<<<g, 256, 0, st>>>(nrows, y, accum ? 1 : 0, guard);
  DS_LAUNCH_CHECK("empty_matrix_kernel");
  return DS_OK;
}

int launch_csr(int64_t nrows, int64_t nnz, const int* off, const int* col, const double* val,
               const int* long_rows, int64_t n_long, int max_len, const double* x, double* y,
               bool accum, const DotOut* dot, cudaStream_t st) {
  if (nrows == 0) return DS_OK;
  if (nnz == 0 && !(dot && dot->fused()))
    return launch_empty_matrix(nrows, y, accum, dot ? dot->guard : nullptr, st);
  const int64_t groups = (nrows + 1) / 2;   // one 8-lane group per row pair
  int64_t blocks = ceil_div(groups * 8, kCsrBlock);
  static int eB = -2, use_g8 = -1;
  if (eB == -2) {
    const char* e = getenv("DS_CSR_BLOCKS_PER_SM");
    eB = e ? atoi(e) : -1;
    use_g8 = getenv("DS_CSR_G8") ? 1 : 0;
  }
  // 8 resident CTAs per SM (measured best: 84 us vs 97 us for a 16-wave grid)
  const int64_t cap = (int64_t)sm_count() * (eB > 0 ? eB : 8);
  if (blocks > cap) blocks = cap;
  const bool skip = (long_rows != nullptr);
  DotOut d = dot ? *dot : DotOut{};
  const bool fuse = d.fused();
  if (fuse && skip && n_long > 0) {
    set_error("fused dot with long rows is not supported");
    return DS_ERR_NOT_SUPPORTED;
  }
  // the TMA pipeline needs the long-row plan (long_rows != NULL, possibly
  // empty): rows > kLongRow are then computed by the long-row kernels
  if (!use_g8 && skip) {
    const int rc = csr_pipe_launch(nrows, nnz, off, col, val, x, y, accum, n_long > 0, max_len, d,
                                   fuse, st);
    if (rc == DS_OK)
      return launch_csr_long(long_rows, n_long, off, col, val, x, y, accum, d.guard, st);
    if (rc != DS_ERR_NOT_SUPPORTED) return rc;
  }
  if (fuse) blocks = d.clamp_grid(blocks);
#define DS_CSR(A, S, F) \
  csr_rows_g8<A, S, F><<<(unsigned)blocks, kCsrBlock, 0, st>>>((int)nrows, off, col, val, x, y, d)
  if (fuse) {
    if (skip && n_long > 0) {
      set_error("fused dot with long rows is not supported");
      return DS_ERR_NOT_SUPPORTED;
    }
    if (accum) DS_CSR(true, false, true); else DS_CSR(false, false, true);
  } else if (skip) {
    if (accum) DS_CSR(true, true, false); else DS_CSR(false, true, false);
  } else {
    if (accum) DS_CSR(true, false, false); else DS_CSR(false, false, false);
  }
#undef DS_CSR
  DS_LAUNCH_CHECK("csr_rows_g8");
  return skip ? launch_csr_long(long_rows, n_long, off, col, val, x, y, accum, d.guard, st)
              : DS_OK;
}

// ===================================================================== DIA ==

constexpr int kDiaBlock = 256;

// Persistent variant: grid = a few CTAs per SM, tile t = blockIdx.x + k*G
// (static, deterministic schedule).  Each CTA keeps S tiles of T rows in
// flight: thread 0 issues one 1-D TMA bulk copy per tile into a ring of S
// shared-memory stages (mbarrier transaction counts signal arrival) and
// refills a stage as soon as the CTA has finished reading it, so HBM
// streaming never waits on the x gathers / add chains of the consumers.
// The fused dot needs only G block partials.
struct DiaPipeCfg {
  int T;        // rows per tile (== blockDim.x, even)
  int S;        // stages
  int stage_bytes;
  int xw_len;   // x window length per offset group (doubles), 0: gather x instead
  int idx_off;  // byte offset in a stage of the per-diagonal window index table
  int xw_off;   // byte offset in a stage of the x windows
  int xw_min_span;   // use the windows only if the offsets span more rows than this
};

// x windows (ND = 27 stencil-like matrices): the sorted offsets fall into
// groups of consecutive values (the 27-point stencil: 9 groups of 3).  For a
// tile of rows [r0, r0+T) group g needs x[r0+first_g .. r0+T+last_g): one
// contiguous window per group, staged by TMA next to the value slab, so the
// 27 gathers per row become shared-memory loads (no L1 misses: at 192^3 a
// plane of x no longer fits the L1 that the stages leave).
constexpr int kXwGroups = 9;
constexpr int kXwSpan = 4;   // max last_g - first_g handled

struct XwPlan {
  int ng;
  int first[kXwGroups], last[kXwGroups];
  int jg[32];   // group of diagonal j
};

// windows of tile t: x copies into `win`, per-diagonal indices into `sidx`.
// Called by all 32 lanes of warp 0 (after griddepcontrol.wait: x may be the
// previous kernel's output): lane g issues group g's copy, lane j < nd writes
// sidx[j]; one arrive carries the summed transaction bytes.  (A single
// issuing thread made this a ~2 us serial section per tile.)
__device__ __forceinline__ void dia_issue_windows(const double* __restrict__ x, int64_t nrows,
                                                  int ncols, int nd, int T, int64_t t,
                                                  const int* s_off, const XwPlan& pl, int wl,
                                                  int* sidx, double* win, uint64_t* bar,
                                                  uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = t * T;
  const int rows = (int)min64(T, nrows - r0);
  const int64_t ce = (int64_t)(ncols & ~1);
  int64_t lo = 0, hi = 0, wlo = 0;
  if (lane < pl.ng) {
    wlo = (r0 + pl.first[lane]) & ~1ll;                   // even: 16-B aligned source
    const int64_t whi = r0 + rows + pl.last[lane];         // exclusive
    const int64_t hi_a = (whi + 1) & ~1ll;
    lo = wlo > 0 ? wlo : 0;
    hi = hi_a < ce ? hi_a : ce;
    if ((ncols & 1) && ncols - 1 >= wlo && ncols - 1 < whi)   // odd tail by hand
      win[lane * wl + (ncols - 1 - wlo)] = x[ncols - 1];
  }
  if (lane < nd) {
    const int g = pl.jg[lane];
    const int64_t wg = (r0 + pl.first[g]) & ~1ll;
    sidx[lane] = (int)(g * wl + (r0 + s_off[lane] - wg));
  }
  uint32_t bytes = (lane < pl.ng && hi > lo) ? (uint32_t)(hi - lo) * 8u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane < pl.ng && hi > lo)
    bulk_g2s(win + lane * wl + (lo - wlo), x + lo, (uint32_t)(hi - lo) * 8u, bar, pol);
}

__device__ __forceinline__ void dia_issue_tile(const double* __restrict__ vals, int64_t nrows,
                                               int nd, int T, int64_t t, double* stage,
                                               uint64_t* bar, uint64_t pol) {
  const int64_t r0 = t * T;
  const int rows = (int)min64(T, nrows - r0);
  const uint32_t bytes = (uint32_t)rows * (uint32_t)nd * 8u;
  const uint32_t bulk = bytes & ~15u;
  if (bulk != bytes) stage[bulk / 8] = vals[r0 * nd + bulk / 8];  // before the arrive (release)
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, bulk);
  if (bulk) bulk_g2s(stage, vals + r0 * nd, bulk, bar, pol);
}

template <bool ACCUM, bool FUSE_DOT, int ND>
__global__ void __launch_bounds__(256, 1)   // 1 CTA/SM: registers for all 27 gathers in flight
    dia_pipe(int nrows, int ncols, int ndiags_rt, const int* __restrict__ offsets,
             const double* __restrict__ vals, const double* __restrict__ x, double* y,
             DiaPipeCfg cfg, DotOut dot) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int nd = ND > 0 ? ND : ndiags_rt;
  const int T = cfg.T, S = cfg.S;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);               // <= 4 barriers
  uint64_t* xfull = full + 4;                                        // x windows, <= 4
  int* s_off = reinterpret_cast<int*>(smem + 64);
  unsigned char* stage0 = smem + 64 + ((nd * 4 + 127) & ~127);
  __shared__ XwPlan s_pl;
  __shared__ int s_xw;
  const int tid = threadIdx.x;
  const int64_t ntiles = (nrows + T - 1) / T;
  const int64_t G = gridDim.x;
  uint64_t pol = 0, pol_x = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&xfull[s], 1);
    }
    fence_barrier_init();
    pol = policy_evict_first();
  }
  if (tid < 32) pol_x = policy_evict_last();   // the lanes issuing x-window copies
  for (int j = tid; j < nd; j += blockDim.x) s_off[j] = offsets[j];
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < S; ++s) {
      const int64_t t = blockIdx.x + s * G;
      if (t < ntiles)
        dia_issue_tile(vals, nrows, nd, T, t,
                       reinterpret_cast<double*>(stage0 + (size_t)s * cfg.stage_bytes), &full[s],
                       pol);
    }
  // offset groups for the x windows (after the first value copies are on
  // their way; only when the launch laid windows out)
  if (ND == 27 && cfg.xw_len > 0) {
  if (tid == 0) {
    int ng = 0, ok = nd <= 32;
    for (int j = 0; ok && j < nd; ++j) {
      if (j == 0 || s_off[j] - s_off[j - 1] > 1) {
        if (ng == kXwGroups) { ok = 0; break; }
        s_pl.first[ng] = s_off[j];
        ++ng;
      }
      s_pl.last[ng - 1] = s_off[j];
      s_pl.jg[j] = ng - 1;
      if (s_pl.last[ng - 1] - s_pl.first[ng - 1] > kXwSpan) ok = 0;
    }
    s_pl.ng = ng;
    // small spans: the gathers hit L1 (104^3: 21.8K-row span, windows 49 vs
    // 43 us); large ones miss it (192^3: 74K rows, windows 267 vs 285 us)
    s_xw = ok && (s_off[nd - 1] - s_off[0]) > cfg.xw_min_span;
  }
  __syncthreads();
  }
  const bool xw = ND == 27 && cfg.xw_len > 0 && s_xw;
  // Programmatic dependent launch (the CG step): the matrix prefetch above
  // depends on nothing the previous kernel writes; everything below does
  // (x, the guard, y and the partials the previous kernel reads).  A no-op
  // for a normal launch.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (dot.skip()) {   // converged: drain the issued copies before exiting
    if (tid == 0)
      for (int s = 0; s < S; ++s)
        if (blockIdx.x + (int64_t)s * G < ntiles) mbar_wait(&full[s], 0);
    return;
  }
  if (xw && tid < 32)   // x windows of the first stages (x is now final)
    for (int s = 0; s < S; ++s) {
      const int64_t t = blockIdx.x + s * G;
      if (t < ntiles) {
        unsigned char* st = stage0 + (size_t)s * cfg.stage_bytes;
        dia_issue_windows(x, nrows, ncols, nd, T, t, s_off, s_pl, cfg.xw_len,
                          reinterpret_cast<int*>(st + cfg.idx_off),
                          reinterpret_cast<double*>(st + cfg.xw_off), &xfull[s], pol_x);
      }
    }
  double dsum = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G) {
    const double* v_stage = reinterpret_cast<const double*>(stage0 + (size_t)s * cfg.stage_bytes);
    mbar_wait(&full[s], ph);
    if (xw) mbar_wait(&xfull[s], ph);
    const int64_t r0 = t * T;
    const int rows = (int)min64(T, nrows - r0);
    if (tid < rows) {
      const int i = (int)r0 + tid;
      const double* v = v_stage + (size_t)tid * nd;
      // Unpredicated gathers (clamped index) so all nd loads are in flight at
      // once; out-of-range slots contribute a selected +0.0.  acc starts at
      // +0.0 and can never become -0.0 (x + (-x) rounds to +0.0), so adding
      // +0.0 is the identity: bitwise equal to skipping the slot
      // (kernels.py:133-138).
      double xv[ND > 0 ? ND : 1];
      double acc = 0.0;
      if (ND > 0) {
        if (xw) {   // from the staged windows (slots outside [0, ncols) are discarded below)
          const unsigned char* stb = stage0 + (size_t)s * cfg.stage_bytes;
          const int* sidx = reinterpret_cast<const int*>(stb + cfg.idx_off);
          const double* win = reinterpret_cast<const double*>(stb + cfg.xw_off);
#pragma unroll
          for (int j = 0; j < (ND > 0 ? ND : 1); ++j) xv[j] = win[sidx[j] + tid];
        } else {
#pragma unroll
          for (int j = 0; j < (ND > 0 ? ND : 1); ++j) {
            const int c = i + s_off[j];
            xv[j] = ld_gather(x + min(max(c, 0), ncols - 1));
          }
        }
#pragma unroll
        for (int j = 0; j < ND; ++j) {
          const int c = i + s_off[j];
          const double pr = mul(v[j], xv[j]);
          acc = add(acc, (c >= 0 && c < ncols) ? pr : 0.0);
        }
      } else {
        for (int j = 0; j < nd; ++j) {
          const int c = i + s_off[j];
          if (c >= 0 && c < ncols) acc = add(acc, mul(v[j], ld_gather(x + c)));
        }
      }
      double out = ACCUM ? add(y[i], acc) : acc;
      if (dot.plus_zero) out = add(out, 0.0);
      y[i] = out;
      if (FUSE_DOT) {
        // p.Ap with p == x (the CG case): x[i] was already gathered for the
        // main diagonal; otherwise load it
        // p.Ap with p == x (the CG case): p[i] was just gathered by this
        // thread for the main diagonal, so this load hits L1 (selecting the
        // gathered value instead costs a compare + select per diagonal)
        const double pi = __ldg(dot.other + i);
        dsum = add(dsum, mul(pi, out));
      }
    }
    __syncthreads();  // stage s fully consumed
    if (tid < 32) {
      const int64_t tn = t + (int64_t)S * G;
      if (tn < ntiles) {
        unsigned char* st = stage0 + (size_t)s * cfg.stage_bytes;
        if (tid == 0)
          dia_issue_tile(vals, nrows, nd, T, tn, reinterpret_cast<double*>(st), &full[s], pol);
        if (xw)
          dia_issue_windows(x, nrows, ncols, nd, T, tn, s_off, s_pl, cfg.xw_len,
                            reinterpret_cast<int*>(st + cfg.idx_off),
                            reinterpret_cast<double*>(st + cfg.xw_off), &xfull[s], pol_x);
      }
    }
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
  if (FUSE_DOT) dot.finish_block<256>(dsum);
}

// Fallback when the slab cannot be staged (huge ndiags or misaligned base):
// one thread per row reading straight from global memory.
template <bool ACCUM, bool FUSE_DOT>
__global__ void __launch_bounds__(kDiaBlock)
    dia_rows_direct(int nrows, int ncols, int ndiags, const int* __restrict__ offsets,
                    const double* __restrict__ vals, const double* __restrict__ x, double* y,
                    DotOut dot) {
  if (dot.skip()) return;
  double dsum = 0.0;
  const int i = blockIdx.x * kDiaBlock + threadIdx.x;
  if (i < nrows) {
    double acc = 0.0;
    const double* v = vals + (size_t)i * ndiags;
    for (int j = 0; j < ndiags; ++j) {
      const int c = i + __ldg(offsets + j);
      if (c >= 0 && c < ncols) acc = add(acc, mul(v[j], ld_gather(x + c)));
    }
    double out = ACCUM ? add(y[i], acc) : acc;
    if (dot.plus_zero) out = add(out, 0.0);
    y[i] = out;
    if (FUSE_DOT) dsum = mul(dot.other[i], out);
  }
  if (FUSE_DOT) dot.finish_block<kDiaBlock>(dsum);
}

template <bool A, bool F, int ND>
static int dia_pipe_launch(int64_t nrows, int64_t ncols, int ndiags, const int* off,
                           const double* val, const double* x, double* y, DotOut d,
                           DiaPipeCfg cfg, size_t smem, int64_t grid, cudaStream_t st) {
  auto k = dia_pipe<A, F, ND>;
  int rc = allow_dynamic_smem(reinterpret_cast<const void*>(k), smem);
  if (rc) return rc;
  static int no_pdl = -1;
  if (no_pdl < 0) no_pdl = getenv("DS_NO_PDL") ? 1 : 0;
  if (F && d.partials_only && !no_pdl) {
    // single-partition CG step: may start while the previous kernel (the
    // fused update/direction) finishes -- the kernel waits (griddepcontrol)
    // before touching anything that kernel writes
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3((unsigned)cfg.T);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    DS_CUDA(cudaLaunchKernelEx(&lc, k, (int)nrows, (int)ncols, ndiags, off, val, x, y, cfg, d));
    return DS_OK;
  }
  k<<<(unsigned)grid, cfg.T, smem, st>>>((int)nrows, (int)ncols, ndiags, off, val, x, y, cfg, d);
  DS_LAUNCH_CHECK("dia_pipe");
  return DS_OK;
}

// tile shape: env DS_DIA_T / DS_DIA_S / DS_DIA_CTAS override (tuning only)
static void dia_shape(int ndiags, int* T, int* S, int* ctas) {
  static int eT = -2, eS = -2, eC = -2;
  if (eT == -2) {
    const char* a = getenv("DS_DIA_T");
    const char* b = getenv("DS_DIA_S");
    const char* c = getenv("DS_DIA_CTAS");
    eT = a ? atoi(a) : -1;
    eS = b ? atoi(b) : -1;
    eC = c ? atoi(c) : -1;
  }
  *T = 256;
  *S = 3;
  *ctas = 1;
  // keep each stage <= ~64 KB
  while (*T > 32 && (int64_t)(*T) * ndiags * 8 > 64 * 1024) *T /= 2;
  if (eT > 0) *T = eT;
  if (eS > 0) *S = eS;
  if (eC > 0) *ctas = eC;
}

int launch_dia(int64_t nrows, int64_t ncols, int ndiags, const int* off, const double* val,
               const double* x, double* y, bool accum, const DotOut* dot, cudaStream_t st) {
  if (nrows == 0) return DS_OK;
  DotOut d = dot ? *dot : DotOut{};
  const bool fuse = d.fused();
  const bool aligned = (reinterpret_cast<uintptr_t>(val) & 15) == 0;
  int T, S, ctas;
  dia_shape(ndiags, &T, &S, &ctas);
  static int no_xw = -1, force_xw = 0;
  if (no_xw < 0) {
    no_xw = getenv("DS_DIA_NO_XWIN") ? 1 : 0;
    force_xw = getenv("DS_DIA_XWIN_FORCE") ? 1 : 0;   // tests: windows at any size
  }
  // x windows next to the value slab (27 diagonals, 16-B aligned x)
  // The window area shrinks the L1 that the gathers of smaller grids live on
  // (104^3: 43 -> 45.5 us standalone, 44 -> 50 us inside the CG step), so it
  // is only laid out for large operators (192^3: 285 -> 267 us); the kernel
  // also checks the offsets' span.
  const bool xwin = !no_xw && ndiags == 27 && (nrows >= (4ll << 20) || force_xw) &&
                    (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int slab = (int)((((int64_t)T * ndiags * 8) + 127) & ~127ll);
  const int wl = (T + kXwSpan + 4 + 1) & ~1;
  const int idx_bytes = xwin ? ((ndiags * 4 + 127) & ~127) : 0;
  const int win_bytes = xwin ? ((kXwGroups * wl * 8 + 127) & ~127) : 0;
  const int stage_bytes = slab + idx_bytes + win_bytes;
  const size_t smem = 64 + ((ndiags * 4 + 127) & ~127) + (size_t)S * stage_bytes;
  if (aligned && ndiags > 0 && S <= 4 && T >= 32 && smem <= (size_t)max_dynamic_smem() - 1024) {
    const int64_t ntiles = ceil_div(nrows, T);
    int64_t grid = (int64_t)sm_count() * ctas;
    if (grid > ntiles) grid = ntiles;
    if (fuse) grid = d.clamp_grid(grid);
    static int span = -2;
    if (span == -2) {
      const char* e = getenv("DS_DIA_XWIN_SPAN");
      span = e ? atoi(e) : 40000;
    }
    DiaPipeCfg cfg{T, S, stage_bytes, xwin ? wl : 0, slab, slab + idx_bytes, span};
#define DS_DIAP(A, F)                                                                           \
  return (ndiags == 27)                                                                         \
             ? dia_pipe_launch<A, F, 27>(nrows, ncols, ndiags, off, val, x, y, d, cfg, smem,    \
                                         grid, st)                                              \
             : dia_pipe_launch<A, F, 0>(nrows, ncols, ndiags, off, val, x, y, d, cfg, smem,     \
                                        grid, st)
    if (accum) {
      if (fuse) DS_DIAP(true, true); else DS_DIAP(true, false);
    } else {
      if (fuse) DS_DIAP(false, true); else DS_DIAP(false, false);
    }
#undef DS_DIAP
  }
  const int64_t blocks = ceil_div(nrows, kDiaBlock);
  if (fuse && d.clamp_grid(blocks) != blocks) {
    set_error("fused dot grid too large");
    return DS_ERR_NOT_SUPPORTED;
  }
#define DS_DIAD(A, F)                                                                   \
  dia_rows_direct<A, F><<<(unsigned)blocks, kDiaBlock, 0, st>>>((int)nrows, (int)ncols, \
                                                               ndiags, off, val, x, y, d)
  if (accum) {
    if (fuse) DS_DIAD(true, true); else DS_DIAD(true, false);
  } else {
    if (fuse) DS_DIAD(false, true); else DS_DIAD(false, false);
  }
#undef DS_DIAD
  DS_LAUNCH_CHECK("dia_rows_direct");
  return DS_OK;
}

// ===================================================================== COO ==

// First entry index >= k that starts a row (rows sorted); k in [0, nnz].
// Called by one full warp: 32 row ids per step, ballot for the first change,
// so a boundary inside a row costs ceil(row_len / 32) coalesced loads.
__device__ __forceinline__ int64_t coo_row_start_at_or_after_warp(const int* rows, int64_t nnz,
                                                                  int64_t k) {
  if (k <= 0) return 0;
  if (k >= nnz) return nnz;
  const int lane = threadIdx.x & 31;
  const int prev = rows[k - 1];
  for (int64_t b = k; b < nnz; b += 32) {
    const int64_t i = b + lane;
    const bool diff = (i < nnz) && (rows[i] != prev);
    const unsigned m = __ballot_sync(0xffffffffu, diff);
    if (m) return b + (__ffs(m) - 1);
  }
  return nnz;
}

template <bool ACCUM>
__device__ __forceinline__ void coo_fill_gap(double* y, int from, int to) {
  for (int r = from; r < to; ++r) y[r] = ACCUM ? add(y[r], 0.0) : 0.0;  // +0.0 either way
}

// ---------------------------------------------------------------------------
// COO v2: warp-centric segments.  Each warp owns row-aligned chunks of
// kCooWarpChunk entries (chunk c = global warp + k * warps, bounds moved
// forward to the next row start with a ballot scan) and walks them in tiles
// of 256 entries: coalesced strided loads (lane + 32 i) of rows / cols /
// vals, the x gathers, products to warp-private shared memory; the NEXT
// tile's loads are issued before the current tile's segments are summed.
// Row segments come from a warp scan of head flags; one lane per segment
// sums sequentially from +0.0 in stored order (np.bincount), a row that
// continues into the next tile is carried.  No block-wide barriers.
constexpr int kCooWarps = 8;
constexpr int kCooWTile = 256;
constexpr int kCooWarpChunk = 4096;

struct CooTileRegs {
  int r[8], c[8];
  double v[8];
};

__device__ __forceinline__ void coo_tile_load(const int* __restrict__ rows,
                                              const int* __restrict__ cols,
                                              const double* __restrict__ vals, int64_t t0,
                                              int cnt, int lane, CooTileRegs& T) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = min(lane + 32 * i, cnt - 1);
    T.r[i] = ld_stream(rows + t0 + k);
    T.c[i] = ld_stream(cols + t0 + k);
    T.v[i] = ld_stream(vals + t0 + k);
  }
}

template <bool ACCUM>
__global__ void __launch_bounds__(32 * kCooWarps)
    coo_warp_segments(int nrows, int64_t nnz, const int* __restrict__ rows,
                      const int* __restrict__ cols, const double* __restrict__ vals,
                      const double* __restrict__ x, double* y, const int* guard, int plus_zero,
                      const int* __restrict__ long_runs, int n_long) {
  if (guard && *guard) return;
  __shared__ double s_p[kCooWarps][kCooWTile];
  __shared__ int s_r[kCooWarps][kCooWTile];
  __shared__ int s_seg[kCooWarps][kCooWTile + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sp = s_p[w];
  int* sr = s_r[w];
  int* sg = s_seg[w];
  const int64_t nchunks = (nnz + kCooWarpChunk - 1) / kCooWarpChunk;
  const int64_t nw = (int64_t)gridDim.x * kCooWarps;
  const int64_t gw = (int64_t)blockIdx.x * kCooWarps + w;
  // empty matrix: warp 0 of block 0 zero-fills (the loop below has no chunks)
  if (nnz == 0) {
    if (gw == 0)
      for (int r = lane; r < nrows; r += 32) {
        double o = ACCUM ? add(y[r], 0.0) : 0.0;
        y[r] = o;
      }
    return;
  }
  for (int64_t c = gw; c < nchunks; c += nw) {
    const int64_t cstart = coo_row_start_at_or_after_warp(rows, nnz, c * kCooWarpChunk);
    const int64_t cend = coo_row_start_at_or_after_warp(rows, nnz, (c + 1) * kCooWarpChunk);
    const int R0 = (cstart == 0) ? 0 : (cstart < nnz ? rows[cstart] : nrows);
    const int R1 = (cend < nnz) ? rows[cend] : nrows;
    int prev_row = R0 - 1, carry_row = -1;
    double carry = 0.0;
    // long runs (whole rows, sorted by start; coo_long_runs_kernel sums them
    // concurrently) are cut out of the chunk: it is processed as the
    // sub-ranges between them
    int lr = 0;
    if (n_long > 0) {
      int lo = 0, hi = n_long;   // first run with start >= cstart
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (long_runs[2 * mid] < cstart) lo = mid + 1; else hi = mid;
      }
      lr = lo;
    }
    int64_t start = cstart;
    for (;;) {
    const int64_t end = (lr < n_long && long_runs[2 * lr] < cend) ? long_runs[2 * lr] : cend;
    CooTileRegs T;
    if (start < end) coo_tile_load(rows, cols, vals, start, (int)min64(kCooWTile, end - start), lane, T);
    for (int64_t t0 = start; t0 < end; t0 += kCooWTile) {
      const int cnt = (int)min64(kCooWTile, end - t0);
      // products of this tile -> warp-private shared memory
#pragma unroll
      for (int i = 0; i < 8; ++i) T.v[i] = mul(T.v[i], ld_gather(x + T.c[i]));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = lane + 32 * i;
        if (k < cnt) sp[k] = T.v[i];
      }
      // segment heads from registers: position k = lane + 32 i, its
      // predecessor is lane-1 of round i (lane 31 of round i-1 for lane 0);
      // one ballot per round gives every head its segment index in order
      int nseg = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int prev_r = __shfl_up_sync(0xffffffffu, T.r[i], 1);
        const int wrap = __shfl_sync(0xffffffffu, T.r[i > 0 ? i - 1 : 0], 31);
        if (lane == 0) prev_r = wrap;
        const int k = lane + 32 * i;
        const bool head = (k < cnt) && (k == 0 || T.r[i] != prev_r);
        const unsigned m = __ballot_sync(0xffffffffu, head);
        if (head) {   // segment start and its row (rows only at heads: 1/8 the stores)
          const int si = nseg + __popc(m & ((1u << lane) - 1u));
          sg[si] = k;
          sr[si] = T.r[i];
        }
        nseg += __popc(m);
      }
      if (lane == 0) sg[nseg] = cnt;
      __syncwarp();
      // prefetch the next tile while this one is reduced
      const int64_t tn = t0 + kCooWTile;
      if (tn < end) coo_tile_load(rows, cols, vals, tn, (int)min64(kCooWTile, end - tn), lane, T);
      const bool more = tn < end;
      const int next_row = more ? rows[tn] : -1;
      int last_row = 0;
      double last_acc = 0.0;
      for (int sgi = lane; sgi < nseg; sgi += 32) {
        const int hs = sg[sgi], he = sg[sgi + 1];
        const int row = sr[sgi];
        const bool cont = (sgi == 0 && row == carry_row);
        double acc = cont ? carry : 0.0;
        int k = hs;
        for (; k + 4 <= he; k += 4) {
          const double p0 = sp[k], p1 = sp[k + 1], p2 = sp[k + 2], p3 = sp[k + 3];
          acc = add(add(add(add(acc, p0), p1), p2), p3);
        }
        for (; k < he; ++k) acc = add(acc, sp[k]);
        const int prev = (sgi == 0) ? prev_row : sr[sgi - 1];
        if (!cont) coo_fill_gap<ACCUM>(y, prev + 1, row);
        if (sgi == nseg - 1) {
          last_row = row;
          last_acc = acc;
        }
        if (!(sgi == nseg - 1 && more && next_row == row)) {
          double out = ACCUM ? add(y[row], acc) : acc;
          if (plus_zero) out = add(out, 0.0);
          y[row] = out;
        }
      }
      const int owner = (nseg - 1) & 31;
      last_row = __shfl_sync(0xffffffffu, last_row, owner);
      last_acc = __shfl_sync(0xffffffffu, last_acc, owner);
      prev_row = last_row;
      if (more && next_row == last_row) {
        carry_row = last_row;
        carry = last_acc;
      } else {
        carry_row = -1;
      }
      __syncwarp();
    }
    if (end == cend) break;
    // skip long run lr: zero the absent rows before it; its own row is
    // written by the long-run kernel
    {
      const int lrow = rows[long_runs[2 * lr]];
      for (int r = prev_row + 1 + lane; r < lrow; r += 32) y[r] = ACCUM ? add(y[r], 0.0) : 0.0;
      prev_row = lrow;
      carry_row = -1;
      start = long_runs[2 * lr + 1];
      ++lr;
      __syncwarp();
    }
    }
    // rows after the chunk's last entry up to the next chunk's first row
    for (int r = prev_row + 1 + lane; r < R1; r += 32) y[r] = ACCUM ? add(y[r], 0.0) : 0.0;
    __syncwarp();
  }
}

// Long runs of a row-sorted COO (rows longer than kCooLongRun entries, e.g.
// the power-law matrix's 14687-entry row): one CTA per run.  All threads form
// the products of a piece of the run into shared memory (coalesced loads,
// every gather in flight), then thread 0 adds them in stored order -- the
// np.bincount chain, carried from piece to piece -- with the next shared
// loads issued ahead of the adds.  Runs on a side stream concurrently with
// coo_warp_segments, which skips these rows.
constexpr int kCooLongRun = 2048;
constexpr int kCooLongPiece = 8192;   // products per shared-memory piece (64 KB)

template <bool ACCUM>
__global__ void __launch_bounds__(512)
    coo_long_runs_kernel(const int* __restrict__ long_runs, int n_long,
                         const int* __restrict__ rows, const int* __restrict__ cols,
                         const double* __restrict__ vals, const double* __restrict__ x,
                         double* y, const int* guard, int plus_zero) {
  if (guard && *guard) return;
  extern __shared__ __align__(16) double s_p[];
  for (int li = blockIdx.x; li < n_long; li += gridDim.x) {
    const int64_t b = long_runs[2 * li], e = long_runs[2 * li + 1];
    double acc = 0.0;
    for (int64_t p0 = b; p0 < e; p0 += kCooLongPiece) {
      const int cnt = (int)min64(kCooLongPiece, e - p0);
      for (int k = threadIdx.x; k < cnt; k += blockDim.x)
        s_p[k] = mul(vals[p0 + k], ld_gather(x + cols[p0 + k]));
      __syncthreads();
      if (threadIdx.x == 0) {
        int k = 0;
        for (; k + 8 <= cnt; k += 8) {
          double q[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) q[j] = s_p[k + j];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc = add(acc, q[j]);
        }
        for (; k < cnt; ++k) acc = add(acc, s_p[k]);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const int row = rows[b];
      double o = ACCUM ? add(y[row], acc) : acc;
      if (plus_zero) o = add(o, 0.0);
      y[row] = o;
    }
  }
}

// ---------------------------------------------------------------------------
// COO v3: persistent TMA pipeline (row-sorted COO).
//
// CTA c owns the row-aligned entry range [s_c, s_{c+1}), s_c = first row
// start at or after c*C, and the rows [R_c, R_{c+1}) (R_0 = 0, R_G = nrows:
// absent rows are written as +0.0 by their owner).  It walks its range in
// tiles of E entries; thread 0 streams each tile's row indices, column
// indices and values into a ring of S stages with three 1-D TMA bulk copies.
//   phase A: thread t takes entries t, t+T, ... (coalesced shared-memory
//            reads, all gathers in flight), writes the products and row ids
//            to a private work buffer -- then the stage is released and
//            refilled while
//   phase B: thread per row (binary search for the row's segment in the
//            tile) sums sequentially in stored order from +0.0, exactly
//            np.bincount (kernels.py:149); the tile's last row is carried
//            into the next tile unless the CTA's range ends there.
struct CooPipeCfg {
  int E;            // entries per tile (multiple of T)
  int S;            // stages (<= 8)
  int stage_bytes;  // 16 * (E + 8), 128-B multiple
};

__device__ __forceinline__ void coo_pipe_issue(const int* __restrict__ rows,
                                               const int* __restrict__ cols,
                                               const double* __restrict__ vals, int64_t nnz,
                                               int64_t a, int64_t b, int E, unsigned char* st,
                                               uint64_t* bar, uint64_t pol) {
  const int64_t ws = a & ~3ll;
  int* s_r = reinterpret_cast<int*>(st);
  int* s_c = s_r + (E + 8);
  double* s_v = reinterpret_cast<double*>(st + 8 * (size_t)(E + 8));
  int64_t ib, vb;  // bulk ends (ints, doubles)
  if (((b + 3) & ~3ll) <= nnz) {
    ib = (b + 3) & ~3ll;
    vb = (b + 1) & ~1ll;
  } else {  // the matrix's last tile: sub-16-byte tails by hand
    ib = b & ~3ll;
    vb = b & ~1ll;
    for (int64_t e = ib; e < b; ++e) {
      s_r[e - ws] = rows[e];
      s_c[e - ws] = cols[e];
    }
    if (vb < b) s_v[vb - ws] = vals[vb];
  }
  const uint32_t ibytes = 4u * (uint32_t)(ib - ws), vbytes = 8u * (uint32_t)(vb - ws);
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, 2 * ibytes + vbytes);
  if (ibytes) {
    bulk_g2s(s_r, rows + ws, ibytes, bar, pol);
    bulk_g2s(s_c, cols + ws, ibytes, bar, pol);
  }
  if (vbytes) bulk_g2s(s_v, vals + ws, vbytes, bar, pol);
}

// first index in w[0, n) with w[i] >= r (w nondecreasing)
__device__ __forceinline__ int lower_bound_smem(const int* w, int n, int r) {
  int lo = 0, len = n;
  while (len > 0) {
    const int h = len >> 1;
    if (w[lo + h] < r) {
      lo += h + 1;
      len -= h + 1;
    } else {
      len = h;
    }
  }
  return lo;
}

// Thread per row (the CSR pipeline's structure: instruction-light, all
// LMAX gathers of a row in flight).  The rows of a tile are [pend, rlast]
// (rlast = the tile's last row, carried into the next tile unless the CTA's
// range ends with this tile, then the range extends to R_{c+1}); thread t
// takes rows pend + t + T*i.  A row's segment is found by binary search in
// the staged row indices; its columns and values are copied to registers and
// its gathers issued before the stage is released (last round only: the
// round count is uniform across the CTA), the sequential sum follows.
template <int LMAX>
struct CooRowRegs {
  int len;
  double v[LMAX];
  double g[LMAX];
};

template <bool ACCUM, int T, int LMAX, int MINB>
__global__ void __launch_bounds__(T, MINB)
    coo_pipe(int nrows, int64_t nnz, const int* __restrict__ rows, const int* __restrict__ cols,
             const double* __restrict__ vals, const double* __restrict__ x, double* y,
             CooPipeCfg cfg, const int* guard, int plus_zero) {
  if (guard && *guard) return;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);          // <= 8 barriers
  int64_t* s_bounds = reinterpret_cast<int64_t*>(smem + 64);   // s_c, s_{c+1}
  int* s_R = reinterpret_cast<int*>(smem + 80);                // R_c, R_{c+1}
  double* s_carry = reinterpret_cast<double*>(smem + 88);
  const int E = cfg.E, S = cfg.S;
  unsigned char* stage0 = smem + 128;
  const int tid = threadIdx.x;
  const int64_t G = gridDim.x;
  const int64_t C = (nnz + G - 1) / G;
  if (tid < 32) {
    const int64_t s0 = coo_row_start_at_or_after_warp(rows, nnz, blockIdx.x * C);
    const int64_t s1 = coo_row_start_at_or_after_warp(rows, nnz, (blockIdx.x + 1) * C);
    if (tid == 0) {
      s_bounds[0] = s0;
      s_bounds[1] = s1;
      s_R[0] = (s0 == 0) ? 0 : (s0 < nnz ? rows[s0] : nrows);
      s_R[1] = (s1 < nnz) ? rows[s1] : nrows;
      for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
      fence_barrier_init();
    }
  }
  __syncthreads();
  const int64_t s0 = s_bounds[0], s1 = s_bounds[1];
  const int Rend = s_R[1];
  const int64_t ntiles = (s1 - s0 + E - 1) / E;
  uint64_t pol = 0;
  if (tid == 0) {
    pol = policy_evict_first();
    for (int s = 0; s < S && s < ntiles; ++s)
      coo_pipe_issue(rows, cols, vals, nnz, s0 + (int64_t)s * E,
                     min64(s0 + (int64_t)(s + 1) * E, s1), E, stage0 + (size_t)s * cfg.stage_bytes,
                     &full[s], pol);
  }
  int pend = s_R[0];    // rows < pend are written
  int carry_row = -1;   // == pend when a partial sum continues
  double carry = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t k = 0; k < ntiles; ++k) {
    const int64_t a = s0 + k * E;
    const int cnt = (int)(min64(a + E, s1) - a);
    const int off = (int)(a - (a & ~3ll));
    unsigned char* st = stage0 + (size_t)s * cfg.stage_bytes;
    const int* s_r = reinterpret_cast<const int*>(st) + off;
    const int* s_c = reinterpret_cast<const int*>(st) + (E + 8) + off;
    const double* s_v = reinterpret_cast<const double*>(st + 8 * (size_t)(E + 8)) + off;
    mbar_wait(&full[s], ph);
    const bool last = (k == ntiles - 1);
    const int rlast = s_r[cnt - 1];
    const int hi = last ? Rend : rlast + 1;
    const int rounds = (hi - pend + T - 1) / T;   // uniform across the CTA
    for (int it = 0; it < rounds; ++it) {
      const int r = pend + tid + T * it;
      CooRowRegs<LMAX> R;
      R.len = 0;
      double acc = (r == carry_row) ? carry : 0.0;
      bool fast = false;
      if (r < hi) {
        int q0, q1;
        if (r > rlast) {   // absent rows after the CTA's last entry
          q0 = q1 = cnt;
        } else {
          q0 = lower_bound_smem(s_r, cnt, r);
          // end: bounded search over the next LMAX+1 entries, else the rest
          const int lim = min(q0 + LMAX + 1, cnt);
          q1 = q0 + lower_bound_smem(s_r + q0, lim - q0, r + 1);
          if (q1 == lim && lim < cnt && s_r[lim] <= r)
            q1 = lim + lower_bound_smem(s_r + lim, cnt - lim, r + 1);
        }
        const int len = q1 - q0;
        if (len == 0) {
          // absent row (or the carried row ending at the tile boundary): acc as is
        } else if (len <= LMAX) {
          fast = true;
          R.len = len;
          const int lst = max(len - 1, 0);
          int c[LMAX];
#pragma unroll
          for (int j = 0; j < LMAX; ++j) c[j] = s_c[q0 + min(j, lst)];
#pragma unroll
          for (int j = 0; j < LMAX; ++j) R.g[j] = ld_gather(x + c[j]);
#pragma unroll
          for (int j = 0; j < LMAX; ++j) R.v[j] = s_v[q0 + min(j, lst)];
        } else {   // long row: sequential from the stage now, 8 gathers in flight
          for (int qb = q0; qb < q1; qb += 8) {
            double gg[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) gg[j] = ld_gather(x + s_c[min(qb + j, q1 - 1)]);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (qb + j < q1) acc = add(acc, mul(s_v[qb + j], gg[j]));
          }
        }
      }
      if (it == rounds - 1) {
        __syncthreads();  // stage consumed: refill it while the gathers land
        if (tid == 0 && k + S < ntiles)
          coo_pipe_issue(rows, cols, vals, nnz, s0 + (k + S) * E,
                         min64(s0 + (k + S + 1) * E, s1), E, st, &full[s], pol);
      }
      if (r < hi) {
        if (fast) {
#pragma unroll
          for (int j = 0; j < LMAX; ++j)
            if (j < R.len) acc = add(acc, mul(R.v[j], R.g[j]));
        }
        if (!last && r == rlast) {
          *s_carry = acc;
        } else {
          double o = ACCUM ? add(y[r], acc) : acc;
          if (plus_zero) o = add(o, 0.0);
          y[r] = o;
        }
      }
    }
    if (rounds == 0) {   // cannot happen (rlast >= pend), kept for the barrier count
      __syncthreads();
      if (tid == 0 && k + S < ntiles)
        coo_pipe_issue(rows, cols, vals, nnz, s0 + (k + S) * E, min64(s0 + (k + S + 1) * E, s1),
                       E, st, &full[s], pol);
    }
    __syncthreads();  // carry published
    if (!last) {
      carry_row = rlast;
      carry = *s_carry;
      pend = rlast;
    }
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
  if (ntiles == 0)   // empty range (only when the matrix has no entries)
    for (int r = pend + tid; r < Rend; r += T) y[r] = ACCUM ? add(y[r], 0.0) : 0.0;
}

template <bool A, int T, int MINB>
static int coo_pipe_launch1(int64_t nrows, int64_t nnz, const int* rows, const int* cols,
                            const double* vals, const double* x, double* y, const int* guard,
                            bool plus_zero, int E, int S, int ctas, cudaStream_t st) {
  CooPipeCfg cfg;
  cfg.E = E;
  cfg.S = S;
  cfg.stage_bytes = (int)((16 * (int64_t)(cfg.E + 8) + 127) & ~127ll);
  const size_t smem = 128 + (size_t)cfg.S * cfg.stage_bytes;
  if (smem > (size_t)max_dynamic_smem() - 1024) return DS_ERR_NOT_SUPPORTED;
  int64_t grid = (int64_t)sm_count() * ctas;
  const int64_t want = ceil_div(nnz, cfg.E);
  if (grid > want) grid = want;
  if (grid < 1) grid = 1;
  auto k = coo_pipe<A, T, 27, MINB>;
  int rc = allow_dynamic_smem(reinterpret_cast<const void*>(k), smem);
  if (rc) return rc;
  k<<<(unsigned)grid, T, smem, st>>>((int)nrows, nnz, rows, cols, vals, x, y, cfg, guard,
                                     (int)plus_zero);
  DS_LAUNCH_CHECK("coo_pipe");
  return DS_OK;
}

// tile shapes (threads, entries per tile, stages, CTAs/SM); DS_COO_CFG picks one
static int coo_pipe_launch(int64_t nrows, int64_t nnz, const int* rows, const int* cols,
                           const double* vals, const double* x, double* y, bool accum,
                           const int* guard, bool plus_zero, cudaStream_t st) {
  static int eC = -2, eS = -2, eN = -2, eE = -2;
  if (eC == -2) {
    const char* a = getenv("DS_COO_CFG");
    const char* b = getenv("DS_COO_S");
    const char* c = getenv("DS_COO_CTAS");
    const char* d = getenv("DS_COO_E");
    eC = a ? atoi(a) : -1;
    eS = b ? atoi(b) : -1;
    eN = c ? atoi(c) : -1;
    eE = d ? atoi(d) : -1;
  }
  if (((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(cols) |
        reinterpret_cast<uintptr_t>(vals)) & 15) != 0 || nnz <= 0 || nnz >= (1ll << 31))
    return DS_ERR_NOT_SUPPORTED;
  const int cfgi = eC >= 0 ? eC : 0;
#define DS_COOP(T, E, S, N)                                                                     \
  return accum ? coo_pipe_launch1<true, T, N>(nrows, nnz, rows, cols, vals, x, y, guard, plus_zero, \
                                           eE > 0 ? eE : E, eS > 0 ? eS : S, eN > 0 ? eN : N, st) \
               : coo_pipe_launch1<false, T, N>(nrows, nnz, rows, cols, vals, x, y, guard,          \
                                            plus_zero, eE > 0 ? eE : E, eS > 0 ? eS : S,        \
                                            eN > 0 ? eN : N, st)
  switch (cfgi) {
    // measured at 104^3 (tools/sweep_coo.sh): 64 threads x 1024 entries x 2
    // stages x 6 CTAs/SM 92.6 us; the register budget (~166 / thread at
    // LMAX 27) caps residency, so the variants bound registers via MINB
    case 0: DS_COOP(64, 1024, 2, 6);
    case 1: DS_COOP(128, 2048, 2, 3);
    case 2: DS_COOP(128, 1536, 2, 4);
    case 3: DS_COOP(64, 1024, 2, 8);
    case 4: DS_COOP(64, 768, 2, 8);
    default: DS_COOP(96, 1536, 2, 5);
  }
#undef DS_COOP
}

__global__ void coo_atomic(int64_t nnz, const int* __restrict__ rows, const int* __restrict__ cols,
                           const double* __restrict__ vals, const double* __restrict__ x,
                           double* y, const int* guard) {
  if (guard && *guard) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(y + rows[k], mul(vals[k], __ldg(x + cols[k])));
}

__global__ void fill_f64(int64_t n, double* y, double v, const int* guard) {
  if (guard && *guard) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = v;
}
__global__ void axpy_inplace(int64_t n, double* y, const double* t, const int* guard) {
  if (guard && *guard) return;  // y = y + t
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = add(y[i], t[i]);
}

int launch_coo(int64_t nrows, int64_t nnz, const int* rows, const int* cols, const double* vals,
               bool sorted, int max_len, const double* x, double* y, bool accum, const int* guard,
               cudaStream_t st, bool plus_zero, const int* long_runs, int n_long) {
  if (nrows == 0) return DS_OK;
  if (nnz == 0) return launch_empty_matrix(nrows, y, accum, guard, st);
  static int coo_warp = -1;
  if (coo_warp < 0) coo_warp = getenv("DS_COO_WARP") ? 1 : 0;
  // thread-per-row pipeline for row-sorted COO whose rows fit its 27-wide
  // register path (the stencil); long rows (power-law) keep the warp kernel,
  // whose parallel products leave only the inherent sequential add chain
  if (sorted && !coo_warp && max_len >= 1 && max_len <= 27) {
    const int rc = coo_pipe_launch(nrows, nnz, rows, cols, vals, x, y, accum, guard, plus_zero, st);
    if (rc != DS_ERR_NOT_SUPPORTED) return rc;
  }
  if (sorted) {
    int64_t blocks = ceil_div(ceil_div(nnz, kCooWarpChunk), kCooWarps);
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const bool split = long_runs != nullptr && n_long > 0;
    cudaEvent_t joined = nullptr;
    if (split) {   // the long runs on a side stream, launched first (fork / join)
      cudaStream_t side;
      cudaEvent_t fork;
      int rc = aux_stream(&side, &fork, &joined);
      if (rc) return rc;
      DS_CUDA(cudaEventRecord(fork, st));
      DS_CUDA(cudaStreamWaitEvent(side, fork, 0));
      const size_t smem = (size_t)kCooLongPiece * 8;
      const void* lk = accum ? (const void*)coo_long_runs_kernel<true>
                             : (const void*)coo_long_runs_kernel<false>;
      rc = allow_dynamic_smem(lk, smem);
      if (rc) return rc;
      const unsigned lg = (unsigned)min64(n_long, (int64_t)sm_count());
      if (accum)
        coo_long_runs_kernel<true><<<lg, 512, smem, side>>>(long_runs, n_long, rows, cols, vals,
                                                            x, y, guard, (int)plus_zero);
      else
        coo_long_runs_kernel<false><<<lg, 512, smem, side>>>(long_runs, n_long, rows, cols, vals,
                                                             x, y, guard, (int)plus_zero);
      DS_LAUNCH_CHECK("coo_long_runs_kernel");
      DS_CUDA(cudaEventRecord(joined, side));
    }
    if (accum)
      coo_warp_segments<true><<<(unsigned)blocks, 32 * kCooWarps, 0, st>>>(
          (int)nrows, nnz, rows, cols, vals, x, y, guard, (int)plus_zero,
          split ? long_runs : nullptr, split ? n_long : 0);
    else
      coo_warp_segments<false><<<(unsigned)blocks, 32 * kCooWarps, 0, st>>>(
          (int)nrows, nnz, rows, cols, vals, x, y, guard, (int)plus_zero,
          split ? long_runs : nullptr, split ? n_long : 0);
    DS_LAUNCH_CHECK("coo_warp_segments");
    if (split) DS_CUDA(cudaStreamWaitEvent(st, joined, 0));
    return DS_OK;
  }
  const unsigned g = (unsigned)min64(ceil_div(nrows, 256), (int64_t)sm_count() * 8);
  double* target = y;
  if (accum) {  // tmp = A x; y += tmp  (kernels.py:196-198)
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&target), nrows * sizeof(double), st));
  }
  fill_f64<<<g, 256, 0, st>>>(nrows, target, 0.0, guard);
  if (nnz > 0) {
    const unsigned ga = (unsigned)min64(ceil_div(nnz, 256), (int64_t)sm_count() * 16);
    coo_atomic<<<ga, 256, 0, st>>>(nnz, rows, cols, vals, x, target, guard);
  }
  if (accum) {
    axpy_inplace<<<g, 256, 0, st>>>(nrows, y, target, guard);
    DS_CUDA(cudaFreeAsync(target, st));
  }
  // atomics start from +0.0, so y + 0.0 is already the identity: plus_zero is free here
  (void)plus_zero;
  DS_LAUNCH_CHECK("coo_atomic");
  return DS_OK;
}

__global__ void coo_flags_kernel(int64_t nnz, const int* __restrict__ rows,
                                 const int* __restrict__ cols, int* bad) {
  // bad[0]: some row decreases; bad[1]: (row, col) not strictly increasing
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = rows[k - 1], r1 = rows[k];
    if (r1 < r0) {
      bad[0] = 1;
      bad[1] = 1;
    } else if (r1 == r0 && cols[k] <= cols[k - 1]) {
      bad[1] = 1;
    }
  }
}

}  // namespace ds

// ============================================================== C ABI ======
using namespace ds;

extern "C" int ds_csr_analyze(int64_t nrows, const int32_t* row_offsets, int32_t* long_rows,
                              int64_t* n_long, int32_t* max_row_len, void* stream) {
  cudaStream_t st = as_stream(stream);
  *n_long = 0;
  if (max_row_len) *max_row_len = 0;
  if (nrows <= 0) return DS_OK;
  int* d = nullptr;  // [count, maxlen]
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 2 * sizeof(int), st));
  DS_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(int), st));
  const unsigned g = (unsigned)min64(ceil_div(nrows, 256), (int64_t)sm_count() * 8);
  csr_find_long<<<g, 256, 0, st>>>((int)nrows, row_offsets, long_rows,
                                   reinterpret_cast<unsigned*>(d), d + 1);
  DS_LAUNCH_CHECK("csr_find_long");
  int h[2];
  DS_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(d, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *n_long = h[0];
  if (max_row_len) *max_row_len = h[1];
  return DS_OK;
}

extern "C" int ds_spmv_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_offsets,
                           const int32_t* col_indices, const double* values,
                           const int32_t* long_rows, int64_t n_long, const double* x, double* y,
                           int accumulate, void* stream) {
  (void)ncols;
  (void)nnz;
  if (nrows < 0 || nrows >= (1ll << 31)) {
    set_error("nrows out of range");
    return DS_ERR_NOT_SUPPORTED;
  }
  return launch_csr(nrows, nnz, row_offsets, col_indices, values, long_rows, n_long, 0, x, y,
                    accumulate != 0, nullptr, as_stream(stream));
}

extern "C" int ds_spmv_dia(int64_t nrows, int64_t ncols, int32_t ndiags, const int32_t* offsets,
                           const double* values, const double* x, double* y, int accumulate,
                           void* stream) {
  if (nrows < 0 || nrows >= (1ll << 31) || ncols >= (1ll << 31)) {
    set_error("dims out of range");
    return DS_ERR_NOT_SUPPORTED;
  }
  return launch_dia(nrows, ncols, ndiags, offsets, values, x, y, accumulate != 0, nullptr,
                    as_stream(stream));
}

extern "C" int ds_spmv_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_indices,
                           const int32_t* col_indices, const double* values, int rows_sorted,
                           const double* x, double* y, int accumulate, void* stream) {
  (void)ncols;
  if (nrows < 0 || nrows >= (1ll << 31)) {
    set_error("nrows out of range");
    return DS_ERR_NOT_SUPPORTED;
  }
  return launch_coo(nrows, nnz, row_indices, col_indices, values, rows_sorted != 0, 0, x, y,
                    accumulate == 1, nullptr, as_stream(stream), accumulate == 2);
}

// Longest run of equal row indices (rows nondecreasing): each run head
// gallops to the end of its run (O(log run) loads), atomicMax of the lengths.
__global__ void coo_max_run_kernel(int64_t nnz, const int* __restrict__ rows, int* out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = rows[k];
    if (k > 0 && rows[k - 1] == r) continue;
    int64_t lo = k, step = 1;   // rows[lo] == r
    while (lo + step < nnz && rows[lo + step] == r) {
      lo += step;
      step <<= 1;
    }
    int64_t hi = min64(lo + step, nnz);   // rows[hi] != r or hi == nnz
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (rows[mid] == r) lo = mid; else hi = mid;
    }
    const int64_t len = lo - k + 1;
    atomicMax(out, (int)min64(len, (int64_t)INT_MAX));
  }
}

extern "C" int ds_coo_max_run(int64_t nnz, const int32_t* row_indices, int32_t* max_run,
                              void* stream) {
  cudaStream_t st = as_stream(stream);
  *max_run = 0;
  if (nnz <= 0) return DS_OK;
  int* d = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(int), st));
  DS_CUDA(cudaMemsetAsync(d, 0, sizeof(int), st));
  const unsigned g = (unsigned)min64(ceil_div(nnz, 256), (int64_t)sm_count() * 8);
  coo_max_run_kernel<<<g, 256, 0, st>>>(nnz, row_indices, d);
  DS_LAUNCH_CHECK("coo_max_run_kernel");
  int h = 0;
  DS_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(d, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *max_run = h;
  return DS_OK;
}

// Runs of equal row index longer than `threshold` (whole rows) as (start,
// end) int32 pairs sorted by start -- the long-run plan of a row-sorted COO.
__global__ void coo_long_runs_find(int64_t nnz, const int* __restrict__ rows, int threshold,
                                   int* out, int64_t capacity, unsigned long long* count) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int r = rows[k];
    if (k > 0 && rows[k - 1] == r) continue;
    if (k + threshold >= nnz || rows[k + threshold] != r) continue;   // run <= threshold
    int64_t lo = k + threshold, step = 1;   // rows[lo] == r: gallop to the run's end
    while (lo + step < nnz && rows[lo + step] == r) {
      lo += step;
      step <<= 1;
    }
    int64_t hi = min64(lo + step, nnz);
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (rows[mid] == r) lo = mid; else hi = mid;
    }
    const unsigned long long slot = atomicAdd(count, 1ull);
    if ((int64_t)slot < capacity) {
      out[2 * slot] = (int)k;
      out[2 * slot + 1] = (int)(lo + 1);
    }
  }
}

extern "C" int ds_coo_long_runs(int64_t nnz, const int32_t* row_indices, int32_t threshold,
                                int32_t* runs, int64_t capacity, int64_t* n_runs, void* stream) {
  cudaStream_t st = as_stream(stream);
  *n_runs = 0;
  if (nnz <= 0 || threshold < 1) return DS_OK;
  unsigned long long* d = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(*d), st));
  DS_CUDA(cudaMemsetAsync(d, 0, sizeof(*d), st));
  const unsigned g = (unsigned)min64(ceil_div(nnz, 256), (int64_t)sm_count() * 8);
  coo_long_runs_find<<<g, 256, 0, st>>>(nnz, row_indices, threshold, runs, capacity, d);
  DS_LAUNCH_CHECK("coo_long_runs_find");
  unsigned long long h = 0;
  DS_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(d, st));
  DS_CUDA(cudaStreamSynchronize(st));
  if ((int64_t)h > capacity) {
    set_error("ds_coo_long_runs: %llu runs exceed the capacity %lld", h, (long long)capacity);
    return DS_ERR_NOT_SUPPORTED;
  }
  if (h > 1) {   // sort the (few) pairs by start on the host
    std::vector<std::pair<int, int>> v(h);
    DS_CUDA(cudaMemcpy(v.data(), runs, h * 2 * sizeof(int), cudaMemcpyDeviceToHost));
    std::sort(v.begin(), v.end());
    DS_CUDA(cudaMemcpy(runs, v.data(), h * 2 * sizeof(int), cudaMemcpyHostToDevice));
  }
  *n_runs = (int64_t)h;
  return DS_OK;
}

extern "C" int ds_coo_long_run_threshold(void) {
  static int e = -2;
  if (e == -2) {
    const char* v = getenv("DS_COO_LONG_RUN");
    e = v ? atoi(v) : -1;
  }
  return e > 0 ? e : kCooLongRun;
}

extern "C" int ds_spmv_coo_sorted(int64_t nrows, int64_t ncols, int64_t nnz,
                                  const int32_t* row_indices, const int32_t* col_indices,
                                  const double* values, int32_t max_row_len, const double* x,
                                  double* y, int accumulate, void* stream) {
  (void)ncols;
  if (nrows < 0 || nrows >= (1ll << 31)) {
    set_error("nrows out of range");
    return DS_ERR_NOT_SUPPORTED;
  }
  return launch_coo(nrows, nnz, row_indices, col_indices, values, true, max_row_len, x, y,
                    accumulate != 0, nullptr, as_stream(stream), false, nullptr, 0);
}

extern "C" int ds_coo_order_flags(int64_t nnz, const int32_t* row_indices,
                                  const int32_t* col_indices, int32_t* flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  *flags = 3;
  if (nnz <= 1) return DS_OK;
  int* d = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 2 * sizeof(int), st));
  DS_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(int), st));
  const unsigned g = (unsigned)min64(ceil_div(nnz, 256), (int64_t)sm_count() * 8);
  coo_flags_kernel<<<g, 256, 0, st>>>(nnz, row_indices, col_indices, d);
  DS_LAUNCH_CHECK("coo_flags_kernel");
  int h[2];
  DS_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(d, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *flags = (h[0] ? 0 : 1) | (h[1] ? 0 : 2);
  return DS_OK;
}
