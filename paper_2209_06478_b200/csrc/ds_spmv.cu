// ds_spmv.cu -- SpMV over CSR / DIA / COO for sm_100a.
//
// Replaces the reference's format-dispatched kernels (kernels.py:102-198):
//   _csr_spmv  kernels.py:102-119   -> csr_rows_g8 (+ csr_long_rows)
//   _dia_spmv  kernels.py:122-140   -> dia_pipe (+ dia_rows_direct)
//   _coo_spmv  kernels.py:143-163   -> coo_sorted_segments / coo_atomic
// Results are bitwise equal to the reference (see include/dynsparse_b200.h)
// except for unsorted COO (atomics; within 1e-13 like the reference's
// threaded COO, kernels.py:13-15).
//
// HBM is the roofline for every kernel here (no tensor cores: SpMV is not a
// dense contraction).  The design goals per format:
//   CSR: 8 lanes per row (the exact numpy pairwise structure), all loads of a
//        row issued before the dependent add chain; matrix arrays streamed
//        with L1::no_allocate, x gathered through L1/L2 (x stays L2-resident).
//   DIA: persistent CTAs stream (T rows x ndiags) value slabs into a ring of
//        shared-memory stages with 1-D TMA bulk copies (cp.async.bulk +
//        mbarrier, L2 evict_first); each thread walks its row from shared
//        memory (odd row stride in 8-B words -> conflict-free) and gathers x.
//   COO: blocks own row-aligned entry ranges; entries are staged to shared
//        memory with their products, then one thread per row segment sums
//        sequentially (np.bincount order), carrying across tiles.
#include <stdlib.h>

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

// One 8-lane group per row; grid-stride over row groups.
template <bool ACCUM, bool SKIP_LONG, bool FUSE_DOT>
__global__ void __launch_bounds__(kCsrBlock)
    csr_rows_g8(int nrows, const int* __restrict__ off, const int* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ x, double* y,
                DotOut dot) {
  if (dot.skip()) return;
  const int lane8 = threadIdx.x & 7;
  const unsigned mask = 0xffu << (threadIdx.x & 24);
  const int groups_per_grid = (gridDim.x * kCsrBlock) >> 3;
  double dsum = 0.0;
  for (int row = (blockIdx.x * kCsrBlock + threadIdx.x) >> 3; row < nrows;
       row += groups_per_grid) {
    const int start = __ldg(off + row);
    const int end = __ldg(off + row + 1);
    const int len = end - start;
    if (SKIP_LONG && len > kLongRow) continue;  // the long-row kernel owns it
    double res = 0.0, p0 = 0.0;
    if (len > 0) {
      if (lane8 == 0) p0 = mul(ld_stream(val + start), ld_gather(x + ld_stream(col + start)));
      if (len <= kLongRow)
        res = csr_leaf_g8(col, val, x, (int64_t)start + 1, len - 1, lane8, mask);
      else
        res = csr_group_pairwise(col, val, x, (int64_t)start + 1, len - 1, lane8, mask);
    }
    if (lane8 == 0) {
      const double s = (len > 0) ? add(p0, res) : 0.0;
      double out = ACCUM ? add(y[row], s) : s;
      if (dot.plus_zero) out = add(out, 0.0);
      y[row] = out;
      if (FUSE_DOT) dsum = add(dsum, mul(dot.other[row], out));
    }
  }
  if (FUSE_DOT) dot.finish_block<kCsrBlock>(dsum);
}

// One CTA per long row: the pairwise recursion tree is cut into subtrees of
// at most kSub addends; each subtree's leaves (64..128 addends each) are
// summed by the CTA's 32 lane-groups in parallel, then thread 0 replays the
// recursion to combine them in numpy's order.
constexpr int kSub = 8192;           // <= 128 leaves per subtree
constexpr int kMaxLeaves = 160;

template <bool ACCUM>
__global__ void __launch_bounds__(kCsrBlock)
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
        double v = csr_leaf_g8(col, val, x, base + s_leaf_lo[l], s_leaf_n[l], lane8, mask);
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

int launch_csr(int64_t nrows, const int* off, const int* col, const double* val,
               const int* long_rows, int64_t n_long, const double* x, double* y, bool accum,
               const DotOut* dot, cudaStream_t st) {
  if (nrows == 0) return DS_OK;
  const int64_t groups = nrows;
  int64_t blocks = ceil_div(groups * 8, kCsrBlock);
  const int64_t cap = (int64_t)sm_count() * 8 * 16;  // grid-stride beyond 16 waves
  if (blocks > cap) blocks = cap;
  const bool skip = (long_rows != nullptr);
  DotOut d = dot ? *dot : DotOut{};
  const bool fuse = d.fused();
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
  if (skip && n_long > 0) {
    int64_t lb = n_long < (int64_t)sm_count() * 8 ? n_long : (int64_t)sm_count() * 8;
    if (accum)
      csr_long_rows<true><<<(unsigned)lb, kCsrBlock, 0, st>>>(long_rows, (int)n_long, off, col,
                                                             val, x, y, d.guard);
    else
      csr_long_rows<false><<<(unsigned)lb, kCsrBlock, 0, st>>>(long_rows, (int)n_long, off, col,
                                                              val, x, y, d.guard);
    DS_LAUNCH_CHECK("csr_long_rows");
  }
  return DS_OK;
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
};

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
  if (dot.skip()) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int nd = ND > 0 ? ND : ndiags_rt;
  const int T = cfg.T, S = cfg.S;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);               // <= 8 barriers
  int* s_off = reinterpret_cast<int*>(smem + 64);
  unsigned char* stage0 = smem + 64 + ((nd * 4 + 127) & ~127);
  const int tid = threadIdx.x;
  const int64_t ntiles = (nrows + T - 1) / T;
  const int64_t G = gridDim.x;
  uint64_t pol = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    pol = policy_evict_first();
  }
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
  double dsum = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += G) {
    const double* v_stage = reinterpret_cast<const double*>(stage0 + (size_t)s * cfg.stage_bytes);
    mbar_wait(&full[s], ph);
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
#pragma unroll
        for (int j = 0; j < ND; ++j) {
          const int c = i + s_off[j];
          xv[j] = ld_gather(x + min(max(c, 0), ncols - 1));
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
      if (FUSE_DOT) dsum = add(dsum, mul(dot.other[i], out));
    }
    __syncthreads();  // stage s fully consumed
    if (tid == 0) {
      const int64_t tn = t + (int64_t)S * G;
      if (tn < ntiles)
        dia_issue_tile(vals, nrows, nd, T, tn,
                       reinterpret_cast<double*>(stage0 + (size_t)s * cfg.stage_bytes), &full[s],
                       pol);
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
  const int stage_bytes = (int)((((int64_t)T * ndiags * 8) + 127) & ~127ll);
  const size_t smem = 64 + ((ndiags * 4 + 127) & ~127) + (size_t)S * stage_bytes;
  if (aligned && ndiags > 0 && S <= 8 && T >= 32 && smem <= (size_t)max_dynamic_smem() - 1024) {
    const int64_t ntiles = ceil_div(nrows, T);
    int64_t grid = (int64_t)sm_count() * ctas;
    if (grid > ntiles) grid = ntiles;
    if (fuse) grid = d.clamp_grid(grid);
    DiaPipeCfg cfg{T, S, stage_bytes};
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

constexpr int kCooBlock = 256;
constexpr int kCooTile = 2048;            // entries staged per tile
constexpr int kCooPerBlock = 4 * kCooTile; // nominal entries per block

// First entry index >= k that starts a row (rows sorted); k in [0, nnz].
__device__ __forceinline__ int64_t coo_row_start_at_or_after(const int* rows, int64_t nnz,
                                                             int64_t k) {
  if (k <= 0) return 0;
  if (k >= nnz) return nnz;
  const int prev = rows[k - 1];
  if (rows[k] != prev) return k;
  // upper_bound of prev in [k, nnz)
  int64_t lo = k, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rows[mid] <= prev) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <bool ACCUM>
__device__ __forceinline__ void coo_fill_gap(double* y, int from, int to) {
  for (int r = from; r < to; ++r) y[r] = ACCUM ? add(y[r], 0.0) : 0.0;  // +0.0 either way
}

template <bool ACCUM>
__global__ void __launch_bounds__(kCooBlock)
    coo_sorted_segments(int nrows, int64_t nnz, const int* __restrict__ rows,
                        const int* __restrict__ cols, const double* __restrict__ vals,
                        const double* __restrict__ x, double* y, const int* guard,
                        int plus_zero) {
  if (guard && *guard) return;
  __shared__ int s_row[kCooTile];
  __shared__ double s_p[kCooTile];
  __shared__ int s_seg[kCooTile + 1];
  __shared__ int s_wsum[kCooBlock / 32];
  __shared__ int s_nseg;
  __shared__ double s_carry;
  __shared__ int s_carry_row, s_prev_row;
  const int tid = threadIdx.x;
  const int64_t start = coo_row_start_at_or_after(rows, nnz, (int64_t)blockIdx.x * kCooPerBlock);
  const int64_t end =
      coo_row_start_at_or_after(rows, nnz, (int64_t)(blockIdx.x + 1) * kCooPerBlock);
  const int R0 = (start == 0) ? 0 : (start < nnz ? rows[start] : nrows);
  const int R1 = (end < nnz) ? rows[end] : nrows;
  if (tid == 0) {
    s_carry_row = -1;
    s_carry = 0.0;
    s_prev_row = R0 - 1;
  }
  __syncthreads();
  for (int64_t t0 = start; t0 < end; t0 += kCooTile) {
    const int cnt = (int)min64(kCooTile, end - t0);
    for (int k = tid; k < cnt; k += kCooBlock) {
      s_row[k] = ld_stream(rows + t0 + k);
      s_p[k] = mul(ld_stream(vals + t0 + k), ld_gather(x + ld_stream(cols + t0 + k)));
    }
    __syncthreads();
    // segment heads: 8 consecutive entries per thread, block exclusive scan
    constexpr int PER = kCooTile / kCooBlock;
    int myh = 0;
    const int k0 = tid * PER;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int k = k0 + q;
      if (k < cnt && (k == 0 || s_row[k] != s_row[k - 1])) ++myh;
    }
    int incl = myh;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((tid & 31) >= o) incl += t;
    }
    if ((tid & 31) == 31) s_wsum[tid >> 5] = incl;
    __syncthreads();
    int wpre = 0;
    for (int w = 0; w < (tid >> 5); ++w) wpre += s_wsum[w];
    int pos = wpre + incl - myh;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int k = k0 + q;
      if (k < cnt && (k == 0 || s_row[k] != s_row[k - 1])) s_seg[pos++] = k;
    }
    if (tid == kCooBlock - 1) {
      s_nseg = wpre + incl;
      s_seg[wpre + incl] = cnt;
    }
    __syncthreads();
    const int nseg = s_nseg;
    const bool more = (t0 + cnt < end);
    const int next_row = more ? rows[t0 + cnt] : -1;
    const double carry_in = s_carry;       // read before any thread rewrites it
    const int carry_row_in = s_carry_row;
    const int prev_row_in = s_prev_row;
    __syncthreads();
    for (int s = tid; s < nseg; s += kCooBlock) {
      const int hs = s_seg[s], he = s_seg[s + 1];
      const int r = s_row[hs];
      const bool cont = (s == 0 && r == carry_row_in);
      double acc = cont ? carry_in : 0.0;
      for (int k = hs; k < he; ++k) acc = add(acc, s_p[k]);
      const int prev = (s == 0) ? prev_row_in : s_row[s_seg[s - 1]];
      if (!cont) coo_fill_gap<ACCUM>(y, prev + 1, r);
      if (s == nseg - 1 && more && next_row == r) {
        s_carry = acc;  // row continues in the next tile
        s_carry_row = r;
      } else {
        double out = ACCUM ? add(y[r], acc) : acc;
        if (plus_zero) out = add(out, 0.0);
        y[r] = out;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const int last = s_row[s_seg[nseg - 1]];
      s_prev_row = last;
      if (!(more && next_row == last)) s_carry_row = -1;
    }
    __syncthreads();
  }
  if (tid == 0) coo_fill_gap<ACCUM>(y, s_prev_row + 1, R1);
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
               bool sorted, const double* x, double* y, bool accum, const int* guard,
               cudaStream_t st, bool plus_zero) {
  if (nrows == 0) return DS_OK;
  if (sorted) {
    const int64_t blocks = nnz == 0 ? 1 : ceil_div(nnz, kCooPerBlock);
    if (accum)
      coo_sorted_segments<true><<<(unsigned)blocks, kCooBlock, 0, st>>>((int)nrows, nnz, rows,
                                                                        cols, vals, x, y, guard, (int)plus_zero);
    else
      coo_sorted_segments<false><<<(unsigned)blocks, kCooBlock, 0, st>>>((int)nrows, nnz, rows,
                                                                         cols, vals, x, y, guard, (int)plus_zero);
    DS_LAUNCH_CHECK("coo_sorted_segments");
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
  return launch_csr(nrows, row_offsets, col_indices, values, long_rows, n_long, x, y,
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
  return launch_coo(nrows, nnz, row_indices, col_indices, values, rows_sorted != 0, x, y,
                    accumulate == 1, nullptr, as_stream(stream), accumulate == 2);
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
