// ds_dia.cu -- DIA SpMV for sm_100a (kernels.py:122-140 _dia_spmv; per row a
// sequential sum from +0.0 over the in-range diagonals, ascending).
//
// dia_pipe: persistent TMA pipeline over row-major value slabs, unpredicated
// gathers (or TMA-staged x windows for large operators), fused p.Ap for the
// CG step (programmatic dependent launch); dia_rows_direct as the fallback.
#include <stdlib.h>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

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
      if (j > 0 && s_off[j] <= s_off[j - 1]) {   // windows need ascending offsets
        ok = 0;
        break;
      }
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
// Measured at 104^3 (one gpurun call, bench CG step / standalone SpMV):
// 128 rows x 3 stages x 2 CTAs/SM 53.7 / 41.2 us, 256 x 3 x 1 55.6 / 43.1,
// 128 x 4 x 2 54.6 / 42.6, 64 x 3-4 x 4 59-62 / 46-47, 2 stages 67-69 in
// the step (the programmatic-launch prefetch wants 3).  Round 2: x gathers
// bypassing L1 (to free it for a 4th stage or a 3rd CTA) 48.9-61 us
// standalone: the gathers need L1 (~70% hits).  An L2 bulk
// prefetch one / two ring rounds beyond the next copy (cp.async.bulk.prefetch.L2)
// was slower: 40.9 -> 44.9 / 47.4 us standalone.  With the x windows
// (>= 4M rows) 256 x 3 x 1 (192^3: 266 us vs 270).
static void dia_shape(int ndiags, int64_t nrows, int* T, int* S, int* ctas) {
  static int eT = -2, eS = -2, eC = -2;
  if (eT == -2) {
    const char* a = getenv("DS_DIA_T");
    const char* b = getenv("DS_DIA_S");
    const char* c = getenv("DS_DIA_CTAS");
    eT = a ? atoi(a) : -1;
    eS = b ? atoi(b) : -1;
    eC = c ? atoi(c) : -1;
  }
  const bool big = nrows >= (4ll << 20);   // the x-window layout (launch_dia)
  *T = big ? 256 : 128;
  *S = 3;
  *ctas = big ? 1 : 2;
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
  dia_shape(ndiags, nrows, &T, &S, &ctas);
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

}  // namespace ds

// ============================================================== C ABI ======
using namespace ds;

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

