// ds_coo.cu -- COO SpMV for sm_100a (kernels.py:143-163 _coo_spmv; per row
// sequential in stored order from +0.0, np.bincount).
//
// coo_pipe (row-sorted, rows <= 27: TMA pipeline, thread per row),
// coo_warp_segments (+ coo_long_runs_kernel on a side stream for rows > 2048)
// for longer rows, coo_atomic for unsorted input (tolerance 1e-13, as the
// reference's threaded COO).
#include <algorithm>
#include <utility>
#include <vector>
#include <stdlib.h>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

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
    // LMAX 27) caps residency, so the variants bound registers via MINB.
    // Round 2 (tools/gpu_coosweep.sh, gpu_coo104.sh): 3-4 stages at 2-5
    // CTAs/SM 121-192 us; row starts scattered to a per-tile slot table (two
    // more barriers) instead of the per-row binary search 127 us -- rejected
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
