// ds_convert.cu -- on-device format conversion through the canonical COO
// proxy (datamove.py:208-295, formats.py:439-479).  Bit-exact with the
// reference:
//   entries:    CSR rows = repeat(arange(n), diff(offsets)); DIA = in-range
//               NONZERO slots (explicit 0.0 / -0.0 dropped, formats.py:463-465)
//   canonical:  stable lexsort((cols, rows)) then duplicate runs summed as
//               np.add.reduceat: first + pairwise(rest) (datamove.py:208-220)
//   COO->CSR:   histogram + scan of row ids (datamove.py:238-243)
//   COO->DIA:   distinct (col - row) ascending; DiaFillOverflow iff
//               ndiags * nrows > fill_limit, tested BEFORE the target is
//               allocated (datamove.py:246-258); scatter.
// Shortcuts that keep the bits: a COO/CSR source that is already strictly
// (row, col)-increasing skips the sort (a stable sort of sorted unique keys is
// the identity); a DIA source yields canonical order directly (row-major walk
// of the slab, columns ascending because offsets ascend).
//
// Integer scans and histograms are hand-written (3-phase block scan); the
// general-case stable sort is ds_sort.cu's onesweep LSD radix sort on
// (row*ncols+col, index) keys limited to the needed bits.
#include <algorithm>
#include <vector>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

struct ds_convert_job {
  cudaStream_t st = nullptr;
  int target = 0;
  int64_t nrows = 0, ncols = 0;
  int64_t nnz = 0;             // canonical entries
  int* r = nullptr;            // canonical COO (device)
  int* c = nullptr;
  double* v = nullptr;
  bool own_r = false, own_c = false, own_v = false;
  bool spec = false;           // speculative CSR -> DIA (diagonal set from sampled tiles)
  int64_t ndiags = 0;          // DIA target
  int* diag_map = nullptr;     // exclusive scan of diagonal presence (nrows+ncols-1)
  int* dia_off = nullptr;      // (ndiags)
  // DIA source, CSR / COO target: the canonical entries are emitted straight
  // into the target at finish (row offsets = the exclusive scan of the row
  // counts), instead of into job buffers that are then copied
  const int* dsrc_off = nullptr;
  const double* dsrc_vals = nullptr;
  int dsrc_nd = 0;
  int64_t dsrc_in_lo = 0, dsrc_in_hi = 0;   // rows whose every diagonal is in range
  int* dsrc_start = nullptr;   // first entry of each row group (ceil(nrows / kDiaGroupRows))
  // canonical CSR source, DIA target: no COO proxy at all; the diagonal
  // census is taken while checking the order, the slab is filled per row
  const int* csr_off = nullptr;
  unsigned char* flags = nullptr;   // diagonal presence (nrows+ncols-1), already marked
  // DIA source (ascending offsets), DIA target: a column selection
  int* dia_jsrc = nullptr;          // (ndiags) source column of each target diagonal
  unsigned char* scratch = nullptr; // begin-phase temporaries (order flag, census), freed with the job
  int* gtmp = nullptr;
};

namespace ds {

constexpr int64_t kDefaultFillLimit = DS_FILL_LIMIT_DEFAULT;
constexpr int kScanBlock = 256;
constexpr int kScanPer = 8;
constexpr int kScanTile = kScanBlock * kScanPer;

// ---------------------------------------------------------------- scans ----
// Exclusive scan of f(k), k in [0, n), into out[0..n) (out may be null) and
// *total.  f returns small non-negative ints; the sum must fit in int32.
template <class F>
__global__ void __launch_bounds__(kScanBlock) scan_reduce_tiles(int64_t n, F f, int* tile_sums) {
  __shared__ int sh[kScanBlock / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int s = 0;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    const int64_t k = base + (int64_t)q * kScanBlock + threadIdx.x;
    if (k < n) s += f(k);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) t += sh[w];
    tile_sums[blockIdx.x] = t;
  }
}

// single block: exclusive scan of tile sums in place, total to *total
__global__ void __launch_bounds__(1024) scan_tile_sums(int64_t ntiles, int* sums, int* total) {
  __shared__ int sh[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < ntiles; b0 += 1024) {
    const int64_t k = b0 + threadIdx.x;
    const int v = (k < ntiles) ? sums[k] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += t;
    }
    if ((threadIdx.x & 31) == 31) sh[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      int w = sh[threadIdx.x];
      int wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, wi, o);
        if (threadIdx.x >= o) wi += t;
      }
      sh[threadIdx.x] = wi - w;  // exclusive warp prefix
    }
    __syncthreads();
    const int excl = carry + sh[threadIdx.x >> 5] + incl - v;
    if (k < ntiles) sums[k] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

template <class F>
__global__ void __launch_bounds__(kScanBlock)
    scan_downsweep(int64_t n, F f, const int* tile_offsets, int* out) {
  __shared__ int sh[kScanBlock / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  // each thread owns kScanPer consecutive elements for the in-tile order
  const int64_t k0 = base + (int64_t)threadIdx.x * kScanPer;
  int v[kScanPer];
  int s = 0;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    v[q] = (k0 + q < n) ? f(k0 + q) : 0;
    s += v[q];
  }
  int incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if ((threadIdx.x & 31) >= o) incl += t;
  }
  if ((threadIdx.x & 31) == 31) sh[threadIdx.x >> 5] = incl;
  __syncthreads();
  int wpre = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wpre += sh[w];
  int run = tile_offsets[blockIdx.x] + wpre + incl - s;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    if (k0 + q < n) out[k0 + q] = run;
    run += v[q];
  }
}

// Returns total on the host (synchronises).  out may be null.
template <class F>
static int exclusive_scan(int64_t n, F f, int* out, int64_t* total_host, cudaStream_t st) {
  const int64_t ntiles = n > 0 ? ceil_div(n, kScanTile) : 0;
  int* sums = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sums), (ntiles + 1) * sizeof(int), st));
  int* dtotal = sums + ntiles;
  if (ntiles > 0) {
    scan_reduce_tiles<<<(unsigned)ntiles, kScanBlock, 0, st>>>(n, f, sums);
    scan_tile_sums<<<1, 1024, 0, st>>>(ntiles, sums, dtotal);
    if (out) scan_downsweep<<<(unsigned)ntiles, kScanBlock, 0, st>>>(n, f, sums, out);
    DS_LAUNCH_CHECK("exclusive_scan");
  } else {
    DS_CUDA(cudaMemsetAsync(dtotal, 0, sizeof(int), st));
  }
  int h = 0;
  DS_CUDA(cudaMemcpyAsync(&h, dtotal, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(sums, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *total_host = h;
  return DS_OK;
}

// --------------------------------------------------------- entry arrays ----
__global__ void csr_expand_rows(int nrows, const int* __restrict__ off, int* rows) {
  // 8 lanes per row write its row id over its slice
  const int lane8 = threadIdx.x & 7;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 3; r < nrows;
       r += (gridDim.x * blockDim.x) >> 3)
    for (int k = off[r] + lane8; k < off[r + 1]; k += 8) rows[k] = r;
}


__global__ void make_keys(int64_t nnz, int64_t ncols, const int* __restrict__ r,
                          const int* __restrict__ c, unsigned long long* keys, int* idx) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    keys[k] = (unsigned long long)r[k] * (unsigned long long)ncols + (unsigned long long)c[k];
    idx[k] = (int)k;
  }
}

struct RunHead {  // 1 at the first entry of each run of equal sorted keys
  const unsigned long long* keys;
  __device__ int operator()(int64_t k) const { return (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0; }
};

// one thread per run head: canonical (row, col, value) with
// value = first + pairwise(rest) in stable (input) order
__global__ void reduce_runs(int64_t nnz, int64_t ncols, const unsigned long long* __restrict__ keys,
                            const int* __restrict__ perm, const int* __restrict__ pos,
                            const double* __restrict__ vals, int* r_out, int* c_out,
                            double* v_out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[k];
    if (k > 0 && keys[k - 1] == key) continue;
    int64_t e = k + 1;
    while (e < nnz && keys[e] == key) ++e;
    const double first = vals[perm[k]];
    double v = first;
    if (e - k > 1) {
      const int* p = perm + k + 1;
      v = add(first, pairwise_serial(e - k - 1, [&](int64_t i) { return vals[p[i]]; }));
    }
    const int o = pos[k];
    r_out[o] = (int)(key / (unsigned long long)ncols);
    c_out[o] = (int)(key % (unsigned long long)ncols);
    v_out[o] = v;
  }
}

// DIA source as a stream compaction.  The offsets ascend, so the canonical
// COO order of a DIA matrix is its row-major slot order filtered by "column
// in range and value != 0" (datamove.py:169-190 via formats.py:239-255).  One
// warp owns kDiaGroupRows consecutive rows, i.e. a contiguous run of slots:
// it reads them 32 at a time (coalesced, 4 chunks in flight) and a ballot
// gives each valid slot its position.  Pass 1 counts per group, an exclusive
// scan over the groups gives each warp its base, pass 2 writes the entries
// (and, for a CSR target, row_offsets[i] = the position of row i's first slot)
// straight into the target arrays.
constexpr int kDiaGroupRows = 32;
constexpr int kDiaChunks = 4;
#ifndef DS_DIA_EMIT_CHUNKS
#define DS_DIA_EMIT_CHUNKS 16
#endif
// slots in flight per lane in the emit walk: latency-bound on the value loads
// (ncu long_scoreboard 13 per issue at 4).  192^3 DIA->COO / DIA->CSR:
// 4: 1.36 / 1.12 ms, 8: 1.34 / 1.12, 12: 1.22 / 1.07, 16: 1.15 / 1.07 (96
// registers), 24: 1.68 / 1.66, 32: 1.33 / 1.29 (tools/gpu_ab_conv.sh)
constexpr int kDiaEmitChunks = DS_DIA_EMIT_CHUNKS;

struct DiaSlots {
  int ncols, nd, q, rmd;   // 32 = q * nd + rmd
  const int* off;
  const double* vals;
  __device__ DiaSlots(int ncols_, int nd_, const int* off_, const double* vals_)
      : ncols(ncols_), nd(nd_), q(32 / nd_), rmd(32 % nd_), off(off_), vals(vals_) {}
  // walk the slots [e_begin, e_end) of one group; f(valid, e, i, j) per lane
  template <int U = kDiaChunks, class F>
  __device__ __forceinline__ void walk(int64_t r0, int64_t e_begin, int64_t e_end, F&& f) const {
    const int lane = threadIdx.x & 31;
    int64_t i = r0 + lane / nd;
    int j = lane % nd;
    for (int64_t e0 = e_begin; e0 < e_end; e0 += 32 * U) {
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + u * 32 + lane;
        x[u] = e < e_end ? __ldg(vals + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + u * 32 + lane;
        const int64_t col = i + __ldg(off + j);
        const bool valid = e < e_end && col >= 0 && col < ncols && x[u] != 0.0;
        f(valid, e < e_end, i, j, (int)col, x[u]);
        i += q;
        j += rmd;
        if (j >= nd) {
          j -= nd;
          ++i;
        }
      }
    }
  }
};

// DIA source -> CSR / COO in ONE pass (ascending offsets, nd <= 32): a warp
// takes the next group of kDiaGroupRows rows (atomic ticket, so every earlier
// group is already resident), keeps the group's 32*nd slots in registers (nd
// per lane), counts the valid ones, publishes the count and sums its
// predecessors' counts by a warp-parallel decoupled look-back, then emits
// straight from the registers -- the slab is read once (the two-pass walk
// reads it twice).  The caller sizes the outputs by the in-range slot count.
constexpr int kDiaOneMaxNd = 32;
constexpr unsigned long long kGrpAgg = 1ull << 62, kGrpIncl = 2ull << 62,
                             kGrpMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(128)
    dia_emit_onepass(int64_t nrows, int ncols, int nd, const int* __restrict__ off,
                     const double* __restrict__ vals, int64_t ngroups,
                     unsigned long long* status, int* ticket, int* row_off, int* r, int* c,
                     double* v, long long* total) {
  __shared__ int s_off[kDiaOneMaxNd];
  for (int j = threadIdx.x; j < nd; j += blockDim.x) s_off[j] = __ldg(off + j);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int qq = 32 / nd, rmd = 32 % nd;
  while (true) {
    int g32 = 0;
    if (lane == 0) g32 = atomicAdd(ticket, 1);
    const int64_t g = __shfl_sync(0xffffffffu, g32, 0);
    if (g >= ngroups) break;
    const int64_t r0 = g * kDiaGroupRows;
    const int64_t r1 = min64(r0 + kDiaGroupRows, nrows);
    const int64_t eb = r0 * nd, ee = r1 * nd;
    double x[kDiaOneMaxNd];
    unsigned valid = 0;
#pragma unroll
    for (int q = 0; q < kDiaOneMaxNd; ++q) {
      const int64_t e = eb + q * 32 + lane;
      x[q] = (q < nd && e < ee) ? __ldg(vals + e) : 0.0;
    }
    int cnt = 0;
    {
      int64_t i = r0 + lane / nd;
      int j = lane % nd;
#pragma unroll
      for (int q = 0; q < kDiaOneMaxNd; ++q) {
        if (q < nd) {
          const int64_t e = eb + q * 32 + lane;
          const int64_t col = i + s_off[j];
          const bool ok = e < ee && col >= 0 && col < ncols && x[q] != 0.0;
          valid |= (unsigned)ok << q;
          cnt += __popc(__ballot_sync(0xffffffffu, ok));
          i += qq;
          j += rmd;
          if (j >= nd) {
            j -= nd;
            ++i;
          }
        }
      }
    }
    // publish, then the warp-parallel look-back over 32 predecessors at a time
    unsigned long long* mine = status + g;
    if (lane == 0)
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mine),
                   "l"((g == 0 ? kGrpIncl : kGrpAgg) | (unsigned long long)cnt) : "memory");
    long long excl = 0;
    for (int64_t p = g - 1; p >= 0; p -= 32) {
      const int64_t pl = p - lane;
      unsigned long long w = 0;
      if (pl >= 0) {
        do {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(status + pl) : "memory");
        } while ((w >> 62) == 0);
      }
      const unsigned incl = __ballot_sync(0xffffffffu, pl >= 0 && (w >> 62) == 2);
      const int stop = incl ? __ffs(incl) - 1 : 31;
      long long val = (pl >= 0 && lane <= stop) ? (long long)(w & kGrpMask) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
      excl += val;
      if (incl) break;
    }
    if (lane == 0 && g > 0)
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mine),
                   "l"(kGrpIncl | (unsigned long long)(excl + cnt)) : "memory");
    // emit from registers
    long long base = excl;
    int64_t i = r0 + lane / nd;
    int j = lane % nd;
#pragma unroll
    for (int q = 0; q < kDiaOneMaxNd; ++q) {
      if (q < nd) {
        const int64_t e = eb + q * 32 + lane;
        const bool ok = (valid >> q) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        const long long pos = base + __popc(m & lt);
        if (row_off && e < ee && j == 0) row_off[i] = (int)pos;
        if (ok) {
          if (r) r[pos] = (int)i;
          c[pos] = (int)(i + s_off[j]);
          v[pos] = x[q];
        }
        base += __popc(m);
        i += qq;
        j += rmd;
        if (j >= nd) {
          j -= nd;
          ++i;
        }
      }
    }
    if (g == ngroups - 1 && lane == 0) {
      if (row_off) row_off[nrows] = (int)(excl + cnt);
      *total = excl + cnt;
    }
  }
}

// DIA -> DIA: the target keeps the source diagonals that hold an entry
// (jsrc[t] = source column of target diagonal t); a slot keeps its value iff
// it is in range and nonzero (-0.0 and padding become +0.0, exactly as the
// canonical COO proxy's zero fill).  Thread per target slot, coalesced stores.
// rows [row0, row1) of the selection
__global__ void dia_copy_diags(int64_t row0, int64_t row1, int ncols, int nd, int nd_out,
                               const int* __restrict__ off, const double* __restrict__ vals,
                               const int* __restrict__ jsrc, double* out) {
  const int64_t total = row1 * nd_out;
  for (int64_t t = row0 * nd_out + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = total < (int64_t(1) << 32) ? (int64_t)((unsigned)t / (unsigned)nd_out)
                                                 : t / nd_out;
    const int j = __ldg(jsrc + (int)(t - i * nd_out));
    const int64_t col = i + __ldg(off + j);
    const double x = __ldg(vals + i * nd + j);
    out[t] = (col >= 0 && col < ncols && x != 0.0) ? x : 0.0;
  }
}

// every diagonal kept, rows whose columns are all in range: the selection
// is the slab itself with -0.0 turned into +0.0 (a 16-B stream over the
// slots [s0, s1); s0 even, values 16-B aligned)
__global__ void dia_copy_interior(int64_t s0, int64_t s1, const double* __restrict__ vals,
                                  double* __restrict__ out) {
  const int64_t n2 = (s1 - s0) >> 1;
  const double2* v2 = reinterpret_cast<const double2*>(vals + s0);
  double2* o2 = reinterpret_cast<double2*>(out + s0);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n2;
       t += (int64_t)gridDim.x * blockDim.x) {
    double2 x = ld_stream2(reinterpret_cast<const double*>(v2 + t));
    x.x = x.x != 0.0 ? x.x : 0.0;
    x.y = x.y != 0.0 ? x.y : 0.0;
    __stcs(o2 + t, x);
  }
  if (((s1 - s0) & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double x = __ldg(vals + s1 - 1);
    out[s1 - 1] = x != 0.0 ? x : 0.0;
  }
}

struct ArrayAt {
  const int* a;
  __device__ int operator()(int64_t k) const { return a[k]; }
};

// present != nullptr (DIA target): also the census of diagonals holding at
// least one entry (L1-cached test-before-set, see the diagonal flags below)
// Rows [in_lo, in_hi) have every diagonal's column inside the matrix: a
// group of them counts the nonzero values of its contiguous slot range with
// 16-B loads and no per-slot offset lookup (the caller passes an empty range
// when the values are not 16-B aligned or `present` is wanted).
// SELECT (DIA -> DIA, nd <= 32): the census as one global bit mask and the
// nonzero count as one global sum (separate 128-B lines), and every warp
// stops once the answer is settled -- every diagonal present and at least
// `need` nonzeros counted (the default fill limit's test; 0 with an
// explicit limit).  The stencil settles after ~10% of the slab; a matrix
// with an empty diagonal is read to the end, as before.
struct DiaSelect {
  unsigned* mask;
  unsigned long long* count;
  unsigned long long need;
  unsigned full;
};

template <bool INTERIOR, bool SELECT = false>
__global__ void dia_group_counts(int64_t nrows, int ncols, int nd, const int* __restrict__ off,
                                 const double* __restrict__ vals, int64_t ngroups, int* gcount,
                                 unsigned char* present, int64_t in_lo, int64_t in_hi,
                                 DiaSelect sel = DiaSelect{}) {
  const DiaSlots s(ncols, nd, off, vals);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned seen = 0;   // SELECT, lane 0: the global mask as last read
  for (; g < ngroups; g += nwarps) {
    if (SELECT) {   // the warps advance together, so the static order is ~ascending
      int stop = 0;
      if (lane == 0) {
        unsigned long long n;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(sel.mask) : "memory");
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(n) : "l"(sel.count) : "memory");
        stop = seen == sel.full && n >= sel.need;
      }
      if (__shfl_sync(0xffffffffu, stop, 0)) break;
    }
    const int64_t r0 = g * kDiaGroupRows;
    const int64_t r1 = r0 + kDiaGroupRows < nrows ? r0 + kDiaGroupRows : nrows;
    if (INTERIOR && r0 >= in_lo && r1 <= in_hi) {
      const int64_t e0 = r0 * nd, e1 = r1 * nd;   // e0 even: r0 is a multiple of 32
      const double2* v2 = reinterpret_cast<const double2*>(vals + e0);
      const int n2 = (int)((e1 - e0) >> 1);
      int cnt = 0;
      // present (DIA target, nd <= 32): lane bit j = a nonzero on diagonal j;
      // a lane's slots advance by 64 per step, so its diagonal advances by 64 % nd
      unsigned mask = 0;
      int j0 = (SELECT || present) ? (2 * lane) % nd : 0;
      const int rm = (SELECT || present) ? 64 % nd : 0;
      for (int t0 = 0; t0 < n2; t0 += 32 * kDiaChunks) {
        double2 x[kDiaChunks];
#pragma unroll
        for (int u = 0; u < kDiaChunks; ++u) {
          const int t = t0 + u * 32 + lane;
          x[u] = t < n2 ? ld_stream2(reinterpret_cast<const double*>(v2 + t)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kDiaChunks; ++u) {
          cnt += (x[u].x != 0.0) + (x[u].y != 0.0);
          if (SELECT || present) {
            const int j1 = j0 + 1 == nd ? 0 : j0 + 1;
            mask |= ((unsigned)(x[u].x != 0.0) << j0) | ((unsigned)(x[u].y != 0.0) << j1);
            j0 += rm;
            if (j0 >= nd) j0 -= nd;
          }
        }
      }
      if (((e1 - e0) & 1) && lane == 0) {   // the odd last slot: diagonal nd - 1
        const bool nz = __ldg(vals + e1 - 1) != 0.0;
        cnt += nz;
        mask |= (unsigned)nz << (nd - 1);
      }
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (SELECT) {
        mask = __reduce_or_sync(0xffffffffu, mask);
        if (lane == 0) {
          atomicAdd(sel.count, (unsigned long long)cnt);
          if ((mask | seen) != seen) atomicOr(sel.mask, mask);
        }
        continue;
      }
      if (lane == 0) gcount[g] = cnt;
      if (present) {
        mask = __reduce_or_sync(0xffffffffu, mask);
        if (lane < nd && ((mask >> lane) & 1u)) {
          unsigned short f;
          asm volatile("ld.global.ca.u8 %0, [%1];" : "=h"(f) : "l"(present + lane));
          if (f == 0) present[lane] = 1;
        }
      }
      continue;
    }
    int cnt = 0;
    unsigned smask = 0;
    s.walk(r0, r0 * nd, r1 * nd, [&](bool valid, bool, int64_t, int j, int, double) {
      cnt += __popc(__ballot_sync(0xffffffffu, valid));
      if (SELECT) {
        if (valid) smask |= 1u << j;
        return;
      }
      if (present && valid) {
        unsigned short f;
        asm volatile("ld.global.ca.u8 %0, [%1];" : "=h"(f) : "l"(present + j));
        if (f == 0) present[j] = 1;
      }
    });
    if (SELECT) {
      smask = __reduce_or_sync(0xffffffffu, smask);
      if (lane == 0) {
        atomicAdd(sel.count, (unsigned long long)cnt);
        if ((smask | seen) != seen) atomicOr(sel.mask, smask);
      }
      continue;
    }
    if ((threadIdx.x & 31) == 0) gcount[g] = cnt;
  }
}

// (Round 2: an interior fast path -- two consecutive slots per lane from one
// 16-B load, offsets in lanes -- was slower, 192^3 DIA->CSR 1.12 -> 1.36 ms:
// each lane's two stores make every warp store touch twice the sectors.)
__global__ void dia_group_emit(int64_t nrows, int ncols, int nd, const int* __restrict__ off,
                               const double* __restrict__ vals, int64_t ngroups,
                               const int* __restrict__ gstart, int* row_off, int* r, int* c,
                               double* v) {
  const DiaSlots s(ncols, nd, off, vals);
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ngroups; g += nwarps) {
    const int64_t r0 = g * kDiaGroupRows;
    const int64_t r1 = r0 + kDiaGroupRows < nrows ? r0 + kDiaGroupRows : nrows;
    int base = gstart[g];
    s.template walk<kDiaEmitChunks>(r0, r0 * nd, r1 * nd, [&](bool valid, bool in, int64_t i, int j, int col, double x) {
      const unsigned m = __ballot_sync(0xffffffffu, valid);
      const int pos = base + __popc(m & lt);
      if (row_off && in && j == 0) row_off[i] = pos;
      if (valid) {
        if (r) r[pos] = (int)i;
        c[pos] = col;
        v[pos] = x;
      }
      base += __popc(m);
    });
  }
}

// ------------------------------------------------------------- targets -----
// offsets[i] = first canonical entry with row >= i  (rows sorted)
__global__ void rows_to_offsets(int64_t nnz, int nrows, const int* __restrict__ r, int* off) {
  if (nnz == 0) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nrows; i += gridDim.x * blockDim.x)
      off[i] = 0;
    return;
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int lo = (k == 0) ? -1 : r[k - 1];
    const int hi = (k == nnz) ? nrows : r[k];
    for (int i = lo + 1; i <= hi; ++i) off[i] = (int)k;
  }
}

// Presence flags of every diagonal (taken by coo_check_mark /
// csr_census_quads / dia_group_counts).  Few distinct diagonals are hit by very
// many entries (27 for the stencil) and same-address stores serialise in L2.
// Each marker tests first with an L1-CACHED load: an SM's own store
// invalidates its L1 line, the next miss brings back the 1, so every SM writes
// each flag about once and all other tests hit L1 (a racing duplicate store
// of 1 is harmless).
// CSR source, DIA target: one pass over the column indices checks the
// canonical order (strictly ascending columns in every row: coo_check_mark's
// test without expanding the rows) and marks the diagonals (csr_census_quads);
// then the DIA slab of a block of rows is zeroed in shared memory, the
// block's entries are dropped into their (row, diagonal) slots and the slab
// is written out with coalesced stores (values are row-major (nrows,
// ndiags)).  The fill walks the entries of a warp's rows 32 at a time
// (coalesced, U chunks of loads in flight), finding each entry's row by a
// shuffle search over the warp's offsets.
// shared-memory caches of diagonal flags / diag_map entries: 2^kFlagTagBits slots
constexpr int kFlagTagBits = 10;
constexpr int kCsrWalkRows = 16;    // rows per warp (<= 31: the offsets live in one lane each)
// Lane t <= r1 - r0 holds off[r0 + t] (the rest INT_MAX): an entry's row is
// found by a 5-step binary search over the lanes (shuffles, no memory).  The
// callers load the next group's offsets before walking the current group.
__device__ __forceinline__ int walk_offsets(const int* __restrict__ off, int nrows, int r0) {
  const int lane = threadIdx.x & 31;
  const int r1 = min(r0 + kCsrWalkRows, nrows);
  return r0 < nrows && lane <= r1 - r0 ? __ldg(off + r0 + lane) : 0x7fffffff;
}
// body(kb, k1, rows[U], loaded[U]): lane's entry of chunk u is kb + 32u + lane
template <int U, class Load, class Body>
__device__ __forceinline__ void csr_warp_walk(int ot, int r0, int r1, Load&& load, Body&& body) {
  const int lane = threadIdx.x & 31;
  const int k1 = __shfl_sync(0xffffffffu, ot, r1 - r0);
  int kb = __shfl_sync(0xffffffffu, ot, 0);
  decltype(load(0)) x[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (kb + 32 * u + lane < k1) x[u] = load(kb + 32 * u + lane);
  for (; kb < k1; kb += 32 * U) {
    decltype(load(0)) xn[U];   // the next chunks' loads in flight while this one is processed
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + 32 * (U + u) + lane;
      if (k < k1) xn[u] = load(k);
    }
    int rr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + 32 * u + lane;
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (__shfl_sync(0xffffffffu, ot, lo + step) <= k) lo += step;
      rr[u] = r0 + lo;
    }
    body(kb, k1, rr, x);
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = xn[u];
  }
}

struct ColVal {
  int c;
  double v;
};

// *bad bits: kBadOrder (not canonical), kBadIndex (a column outside [0, ncols):
// nothing is marked for it, the caller raises IndexOutOfRange)
constexpr int kBadOrder = 1, kBadIndex = 2, kBadRowOrder = 4;   // 4: rows decrease somewhere
constexpr int kBadMiss = 8;   // a diagonal outside the speculative set (dia_fill_csr<true>)


// diag_map cache of the DIA fills: the target's nd diagonals (dia_off) are
// entered by one thread before the walk ((j << 32) | d words, a later
// diagonal taking a colliding slot), so the walk only reads it; a miss reads
// diag_map itself.  Returns after the block barrier.
__device__ __forceinline__ void preload_map_cache(unsigned long long* mc, const int* dia_off,
                                                  int nd, int nrows) {
  for (int i = threadIdx.x; i < (1 << kFlagTagBits); i += blockDim.x) mc[i] = ~0ull;
  __syncthreads();
  if (threadIdx.x == 0 && nd <= 256)   // wider sets: every lookup reads diag_map
    for (int j = 0; j < nd; ++j) {
      const unsigned d = (unsigned)__ldg(dia_off + j) + (unsigned)(nrows - 1);
      mc[(d * 0x9E3779B1u) >> (32 - kFlagTagBits)] = ((unsigned long long)(unsigned)j << 32) | d;
    }
  __syncthreads();
}

// CHECK (the speculative CSR -> DIA, ds_convert_begin_csr_dia_spec): the
// walk also checks the order ((row, col) strictly increasing in every row),
// the column range and that every entry's diagonal is in `map` (the
// exclusive scan of the sampled presence: d present iff map[d+1] > map[d]),
// setting kBadOrder / kBadIndex / kBadMiss in *bad instead of storing.
#ifndef DS_FILL_U
#define DS_FILL_U 4
#endif
// 32-entry chunks in flight per warp in the slab fill; 192^3 CSR->DIA
// (speculative path) 2: 1.09-1.10 ms, 4: 1.04-1.05, 8: 1.42 (90 registers)
constexpr int kFillU = DS_FILL_U;
template <bool CHECK>
__global__ void dia_fill_csr(int nrows, int nd, int R, const int* __restrict__ off,
                             const int* __restrict__ c, const double* __restrict__ v,
                             const int* __restrict__ map, const int* __restrict__ dia_off,
                             double* vals, int ncols = 0, int* bad = nullptr) {
  extern __shared__ double slab[];   // R * nd, R = kCsrWalkRows * warps per block
  __shared__ unsigned long long mcache[1 << kFlagTagBits];
  preload_map_cache(mcache, dia_off, nd, nrows);
  const int warp = threadIdx.x >> 5;
  const unsigned D = (unsigned)nrows + (unsigned)ncols - 1u;
  int mybad = 0;
  int ot = walk_offsets(off, nrows, blockIdx.x * R + warp * kCsrWalkRows);
  for (int b0 = blockIdx.x * R; b0 < nrows; b0 += gridDim.x * R) {
    const int rows = min(R, nrows - b0);
    const int total = rows * nd;
    const int r0 = b0 + warp * kCsrWalkRows;
    const int ot_next = walk_offsets(off, nrows, r0 + gridDim.x * R);
    for (int t = threadIdx.x; t < total; t += blockDim.x) slab[t] = 0.0;
    __syncthreads();
    if (r0 < b0 + rows) {
      const int r1 = min(r0 + kCsrWalkRows, b0 + rows);
      int carry = -1, carry_row = -1;   // CHECK: the previous chunk's last entry (lane 31)
      csr_warp_walk<kFillU>(ot, r0, r1, [&](int k) { return ColVal{__ldg(c + k), __ldg(v + k)}; },
                       [&](int kb, int k1, const int (&rr)[kFillU], const ColVal (&e)[kFillU]) {
                         const int lane = threadIdx.x & 31;
                         int j[kFillU];
                         bool ok[kFillU];
#pragma unroll
                         for (int u = 0; u < kFillU; ++u) {
                           j[u] = 0;
                           ok[u] = kb + 32 * u + lane < k1;
                           if (CHECK) {
                             int prev = __shfl_up_sync(0xffffffffu, e[u].c, 1);
                             int prev_row = __shfl_up_sync(0xffffffffu, rr[u], 1);
                             if (lane == 0) {
                               prev = carry;
                               prev_row = carry_row;
                             }
                             carry = __shfl_sync(0xffffffffu, e[u].c, 31);
                             carry_row = __shfl_sync(0xffffffffu, rr[u], 31);
                             if (ok[u]) {
                               // an entry out of order is not stored (its
                               // duplicate's slot stays single-writer)
                               if (prev_row == rr[u] && prev >= e[u].c) {
                                 mybad |= kBadOrder;
                                 ok[u] = false;
                               }
                               if ((unsigned)e[u].c >= (unsigned)ncols) {
                                 mybad |= kBadIndex;
                                 ok[u] = false;
                               }
                             }
                           }
                           if (ok[u]) {
                             const unsigned d = (unsigned)e[u].c - (unsigned)rr[u] + (unsigned)(nrows - 1);
                             const unsigned h = (d * 0x9E3779B1u) >> (32 - kFlagTagBits);
                             const unsigned long long m = mcache[h];
                             if ((unsigned)m == d) {
                               j[u] = (int)(m >> 32);
                             } else {
                               j[u] = __ldg(map + d);
                               if (CHECK) {
                                 const int jn = d + 1 < D ? __ldg(map + d + 1) : nd;
                                 if (jn == j[u]) j[u] = -1;
                               }
                             }
                             if (CHECK && j[u] < 0) {
                               mybad |= kBadMiss;
                               ok[u] = false;
                             }
                           }
                         }
#pragma unroll
                         for (int u = 0; u < kFillU; ++u)
                           if (ok[u]) slab[(rr[u] - b0) * nd + j[u]] = e[u].v;
                       });
    }
    __syncthreads();
    double* out = vals + (int64_t)b0 * nd;
    for (int t = threadIdx.x; t < total; t += blockDim.x) out[t] = slab[t];
    __syncthreads();
    ot = ot_next;
  }
  if (CHECK) {
    mybad = __reduce_or_sync(0xffffffffu, mybad);
    if ((threadIdx.x & 31) == 0 && mybad) atomicOr(bad, mybad);
  }
}

// Slot-parallel DIA fill (nd <= 32; datamove.py:238-258 places entry (r, c)
// at slot (r, j) with dia_off[j] = c - r).  A warp takes 32 consecutive rows
// and walks their 32 * nd target slots flat, lane per slot (coalesced
// stores, kFillSlotsU slots per lane in flight).  A row holding exactly nd
// entries ("full": the stencil's interior) needs no diag_map lookup: its
// slot j is entry off[r] + j, checked by one compare (column == r +
// dia_off[j], in range -- which also proves the row strictly increasing).
// Rows that are not full -- and every row of a chunk where a compare failed
// -- are then rewritten one at a time by the warp: zeroed, and their entries
// scattered through diag_map (or, without one, a 5-step shuffle search of
// the lanes' offsets) with dia_fill_csr<CHECK>'s checks (order, column
// range, membership; an out-of-order entry is not stored).
// Measured (tools/gpu_fillab.sh, same box, 192^3 wall): CSR -> DIA 1.04 ms
// (the slab walk, DS_DIA_FILL_ROWS=0) -> 0.93 ms, COO -> DIA 1.62 -> 1.28 ms
// (with coo_offsets_check).  Slots per lane 6 (64 registers); 8: 1.07 ms,
// 12: 1.39, 16: 1.22; a bulk L2 prefetch of the next chunk's entries: 1.19
// vs 0.98; the slot state recomputed in the store loop instead of kept per
// slot (6 / 8 / 10 slots): 0.98 / 1.04 / 0.95.  Rejected: a warp per row (~57 warp instructions per row, 852 us
// cold for the fill kernel, the same as the slab walk) and the same walk
// TMA-staged at 1 CTA/SM (1.49 ms, issue-latency bound).
#ifndef DS_FILL_SLOTS_U
#define DS_FILL_SLOTS_U 6
#endif
constexpr int kFillSlotsU = DS_FILL_SLOTS_U;
template <bool CHECK>
__global__ void __launch_bounds__(256)
    dia_fill_rows(int nrows, int nd, const int* __restrict__ off, const int* __restrict__ c,
                  const double* __restrict__ v, const int* __restrict__ map,
                  const int* __restrict__ dia_off, double* vals, int ncols, int* bad) {
  constexpr int U = kFillSlotsU;
  const int lane = threadIdx.x & 31;
  const int myoff = lane < nd ? __ldg(dia_off + lane) : 0;
  const unsigned D = (unsigned)nrows + (unsigned)ncols - 1u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int qq = 32 / nd, rmd = 32 % nd;   // a lane's slot advances by 32: rows qq, slots rmd
  int mybad = 0;
  for (int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; r0 < nrows;
       r0 += nw * 32) {
    const int nr = (int)min64(32, nrows - r0);
    int oa = 0, ob = 0;
    if (lane < nr) {
      oa = __ldg(off + r0 + lane);
      ob = __ldg(off + r0 + lane + 1);
    }
    const unsigned full = __ballot_sync(0xffffffffu, lane < nr && ob - oa == nd);
    const int total = nr * nd;
    double* out = vals + r0 * nd;
    int row = lane / nd, j = lane % nd;
    bool mism = false;
    for (int q0 = 0; q0 < total; q0 += 32 * U) {
      int col[U];
      double val[U];
      bool f[U];
      int rw[U], jj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + 32 * u + lane;
        rw[u] = row;
        jj[u] = j;
        const int k = __shfl_sync(0xffffffffu, oa, row & 31) + j;
        f[u] = q < total && ((full >> (row & 31)) & 1u);
        col[u] = -1;
        val[u] = 0.0;
        if (f[u]) {
          col[u] = __ldg(c + k);
          val[u] = __ldg(v + k);
        }
        row += qq;
        j += rmd;
        if (j >= nd) {
          j -= nd;
          ++row;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int doff = __shfl_sync(0xffffffffu, myoff, jj[u]);
        if (f[u]) {
          if (col[u] == (int)r0 + rw[u] + doff && (unsigned)col[u] < (unsigned)ncols)
            out[q0 + 32 * u + lane] = val[u];
          else
            mism = true;
        }
      }
    }
    // rows the slot walk did not (validly) write
    unsigned redo = __any_sync(0xffffffffu, mism) ? 0xffffffffu : ~full;
    if (nr < 32) redo &= (1u << nr) - 1u;
    if (redo) __syncwarp();
    while (redo) {
      const int i = __ffs(redo) - 1;
      redo &= redo - 1;
      const int r = (int)r0 + i;
      const int k0 = __shfl_sync(0xffffffffu, oa, i), k1 = __shfl_sync(0xffffffffu, ob, i);
      double* rowp = vals + (int64_t)r * nd;
      if (lane < nd) rowp[lane] = 0.0;
      __syncwarp();
      for (int kb = k0; kb < k1; kb += 32) {   // warp-uniform trips: the search shuffles
        const int k = kb + lane;
        bool ok = k < k1;
        const int ck = ok ? __ldg(c + k) : 0;
        if (CHECK && ok) {
          if (k > k0 && __ldg(c + k - 1) >= ck) {   // not strictly increasing
            mybad |= kBadOrder;
            ok = false;
          } else if ((unsigned)ck >= (unsigned)ncols) {
            mybad |= kBadIndex;
            ok = false;
          }
        }
        int jd = 0;
        if (map) {
          if (ok) {
            const unsigned d = (unsigned)ck - (unsigned)r + (unsigned)(nrows - 1);
            jd = __ldg(map + d);
            if (CHECK && (d + 1 < D ? __ldg(map + d + 1) : nd) == jd) {
              mybad |= kBadMiss;
              ok = false;
            }
          }
        } else {   // no diag_map (the small speculative set): search the lanes' offsets
          const int o = ck - r;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int idx = jd + step;
            const int val = __shfl_sync(0xffffffffu, myoff, idx & 31);
            if (idx < nd && val <= o) jd = idx;
          }
          const int hit = __shfl_sync(0xffffffffu, myoff, jd);
          if (ok && hit != o) {
            mybad |= kBadMiss;
            ok = false;
          }
        }
        if (ok) rowp[jd] = __ldg(v + k);
      }
      __syncwarp();
    }
  }
  if (CHECK) {
    mybad = __reduce_or_sync(0xffffffffu, mybad);
    if (lane == 0 && mybad) atomicOr(bad, mybad);
  }
}

// The sampled census's diagonals when there are at most kSmallDiags (the
// slot fill's case, which then needs no D-long diag_map): flag bytes read
// 16 at a time, set ones appended to a short list; one warp sorts it.
constexpr int kSmallDiags = 32;
__global__ void flags_collect(int64_t D, const unsigned char* __restrict__ flags, int* list,
                              int* count) {
  const int64_t n16 = D >> 4;
  const uint4* w16 = reinterpret_cast<const uint4*>(flags);
  auto put = [&](int64_t d) {
    const int k = atomicAdd(count, 1);
    if (k < kSmallDiags) list[k] = (int)d;
  };
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = __ldg(w16 + i);
    if (w.x | w.y | w.z | w.w) {
      const unsigned q[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if ((q[b >> 2] >> (8 * (b & 3))) & 0xffu) put(i * 16 + b);
    }
  }
  if (blockIdx.x == 0)
    for (int64_t d = n16 * 16 + threadIdx.x; d < D; d += blockDim.x)
      if (flags[d]) put(d);
}

// one warp: offsets[rank of list[l]] = list[l] - (nrows - 1), n <= 32 distinct
__global__ void small_diags_sort(int nrows, const int* __restrict__ list,
                                 const int* __restrict__ count, int* offsets) {
  const int lane = threadIdx.x;
  const int n = min(*count, kSmallDiags);
  const int mine = lane < n ? list[lane] : INT_MAX;
  int rank = 0;
  for (int l = 0; l < n; ++l) rank += __shfl_sync(0xffffffffu, mine, l) < mine;
  if (lane < n) offsets[rank] = mine - (nrows - 1);
}

// Row offsets of a COO source for the row-slot fill (the speculative COO ->
// DIA): off[i] = first entry with row >= i, checking the row order (kBadOrder
// | kBadRowOrder) and range (kBadIndex).  off must be zeroed first: with
// unsorted rows some offsets stay unwritten, and every written or zero value
// lies in [0, nnz], so the fill that runs before the host sees `bad` only
// reads inside the arrays.
__device__ __forceinline__ void coo_offsets_span(int64_t k, int lo, int hi, int nrows, int* off) {
  lo = min(max(lo, -1), nrows);
  hi = min(max(hi, -1), nrows);
  for (int i = lo + 1; i <= hi; ++i) off[i] = (int)k;
}

// entries taken as 16-B quads (rows 16-B aligned), two quads in flight per
// thread; the boundary k == nnz and a ragged tail by the last thread
// (Rejected, 192^3: 4 quads per thread with the previous row from a shuffle,
// 360 us; the same plus a compare-only path for quads without a row change,
// 366 us -- against this kernel's 343 us; ncu: 884 MB read for 757 MB, L2
// hit rate 26%, sm__throughput 76%.)
__global__ void coo_offsets_check(int64_t nnz, int nrows, const int* __restrict__ r, int* off,
                                  int* bad) {
  int mybad = 0;
  const int64_t nq = nnz >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto quad = [&](int64_t q, int4 x) {
    const int64_t k = q * 4;
    const int p = k > 0 ? __ldg(r + k - 1) : -1;
    const int rr[4] = {x.x, x.y, x.z, x.w};
    int prev = p;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((unsigned)rr[u] >= (unsigned)nrows) mybad |= kBadIndex;
      if (rr[u] < prev) mybad |= kBadOrder | kBadRowOrder;
      if (rr[u] != prev) coo_offsets_span(k + u, prev, rr[u], nrows, off);
      prev = rr[u];
    }
  };
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; q + stride < nq; q += 2 * stride) {
    const int4 x0 = ld_stream4(r + q * 4), x1 = ld_stream4(r + (q + stride) * 4);
    quad(q, x0);
    quad(q + stride, x1);
  }
  if (q < nq) quad(q, ld_stream4(r + q * 4));
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // the tail entries and the end k == nnz
    int prev = nq * 4 > 0 ? __ldg(r + nq * 4 - 1) : -1;
    for (int64_t k = nq * 4; k < nnz; ++k) {
      const int x = __ldg(r + k);
      if ((unsigned)x >= (unsigned)nrows) mybad |= kBadIndex;
      if (x < prev) mybad |= kBadOrder | kBadRowOrder;
      coo_offsets_span(k, prev, x, nrows, off);
      prev = x;
    }
    coo_offsets_span(nnz, prev, nrows, nrows, off);
  }
  mybad = __reduce_or_sync(0xffffffffu, mybad);
  if ((threadIdx.x & 31) == 0 && mybad) atomicOr(bad, mybad);
}

// ------------------------------------------------- CSR tiles with row ids --
// Entry-parallel walks of a CSR source: a CTA takes kRT consecutive rows and
// scatters each row's tile-local id over the tile's entries in shared memory
// (one thread per row; chunks of kRtCap entries when the rows are long), then
// every thread reads consecutive entries -- coalesced loads, no per-entry
// search of the offsets (the warp walks above spend their issue slots on it).
constexpr int kRT = 128;
constexpr int kRtCap = 4096;

struct RowIds {
  int off[kRT + 1];
  unsigned char rid[kRtCap];
};

// body(kb, k0, kend): entries kb + u * blockDim.x + threadIdx.x (u < kRtU) of
// the chunk [k0, kend) -- kRtU loads in flight per thread; the trip count is
// uniform across the block (lanes past kend see k >= kend)
constexpr int kRtU = 8;
template <class Body>
__device__ __forceinline__ void csr_rowid_tile(int nrows, const int* __restrict__ off, int r0,
                                               RowIds& ids, Body&& body) {
  const int nr = min(kRT, nrows - r0);
  for (int t = threadIdx.x; t <= nr; t += blockDim.x) ids.off[t] = __ldg(off + r0 + t);
  __syncthreads();
  const int e0 = ids.off[0], e1 = ids.off[nr];
  for (int k0 = e0; k0 < e1; k0 += kRtCap) {
    const int kend = min(k0 + kRtCap, e1);
    for (int t = threadIdx.x; t < nr; t += blockDim.x) {
      const int lo = max(ids.off[t], k0), hi = min(ids.off[t + 1], kend);
      for (int k = lo; k < hi; ++k) ids.rid[k - k0] = (unsigned char)t;
    }
    __syncthreads();
    for (int kb = k0; kb < kend; kb += blockDim.x * kRtU) body(kb, k0, kend);
    __syncthreads();
  }
}

// order check ((row, col) strictly increasing inside every row), index range
// and the diagonal census of a CSR source.  Round 2 (tools/gpu_ab_conv.sh):
// a row-uniform warp walk (a warp takes 32 rows one row at a time, no row-id
// lookup per entry, 8 rows' columns in flight) was slower -- 192^3 census
// 1.13 -> 1.26 ms wall, and with the matching slab-per-row DIA fill CSR->DIA
// 1.46 -> 1.85 ms: latency-bound on the per-row chain.  The entry-at-a-time
// row-id tile walk (csr_census_tiles, round 2 first pass) was issue-bound at
// ~2 warp instructions per entry; csr_census_quads below replaces it.

// The same census, entries taken four at a time (round 2, second pass): a
// thread loads one 16-B aligned quad of columns and the quad's four row ids
// with one 32-bit shared load, so the per-entry work is the order compare,
// the range check and the flag test (~12 instructions per entry, was ~40:
// csr_census_tiles was issue-bound, ncu sm__throughput 62-69% at 2 warp
// instructions per entry).  "Same row as the previous entry" is a row-id
// compare inside the quad and `k > off[row]` at its first entry; the previous
// column comes from the lane before (lane 0: one scalar load).  Quads that
// straddle the array bounds or a chunk edge load their entries one by one.
// The next tile's offsets are loaded before the current tile is walked.
constexpr int kCqU = 4;             // quads in flight per thread
constexpr int kCqCap = 8192;        // entries per row-id chunk (multiple of 4)
struct QuadIds {
  int off[kRT + 1];
  unsigned char rid[kCqCap + 4];
};


// flag test of one entry: a per-CTA shared-memory tag table of recently set
// diagonals first (the stencil's 27 diagonals stay resident: one shared
// atomic per entry -- atomics, so the racing tag updates are not data races),
// then the L1-cached global test-before-set.  A tag is written only after its
// flag was tested / set, so a tag hit always means the flag is set.
__device__ __forceinline__ void census_flag(unsigned char* flags, unsigned d, bool ok,
                                            unsigned* tags) {
  const unsigned h = (d * 0x9E3779B1u) >> (32 - kFlagTagBits);
  if (ok && atomicOr(&tags[h], 0u) != d) {
    unsigned short f;
    asm volatile("ld.global.ca.u8 %0, [%1];" : "=h"(f) : "l"(flags + d));
    if (f == 0) flags[d] = 1;
    atomicExch(&tags[h], d);
  }
}

// COPY (ds_convert_direct, a canonical CSR source to a COO / CSR target):
// the same walk also writes the columns, values and -- ROWS -- the row index
// of every entry (tile row + row id) into the target, so the source is read
// once; the caller discards the target if the census finds the source not
// canonical.  Needs 16-B aligned columns / values / targets (s == 0).
template <bool FLAGS, bool COPY = false, bool ROWS = false>
__global__ void __launch_bounds__(256)
    csr_census_quads(int nrows, int ncols, int64_t nnz, const int* __restrict__ off,
                     const int* __restrict__ c, unsigned char* flags, int* bad,
                     const double* __restrict__ v = nullptr, int* __restrict__ orow = nullptr,
                     int* __restrict__ ocol = nullptr, double* __restrict__ oval = nullptr,
                     int tile0 = 0, int tile_step = 1) {
  constexpr bool LOADV = COPY;
  constexpr int U = LOADV ? 2 : kCqU;
  __shared__ QuadIds ids;
  __shared__ unsigned tags[FLAGS ? 1 << kFlagTagBits : 1];
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  if (FLAGS)
    for (int i = tid; i < (1 << kFlagTagBits); i += blockDim.x) tags[i] = 0xffffffffu;
  // (the tile loop's first barrier orders the tag reset before any lookup)
  // entry k lives in address quad (k + s) >> 2
  const int s = (int)((reinterpret_cast<uintptr_t>(c) >> 2) & 3);
  int mybad = 0;
  const int ntiles = (nrows + kRT - 1) / kRT;
  int tile = tile0 + (int)blockIdx.x * tile_step;
  int o_next = 0;
  if (tile < ntiles && tid <= min(kRT, nrows - tile * kRT)) o_next = __ldg(off + tile * kRT + tid);
  for (; tile < ntiles; tile += (int)gridDim.x * tile_step) {
    const int r0 = tile * kRT;
    const int nr = min(kRT, nrows - r0);
    if (tid <= nr) ids.off[tid] = o_next;
    {
      const int nt = tile + (int)gridDim.x * tile_step;
      if (nt < ntiles && tid <= min(kRT, nrows - nt * kRT)) o_next = __ldg(off + nt * kRT + tid);
    }
    __syncthreads();
    const int e0 = ids.off[0], e1 = ids.off[nr];
    // d = column - row + nrows - 1 = column - t + dbase for tile-local row t
    const unsigned dbase = (unsigned)(nrows - 1) - (unsigned)r0;
    for (int kq0 = ((e0 + s) & ~3) - s; kq0 < e1; kq0 += kCqCap) {
      const int k0 = max(kq0, e0), kend = min(kq0 + kCqCap, e1);
      for (int t = tid; t < nr; t += blockDim.x) {
        const int lo = max(ids.off[t], k0), hi = min(ids.off[t + 1], kend);
        for (int k = lo; k < hi; ++k) ids.rid[k - kq0] = (unsigned char)t;
      }
      if (tid < k0 - kq0) ids.rid[tid] = 0xff;   // head entries before the tile: no row
      __syncthreads();
      const int nq = (kend - kq0 + 3) >> 2;
      const int4* cq = reinterpret_cast<const int4*>(c + kq0);   // 16-B aligned: (kq0 + s) % 4 == 0
      for (int qb = 0; qb < nq; qb += (int)blockDim.x * U) {
        int4 cv[U];
        int pv[U];
        double ve[LOADV ? U : 1][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = qb + u * (int)blockDim.x + tid;
          const int kq = kq0 + 4 * q;
          if (q < nq && kq >= k0 && kq + 3 < kend) {
            cv[u] = ld_stream4(reinterpret_cast<const int*>(cq + q));
            if (LOADV) {
              const double2 a = ld_stream2(v + kq), b = ld_stream2(v + kq + 2);
              ve[u][0] = a.x; ve[u][1] = a.y; ve[u][2] = b.x; ve[u][3] = b.y;
            }
          } else {
            cv[u] = make_int4(0, 0, 0, 0);
            if (LOADV) ve[u][0] = ve[u][1] = ve[u][2] = ve[u][3] = 0.0;
            if (q < nq) {   // a quad across the chunk's head or tail: entries one by one
              if (kq >= k0) cv[u].x = ld_stream(c + kq);
              if (kq + 1 >= k0 && kq + 1 < kend) cv[u].y = ld_stream(c + kq + 1);
              if (kq + 2 >= k0 && kq + 2 < kend) cv[u].z = ld_stream(c + kq + 2);
              if (kq + 3 < kend) cv[u].w = ld_stream(c + kq + 3);
              if (LOADV) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (kq + e >= k0 && kq + e < kend) ve[u][e] = ld_stream(v + kq + e);
              }
            }
          }
          pv[u] = (lane == 0 && q < nq && kq > 0) ? __ldg(c + kq - 1) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = qb + u * (int)blockDim.x + tid;
          const int kq = kq0 + 4 * q;
          int prev = __shfl_up_sync(0xffffffffu, cv[u].w, 1);
          if (lane == 0) prev = pv[u];
          if (q < nq) {
            const unsigned r4 = *reinterpret_cast<const unsigned*>(&ids.rid[4 * q]);
            const int ce[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
            const bool full = kq >= k0 && kq + 3 < kend;
            int tprev = -1, pc = prev;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = kq + e;
              const int t = (int)((r4 >> (8 * e)) & 0xffu);
              const bool valid = full || (k >= k0 && k < kend);
              // an entry continues its row unless it is the row's first;
              // entries before k0 carry row id 0xff (no row)
              const bool same = e == 0 ? (valid && k > ids.off[t & 0x7f]) : t == tprev;
              const bool inr = (unsigned)ce[e] < (unsigned)ncols;
              mybad |= (valid && same && pc >= ce[e]) ? kBadOrder : 0;
              mybad |= (valid && !inr) ? kBadIndex : 0;
              if (FLAGS) census_flag(flags, (unsigned)ce[e] - (unsigned)t + dbase, valid && inr, tags);
              if (COPY && !full && valid) {
                ocol[k] = ce[e];
                __stcs(oval + k, ve[u][e]);
                if (ROWS) orow[k] = r0 + t;
              }
              tprev = t;
              pc = ce[e];
            }
            if (COPY && full) {
              __stcs(reinterpret_cast<int4*>(ocol + kq), cv[u]);
              __stcs(reinterpret_cast<double2*>(oval + kq), make_double2(ve[u][0], ve[u][1]));
              __stcs(reinterpret_cast<double2*>(oval + kq + 2), make_double2(ve[u][2], ve[u][3]));
              if (ROWS)
                __stcs(reinterpret_cast<int4*>(orow + kq),
                       make_int4(r0 + (int)(r4 & 0xffu), r0 + (int)((r4 >> 8) & 0xffu),
                                 r0 + (int)((r4 >> 16) & 0xffu), r0 + (int)(r4 >> 24)));
            }
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();   // ids.off[0] / ids.off[nr] read above (a tile without entries skips the chunk loop)
  }
  mybad = __reduce_or_sync(0xffffffffu, mybad);
  if (lane == 0 && mybad) atomicOr(bad, mybad);
}

// COO source, canonical ((row, col) strictly increasing, every index in
// range) -> COO / CSR target in one pass (ds_convert_direct): one address
// quad of entries per lane, the previous entry from the lane before (lane 0:
// scalar loads); the CSR offsets are written at row changes (rows_to_offsets'
// rule, clamped so that a non-canonical source stays in bounds -- its target
// is discarded).  Needs 16-B aligned arrays.
template <bool ROWS_OUT, bool OFF_OUT>
__global__ void __launch_bounds__(256)
    coo_direct_kernel(int64_t nnz, int nrows, int ncols, const int* __restrict__ r,
                      const int* __restrict__ c, const double* __restrict__ v,
                      int* __restrict__ orow, int* __restrict__ ocol, double* __restrict__ oval,
                      int* __restrict__ ooff, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nqa = (nnz + 3) >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int mybad = 0;
  for (int64_t qw = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); qw < nqa; qw += stride) {
    const int64_t q = qw + lane;   // the warp's quads are consecutive
    const int64_t kq = 4 * q;
    const bool full = kq + 3 < nnz;
    int4 rv = make_int4(0, 0, 0, 0), cv = make_int4(0, 0, 0, 0);
    double ve[4] = {0.0, 0.0, 0.0, 0.0};
    if (full) {
      rv = ld_stream4(r + kq);
      cv = ld_stream4(c + kq);
      const double2 a = ld_stream2(v + kq), b = ld_stream2(v + kq + 2);
      ve[0] = a.x; ve[1] = a.y; ve[2] = b.x; ve[3] = b.y;
    } else if (kq < nnz) {
      rv.x = ld_stream(r + kq); cv.x = ld_stream(c + kq); ve[0] = ld_stream(v + kq);
      if (kq + 1 < nnz) { rv.y = ld_stream(r + kq + 1); cv.y = ld_stream(c + kq + 1); ve[1] = ld_stream(v + kq + 1); }
      if (kq + 2 < nnz) { rv.z = ld_stream(r + kq + 2); cv.z = ld_stream(c + kq + 2); ve[2] = ld_stream(v + kq + 2); }
    }
    int pr = __shfl_up_sync(0xffffffffu, rv.w, 1), pc = __shfl_up_sync(0xffffffffu, cv.w, 1);
    if (lane == 0 && kq > 0 && kq < nnz) {
      pr = __ldg(r + kq - 1);
      pc = __ldg(c + kq - 1);
    }
    const int re[4] = {rv.x, rv.y, rv.z, rv.w}, ce[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t k = kq + e;
      if (k < nnz) {
        const int rk = re[e], ck = ce[e];
        if (k > 0) {
          if (rk < pr) mybad |= kBadOrder | kBadRowOrder;
          else if (rk == pr && ck <= pc) mybad |= kBadOrder;
        }
        if ((unsigned)rk >= (unsigned)nrows || (unsigned)ck >= (unsigned)ncols) mybad |= kBadIndex;
        if (OFF_OUT) {
          // off[i] = k for the rows i in (r[k-1], r[k]]; the last entry also
          // closes (r[nnz-1], nrows]
          const int lo = k == 0 ? 0 : max(pr + 1, 0), hi = min(rk, nrows);
          for (int i = lo; i <= hi; ++i) ooff[i] = (int)k;
          if (k == nnz - 1)
            for (int i = max(rk + 1, 0); i <= nrows; ++i) ooff[i] = (int)nnz;
        }
        if (!full) {
          ocol[k] = ck;
          __stcs(oval + k, ve[e]);
          if (ROWS_OUT) orow[k] = rk;
        }
        pr = rk;
        pc = ck;
      }
    }
    if (full) {
      __stcs(reinterpret_cast<int4*>(ocol + kq), cv);
      __stcs(reinterpret_cast<double2*>(oval + kq), make_double2(ve[0], ve[1]));
      __stcs(reinterpret_cast<double2*>(oval + kq + 2), make_double2(ve[2], ve[3]));
      if (ROWS_OUT) __stcs(reinterpret_cast<int4*>(orow + kq), rv);
    }
  }
  mybad = __reduce_or_sync(0xffffffffu, mybad);
  if (lane == 0 && mybad) atomicOr(bad, mybad);
}

// canonical CSR -> DIA: the tile's (kRT x nd) slab zeroed in shared memory,
// entries dropped into (row, diag_map[col - row]) slots, the slab written out
// contiguously (values are row-major (nrows, nd))
__global__ void __launch_bounds__(256)
    csr_dia_fill_tiles(int nrows, int nd, const int* __restrict__ off,
                       const int* __restrict__ c, const double* __restrict__ v,
                       const int* __restrict__ map, double* __restrict__ vals) {
  extern __shared__ double slab[];   // kRT * nd
  __shared__ RowIds ids;
  const int ntiles = (nrows + kRT - 1) / kRT;
  const uint64_t pol = policy_evict_first();
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int r0 = tile * kRT;
    const int total = min(kRT, nrows - r0) * nd;
    for (int i = threadIdx.x; i < total; i += blockDim.x) slab[i] = 0.0;
    // (csr_rowid_tile's first barrier orders the zeroing before the drops)
    csr_rowid_tile(nrows, off, r0, ids, [&](int kb, int k0, int kend) {
      int ck[kRtU];
      double vk[kRtU];
#pragma unroll
      for (int u = 0; u < kRtU; ++u) {
        const int k = kb + u * (int)blockDim.x + (int)threadIdx.x;
        ck[u] = k < kend ? ld_hint(c + k, pol) : 0;
        vk[u] = k < kend ? ld_hint(v + k, pol) : 0.0;
      }
      int j[kRtU];
#pragma unroll
      for (int u = 0; u < kRtU; ++u) {
        const int k = kb + u * (int)blockDim.x + (int)threadIdx.x;
        j[u] = k < kend ? __ldg(map + ((int64_t)ck[u] - (r0 + ids.rid[k - k0]) + nrows - 1)) : 0;
      }
#pragma unroll
      for (int u = 0; u < kRtU; ++u) {
        const int k = kb + u * (int)blockDim.x + (int)threadIdx.x;
        if (k < kend) slab[ids.rid[k - k0] * nd + j[u]] = vk[u];
      }
    });
    double* out = vals + (int64_t)r0 * nd;
    for (int i = threadIdx.x; i < total; i += blockDim.x) __stcs(out + i, slab[i]);
    __syncthreads();
  }
}

// row index of every entry (COO target from a canonical CSR source)
__global__ void csr_rows_walk(int nrows, const int* __restrict__ off, int* rows) {
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kCsrWalkRows;
  int ot = walk_offsets(off, nrows, r0);
  for (; r0 < nrows; r0 += nwarps * kCsrWalkRows) {
    const int ot_next = walk_offsets(off, nrows, r0 + nwarps * kCsrWalkRows);
    csr_warp_walk<4>(ot, r0, min(r0 + kCsrWalkRows, nrows), [](int) { return 0; },
                     [&](int kb, int k1, const int (&rr)[4], const int (&)[4]) {
                       const int lane = threadIdx.x & 31;
#pragma unroll
                       for (int u = 0; u < 4; ++u)
                         if (kb + 32 * u + lane < k1) rows[kb + 32 * u + lane] = rr[u];
                     });
    ot = ot_next;
  }
}

// (Round 2: a quad-per-lane variant with the row offsets of a canonical
// source written in the same pass -- so COO -> DIA could use the CSR slab fill
// instead of zero + scatter -- ran 0.76 ms against this kernel's 0.56 at
// 192^3, ~2.7 warp instructions per entry: no net gain.)
__global__ void coo_check_mark(int64_t nnz, int nrows, int ncols, const int* __restrict__ r,
                               const int* __restrict__ c, unsigned char* flags, int* bad) {
  int mybad = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int rk = __ldg(r + k), ck = __ldg(c + k);
    if (k > 0) {
      const int rp = __ldg(r + k - 1), cp = __ldg(c + k - 1);
      if (rk < rp) mybad |= kBadOrder | kBadRowOrder;
      else if (rk == rp && ck <= cp) mybad |= kBadOrder;
    }
    if ((unsigned)rk >= (unsigned)nrows || (unsigned)ck >= (unsigned)ncols) {
      mybad |= kBadIndex;
    } else if (flags) {
      const int64_t d = (int64_t)ck - rk + nrows - 1;
      unsigned short f;
      asm volatile("ld.global.ca.u8 %0, [%1];" : "=h"(f) : "l"(flags + d));
      if (f == 0) flags[d] = 1;
    }
  }
  mybad = __reduce_or_sync(0xffffffffu, mybad);
  if ((threadIdx.x & 31) == 0 && mybad) atomicOr(bad, mybad);
}

static int index_error(int64_t nrows, int64_t ncols) {
  set_error("an entry's row or column lies outside the %lld x %lld shape", (long long)nrows,
            (long long)ncols);
  return DS_ERR_INDEX_OUT_OF_RANGE;
}

struct FlagAt {
  const unsigned char* f;
  __device__ int operator()(int64_t k) const { return f[k]; }
};
__global__ void diag_offsets_kernel(int64_t D, int nrows, const unsigned char* __restrict__ flags,
                                    const int* __restrict__ map, int* offsets) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D;
       d += (int64_t)gridDim.x * blockDim.x)
    if (flags[d]) offsets[map[d]] = (int)(d - (nrows - 1));
}
__global__ void zero_f64(int64_t n, double* p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}
// CHECK (the speculative COO -> DIA, ds_convert_begin_coo_dia_spec): the
// scatter also checks the canonical order against the previous entry, the
// index range and that the entry's diagonal is in `map` (the exclusive scan
// of the sampled presence: d present iff map[d+1] > map[d]), setting
// kBadOrder / kBadIndex / kBadMiss in *bad instead of storing.  The map
// lookups go through the preloaded shared-memory cache (preload_map_cache).
// (Round 2: 4 warp-uniform groups of 32 entries in flight per thread with the
// previous entry from a shuffle ran 192^3 COO->DIA 1.62 -> 2.19 ms.)
template <bool CHECK>
__global__ void dia_scatter(int64_t nnz, int nrows, int64_t nd, const int* __restrict__ r,
                            const int* __restrict__ c, const double* __restrict__ v,
                            const int* __restrict__ map, const int* __restrict__ dia_off,
                            double* vals, int ncols = 0, int* bad = nullptr) {
  __shared__ unsigned long long mcache[1 << kFlagTagBits];
  preload_map_cache(mcache, dia_off, (int)nd, nrows);
  const unsigned D = (unsigned)nrows + (unsigned)ncols - 1u;
  int mybad = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int rk = __ldg(r + k), ck = __ldg(c + k);
    if (CHECK) {
      if (k > 0) {
        const int rp = __ldg(r + k - 1), cp = __ldg(c + k - 1);
        if (rk < rp || (rk == rp && ck <= cp)) {
          mybad |= kBadOrder;
          continue;   // not stored: a duplicate's slot stays single-writer
        }
      }
      if ((unsigned)rk >= (unsigned)nrows || (unsigned)ck >= (unsigned)ncols) {
        mybad |= kBadIndex;
        continue;
      }
    }
    const unsigned d = (unsigned)ck - (unsigned)rk + (unsigned)(nrows - 1);
    const unsigned h = (d * 0x9E3779B1u) >> (32 - kFlagTagBits);
    const unsigned long long m = mcache[h];
    int j;
    if ((unsigned)m == d) {
      j = (int)(m >> 32);
    } else {
      j = __ldg(map + d);
      if (CHECK) {
        const int jn = d + 1 < D ? __ldg(map + d + 1) : (int)nd;
        if (jn == j) j = -1;
      }
    }
    if (CHECK && j < 0) {
      mybad |= kBadMiss;
      continue;
    }
    vals[(int64_t)rk * nd + j] = __ldg(v + k);
  }
  if (CHECK) {
    mybad = __reduce_or_sync(0xffffffffu, mybad);
    if ((threadIdx.x & 31) == 0 && mybad) atomicOr(bad, mybad);
  }
}

// the sampled census of a COO source: block b marks the diagonals of the
// entries in chunk b * step (the last block: the last chunk)
__global__ void coo_census_sample(int64_t nnz, int nrows, int ncols, int64_t chunk, int64_t step,
                                  const int* __restrict__ r, const int* __restrict__ c,
                                  unsigned char* flags) {
  const int64_t nchunks = (nnz + chunk - 1) / chunk;
  const int64_t ci = blockIdx.x + 1 == gridDim.x ? nchunks - 1 : (int64_t)blockIdx.x * step;
  const int64_t k1 = min64((ci + 1) * chunk, nnz);
  for (int64_t k = ci * chunk + threadIdx.x; k < k1; k += blockDim.x) {
    const int rk = __ldg(r + k), ck = __ldg(c + k);
    if ((unsigned)rk < (unsigned)nrows && (unsigned)ck < (unsigned)ncols) {
      const unsigned d = (unsigned)ck - (unsigned)rk + (unsigned)(nrows - 1);
      unsigned short f;
      asm volatile("ld.global.ca.u8 %0, [%1];" : "=h"(f) : "l"(flags + d));
      if (f == 0) flags[d] = 1;
    }
  }
}

static unsigned grid1d(int64_t n) {
  int64_t g = ceil_div(n, 256);
  const int64_t cap = (int64_t)sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

static int bits_for(unsigned long long maxkey) {
  int b = 0;
  while (b < 64 && (maxkey >> b) != 0ull) ++b;
  return b < 1 ? 1 : b;
}

static int tile_plan(int64_t nrows, const int* off, int lng, int target, int* tiles,
                     int64_t* ntiles, cudaStream_t st);

// canonicalise raw (rows, cols, vals) into job->{r,c,v}.  Owned rows hang on
// the job from the start, so every error return frees them with it.
// row_off: the CSR source's offsets (rows then known to be sorted), or null.
static int canonicalize(ds_convert_job* job, int64_t nnz, const int* rows, const int* cols,
                        const double* vals, bool rows_owned, const int* row_off = nullptr) {
  cudaStream_t st = job->st;
  if (rows_owned) {
    job->r = const_cast<int*>(rows);
    job->own_r = true;
  }
  if (nnz == 0) {
    job->nnz = 0;
    return DS_OK;
  }
  // one pass: the order check ((row, col) strictly ascending), the index range
  // and, for a DIA target, the diagonal census -- the set of diagonals does not
  // depend on the order or on duplicates (their sums are kept even when zero)
  const bool dia = job->target == DS_FMT_DIA;
  const int64_t flag_bytes = dia ? (job->nrows + job->ncols - 1 + 3) & ~int64_t(3) : 0;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->scratch), flag_bytes + 4, st));
  DS_CUDA(cudaMemsetAsync(job->scratch, 0, flag_bytes + 4, st));
  int* bad_d = reinterpret_cast<int*>(job->scratch + flag_bytes);
  coo_check_mark<<<grid1d(nnz), 256, 0, st>>>(nnz, (int)job->nrows, (int)job->ncols, rows, cols,
                                               dia ? job->scratch : nullptr, bad_d);
  DS_LAUNCH_CHECK("coo_check_mark");
  int bad = 1;
  DS_CUDA(cudaMemcpyAsync(&bad, bad_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaStreamSynchronize(st));
  if (bad & kBadIndex) return index_error(job->nrows, job->ncols);
  if (dia) {
    job->flags = job->scratch;
  } else {
    DS_CUDA(cudaFreeAsync(job->scratch, st));
  }
  job->scratch = nullptr;
  int rc = DS_OK;
  if (bad == 0) {  // already canonical: borrow (copied into the target at finish)
    job->nnz = nnz;
    job->r = const_cast<int*>(rows);
    job->own_r = rows_owned;
    job->c = const_cast<int*>(cols);
    job->v = const_cast<double*>(vals);
    return DS_OK;
  }
  // the stable (row, col) sort (np.lexsort((cols, rows)) is stable,
  // datamove.py:212): rows already non-decreasing -> a sort inside each row
  // (ds_sort.cu segmented_sort_rows); otherwise the onesweep LSD radix sort,
  // which builds the keys from the index arrays in its first pass
  unsigned long long* keys_s = nullptr;
  int *perm = nullptr, *pos = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys_s), nnz * 8, st));
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&perm), nnz * 4, st));
  rc = DS_ERR_NOT_SUPPORTED;
  static int no_seg = -1;
  if (no_seg < 0) no_seg = getenv("DS_SORT_NO_SEGMENTED") ? 1 : 0;
  if (!(bad & kBadRowOrder) && !no_seg) {
    int *off = nullptr, *tiles = nullptr;
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tiles), (job->nrows + 1) * 4, st));
    if (!row_off) {
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&off), (job->nrows + 1) * 4, st));
      rows_to_offsets<<<grid1d(nnz + 1 > job->nrows + 1 ? nnz + 1 : job->nrows + 1), 256, 0, st>>>(
          nnz, (int)job->nrows, rows, off);
      row_off = off;
    }
    int64_t nt = 0;
    rc = tile_plan(job->nrows, row_off, 128, 128, tiles, &nt, st);
    if (!rc)
      rc = segmented_sort_rows(row_off, rows, cols, (unsigned long long)job->ncols, tiles, nt,
                               keys_s, perm, st);
    cudaFreeAsync(tiles, st);
    if (off) cudaFreeAsync(off, st);
    if (rc && rc != DS_ERR_NOT_SUPPORTED) {
      cudaFreeAsync(keys_s, st);
      cudaFreeAsync(perm, st);
      return rc;
    }
  }
  if (rc == DS_ERR_NOT_SUPPORTED) {
    const unsigned long long maxkey = (unsigned long long)(job->nrows > 0 ? job->nrows : 1) *
                                          (unsigned long long)(job->ncols > 0 ? job->ncols : 1) -
                                      1ull;
    rc = radix_sort_pairs(nullptr, rows, cols, (unsigned long long)job->ncols, nnz, maxkey,
                          keys_s, perm, st);
  }
  if (rc) {
    cudaFreeAsync(keys_s, st);
    cudaFreeAsync(perm, st);
    return rc;
  }
  if (rows_owned) {
    job->r = nullptr;
    job->own_r = false;
    DS_CUDA(cudaFreeAsync(const_cast<int*>(rows), st));
  }
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pos), nnz * 4, st));
  int64_t nc = 0;
  rc = exclusive_scan(nnz, RunHead{keys_s}, pos, &nc, st);
  if (rc) return rc;
  job->nnz = nc;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->r), nc * 4, st));
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->c), nc * 4, st));
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->v), nc * 8, st));
  job->own_r = job->own_c = job->own_v = true;
  reduce_runs<<<grid1d(nnz), 256, 0, st>>>(nnz, job->ncols, keys_s, perm, pos, vals, job->r,
                                           job->c, job->v);
  DS_LAUNCH_CHECK("reduce_runs");
  DS_CUDA(cudaFreeAsync(keys_s, st));
  DS_CUDA(cudaFreeAsync(perm, st));
  DS_CUDA(cudaFreeAsync(pos, st));
  return DS_OK;
}

static void free_job(ds_convert_job* job) {
  if (!job) return;
  cudaStream_t st = job->st;
  if (job->own_r && job->r) cudaFreeAsync(job->r, st);
  if (job->own_c && job->c) cudaFreeAsync(job->c, st);
  if (job->own_v && job->v) cudaFreeAsync(job->v, st);
  if (job->diag_map) cudaFreeAsync(job->diag_map, st);
  if (job->dia_off) cudaFreeAsync(job->dia_off, st);
  if (job->dsrc_start) cudaFreeAsync(job->dsrc_start, st);
  if (job->flags) cudaFreeAsync(job->flags, st);
  if (job->dia_jsrc) cudaFreeAsync(job->dia_jsrc, st);
  if (job->scratch) cudaFreeAsync(job->scratch, st);
  if (job->gtmp) cudaFreeAsync(job->gtmp, st);
  delete job;
}

// size the target; DIA: presence flags -> ndiags -> fill check before alloc
// size_target for a speculative DIA target whose sampled set is small: the
// offsets straight from the flags (no D-long scan / diag_map; the slot fill
// then searches the offsets).  *small = false (flags kept) when the set has
// more than kSmallDiags diagonals: the caller runs size_target.
static int size_target_small(ds_convert_job* job, int64_t fill_limit, int64_t* out_ndiags,
                             bool* small) {
  cudaStream_t st = job->st;
  *small = false;
  *out_ndiags = 0;
  const int64_t D = job->nrows + job->ncols - 1;
  if (D <= 0 || job->nnz <= 0 || !job->flags) return DS_OK;
  int* tmp = nullptr;   // list[kSmallDiags] | count; on the job until freed (free_job on errors)
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), (kSmallDiags + 1) * sizeof(int), st));
  job->scratch = reinterpret_cast<unsigned char*>(tmp);
  DS_CUDA(cudaMemsetAsync(tmp + kSmallDiags, 0, sizeof(int), st));
  flags_collect<<<grid1d(ceil_div(D, 16)), 256, 0, st>>>(D, job->flags, tmp, tmp + kSmallDiags);
  DS_LAUNCH_CHECK("flags_collect");
  int n = 0;
  DS_CUDA(cudaMemcpyAsync(&n, tmp + kSmallDiags, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaStreamSynchronize(st));
  if (n < 1 || n > kSmallDiags) {
    job->scratch = nullptr;
    DS_CUDA(cudaFreeAsync(tmp, st));
    return DS_OK;
  }
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->dia_off), n * sizeof(int), st));
  small_diags_sort<<<1, 32, 0, st>>>((int)job->nrows, tmp, tmp + kSmallDiags, job->dia_off);
  DS_LAUNCH_CHECK("small_diags_sort");
  job->scratch = nullptr;
  DS_CUDA(cudaFreeAsync(tmp, st));
  DS_CUDA(cudaFreeAsync(job->flags, st));
  job->flags = nullptr;
  *small = true;
  job->ndiags = n;
  *out_ndiags = n;
  const __int128 slots = (__int128)n * (__int128)job->nrows;
  if (slots > (__int128)fill_limit) {
    set_error("%lld diagonals x %lld rows = %lld value slots exceed the fill limit of %lld",
              (long long)n, (long long)job->nrows, (long long)(n * job->nrows),
              (long long)fill_limit);
    return DS_ERR_DIA_FILL_OVERFLOW;
  }
  return DS_OK;
}

static int size_target(ds_convert_job* job, int64_t fill_limit, int64_t* out_nnz,
                       int64_t* out_ndiags) {
  cudaStream_t st = job->st;
  *out_nnz = job->nnz;
  *out_ndiags = 0;
  if (job->target != DS_FMT_DIA) return DS_OK;
  const int64_t D = job->nrows + job->ncols - 1;
  int64_t nd = 0;
  if (D > 0 && job->nnz > 0) {
    unsigned char* flags = job->flags;   // marked by the order-check pass
    job->flags = nullptr;
    if (!flags) {
      set_error("conversion job without a diagonal census");
      return DS_ERR_CUDA;
    }
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->diag_map), D * sizeof(int), st));
    int rc = exclusive_scan(D, FlagAt{flags}, job->diag_map, &nd, st);
    if (rc) return rc;
    if (nd > 0) {
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->dia_off), nd * sizeof(int), st));
      diag_offsets_kernel<<<grid1d(D), 256, 0, st>>>(D, (int)job->nrows, flags, job->diag_map,
                                                      job->dia_off);
      DS_LAUNCH_CHECK("diag_offsets_kernel");
    }
    DS_CUDA(cudaFreeAsync(flags, st));
  }
  job->ndiags = nd;
  *out_ndiags = nd;
  const __int128 slots = (__int128)nd * (__int128)job->nrows;
  if (slots > (__int128)fill_limit) {
    set_error("%lld diagonals x %lld rows = %lld value slots exceed the fill limit of %lld",
              (long long)nd, (long long)job->nrows, (long long)(nd * job->nrows),
              (long long)fill_limit);
    return DS_ERR_DIA_FILL_OVERFLOW;
  }
  return DS_OK;
}

}  // namespace ds

using namespace ds;

// ---------------------------------------------------------------- CSR bins --
__device__ __forceinline__ int csr_bin_of(int len) {
  if (len == 0) return 0;
  if (len <= 9) return 1;
  if (len <= 17) return 2;
  if (len <= 25) return 3;
  if (len <= 33) return 4;
  if (len <= 129) return 5;
  if (len <= kCsrWarpRow) return 6;
  return 7;
}
struct IsBin {
  const int* off;
  int b;
  __device__ int operator()(int64_t r) const { return csr_bin_of(off[r + 1] - off[r]) == b; }
};
__global__ void bin_scatter(int nrows, const int* __restrict__ off, int b, const int* __restrict__ pos,
                            int64_t base, int* perm) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x)
    if (csr_bin_of(off[r + 1] - off[r]) == b) perm[base + pos[r]] = r;
}

// ---------------------------------------------------------------- CSR tiles --
namespace ds {
// A tile starts at row 0, at every row longer than `lng` entries, right after
// one, and where off[r] crosses a multiple of `target`: a tile of rows of at
// most `lng` entries then holds fewer than target + lng entries.
__device__ __forceinline__ int tile_head(int r, const int* __restrict__ off, int lng, int target) {
  if (r == 0) return 1;
  const int a = off[r - 1], b = off[r], c = off[r + 1];
  return c - b > lng || b - a > lng || (b / target != a / target);
}
struct TileHead {
  const int* off;
  int lng, target;
  __device__ int operator()(int64_t r) const { return tile_head((int)r, off, lng, target); }
};
__global__ void tile_scatter(int nrows, const int* __restrict__ off, int lng, int target,
                             const int* __restrict__ pos, int* tiles) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x)
    if (tile_head(r, off, lng, target)) tiles[pos[r]] = r;
}
__global__ void tile_close(int* tiles, int64_t ntiles, int nrows) { tiles[ntiles] = nrows; }

static int tile_plan(int64_t nrows, const int* off, int lng, int target, int* tiles,
                     int64_t* ntiles, cudaStream_t st) {
  *ntiles = 0;
  if (nrows <= 0) return DS_OK;
  int* pos = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pos), nrows * sizeof(int), st));
  int64_t nt = 0;
  int rc = exclusive_scan(nrows, TileHead{off, lng, target}, pos, &nt, st);
  if (rc) {
    cudaFreeAsync(pos, st);
    return rc;
  }
  tile_scatter<<<grid1d(nrows), 256, 0, st>>>((int)nrows, off, lng, target, pos, tiles);
  tile_close<<<1, 1, 0, st>>>(tiles, nt, (int)nrows);
  DS_LAUNCH_CHECK("tile_scatter");
  DS_CUDA(cudaFreeAsync(pos, st));
  *ntiles = nt;
  return DS_OK;
}
}  // namespace ds

namespace ds {
// ---- the SpMV tile plan of an irregular CSR (csr_tile_kernel, ds_csr.cu) ----
// Layout (int32 words), see include/dynsparse_b200.h ds_csr_tiles:
//   [0..7] header: total tiles, leaves, long rows, LV, LR, SCR (word offsets), row tiles
//   [8 ..) one int4 per tile {A, B, E0, E1}: a row tile (A >= 0) holds rows
//          [A, B) and entries [E0, E1); a leaf tile (A < 0) holds the B
//          consecutive pairwise leaves -A-1 .. -A-2+B of one long row, entries [E0, E1)
//   LV: (start, len) of every leaf;  LR: (row, first leaf) of every long row
//   SCR: one double per leaf (the leaf sums, written by every SpMV)
// A long row (> 129 entries) is reduced by np.add.reduceat as p[first] +
// pairwise(p[first+1 .. end]); pairwise splits n > 128 addends at
// n/2 - (n/2)%8, so its leaves hold 64..128 addends.  They become leaf tiles
// of <= 4 leaves (<= 512 entries), spread over the whole grid with the row
// tiles; a small kernel then replays the recursion over the leaf sums.
constexpr int kLeavesPerTile = kCsrTileMax / 128;
constexpr int kPlanHeader = 8;

__device__ __forceinline__ int pw_split(int n) {
  const int n2 = n / 2;
  return n2 - n2 % 8;
}
__device__ int pw_count_leaves(int m) {
  int stack[48], sp = 0, cnt = 0;
  stack[sp++] = m;
  while (sp) {
    const int n = stack[--sp];
    if (n <= 128) {
      ++cnt;
      continue;
    }
    const int n2 = pw_split(n);
    stack[sp++] = n - n2;   // right pushed first: the left half is visited first
    stack[sp++] = n2;
  }
  return cnt;
}
struct IsLongRow {
  const int* off;
  __device__ int operator()(int64_t r) const { return off[r + 1] - off[r] > 129 ? 1 : 0; }
};
struct TilesOf {
  const int* a;
  __device__ int operator()(int64_t k) const { return (a[k] + kLeavesPerTile - 1) / kLeavesPerTile; }
};
__global__ void long_rows_scatter(int nrows, const int* __restrict__ off, const int* __restrict__ pos,
                                  int* longs) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x)
    if (off[r + 1] - off[r] > 129) longs[pos[r]] = r;
}
__global__ void long_rows_leaf_counts(int64_t nlong, const int* __restrict__ longs,
                                      const int* __restrict__ off, int* cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlong;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = longs[i];
    cnt[i] = pw_count_leaves(off[r + 1] - off[r] - 1);
  }
}
__global__ void row_tiles_write(int64_t nt, const int* __restrict__ rs, const int* __restrict__ off,
                                int4* plan4) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = rs[t], r1 = rs[t + 1], e0 = off[r0], e1 = off[r1];
    // a long row's own tile stays as an empty placeholder: its leaf tiles carry it
    plan4[t] = (r1 - r0 == 1 && e1 - e0 > 129) ? make_int4(r0, r0, e0, e0)
                                                : make_int4(r0, r1, e0, e1);
  }
}
// one thread per long row: its leaves in recursion order, its leaf tiles
__global__ void long_rows_leaves(int64_t nlong, const int* __restrict__ longs,
                                 const int* __restrict__ off, const int* __restrict__ leaf0,
                                 const int* __restrict__ tile0, int64_t nt, int4* plan4, int* lv,
                                 int* lr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlong;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = longs[i], first = off[r];
    const int L0 = leaf0[i];
    lr[2 * i] = r;
    lr[2 * i + 1] = L0;
    int st_s[48], st_n[48], sp = 0, k = 0, tstart = 0, tlo = 0;
    int64_t tj = nt + tile0[i];
    st_s[sp] = first + 1;
    st_n[sp++] = off[r + 1] - first - 1;
    while (sp) {
      --sp;
      const int a = st_s[sp], n = st_n[sp];
      if (n <= 128) {
        lv[2 * (L0 + k)] = a;
        lv[2 * (L0 + k) + 1] = n;
        if (k % kLeavesPerTile == 0) {
          tstart = a;
          tlo = k;
        }
        ++k;
        const bool last = sp == 0;
        if (k % kLeavesPerTile == 0 || last) {
          plan4[tj++] = make_int4(-(L0 + tlo) - 1, k - tlo, tstart, a + n);
        }
        continue;
      }
      const int n2 = pw_split(n);
      st_s[sp] = a + n2;
      st_n[sp++] = n - n2;
      st_s[sp] = a;
      st_n[sp++] = n2;
    }
  }
}
__global__ void plan_header(int* h, int a, int b, int c, int d, int e, int f, int g) {
  h[0] = a; h[1] = b; h[2] = c; h[3] = d; h[4] = e; h[5] = f; h[6] = g; h[7] = 0;
}
}  // namespace ds

extern "C" int64_t ds_csr_tiles_capacity(int64_t nrows, int64_t nnz) {
  const int64_t leaves = nnz / 64 + 1, longs = nnz / 130 + 1;
  return kPlanHeader + 4 * (nrows + 1 + leaves) + 2 * leaves + 2 * longs + 2 * leaves + 2;
}

extern "C" int ds_csr_tiles(int64_t nrows, const int32_t* row_offsets, int32_t* plan,
                            int64_t capacity, int64_t* ntiles, int64_t* words, void* stream) {
  cudaStream_t st = as_stream(stream);
  *ntiles = 0;
  if (words) *words = 0;
  if (nrows <= 0) return DS_OK;
  int64_t nnz = 0;
  {
    int h = 0;
    DS_CUDA(cudaMemcpyAsync(&h, row_offsets + nrows, sizeof(int), cudaMemcpyDeviceToHost, st));
    DS_CUDA(cudaStreamSynchronize(st));
    nnz = h;
  }
  if (capacity < ds_csr_tiles_capacity(nrows, nnz)) {
    set_error("ds_csr_tiles: capacity %lld < %lld words", (long long)capacity,
              (long long)ds_csr_tiles_capacity(nrows, nnz));
    return DS_ERR_INVALID_ARGUMENT;
  }
  // scratch: row starts of the row tiles, long rows, per-long-row leaf / tile counts and starts
  int* tmp = nullptr;
  const int64_t lcap = nnz / 130 + 1;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), (nrows + 1 + 5 * lcap) * sizeof(int), st));
  int *rs = tmp, *longs = rs + nrows + 1, *cnt = longs + lcap, *leaf0 = cnt + lcap,
      *tile0 = leaf0 + lcap, *pos = tile0 + lcap;
  int64_t nt = 0, nlong = 0, nleaves = 0, nlt = 0;
  int rc = tile_plan(nrows, row_offsets, 129, kCsrTileTarget, rs, &nt, st);
  int* rpos = nullptr;
  if (!rc) {
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rpos), nrows * sizeof(int), st));
    rc = exclusive_scan(nrows, IsLongRow{row_offsets}, rpos, &nlong, st);
  }
  if (!rc && nlong > 0) {
    long_rows_scatter<<<grid1d(nrows), 256, 0, st>>>((int)nrows, row_offsets, rpos, longs);
    long_rows_leaf_counts<<<grid1d(nlong), 256, 0, st>>>(nlong, longs, row_offsets, cnt);
    DS_LAUNCH_CHECK("long_rows_leaf_counts");
    rc = exclusive_scan(nlong, ArrayAt{cnt}, leaf0, &nleaves, st);
    if (!rc) rc = exclusive_scan(nlong, TilesOf{cnt}, tile0, &nlt, st);
  }
  (void)pos;
  if (rpos) cudaFreeAsync(rpos, st);
  if (rc) {
    cudaFreeAsync(tmp, st);
    return rc;
  }
  const int64_t LV = kPlanHeader + 4 * (nt + nlt);
  const int64_t LR = LV + 2 * nleaves;
  const int64_t SCR = (LR + 2 * nlong + 1) & ~int64_t(1);
  const int64_t used = SCR + 2 * nleaves;
  if (used > (int64_t)INT32_MAX) {   // the header holds int32 word offsets
    cudaFreeAsync(tmp, st);
    set_error("ds_csr_tiles: a plan of %lld words exceeds int32 offsets", (long long)used);
    return DS_ERR_NOT_SUPPORTED;
  }
  if (used > capacity) {   // cannot happen with ds_csr_tiles_capacity
    cudaFreeAsync(tmp, st);
    set_error("ds_csr_tiles: plan needs %lld words", (long long)used);
    return DS_ERR_INVALID_ARGUMENT;
  }
  int4* plan4 = reinterpret_cast<int4*>(plan + kPlanHeader);
  if (nt > 0) row_tiles_write<<<grid1d(nt), 256, 0, st>>>(nt, rs, row_offsets, plan4);
  if (nlong > 0)
    long_rows_leaves<<<grid1d(nlong), 128, 0, st>>>(nlong, longs, row_offsets, leaf0, tile0, nt,
                                                    plan4, plan + LV, plan + LR);
  plan_header<<<1, 1, 0, st>>>(plan, (int)(nt + nlt), (int)nleaves, (int)nlong, (int)LV, (int)LR,
                               (int)SCR, (int)nt);
  DS_LAUNCH_CHECK("ds_csr_tiles");
  DS_CUDA(cudaFreeAsync(tmp, st));
  DS_CUDA(cudaStreamSynchronize(st));
  *ntiles = nt + nlt;
  if (words) *words = used;
  return DS_OK;
}

extern "C" int ds_csr_bins(int64_t nrows, const int32_t* row_offsets, int32_t* perm, int64_t* bins,
                           void* stream) {
  cudaStream_t st = as_stream(stream);
  for (int b = 0; b <= kCsrBinCount; ++b) bins[b] = 0;
  if (nrows <= 0) return DS_OK;
  int* pos = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pos), nrows * sizeof(int), st));
  int64_t base = 0;
  for (int b = 0; b < kCsrBinCount; ++b) {   // stable: rows ascending inside every bin
    int64_t cnt = 0;
    int rc = exclusive_scan(nrows, IsBin{row_offsets, b}, pos, &cnt, st);
    if (rc) return rc;
    bins[b] = base;
    if (cnt) {
      bin_scatter<<<grid1d(nrows), 256, 0, st>>>((int)nrows, row_offsets, b, pos, base, perm);
      DS_LAUNCH_CHECK("bin_scatter");
    }
    base += cnt;
  }
  bins[kCsrBinCount] = base;
  DS_CUDA(cudaFreeAsync(pos, st));
  DS_CUDA(cudaStreamSynchronize(st));
  return DS_OK;
}

// ------------------------------------------------------- stencil generator --
// On-device generate_problem for one partition (stencil.py:143-253): 27-point
// couplings, x-fastest local numbering, rank = cx + px*(cy + py*cz), ghosts
// numbered by sorted (owner*n + owner_local) keys, columns ascending per row,
// values 26 / -1, b = 27 - row_len (exact row sums).  Integer-exact, so the
// arrays are bitwise those of the host generator (tested).
struct StencilGrid {
  int nx, ny, nz, px, py, pz, rank;
};

__device__ __forceinline__ bool stencil_nbr(const StencilGrid& g, int64_t i, int t, int64_t n,
                                            int& owner, int& oloc) {
  const int dz = t / 9 - 1, dy = (t / 3) % 3 - 1, dx = t % 3 - 1;
  const int cx = g.rank % g.px, cy = (g.rank / g.px) % g.py, cz = g.rank / (g.px * g.py);
  const int lx = (int)(i % g.nx), ly = (int)((i / g.nx) % g.ny), lz = (int)(i / ((int64_t)g.nx * g.ny));
  const int tx = lx + cx * g.nx + dx, ty = ly + cy * g.ny + dy, tz = lz + cz * g.nz + dz;
  if (tx < 0 || ty < 0 || tz < 0 || tx >= g.nx * g.px || ty >= g.ny * g.py || tz >= g.nz * g.pz)
    return false;
  const int ox = tx / g.nx, oy = ty / g.ny, oz = tz / g.nz;
  owner = ox + g.px * (oy + g.py * oz);
  oloc = (tx - ox * g.nx) + g.nx * ((ty - oy * g.ny) + g.ny * (tz - oz * g.nz));
  (void)n;
  return true;
}

struct StencilCount {
  StencilGrid g;
  int64_t n;
  int ghosts_only;
  __device__ int operator()(int64_t i) const {
    int c = 0, ow, ol;
    for (int t = 0; t < 27; ++t)
      if (stencil_nbr(g, i, t, n, ow, ol) && (!ghosts_only || ow != g.rank)) ++c;
    return c;
  }
};

__global__ void stencil_ghost_keys(StencilGrid g, int64_t n, const int* __restrict__ gpos,
                                   unsigned long long* keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int o = gpos[i], ow, ol;
    for (int t = 0; t < 27; ++t)
      if (stencil_nbr(g, i, t, n, ow, ol) && ow != g.rank)
        keys[o++] = (unsigned long long)ow * (unsigned long long)n + (unsigned long long)ol;
  }
}

struct KeyHead {
  const unsigned long long* k;
  __device__ int operator()(int64_t i) const { return (i == 0 || k[i] != k[i - 1]) ? 1 : 0; }
};
__global__ void compact_keys(int64_t m, const unsigned long long* __restrict__ k,
                             const int* __restrict__ pos, unsigned long long* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    if (i == 0 || k[i] != k[i - 1]) out[pos[i]] = k[i];
}

__global__ void stencil_fill(StencilGrid g, int64_t n, const int* __restrict__ off,
                             const unsigned long long* __restrict__ ukeys, int64_t G, int* cols,
                             double* vals, double* b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[27];
    int cnt = 0, ow, ol;
    for (int t = 0; t < 27; ++t) {
      if (!stencil_nbr(g, i, t, n, ow, ol)) continue;
      int64_t col;
      if (ow == g.rank) {
        col = ol;
      } else {  // n + rank of the key among the sorted unique ghost keys
        const unsigned long long key = (unsigned long long)ow * (unsigned long long)n + ol;
        int64_t lo = 0, hi = G;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (ukeys[mid] < key) lo = mid + 1; else hi = mid;
        }
        col = n + lo;
      }
      int j = cnt++;  // insertion sort (<= 27 entries)
      while (j > 0 && c[j - 1] > col) {
        c[j] = c[j - 1];
        --j;
      }
      c[j] = col;
    }
    const int o = off[i];
    for (int j = 0; j < cnt; ++j) {
      cols[o + j] = (int)c[j];
      vals[o + j] = (c[j] == i) ? 26.0 : -1.0;
    }
    b[i] = (double)(27 - cnt);
  }
}

struct ds_stencil_job {
  cudaStream_t st;
  StencilGrid g;
  int64_t n, nnz, G;
  int* offsets;                 // n+1 (owned by the job until finish)
  unsigned long long* ukeys;    // G
};

extern "C" int ds_stencil_begin(int nx, int ny, int nz, int px, int py, int pz, int rank,
                                void* stream, ds_stencil_job** job, int64_t* nnz,
                                int64_t* nghosts) {
  *job = nullptr;
  cudaStream_t st = as_stream(stream);
  const int64_t n = (int64_t)nx * ny * nz;
  if (n <= 0 || n * 27 >= (1ll << 31) || (int64_t)px * py * pz * n >= (1ll << 62)) {
    set_error("grid too large for int32 device indices");
    return DS_ERR_NOT_SUPPORTED;
  }
  StencilGrid g{nx, ny, nz, px, py, pz, rank};
  ds_stencil_job* j = new ds_stencil_job{st, g, n, 0, 0, nullptr, nullptr};
  int* gpos = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->offsets), (n + 1) * sizeof(int), st));
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&gpos), n * sizeof(int), st));
  int64_t total = 0, gtotal = 0;
  int rc = exclusive_scan(n, StencilCount{g, n, 0}, j->offsets, &total, st);
  if (!rc) rc = exclusive_scan(n, StencilCount{g, n, 1}, gpos, &gtotal, st);
  if (rc) return rc;
  const int tot32 = (int)total;
  DS_CUDA(cudaMemcpyAsync(j->offsets + n, &tot32, sizeof(int), cudaMemcpyHostToDevice, st));
  int64_t G = 0;
  if (gtotal > 0) {
    unsigned long long *keys = nullptr, *sorted = nullptr;
    int* pos = nullptr;
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys), gtotal * 8, st));
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sorted), gtotal * 8, st));
    int* perm_unused = nullptr;
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&perm_unused), gtotal * 4, st));
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pos), gtotal * 4, st));
    stencil_ghost_keys<<<grid1d(n), 256, 0, st>>>(g, n, gpos, keys);
    DS_LAUNCH_CHECK("stencil_ghost_keys");
    // ghost keys = owner * n + owner-local < P * n
    rc = radix_sort_pairs(keys, nullptr, nullptr, 0, gtotal,
                          (unsigned long long)(px * py * pz) * (unsigned long long)n - 1ull, sorted,
                          perm_unused, st);
    if (rc) return rc;
    DS_CUDA(cudaFreeAsync(perm_unused, st));
    rc = exclusive_scan(gtotal, KeyHead{sorted}, pos, &G, st);
    if (rc) return rc;
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->ukeys), (G > 0 ? G : 1) * 8, st));
    compact_keys<<<grid1d(gtotal), 256, 0, st>>>(gtotal, sorted, pos, j->ukeys);
    DS_LAUNCH_CHECK("compact_keys");
    DS_CUDA(cudaFreeAsync(keys, st));
    DS_CUDA(cudaFreeAsync(sorted, st));
    DS_CUDA(cudaFreeAsync(pos, st));
  }
  DS_CUDA(cudaFreeAsync(gpos, st));
  j->nnz = total;
  j->G = G;
  *nnz = total;
  *nghosts = G;
  *job = j;
  return DS_OK;
}

extern "C" int ds_stencil_finish(ds_stencil_job* j, int32_t* row_offsets, int32_t* cols,
                                 double* vals, double* b, int64_t* ghost_keys) {
  cudaStream_t st = j->st;
  stencil_fill<<<grid1d(j->n), 256, 0, st>>>(j->g, j->n, j->offsets, j->ukeys, j->G, cols, vals,
                                              b);
  DS_LAUNCH_CHECK("stencil_fill");
  DS_CUDA(cudaMemcpyAsync(row_offsets, j->offsets, (j->n + 1) * sizeof(int),
                          cudaMemcpyDeviceToDevice, st));
  if (j->G > 0 && ghost_keys)
    DS_CUDA(cudaMemcpyAsync(ghost_keys, j->ukeys, j->G * 8, cudaMemcpyDeviceToDevice, st));
  DS_CUDA(cudaFreeAsync(j->offsets, st));
  if (j->ukeys) DS_CUDA(cudaFreeAsync(j->ukeys, st));
  delete j;
  return DS_OK;
}

// -------------------------------------------------------- local/remote split --
// split_local_remote (stencil.py:256-277): columns < n_owned form the local
// (square) part, the rest the remote part re-based by -n_owned.  Columns are
// sorted per row, so each row's local entries are a prefix.
struct LocalCount {
  const int* off;
  const int* cols;
  int n_owned;
  __device__ int operator()(int64_t i) const {
    int c = 0;
    for (int k = off[i]; k < off[i + 1] && cols[k] < n_owned; ++k) ++c;
    return c;
  }
};

__global__ void split_fill(int nrows, int n_owned, const int* __restrict__ off,
                           const int* __restrict__ cols, const double* __restrict__ vals,
                           const int* __restrict__ loc_off, int* loc_cols, double* loc_vals,
                           int* rem_off, int* rem_cols, double* rem_vals, int nnz_loc,
                           int nnz_total) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nrows; i += gridDim.x * blockDim.x) {
    const int lo = (i < nrows) ? loc_off[i] : nnz_loc;
    const int ro = ((i < nrows) ? off[i] : nnz_total) - lo;
    rem_off[i] = ro;
    if (i == nrows) break;
    int k = off[i], o = lo;
    const int e = off[i + 1];
    for (; k < e && cols[k] < n_owned; ++k, ++o) {
      loc_cols[o] = cols[k];
      loc_vals[o] = vals[k];
    }
    for (int r = ro; k < e; ++k, ++r) {
      rem_cols[r] = cols[k] - n_owned;
      rem_vals[r] = vals[k];
    }
  }
}

extern "C" int ds_csr_split_count(int64_t nrows, int64_t n_owned, const int32_t* row_offsets,
                                  const int32_t* cols, int32_t* loc_off, int64_t* nnz_local,
                                  void* stream) {
  cudaStream_t st = as_stream(stream);
  int64_t tot = 0;
  int rc = exclusive_scan(nrows, LocalCount{row_offsets, cols, (int)n_owned}, loc_off, &tot, st);
  if (rc) return rc;
  const int t32 = (int)tot;
  DS_CUDA(cudaMemcpyAsync(loc_off + nrows, &t32, sizeof(int), cudaMemcpyHostToDevice, st));
  *nnz_local = tot;
  return DS_OK;
}

extern "C" int ds_csr_split_fill(int64_t nrows, int64_t n_owned, int64_t nnz,
                                 const int32_t* row_offsets, const int32_t* cols,
                                 const double* vals, const int32_t* loc_off, int64_t nnz_local,
                                 int32_t* loc_cols, double* loc_vals, int32_t* rem_off,
                                 int32_t* rem_cols, double* rem_vals, void* stream) {
  cudaStream_t st = as_stream(stream);
  split_fill<<<grid1d(nrows + 1), 256, 0, st>>>((int)nrows, (int)n_owned, row_offsets, cols, vals,
                                                loc_off, loc_cols, loc_vals, rem_off, rem_cols,
                                                rem_vals, (int)nnz_local, (int)nnz);
  DS_LAUNCH_CHECK("split_fill");
  return DS_OK;
}

static ds_convert_job* new_job(int64_t nrows, int64_t ncols, int target, void* stream) {
  ds_convert_job* job = new ds_convert_job;
  job->st = as_stream(stream);
  job->nrows = nrows;
  job->ncols = ncols;
  job->target = target;
  return job;
}

static bool dims_ok(int64_t nrows, int64_t ncols, int64_t nnz) {
  if (nrows < 0 || ncols < 0 || nrows >= (1ll << 31) || ncols >= (1ll << 31) ||
      nnz >= (1ll << 31)) {
    set_error("dimensions must be < 2^31");
    return false;
  }
  return true;
}

// Every begin_* wrapper owns the job: the *_impl bodies never free it, so
// every failure after new_job -- a DS_CUDA early return included -- lands in
// one free_job (the pool allocations hung on the job go back with it).
static int begin_coo_impl(ds_convert_job* j, int64_t nnz, const int32_t* rows, const int32_t* cols,
                          const double* values, int64_t fill_limit, int64_t* out_nnz,
                          int64_t* out_ndiags) {
  int rc = canonicalize(j, nnz, rows, cols, values, false);
  if (rc) return rc;
  return size_target(j, fill_limit, out_nnz, out_ndiags);
}

extern "C" int ds_convert_begin_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                                    const int32_t* cols, const double* values, int target,
                                    int64_t fill_limit, void* stream, ds_convert_job** job,
                                    int64_t* out_nnz, int64_t* out_ndiags) {
  *job = nullptr;
  if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nnz, nrows);   // datamove.py:55-57
  if (!dims_ok(nrows, ncols, nnz)) return DS_ERR_NOT_SUPPORTED;
  ds_convert_job* j = new_job(nrows, ncols, target, stream);
  const int rc = begin_coo_impl(j, nnz, rows, cols, values, fill_limit, out_nnz, out_ndiags);
  if (rc) {
    free_job(j);
    return rc;
  }
  *job = j;
  return DS_OK;
}

static unsigned rt_grid(int64_t nrows, int per_sm) {   // kRT-row tiles, persistent
  return (unsigned)std::max<int64_t>(1, min64(ceil_div(nrows, kRT), (int64_t)sm_count() * per_sm));
}

static unsigned csr_walk_grid(int64_t nrows) {   // 8 warps per block
  return (unsigned)std::max<int64_t>(
      1, min64(ceil_div(nrows, kCsrWalkRows * 8), (int64_t)sm_count() * 8));
}

// the slot-parallel fill (dia_fill_rows) for nd <= 32; DS_DIA_FILL_ROWS=0
// keeps the shared-memory slab walk (dia_fill_csr) for A/B runs
static bool use_fill_rows(int64_t nd) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("DS_DIA_FILL_ROWS");
    on = e ? atoi(e) != 0 : 1;
  }
  return on && nd >= 1 && nd <= 32;
}

// entries of row r: [off[r], off[r + 1]) of (c, v); bad may be null when !CHECK
template <bool CHECK>
static int launch_fill_rows(int64_t nrows, int64_t ncols, int64_t nd, const int* off,
                            const int* c, const double* v, const int* map, const int* dia_off,
                            double* values, int* bad, cudaStream_t st) {
  const unsigned grid = (unsigned)std::max<int64_t>(   // 8 warps per block, 32 rows per warp
      1, min64(ceil_div(nrows, 32 * 8), (int64_t)sm_count() * 8));
  dia_fill_rows<CHECK><<<grid, 256, 0, st>>>((int)nrows, (int)nd, off, c, v, map, dia_off, values,
                                             (int)ncols, bad);
  DS_LAUNCH_CHECK("dia_fill_rows");
  return DS_OK;
}

static int begin_csr_impl(ds_convert_job* j, int64_t nnz, const int32_t* row_offsets,
                          const int32_t* cols, const double* values, int64_t fill_limit,
                          int64_t* out_nnz, int64_t* out_ndiags) {
  const int64_t nrows = j->nrows, ncols = j->ncols;
  const int target = j->target;
  cudaStream_t st = j->st;
  if (nnz > 0 && nrows > 0) {
    // canonical already (the common case)?  then no COO proxy at all: a DIA
    // target takes its diagonal census in the same pass, a CSR / COO target
    // copies (expands) the source at finish
    const bool dia = target == DS_FMT_DIA;
    const int64_t flag_bytes = dia ? (nrows + ncols - 1 + 3) & ~int64_t(3) : 0;
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->scratch), flag_bytes + 4, st));
    DS_CUDA(cudaMemsetAsync(j->scratch, 0, flag_bytes + 4, st));
    int* bad = reinterpret_cast<int*>(j->scratch + flag_bytes);
    if (dia)
      csr_census_quads<true><<<rt_grid(nrows, 8), 256, 0, st>>>((int)nrows, (int)ncols, nnz,
                                                               row_offsets, cols, j->scratch, bad);
    else
      csr_census_quads<false><<<rt_grid(nrows, 8), 256, 0, st>>>((int)nrows, (int)ncols, nnz,
                                                                row_offsets, cols, nullptr, bad);
    DS_LAUNCH_CHECK("csr_census_quads");
    int bad_h = 1;
    DS_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    DS_CUDA(cudaStreamSynchronize(st));
    if (bad_h & kBadIndex) return index_error(nrows, ncols);
    if (!bad_h) {
      j->nnz = nnz;
      j->csr_off = row_offsets;
      j->c = const_cast<int*>(cols);
      j->v = const_cast<double*>(values);
      if (dia) {   // the census becomes the job's diagonal flags
        j->flags = j->scratch;
        j->scratch = nullptr;
      }
      return size_target(j, fill_limit, out_nnz, out_ndiags);
    }
    DS_CUDA(cudaFreeAsync(j->scratch, st));   // not canonical: the general path
    j->scratch = nullptr;
  }
  int* rows = nullptr;
  if (nnz > 0) {
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rows), nnz * 4, st));
    csr_expand_rows<<<grid1d(nrows * 8), 256, 0, st>>>((int)nrows, row_offsets, rows);
    DS_LAUNCH_CHECK("csr_expand_rows");
  }
  int rc = canonicalize(j, nnz, rows, cols, values, true, row_offsets);
  if (rc) return rc;
  return size_target(j, fill_limit, out_nnz, out_ndiags);
}

extern "C" int ds_convert_begin_csr(int64_t nrows, int64_t ncols, int64_t nnz,
                                    const int32_t* row_offsets, const int32_t* cols,
                                    const double* values, int target, int64_t fill_limit,
                                    void* stream, ds_convert_job** job, int64_t* out_nnz,
                                    int64_t* out_ndiags) {
  *job = nullptr;
  if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nnz, nrows);   // datamove.py:55-57
  if (!dims_ok(nrows, ncols, nnz)) return DS_ERR_NOT_SUPPORTED;
  ds_convert_job* j = new_job(nrows, ncols, target, stream);
  const int rc = begin_csr_impl(j, nnz, row_offsets, cols, values, fill_limit, out_nnz,
                                out_ndiags);
  if (rc) {
    free_job(j);
    return rc;
  }
  *job = j;
  return DS_OK;
}

// ------------------------------------------- speculative CSR -> DIA ------
// The census pass exists only to learn the diagonal set before the slab is
// sized.  Speculation: take the census of a sample of row tiles (every
// ntiles/256-th and the last), size the target by it, and let finish_dia run
// ONE pass that checks the order, the index range and that every entry's
// diagonal is in the sampled set while it fills the slab.  A sampled set is
// a subset of the true one, so "no entry outside it" means they are equal;
// otherwise finish returns DS_ERR_RETRY and the caller runs begin_csr /
// finish_dia (the census path).  A fill-limit overflow of the sample also
// returns DS_ERR_RETRY (the census path raises it with the true count).
extern "C" int ds_convert_begin_csr_dia_spec(int64_t nrows, int64_t ncols, int64_t nnz,
                                             const int32_t* row_offsets, const int32_t* cols,
                                             const double* values, int64_t fill_limit,
                                             void* stream, ds_convert_job** job,
                                             int64_t* out_ndiags) {
  *job = nullptr;
  *out_ndiags = 0;
  if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nnz, nrows);   // datamove.py:55-57
  if (!dims_ok(nrows, ncols, nnz)) return DS_ERR_NOT_SUPPORTED;
  if (nnz <= 0 || nrows <= 0 || (reinterpret_cast<uintptr_t>(values) & 15) ||
      (reinterpret_cast<uintptr_t>(cols) & 15))
    return DS_ERR_RETRY;
  ds_convert_job* j = new_job(nrows, ncols, DS_FMT_DIA, stream);
  cudaStream_t st = j->st;
  const int64_t flag_bytes = (nrows + ncols - 1 + 3) & ~int64_t(3);
  int rc = DS_OK;
  do {
    if (cudaMallocAsync(reinterpret_cast<void**>(&j->flags), flag_bytes + 4, st) != cudaSuccess ||
        cudaMemsetAsync(j->flags, 0, flag_bytes + 4, st) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "speculative census flags");
      break;
    }
    int* bad = reinterpret_cast<int*>(j->flags + flag_bytes);   // ignored: finish re-checks
    const int ntiles = (int)ceil_div(nrows, kRT);
    const int S = std::min(ntiles, 256), step = std::max(1, ntiles / S);
    csr_census_quads<true><<<S, 256, 0, st>>>((int)nrows, (int)ncols, nnz, row_offsets, cols,
                                             j->flags, bad, nullptr, nullptr, nullptr, nullptr, 0,
                                             step);
    csr_census_quads<true><<<1, 256, 0, st>>>((int)nrows, (int)ncols, nnz, row_offsets, cols,
                                             j->flags, bad, nullptr, nullptr, nullptr, nullptr,
                                             ntiles - 1, 1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "csr_census_quads(sample)");
      break;
    }
    j->nnz = nnz;
    j->csr_off = row_offsets;
    j->c = const_cast<int*>(cols);
    j->v = const_cast<double*>(values);
    j->spec = true;
    int64_t nnz_out = 0;
    bool small = false;   // the slot fill's case: no diag_map (finish_dia_impl)
    if (use_fill_rows(kSmallDiags)) rc = size_target_small(j, fill_limit, out_ndiags, &small);
    if (rc == DS_OK && !small) rc = size_target(j, fill_limit, &nnz_out, out_ndiags);
    if (rc == DS_ERR_DIA_FILL_OVERFLOW) rc = DS_ERR_RETRY;
    // the fill keeps a 128-row slab in shared memory
    if (rc == DS_OK && (*out_ndiags < 1 || *out_ndiags * kCsrWalkRows * 8 * 8 > 160 * 1024))
      rc = DS_ERR_RETRY;
  } while (false);
  if (rc) {
    free_job(j);
    *out_ndiags = 0;
    return rc;
  }
  *job = j;
  return DS_OK;
}


// The same speculation for a COO source: the census of 256 evenly spaced
// 4096-entry chunks and the last one; finish_dia clears the slab and runs
// the checked scatter (dia_scatter<true>).
extern "C" int ds_convert_begin_coo_dia_spec(int64_t nrows, int64_t ncols, int64_t nnz,
                                             const int32_t* rows, const int32_t* cols,
                                             const double* values, int64_t fill_limit,
                                             void* stream, ds_convert_job** job,
                                             int64_t* out_ndiags) {
  *job = nullptr;
  *out_ndiags = 0;
  if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nnz, nrows);   // datamove.py:55-57
  if (!dims_ok(nrows, ncols, nnz)) return DS_ERR_NOT_SUPPORTED;
  if (nnz <= 0 || nrows <= 0) return DS_ERR_RETRY;
  ds_convert_job* j = new_job(nrows, ncols, DS_FMT_DIA, stream);
  cudaStream_t st = j->st;
  const int64_t flag_bytes = (nrows + ncols - 1 + 3) & ~int64_t(3);
  int rc = DS_OK;
  do {
    if (cudaMallocAsync(reinterpret_cast<void**>(&j->flags), flag_bytes, st) != cudaSuccess ||
        cudaMemsetAsync(j->flags, 0, flag_bytes, st) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "speculative census flags");
      break;
    }
    const int64_t chunk = 4096, nchunks = ceil_div(nnz, chunk);
    const int64_t S = std::min<int64_t>(nchunks, 256), step = std::max<int64_t>(1, nchunks / S);
    coo_census_sample<<<(unsigned)S + 1, 256, 0, st>>>(nnz, (int)nrows, (int)ncols, chunk, step,
                                                      rows, cols, j->flags);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "coo_census_sample");
      break;
    }
    j->nnz = nnz;
    j->r = const_cast<int*>(rows);
    j->c = const_cast<int*>(cols);
    j->v = const_cast<double*>(values);
    j->spec = true;
    int64_t nnz_out = 0;
    bool small = false;   // the slot fill's case: no diag_map (finish_dia_impl)
    if (use_fill_rows(kSmallDiags) && nnz < INT32_MAX && (reinterpret_cast<uintptr_t>(rows) & 15) == 0)
      rc = size_target_small(j, fill_limit, out_ndiags, &small);
    if (rc == DS_OK && !small) rc = size_target(j, fill_limit, &nnz_out, out_ndiags);
    if (rc == DS_ERR_DIA_FILL_OVERFLOW) rc = DS_ERR_RETRY;
    if (rc == DS_OK && *out_ndiags < 1) rc = DS_ERR_RETRY;
  } while (false);
  if (rc) {
    free_job(j);
    *out_ndiags = 0;
    return rc;
  }
  *job = j;
  return DS_OK;
}

// ---------------------------------------- one-pass canonical conversions --
// A canonical COO / CSR source to a COO / CSR target: the order / range
// check and the target writes in one pass over the source (the begin /
// finish pair reads it twice and copies with cudaMemcpy).  *done = 0 when
// the path does not apply (empty, misaligned arrays) or the source is not
// canonical -- the caller then runs begin / finish; the target arrays may
// have been written either way.
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int ds_convert_direct(int src_format, int target, int64_t nrows, int64_t ncols,
                                 int64_t nnz, const int32_t* src_idx, const int32_t* cols,
                                 const double* values, int32_t* out_idx, int32_t* out_cols,
                                 double* out_values, void* stream, int* done) {
  *done = 0;
  if ((src_format != DS_FMT_COO && src_format != DS_FMT_CSR) ||
      (target != DS_FMT_COO && target != DS_FMT_CSR))
    return DS_ERR_INVALID_ARGUMENT;
  if (!dims_ok(nrows, ncols, nnz)) return DS_ERR_NOT_SUPPORTED;
  if (nnz <= 0 || nrows <= 0) return DS_OK;
  if (!aligned16(cols) || !aligned16(values) || !aligned16(out_cols) || !aligned16(out_values))
    return DS_OK;
  if (src_format == DS_FMT_COO && !aligned16(src_idx)) return DS_OK;
  if (target == DS_FMT_COO && !aligned16(out_idx)) return DS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* bad = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), st));
  DS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const int nr = (int)nrows, nc = (int)ncols;
  if (src_format == DS_FMT_CSR) {
    if (target == DS_FMT_COO)
      csr_census_quads<false, true, true><<<rt_grid(nrows, 4), 256, 0, st>>>(
          nr, nc, nnz, src_idx, cols, nullptr, bad, values, out_idx, out_cols, out_values);
    else
      csr_census_quads<false, true, false><<<rt_grid(nrows, 4), 256, 0, st>>>(
          nr, nc, nnz, src_idx, cols, nullptr, bad, values, nullptr, out_cols, out_values);
    DS_LAUNCH_CHECK("csr_census_quads(copy)");
    if (target == DS_FMT_CSR)
      DS_CUDA(cudaMemcpyAsync(out_idx, src_idx, (nrows + 1) * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, st));
  } else {
    const unsigned g = (unsigned)std::max<int64_t>(
        1, min64(ceil_div(ceil_div(nnz, 4), 256), (int64_t)sm_count() * 4));
    if (target == DS_FMT_COO)
      coo_direct_kernel<true, false><<<g, 256, 0, st>>>(nnz, nr, nc, src_idx, cols, values,
                                                         out_idx, out_cols, out_values, nullptr, bad);
    else
      coo_direct_kernel<false, true><<<g, 256, 0, st>>>(nnz, nr, nc, src_idx, cols, values,
                                                         nullptr, out_cols, out_values, out_idx, bad);
    DS_LAUNCH_CHECK("coo_direct_kernel");
  }
  int bad_h = 1;
  DS_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  DS_CUDA(cudaFreeAsync(bad, st));
  DS_CUDA(cudaStreamSynchronize(st));
  if (bad_h & kBadIndex) return index_error(nrows, ncols);
  *done = bad_h == 0;
  return DS_OK;
}

static unsigned dia_walk_grid(int64_t ngroups) {   // 8 warps (groups) per block
  return (unsigned)std::max<int64_t>(1, min64(ceil_div(ngroups, 8), (int64_t)sm_count() * 8));
}

// entries of a DIA source straight into the target (row_offsets: CSR target)
static int dia_emit_into(ds_convert_job* job, int* row_off, int* rows, int* cols, double* values) {
  const int64_t ngroups = ceil_div(job->nrows, kDiaGroupRows);
  dia_group_emit<<<dia_walk_grid(ngroups), 256, 0, job->st>>>(
      job->nrows, (int)job->ncols, job->dsrc_nd, job->dsrc_off, job->dsrc_vals, ngroups,
      job->dsrc_start, row_off, rows, cols, values);
  DS_LAUNCH_CHECK("dia_group_emit");
  return DS_OK;
}

static int begin_dia_impl(ds_convert_job* j, int32_t ndiags, const int32_t* offsets,
                          const double* values, int64_t fill_limit, int64_t* out_nnz,
                          int64_t* out_ndiags) {
  const int64_t nrows = j->nrows, ncols = j->ncols;
  const int target = j->target;
  cudaStream_t st = j->st;
  int64_t nc = 0;
  if (nrows > 0 && ndiags > 0) {
    const int64_t ngroups = ceil_div(nrows, kDiaGroupRows);
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->gtmp), ngroups * sizeof(int), st));
    DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->dsrc_start), ngroups * sizeof(int), st));
    // slot order is canonical only for strictly ascending offsets; otherwise
    // (unsorted or repeated diagonals) the entries go through the proxy's sort
    // and duplicate sums like any other source (datamove.py:208-235)
    std::vector<int> h_off(ndiags);
    DS_CUDA(cudaMemcpyAsync(h_off.data(), offsets, ndiags * sizeof(int), cudaMemcpyDeviceToHost, st));
    DS_CUDA(cudaStreamSynchronize(st));
    bool ascending = true;
    for (int q = 1; q < ndiags; ++q) ascending = ascending && h_off[q - 1] < h_off[q];
    const bool select = target == DS_FMT_DIA && ascending;   // DIA -> DIA: a column selection
    if (select && ndiags > 32) {   // census of the source diagonals holding an entry
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->scratch), ndiags, st));
      DS_CUDA(cudaMemsetAsync(j->scratch, 0, ndiags, st));
    }
    // rows whose every diagonal lands inside the matrix (the counts' fast path)
    int64_t in_lo = 0, in_hi = 0;
    if ((!select || ndiags <= 32) && (reinterpret_cast<uintptr_t>(values) & 15) == 0) {
      const int64_t omin = *std::min_element(h_off.begin(), h_off.end());
      const int64_t omax = *std::max_element(h_off.begin(), h_off.end());
      in_lo = std::max<int64_t>(0, -omin);
      in_hi = std::min<int64_t>(nrows, ncols - omax);
    }
    // DIA -> DIA with <= 32 diagonals: the census alone, stopping once settled
    const bool settle = select && ndiags <= 32;
    std::vector<unsigned char> h_present(ndiags);
    if (settle) {
      unsigned char* sc = nullptr;   // mask | count, a 128-B line each (freed with the job)
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc), 256, st));
      j->scratch = sc;
      DS_CUDA(cudaMemsetAsync(sc, 0, 256, st));
      DiaSelect sel;
      sel.mask = reinterpret_cast<unsigned*>(sc);
      sel.count = reinterpret_cast<unsigned long long*>(sc + 128);
      sel.full = ndiags == 32 ? ~0u : (1u << ndiags) - 1u;
      // the default limit passes once 10 * nnz >= ndiags * nrows (all present)
      sel.need = (fill_limit == kDefaultFillLimit && ndiags > 10)
                     ? (unsigned long long)ceil_div((int64_t)ndiags * nrows, 10)
                     : 0ull;
      if (in_hi > in_lo)
        dia_group_counts<true, true><<<dia_walk_grid(ngroups), 256, 0, st>>>(
            nrows, (int)ncols, ndiags, offsets, values, ngroups, nullptr, nullptr, in_lo, in_hi,
            sel);
      else
        dia_group_counts<false, true><<<dia_walk_grid(ngroups), 256, 0, st>>>(
            nrows, (int)ncols, ndiags, offsets, values, ngroups, nullptr, nullptr, 0, 0, sel);
      DS_LAUNCH_CHECK("dia_group_counts(select)");
      unsigned long long h[32] = {};
      DS_CUDA(cudaMemcpyAsync(h, sc, 256, cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaStreamSynchronize(st));
      const unsigned m = (unsigned)h[0];
      for (int q = 0; q < ndiags; ++q) h_present[q] = (m >> q) & 1u;
      nc = (int64_t)h[16];   // exact unless the walk stopped early (then >= need)
    } else {
      if (in_hi > in_lo)
        dia_group_counts<true><<<dia_walk_grid(ngroups), 256, 0, st>>>(
            nrows, (int)ncols, ndiags, offsets, values, ngroups, j->gtmp, j->scratch, in_lo, in_hi);
      else
        dia_group_counts<false><<<dia_walk_grid(ngroups), 256, 0, st>>>(
            nrows, (int)ncols, ndiags, offsets, values, ngroups, j->gtmp, j->scratch, 0, 0);
      DS_LAUNCH_CHECK("dia_group_counts");
      int rc = exclusive_scan(ngroups, ArrayAt{j->gtmp}, j->dsrc_start, &nc, st);
      if (rc) return rc;
    }
    DS_CUDA(cudaFreeAsync(j->gtmp, st));
    j->gtmp = nullptr;
    j->dsrc_off = offsets;
    j->dsrc_vals = values;
    j->dsrc_nd = ndiags;
    j->dsrc_in_lo = in_lo;
    j->dsrc_in_hi = in_hi;
    int rc = DS_OK;
    if (select) {
      if (!settle) {
        DS_CUDA(cudaMemcpyAsync(h_present.data(), j->scratch, ndiags, cudaMemcpyDeviceToHost, st));
        DS_CUDA(cudaStreamSynchronize(st));
      }
      if (j->scratch) DS_CUDA(cudaFreeAsync(j->scratch, st));
      j->scratch = nullptr;
      DS_CUDA(cudaFreeAsync(j->dsrc_start, st));
      j->dsrc_start = nullptr;
      std::vector<int> jsrc, off_out;
      for (int q = 0; q < ndiags; ++q)
        if (h_present[q]) {
          jsrc.push_back(q);
          off_out.push_back(h_off[q]);
        }
      const int64_t nd_out = (int64_t)jsrc.size();
      if (nd_out > 0) {
        DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->dia_off), nd_out * 4, st));
        DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&j->dia_jsrc), nd_out * 4, st));
        DS_CUDA(cudaMemcpyAsync(j->dia_off, off_out.data(), nd_out * 4, cudaMemcpyHostToDevice, st));
        DS_CUDA(cudaMemcpyAsync(j->dia_jsrc, jsrc.data(), nd_out * 4, cudaMemcpyHostToDevice, st));
        DS_CUDA(cudaStreamSynchronize(st));   // the host vectors die here
      }
      j->nnz = nc;
      j->ndiags = nd_out;
      *out_nnz = nc;
      *out_ndiags = nd_out;
      if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nc, nrows);
      if ((__int128)nd_out * (__int128)nrows > (__int128)fill_limit) {
        set_error("%lld diagonals x %lld rows = %lld value slots exceed the fill limit of %lld",
                  (long long)nd_out, (long long)nrows, (long long)(nd_out * nrows),
                  (long long)fill_limit);
        return DS_ERR_DIA_FILL_OVERFLOW;
      }
      return DS_OK;
    }
    if (target == DS_FMT_DIA || !ascending) {   // materialise the (slot-order) COO
      int *tr = nullptr, *tc = nullptr;
      double* tv = nullptr;
      if (nc > 0) {   // hung on the job at once: freed with it on any error
        DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tr), nc * 4, st));
        j->r = tr;
        j->own_r = true;
        DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tc), nc * 4, st));
        j->c = tc;
        j->own_c = true;
        DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tv), nc * 8, st));
        j->v = tv;
        j->own_v = true;
        j->nnz = nc;
        rc = dia_emit_into(j, nullptr, tr, tc, tv);
        if (rc) return rc;
      }
      DS_CUDA(cudaFreeAsync(j->dsrc_start, st));
      j->dsrc_start = nullptr;
      if (!ascending) {
        // the proxy's sort: canonicalize adopts tr (own_r) and builds fresh c / v
        j->r = nullptr;
        j->c = nullptr;
        j->v = nullptr;
        j->own_r = j->own_c = j->own_v = false;
        rc = canonicalize(j, nc, tr, tc, tv, true);
        if (j->c == tc) j->own_c = true;
        else if (tc) cudaFreeAsync(tc, st);
        if (j->v == tv) j->own_v = true;
        else if (tv) cudaFreeAsync(tv, st);
        if (rc) return rc;
        if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nc, nrows);
        nc = j->nnz;
      }
    }
  }
  j->nnz = nc;
  if (fill_limit == kDefaultFillLimit) fill_limit = 10 * std::max(nc, nrows);   // DIA nnz = the compacted count
  return size_target(j, fill_limit, out_nnz, out_ndiags);
}

extern "C" int ds_convert_begin_dia(int64_t nrows, int64_t ncols, int32_t ndiags,
                                    const int32_t* offsets, const double* values, int target,
                                    int64_t fill_limit, void* stream, ds_convert_job** job,
                                    int64_t* out_nnz, int64_t* out_ndiags) {
  *job = nullptr;
  if (!dims_ok(nrows, ncols, 0)) return DS_ERR_NOT_SUPPORTED;
  ds_convert_job* j = new_job(nrows, ncols, target, stream);
  const int rc = begin_dia_impl(j, ndiags, offsets, values, fill_limit, out_nnz, out_ndiags);
  if (rc) {
    free_job(j);
    return rc;
  }
  *job = j;
  return DS_OK;
}

__global__ void set_last_offset(int* off, int64_t nrows, int64_t nnz) { off[nrows] = (int)nnz; }

static int finish_coo_impl(ds_convert_job* job, int32_t* rows, int32_t* cols,
                                     double* values) {
  cudaStream_t st = job->st;
  if (job->dsrc_start) {
    return job->nnz > 0 ? dia_emit_into(job, nullptr, rows, cols, values) : DS_OK;
  }
  if (job->csr_off && job->nnz > 0) {   // canonical CSR source: expand the rows in place
    csr_rows_walk<<<csr_walk_grid(job->nrows), 256, 0, st>>>((int)job->nrows, job->csr_off, rows);
    DS_LAUNCH_CHECK("csr_rows_walk");
    DS_CUDA(cudaMemcpyAsync(cols, job->c, job->nnz * 4, cudaMemcpyDeviceToDevice, st));
    DS_CUDA(cudaMemcpyAsync(values, job->v, job->nnz * 8, cudaMemcpyDeviceToDevice, st));
    return DS_OK;
  }
  if (job->nnz > 0) {
    DS_CUDA(cudaMemcpyAsync(rows, job->r, job->nnz * 4, cudaMemcpyDeviceToDevice, st));
    DS_CUDA(cudaMemcpyAsync(cols, job->c, job->nnz * 4, cudaMemcpyDeviceToDevice, st));
    DS_CUDA(cudaMemcpyAsync(values, job->v, job->nnz * 8, cudaMemcpyDeviceToDevice, st));
  }
  return DS_OK;
}

static int finish_csr_impl(ds_convert_job* job, int32_t* row_offsets, int32_t* cols,
                                     double* values) {
  cudaStream_t st = job->st;
  if (job->dsrc_start) {   // row offsets written by the emit pass
    set_last_offset<<<1, 1, 0, st>>>(row_offsets, job->nrows, job->nnz);
    DS_LAUNCH_CHECK("set_last_offset");
    return dia_emit_into(job, row_offsets, nullptr, cols, values);
  }
  if (job->csr_off) {   // canonical CSR source: a copy
    DS_CUDA(cudaMemcpyAsync(row_offsets, job->csr_off, (job->nrows + 1) * 4,
                            cudaMemcpyDeviceToDevice, st));
    if (job->nnz > 0) {
      DS_CUDA(cudaMemcpyAsync(cols, job->c, job->nnz * 4, cudaMemcpyDeviceToDevice, st));
      DS_CUDA(cudaMemcpyAsync(values, job->v, job->nnz * 8, cudaMemcpyDeviceToDevice, st));
    }
    return DS_OK;
  }
  rows_to_offsets<<<grid1d(job->nnz + 1 > job->nrows + 1 ? job->nnz + 1 : job->nrows + 1), 256, 0,
                    st>>>(job->nnz, (int)job->nrows, job->r, row_offsets);
  DS_LAUNCH_CHECK("rows_to_offsets");
  if (job->nnz > 0) {
    DS_CUDA(cudaMemcpyAsync(cols, job->c, job->nnz * 4, cudaMemcpyDeviceToDevice, st));
    DS_CUDA(cudaMemcpyAsync(values, job->v, job->nnz * 8, cudaMemcpyDeviceToDevice, st));
  }
  return DS_OK;
}

static int finish_dia_impl(ds_convert_job* job, int32_t* offsets, double* values) {
  cudaStream_t st = job->st;
  const int64_t nd = job->ndiags;
  if (nd > 0) {
    DS_CUDA(cudaMemcpyAsync(offsets, job->dia_off, nd * sizeof(int), cudaMemcpyDeviceToDevice,
                            st));
    const int64_t slots = nd * job->nrows;
    if (job->spec && !job->csr_off) {   // COO: a miss / disorder -> DS_ERR_RETRY
      const bool rows_fill = use_fill_rows(nd) && job->nnz < INT32_MAX &&
                             (reinterpret_cast<uintptr_t>(job->r) & 15) == 0;
      const size_t obytes = rows_fill ? (size_t)(job->nrows + 1) * 4 : 0;
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->scratch), 16 + obytes, st));
      DS_CUDA(cudaMemsetAsync(job->scratch, 0, 16 + obytes, st));
      int* bad = reinterpret_cast<int*>(job->scratch);
      if (rows_fill) {   // row offsets (checking the rows), then the CSR row-slot fill
        int* roff = reinterpret_cast<int*>(job->scratch + 16);
        coo_offsets_check<<<grid1d((job->nnz + 7) / 8), 256, 0, st>>>(job->nnz, (int)job->nrows,
                                                                      job->r, roff, bad);
        DS_LAUNCH_CHECK("coo_offsets_check");
        const int rc = launch_fill_rows<true>(job->nrows, job->ncols, nd, roff, job->c,
                                              job->v, job->diag_map, job->dia_off, values, bad, st);
        if (rc) return rc;
      } else {   // zero + checked scatter
        DS_CUDA(cudaMemsetAsync(values, 0, slots * sizeof(double), st));   // +0.0
        dia_scatter<true><<<grid1d(job->nnz), 256, 0, st>>>(job->nnz, (int)job->nrows, nd, job->r,
                                                            job->c, job->v, job->diag_map,
                                                            job->dia_off, values, (int)job->ncols,
                                                            bad);
        DS_LAUNCH_CHECK("dia_scatter(check)");
      }
      int bad_h = 1;
      DS_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaStreamSynchronize(st));
      if (bad_h & kBadIndex) return index_error(job->nrows, job->ncols);
      if (bad_h) {
        set_error("speculative COO -> DIA: diagonal set or order differs; use the census path");
        return DS_ERR_RETRY;
      }
      return DS_OK;
    }
    if (job->spec) {   // one pass: order check + fill; a miss -> DS_ERR_RETRY
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->scratch), 4, st));
      DS_CUDA(cudaMemsetAsync(job->scratch, 0, 4, st));
      int* bad = reinterpret_cast<int*>(job->scratch);
      if (use_fill_rows(nd)) {
        const int rc = launch_fill_rows<true>(job->nrows, job->ncols, nd, job->csr_off,
                                              job->c, job->v, job->diag_map, job->dia_off, values,
                                              bad, st);
        if (rc) return rc;
      } else {
        const int R = kCsrWalkRows * 8;   // 8 warps
        const size_t smem = (size_t)R * nd * 8;
        int rc = allow_dynamic_smem((const void*)dia_fill_csr<true>, smem);
        if (rc) return rc;
        dia_fill_csr<true><<<csr_walk_grid(job->nrows), 256, smem, st>>>(
            (int)job->nrows, (int)nd, R, job->csr_off, job->c, job->v, job->diag_map, job->dia_off,
            values, (int)job->ncols, bad);
        DS_LAUNCH_CHECK("dia_fill_csr(check)");
      }
      int bad_h = 1;
      DS_CUDA(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaStreamSynchronize(st));
      if (bad_h & kBadIndex) return index_error(job->nrows, job->ncols);
      if (bad_h) {
        set_error("speculative CSR -> DIA: diagonal set or order differs; use the census path");
        return DS_ERR_RETRY;
      }
      return DS_OK;
    }
    if (job->dia_jsrc) {   // DIA source: the selected columns, masked
      // every diagonal kept: the in-range rows are a plain stream of the slab
      const bool all = nd == job->dsrc_nd && job->dsrc_in_hi > job->dsrc_in_lo &&
                       (reinterpret_cast<uintptr_t>(values) & 15) == 0;
      const int64_t lo = all ? job->dsrc_in_lo : job->nrows, hi = all ? job->dsrc_in_hi : job->nrows;
      if (all) {
        const int64_t a = lo * nd + ((lo * nd) & 1), b = hi * nd;   // even start
        dia_copy_interior<<<grid1d((b - a) / 2), 256, 0, st>>>(a, b, job->dsrc_vals, values);
        DS_LAUNCH_CHECK("dia_copy_interior");
        if (a > lo * nd)   // the odd first slot of the interior goes with the head rows
          dia_copy_diags<<<1, 32, 0, st>>>(lo, lo + 1, (int)job->ncols, job->dsrc_nd, (int)nd,
                                           job->dsrc_off, job->dsrc_vals, job->dia_jsrc, values);
      }
      if (lo > 0)
        dia_copy_diags<<<grid1d(lo * nd), 256, 0, st>>>(0, lo, (int)job->ncols, job->dsrc_nd,
                                                        (int)nd, job->dsrc_off, job->dsrc_vals,
                                                        job->dia_jsrc, values);
      if (hi < job->nrows)
        dia_copy_diags<<<grid1d((job->nrows - hi) * nd), 256, 0, st>>>(
            hi, job->nrows, (int)job->ncols, job->dsrc_nd, (int)nd, job->dsrc_off, job->dsrc_vals,
            job->dia_jsrc, values);
      DS_LAUNCH_CHECK("dia_copy_diags");
      return DS_OK;
    }
    static int fill_tiles = -1;   // measured slower at 192^3 (1.28 vs 0.81 ms): opt-in
    if (fill_tiles < 0) fill_tiles = getenv("DS_DIA_FILL_TILES") ? 1 : 0;
    if (fill_tiles && job->csr_off && (int64_t)kRT * nd * 8 <= 96 * 1024) {
      const size_t smem = (size_t)kRT * nd * 8;
      int rc = allow_dynamic_smem((const void*)csr_dia_fill_tiles, smem);
      if (rc) return rc;
      csr_dia_fill_tiles<<<rt_grid(job->nrows, 6), 256, smem, st>>>(
          (int)job->nrows, (int)nd, job->csr_off, job->c, job->v, job->diag_map, values);
      DS_LAUNCH_CHECK("csr_dia_fill_tiles");
      return DS_OK;
    }
    if (job->csr_off && use_fill_rows(nd)) {
      return launch_fill_rows<false>(job->nrows, job->ncols, nd, job->csr_off, job->c,
                                     job->v, job->diag_map, job->dia_off, values, nullptr, st);
    }
    const int R = kCsrWalkRows * 8;   // 8 warps
    if (job->csr_off && (int64_t)R * nd * 8 <= 48 * 1024) {
      if ((int64_t)R * nd * 8 > 40 * 1024) {   // + the 8 KB map cache
        int rc = allow_dynamic_smem((const void*)dia_fill_csr<false>, (size_t)R * nd * 8);
        if (rc) return rc;
      }
      dia_fill_csr<false><<<csr_walk_grid(job->nrows), 256, (size_t)R * nd * 8, st>>>(
          (int)job->nrows, (int)nd, R, job->csr_off, job->c, job->v, job->diag_map, job->dia_off,
          values);
      DS_LAUNCH_CHECK("dia_fill_csr");
      return DS_OK;
    }
    if (job->csr_off && job->nnz > 0) {   // slab too wide for shared memory: expand the rows
      DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&job->r), job->nnz * 4, st));
      job->own_r = true;
      csr_expand_rows<<<grid1d(job->nrows * 8), 256, 0, st>>>((int)job->nrows, job->csr_off,
                                                               job->r);
      DS_LAUNCH_CHECK("csr_expand_rows");
    }
    zero_f64<<<grid1d(slots), 256, 0, st>>>(slots, values);
    dia_scatter<false><<<grid1d(job->nnz), 256, 0, st>>>(job->nnz, (int)job->nrows, nd, job->r,
                                                         job->c, job->v, job->diag_map,
                                                         job->dia_off, values);
    DS_LAUNCH_CHECK("dia_scatter");
  }
  return DS_OK;
}

// finish_* frees the job on every path (a DS_CUDA early return included)
extern "C" int ds_convert_finish_coo(ds_convert_job* job, int32_t* rows, int32_t* cols,
                                     double* values) {
  const int rc = finish_coo_impl(job, rows, cols, values);
  free_job(job);
  return rc;
}

extern "C" int ds_convert_finish_csr(ds_convert_job* job, int32_t* row_offsets, int32_t* cols,
                                     double* values) {
  const int rc = finish_csr_impl(job, row_offsets, cols, values);
  free_job(job);
  return rc;
}

extern "C" int ds_convert_finish_dia(ds_convert_job* job, int32_t* offsets, double* values) {
  const int rc = finish_dia_impl(job, offsets, values);
  free_job(job);
  return rc;
}

extern "C" void ds_convert_abort(ds_convert_job* job) { free_job(job); }

extern "C" int ds_dia_to_entries(int64_t nrows, int64_t ncols, int32_t ndiags,
                                 const int32_t* offsets, const double* values, int target,
                                 int32_t* row_idx, int32_t* cols, double* vals, int64_t* nnz,
                                 void* stream) {
  cudaStream_t st = as_stream(stream);
  *nnz = 0;
  if (!dims_ok(nrows, ncols, 0)) return DS_ERR_NOT_SUPPORTED;
  if (target != DS_FMT_CSR && target != DS_FMT_COO) {
    set_error("ds_dia_to_entries: CSR or COO target only");
    return DS_ERR_INVALID_ARGUMENT;
  }
  if (ndiags > kDiaOneMaxNd || ndiags < 1 || nrows == 0) {
    set_error("ds_dia_to_entries: 1 <= ndiags <= %d and nrows > 0", kDiaOneMaxNd);
    return DS_ERR_NOT_SUPPORTED;
  }
  const int64_t ngroups = ceil_div(nrows, kDiaGroupRows);
  unsigned char* scratch = nullptr;   // ticket | total | status[ngroups]
  const size_t bytes = 16 + (size_t)ngroups * 8;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), bytes, st));
  int rc = DS_OK;
  long long h_total = 0;
  do {
    if (cudaMemsetAsync(scratch, 0, bytes, st) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "dia one-pass scratch");
      break;
    }
    const unsigned grid = (unsigned)std::max<int64_t>(
        1, min64(ceil_div(ngroups, 4), (int64_t)sm_count() * 4));
    dia_emit_onepass<<<grid, 128, 0, st>>>(
        nrows, (int)ncols, ndiags, offsets, values, ngroups,
        reinterpret_cast<unsigned long long*>(scratch + 16), reinterpret_cast<int*>(scratch),
        target == DS_FMT_CSR ? row_idx : nullptr, target == DS_FMT_COO ? row_idx : nullptr,
        cols, vals, reinterpret_cast<long long*>(scratch + 8));
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_total, scratch + 8, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "dia_emit_onepass");
  } while (false);
  cudaFreeAsync(scratch, st);
  *nnz = h_total;
  return rc;
}
