// ds_sort.cu -- stable LSD radix sort of (64-bit key, 32-bit index) pairs:
// the stable np.lexsort((cols, rows)) of the COO canonicalisation
// (datamove.py:208-220, lexsort at :212) and the ghost-key sort of the
// stencil generator (stencil.py:198-209).  Hand-written; no library sort.
//
// Keys are limited to the bits the data needs (row * ncols + col < 2^bits),
// 8 bits per pass.  One histogram kernel counts every pass's digits up front
// (the digit counts do not depend on the order), a 1-block kernel turns them
// into each pass's global digit bases, then ONE kernel per pass ranks and
// scatters (a "onesweep" pass):
//   * a CTA takes the next tile of 4096 keys (tile ids from an atomic
//     counter, so every earlier tile is already resident -- the look-back
//     below always makes progress);
//   * keys are held warp-striped (warp w, item i, lane l = tile position
//     w*512 + i*32 + l), so ranking items in (i, lane) order per warp with
//     __match_any_sync + per-warp digit counters, then offsetting by the
//     earlier warps' counts, is exactly stable;
//   * the tile publishes its per-digit counts and finds the counts of all
//     earlier tiles by decoupled look-back (one thread per digit; a status
//     word = pass tag | aggregate / inclusive flag | count, so the status
//     array is zeroed once for all passes);
//   * the tile is staged in digit order in shared memory and written out
//     with consecutive threads on consecutive output positions (runs of one
//     digit are contiguous in the output).
// The first pass builds the keys from the (row, col) arrays and the identity
// index on the fly, so neither is ever materialised.
#include <algorithm>

#include "ds_common.cuh"

namespace ds {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;   // 4096
constexpr int kRadix = 256;
constexpr int kMaxPasses = 8;

typedef unsigned long long u64;

struct SortSrc {
  const u64* keys;    // pass input keys, or nullptr: key = rows[k] * ncols + cols[k]
  const int* rows;
  const int* cols;
  u64 ncols;
  __device__ __forceinline__ u64 key(int64_t k) const {
    return keys ? keys[k] : (u64)(unsigned)rows[k] * ncols + (u64)(unsigned)cols[k];
  }
};

__global__ void __launch_bounds__(kSortThreads) radix_histogram(SortSrc src, int64_t n,
                                                                int passes, unsigned* hist) {
  __shared__ unsigned h[kMaxPasses * kRadix];
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const u64 key = src.key(k);
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * kRadix + ((key >> (8 * p)) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// exclusive scan of 256 values held one per thread (block of 256)
__device__ __forceinline__ long long block_exclusive_scan256(long long v, long long* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  long long before = 0;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  __syncthreads();
  return before + inc - v;
}

__global__ void __launch_bounds__(kRadix) radix_bases(const unsigned* hist, int passes,
                                                      long long* bases) {
  __shared__ long long wt[kRadix / 32];
  for (int p = 0; p < passes; ++p)
    bases[p * kRadix + threadIdx.x] =
        block_exclusive_scan256(hist[p * kRadix + threadIdx.x], wt);
}

// status word: [63:62] kind (1 aggregate, 2 inclusive) | [61:56] pass tag | [55:0] count
constexpr u64 kAgg = 1ull << 62, kIncl = 2ull << 62, kCountMask = (1ull << 56) - 1;

__device__ __forceinline__ void st_status(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_status(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct SortSmem {
  u64 key[kSortTile];
  int idx[kSortTile];
  int wcnt[kSortWarps * kRadix];   // per-warp digit counts -> exclusive over warps
  int tstart[kRadix];              // digit start inside the tile (digit order)
  long long gpos[kRadix];          // output position of tile slot j with digit d = gpos[d] + j
  long long wtot[kRadix / 32];
  int tile;
};

__global__ void __launch_bounds__(kSortThreads, 2)
    radix_onesweep(SortSrc src, const int* __restrict__ idx_in, u64* __restrict__ keys_out,
                   int* __restrict__ idx_out, int64_t n, int shift, u64 tag,
                   const long long* __restrict__ gbase, u64* status, int* tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) S.tile = atomicAdd(tile_counter, 1);
  for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) S.wcnt[i] = 0;
  __syncthreads();
  const int64_t tile = S.tile;
  const int64_t t0 = tile * kSortTile;
  const int64_t wbase = t0 + (int64_t)warp * 32 * kSortItems;

  u64 key[kSortItems];
  int idv[kSortItems];
  int rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t k = wbase + i * 32 + lane;
    if (k < n) {
      key[i] = src.key(k);
      idv[i] = idx_in ? __ldg(idx_in + k) : (int)k;
    } else {
      key[i] = ~0ull;
      idv[i] = -1;
    }
  }
  // stable rank inside the warp: items in (i, lane) order
  const unsigned lt = (1u << lane) - 1u;
  int* wc = S.wcnt + warp * kRadix;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const int d = valid ? (int)((key[i] >> shift) & 255) : kRadix;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int before = valid ? wc[d] : 0;
    __syncwarp();
    rank[i] = before + __popc(peers & lt);
    if (valid && (peers & lt) == 0) wc[d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // thread d: offsets of each warp inside digit d, the tile's count of d
  const int d = tid;
  int total = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    const int c = S.wcnt[w * kRadix + d];
    S.wcnt[w * kRadix + d] = total;
    total += c;
  }
  u64* my_status = status + tile * kRadix + d;
  st_status(my_status, (tile == 0 ? kIncl : kAgg) | tag | (u64)total);
  const int tstart = (int)block_exclusive_scan256(total, S.wtot);
  S.tstart[d] = tstart;
  // decoupled look-back over the earlier tiles' counts of digit d
  long long excl = 0;
  if (tile > 0) {
    for (int64_t t = tile - 1; t >= 0; --t) {
      const u64* p = status + t * kRadix + d;
      u64 w;
      do {
        w = ld_status(p);
      } while ((w & (63ull << 56)) != tag);
      excl += (long long)(w & kCountMask);
      if ((w >> 62) == 2) break;
    }
    st_status(my_status, kIncl | tag | (u64)(excl + total));
  }
  S.gpos[d] = gbase[d] + excl - tstart;
  __syncthreads();
  // stage the tile in digit order
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    if (wbase + i * 32 + lane < n) {
      const int dd = (int)((key[i] >> shift) & 255);
      const int j = S.tstart[dd] + S.wcnt[warp * kRadix + dd] + rank[i];
      S.key[j] = key[i];
      S.idx[j] = idv[i];
    }
  }
  __syncthreads();
  const int cnt = (int)min64(kSortTile, n - t0);
  for (int j = tid; j < cnt; j += kSortThreads) {
    const u64 kk = S.key[j];
    const long long pos = S.gpos[(kk >> shift) & 255] + j;
    keys_out[pos] = kk;
    idx_out[pos] = S.idx[j];
  }
}

static int bits_needed(u64 maxkey) {
  int b = 0;
  while (b < 64 && (maxkey >> b) != 0ull) ++b;
  return b < 1 ? 1 : b;
}

// Sorted keys into keys_out and the stable permutation into perm_out (both
// n long).  Keys from `keys` or, when null, rows[k] * ncols + cols[k];
// max_key bounds them (inclusive).  Temporaries come from the stream pool.
int radix_sort_pairs(const u64* keys, const int* rows, const int* cols, u64 ncols, int64_t n,
                     u64 max_key, u64* keys_out, int* perm_out, cudaStream_t st) {
  if (n <= 0) return DS_OK;
  if (n >= (1ll << 31)) {
    set_error("radix sort: %lld keys (at most 2^31 - 1)", (long long)n);
    return DS_ERR_NOT_SUPPORTED;
  }
  const int bits = bits_needed(max_key);
  const int passes = (bits + 7) / 8;
  const int64_t ntiles = ceil_div(n, kSortTile);
  // one scratch block: hist | bases | tile counters | status (zeroed once)
  const size_t hist_b = (size_t)kMaxPasses * kRadix * sizeof(unsigned);
  const size_t base_b = (size_t)kMaxPasses * kRadix * sizeof(long long);
  const size_t ctr_b = 64;
  const size_t stat_b = (size_t)ntiles * kRadix * sizeof(u64);
  const size_t scratch_b = hist_b + base_b + ctr_b + stat_b;
  unsigned char* scratch = nullptr;
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), scratch_b, st));
  unsigned* hist = reinterpret_cast<unsigned*>(scratch);
  long long* bases = reinterpret_cast<long long*>(scratch + hist_b);
  int* counters = reinterpret_cast<int*>(scratch + hist_b + base_b);
  u64* status = reinterpret_cast<u64*>(scratch + hist_b + base_b + ctr_b);
  int rc = DS_OK;
  u64 *kbuf = nullptr;
  int* ibuf = nullptr;
  do {
    if (cudaMemsetAsync(scratch, 0, scratch_b, st) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "radix scratch memset");
      break;
    }
    SortSrc src0{keys, rows, cols, ncols};
    const unsigned hg = (unsigned)std::max<int64_t>(1, min64(ceil_div(n, 256 * 8), (int64_t)sm_count() * 8));
    radix_histogram<<<hg, 256, 0, st>>>(src0, n, passes, hist);
    radix_bases<<<1, kRadix, 0, st>>>(hist, passes, bases);
    if ((rc = allow_dynamic_smem((const void*)radix_onesweep, sizeof(SortSmem)))) break;
    // ping-pong: pass p writes (keys, idx) to the buffer that makes the last
    // pass land in keys_out / perm_out
    if (passes > 1) {
      if (cudaMallocAsync(reinterpret_cast<void**>(&kbuf), n * sizeof(u64), st) != cudaSuccess ||
          cudaMallocAsync(reinterpret_cast<void**>(&ibuf), n * sizeof(int), st) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError(), "radix ping-pong buffers");
        break;
      }
    }
    const u64* kin = nullptr;
    const int* iin = nullptr;
    for (int p = 0; p < passes; ++p) {
      const bool to_final = ((passes - 1 - p) % 2) == 0;
      u64* kout = to_final ? keys_out : kbuf;
      int* iout = to_final ? perm_out : ibuf;
      SortSrc src = p == 0 ? src0 : SortSrc{kin, nullptr, nullptr, ncols};
      radix_onesweep<<<(unsigned)ntiles, kSortThreads, sizeof(SortSmem), st>>>(
          src, iin, kout, iout, n, 8 * p, (u64)(p + 1) << 56, bases + p * kRadix, status,
          counters + p);
      kin = kout;
      iin = iout;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "radix_onesweep");
  } while (false);
  if (kbuf) cudaFreeAsync(kbuf, st);
  if (ibuf) cudaFreeAsync(ibuf, st);
  cudaFreeAsync(scratch, st);
  return rc;
}

// ------------------------------------------------------ row-sorted input --
// When the rows are already non-decreasing (a CSR source; a COO built row by
// row, like the power-law matrix) the stable (row, col) sort is a sort INSIDE
// each row: one read and one write of the entries instead of 8-bit LSD
// passes over row AND column bits.  Rows are cut into warp tiles of at most
// kSegTile entries (rows of up to kSegShort entries, grouped); a warp sorts
// its tile in shared memory with a bitonic network over unique composite keys
// (local row | column | local index -- unique, so the unstable network
// yields the stable order).  Longer rows (up to kSegLong) are sorted one per
// CTA the same way with (column | local index) keys.
constexpr int kSegShort = 128;          // rows up to this many entries share warp tiles
constexpr int kSegTile = 2 * kSegShort; // entries per warp tile (< kSegShort + 129)
constexpr int kSegLong = 16384;         // longest row the CTA kernel sorts in shared memory
constexpr int kSegWarps = 8;

__device__ __forceinline__ void bitonic_warp(u64* s, int n2) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < (n2 >> 1); t += 32) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const u64 a = s[i], b = s[i + j];
        if ((a > b) == ((i & k) == 0)) {
          s[i] = b;
          s[i + j] = a;
        }
      }
      __syncwarp();
    }
}

__global__ void __launch_bounds__(32 * kSegWarps)
    seg_sort_tiles(int64_t ntiles, const int* __restrict__ tiles, const int* __restrict__ off,
                   const int* __restrict__ rows, const int* __restrict__ cols, u64 ncols,
                   u64* __restrict__ keys_out, int* __restrict__ perm_out) {
  __shared__ u64 sk_all[kSegWarps][kSegTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64* sk = sk_all[warp];
  for (int64_t t = (int64_t)blockIdx.x * kSegWarps + warp; t < ntiles;
       t += (int64_t)gridDim.x * kSegWarps) {
    const int r0 = __ldg(tiles + t), r1 = __ldg(tiles + t + 1);
    const int e0 = __ldg(off + r0), cnt = __ldg(off + r1) - e0;
    if (r1 - r0 == 1 && cnt > kSegShort) continue;   // a long row: the CTA kernel sorts it
    if (cnt <= 1) {   // nothing to sort (the entry's row need not be r0: empty rows lead)
      if (lane < cnt) {
        keys_out[e0] = (u64)(unsigned)__ldg(rows + e0) * ncols + (u64)(unsigned)__ldg(cols + e0);
        perm_out[e0] = e0;
      }
      continue;
    }
    int n2 = 32;
    while (n2 < cnt) n2 <<= 1;
    for (int k = lane; k < n2; k += 32) {
      u64 key = ~0ull;
      if (k < cnt) {
        const u64 lr = (u64)(unsigned)(__ldg(rows + e0 + k) - r0);
        key = (lr << 40) | ((u64)(unsigned)__ldg(cols + e0 + k) << 8) | (u64)k;
      }
      sk[k] = key;
    }
    __syncwarp();
    bitonic_warp(sk, n2);
    for (int k = lane; k < cnt; k += 32) {
      const u64 key = sk[k];
      const u64 r = (u64)(unsigned)r0 + (key >> 40);
      keys_out[e0 + k] = r * ncols + ((key >> 8) & 0xffffffffull);
      perm_out[e0 + k] = e0 + (int)(key & 255);
    }
    __syncwarp();
  }
}

// one CTA per long row: bitonic sort of (column << 32 | local index) in
// shared memory (next power of two of the row length, padded with ~0)
__global__ void __launch_bounds__(512)
    seg_sort_long(const int* __restrict__ long_rows, const int* __restrict__ off,
                  const int* __restrict__ cols, u64 ncols, u64* __restrict__ keys_out,
                  int* __restrict__ perm_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* sk = reinterpret_cast<u64*>(smem_raw);
  const int r = __ldg(long_rows + blockIdx.x);
  const int e0 = __ldg(off + r), len = __ldg(off + r + 1) - e0;
  int n2 = 1;
  while (n2 < len) n2 <<= 1;
  for (int k = threadIdx.x; k < n2; k += blockDim.x)
    sk[k] = k < len ? (((u64)(unsigned)__ldg(cols + e0 + k) << 32) | (u64)k) : ~0ull;
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (n2 >> 1); t += blockDim.x) {
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const u64 a = sk[i], b = sk[i + j];
        if ((a > b) == ((i & k) == 0)) {
          sk[i] = b;
          sk[i + j] = a;
        }
      }
      __syncthreads();
    }
  const u64 rb = (u64)(unsigned)r * ncols;
  for (int k = threadIdx.x; k < len; k += blockDim.x) {
    const u64 key = sk[k];
    keys_out[e0 + k] = rb + (key >> 32);
    perm_out[e0 + k] = e0 + (int)(key & 0xffffffffull);
  }
}

// the long rows of a tile plan (tiles of one row with more than kSegShort entries)
__global__ void seg_collect_long(int64_t ntiles, const int* __restrict__ tiles,
                                 const int* __restrict__ off, int* long_rows, int* count,
                                 int* max_len) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = tiles[t], r1 = tiles[t + 1];
    const int len = off[r1] - off[r0];
    if (r1 - r0 == 1 && len > kSegShort) {
      long_rows[atomicAdd(count, 1)] = r0;
      atomicMax(max_len, len);
    }
  }
}

int segmented_sort_rows(const int* off, const int* rows, const int* cols, u64 ncols,
                        const int* tiles, int64_t ntiles, u64* keys_out, int* perm_out,
                        cudaStream_t st) {
  if (ntiles <= 0) return DS_OK;
  int* scratch = nullptr;   // [count, max_len, long rows ...]
  DS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), (ntiles + 2) * sizeof(int), st));
  int rc = DS_OK;
  do {
    if (cudaMemsetAsync(scratch, 0, 2 * sizeof(int), st) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "segmented sort scratch");
      break;
    }
    const unsigned g = (unsigned)std::max<int64_t>(1, min64(ceil_div(ntiles, 256),
                                                              (int64_t)sm_count() * 4));
    seg_collect_long<<<g, 256, 0, st>>>(ntiles, tiles, off, scratch + 2, scratch, scratch + 1);
    int h[2] = {0, 0};
    if (cudaMemcpyAsync(h, scratch, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "segmented sort plan");
      break;
    }
    if (h[1] > kSegLong) {   // a row too long for shared memory: the caller falls back
      set_error("row of %d entries exceeds the segmented sort's %d", h[1], kSegLong);
      rc = DS_ERR_NOT_SUPPORTED;
      break;
    }
    if (h[0] > 0) {
      int n2 = 1;
      while (n2 < h[1]) n2 <<= 1;
      const size_t smem = (size_t)n2 * sizeof(u64);
      if ((rc = allow_dynamic_smem((const void*)seg_sort_long, smem))) break;
      seg_sort_long<<<(unsigned)h[0], 512, smem, st>>>(scratch + 2, off, cols, ncols, keys_out,
                                                       perm_out);
    }
    const unsigned gt = (unsigned)std::max<int64_t>(
        1, min64(ceil_div(ntiles, kSegWarps), (int64_t)sm_count() * 8));
    seg_sort_tiles<<<gt, 32 * kSegWarps, 0, st>>>(ntiles, tiles, off, rows, cols, ncols, keys_out,
                                                  perm_out);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "segmented sort");
  } while (false);
  cudaFreeAsync(scratch, st);
  return rc;
}

}  // namespace ds

using namespace ds;

// Exposed for the tests: sort n 64-bit keys (stable), keys < 2^bits.
extern "C" int ds_radix_sort_pairs(const unsigned long long* keys_in, int64_t n, int bits,
                                   unsigned long long* keys_out, int32_t* perm_out,
                                   void* stream) {
  if (bits < 1 || bits > 64) {
    set_error("bits must be in [1, 64]");
    return DS_ERR_INVALID_ARGUMENT;
  }
  const u64 max_key = bits == 64 ? ~0ull : ((1ull << bits) - 1ull);
  return radix_sort_pairs(keys_in, nullptr, nullptr, 0, n, max_key, keys_out, perm_out,
                          as_stream(stream));
}
