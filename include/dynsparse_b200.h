/*
 * dynsparse_b200.h -- C ABI of the B200-native dynsparse hot path.
 *
 * One shared library (libdynsparse_b200.so, sm_100a) exports these symbols.
 * Every entry point takes plain device pointers + sizes and a CUDA stream
 * (cudaStream_t passed as void*; NULL = legacy default stream), enqueues
 * stream-ordered work and returns an int status (DS_OK = 0).  No torch types
 * cross the boundary.  Buffers are owned by the caller; the library borrows
 * them for the duration of the stream-ordered call.  Internal temporaries use
 * the stream-ordered allocator (cudaMallocAsync) and are released on the same
 * stream.
 *
 * Index arrays are int32 on the device (the reference stores int64,
 * formats.py:82-83; the host layer narrows on upload after checking every
 * dimension is < 2^31 and widens on download).  Values are IEEE float64.
 *
 * Each block cites the reference interface it replaces (file:line relative
 * to the reference's pkg/src/dynsparse/).  Status codes map 1:1 onto the
 * reference's exception classes (errors.py).
 */
#ifndef DYNSPARSE_B200_H
#define DYNSPARSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 1

/* ---- status codes (errors.py) ------------------------------------------ */
enum {
  DS_OK = 0,
  DS_ERR_INVALID_ARGUMENT = 1,          /* ValueError / DimensionMismatch (host-checked) */
  DS_ERR_CUDA = 2,                      /* DeviceError (new): a CUDA runtime failure     */
  DS_ERR_DIA_FILL_OVERFLOW = 3,         /* DiaFillOverflow        errors.py:52-53        */
  DS_ERR_STRUCTURALLY_ABSENT_DIAG = 4,  /* StructurallyAbsentDiagonal errors.py:73-78    */
  DS_ERR_BREAKDOWN = 5,                 /* BreakdownZeroCurvature errors.py:81-82        */
  DS_ERR_NOT_SUPPORTED = 6,             /* dims >= 2^31 or a layout the kernels refuse   */
  DS_ERR_INDEX_OUT_OF_RANGE = 7,        /* IndexOutOfRange errors.py:17: an entry's row /
                                           column outside the shape (conversion sources)  */
  DS_ERR_RETRY = 8                      /* a speculative fast path did not apply: run the
                                           general entry point (never surfaces in Python) */
};

/* Message of the last failing call on this host thread ("" if none). */
const char* ds_last_error(void);
int ds_abi_version(void);
/* SM count of the current device (grid sizing is a multiple of it). */
int ds_device_sm_count(int* out);

/* ---- SpMV: replaces kernels._SPMV_KERNELS (kernels.py:166-170) behind
 *      spmv (kernels.py:173-186, accumulate=0: y = A x) and
 *      spmv_add (kernels.py:189-198, accumulate=1: y = y + (A x)).
 * Rounding contract (bitwise equal to the reference on the same inputs):
 *   CSR: y[i] = p[first] + pairwise8(p[first+1:end])   (np.add.reduceat)
 *   DIA: y[i] = ((0 + p_0) + p_1) + ...  over in-range diagonals ascending
 *   COO (rows nondecreasing): sequential per row in stored order from 0.0 (np.bincount)
 *   COO (unsorted): atomics, within 1e-13 relative (as the reference's threaded COO)
 * with every product rounded before the add (no FMA).                       */

/* Rows longer than 129 entries need the pairwise recursion; ds_csr_analyze
 * lists them so ds_spmv_csr can hand them to a CTA-per-row kernel.
 * long_rows must hold nrows int32; *n_long is written (host, synchronises). */
int ds_csr_analyze(int64_t nrows, const int32_t* row_offsets, int32_t* long_rows,
                   int64_t* n_long, int32_t* max_row_len, void* stream);

/* long_rows may be NULL: the matrix is then treated as un-analysed and every
 * row is handled in-line (correct, slower).  A non-NULL long_rows (even with
 * n_long == 0) enables the TMA-tiled kernel, which leaves rows > 129 entries
 * to a CTA-per-row kernel.  n_long is the count from ds_csr_analyze.        */
int ds_spmv_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_offsets,
                const int32_t* col_indices, const double* values,
                const int32_t* long_rows, int64_t n_long,
                const double* x, double* y, int accumulate, void* stream);

/* values: row-major (nrows, ndiags), entry (i, i+offsets[j]) at values[i*ndiags+j]
 * (formats.py:217-258); offsets strictly increasing, on the device.         */
int ds_spmv_dia(int64_t nrows, int64_t ncols, int32_t ndiags, const int32_t* offsets,
                const double* values, const double* x, double* y, int accumulate,
                void* stream);

/* rows_sorted != 0 promises row indices are nondecreasing (canonical COO). */
int ds_spmv_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_indices,
                const int32_t* col_indices, const double* values, int rows_sorted,
                const double* x, double* y, int accumulate, void* stream);

/* Row-sorted COO with a known longest row (ds_coo_max_run): rows of at most
 * 27 entries run on the TMA-pipelined thread-per-row kernel; max_row_len 0
 * (unknown) or longer rows use the warp-segment kernel.  Same result bits
 * as ds_spmv_coo with rows_sorted = 1 (np.bincount order).                 */
int ds_spmv_coo_sorted(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_indices,
                       const int32_t* col_indices, const double* values, int32_t max_row_len,
                       const double* x, double* y, int accumulate, void* stream);

/* Long-run plan of a row-sorted COO: the runs of equal row index longer than
 * `threshold` entries (ds_coo_long_run_threshold() is the kernel's) as int32
 * (start, end) pairs sorted by start; pass them in ds_matrix.long_rows with
 * n_long = the number of runs: those rows are summed by a CTA each on a side
 * stream while the warp kernel skips them.  `runs` holds 2*capacity int32
 * (capacity >= nnz / threshold + 1 suffices).  Host count, synchronises.   */
int ds_coo_long_runs(int64_t nnz, const int32_t* row_indices, int32_t threshold, int32_t* runs,
                     int64_t capacity, int64_t* n_runs, void* stream);
int ds_coo_long_run_threshold(void);

/* Longest run of equal row indices of a row-sorted COO (host, synchronises). */
int ds_coo_max_run(int64_t nnz, const int32_t* row_indices, int32_t* max_run, void* stream);

/* flags bit0: rows nondecreasing; bit1: (row, col) strictly increasing
 * (already canonical).  Written to host memory (synchronises).              */
int ds_coo_order_flags(int64_t nnz, const int32_t* row_indices, const int32_t* col_indices,
                       int32_t* flags, void* stream);

/* ---- dense-vector kernels (kernels.py:205-235) -------------------------- */
/* Deterministic two-level tree reduction (fixed for a given n); result to
 * device memory.  workspace: ds_dot_workspace_bytes() bytes of device memory
 * (zeroed once before first use; the kernel leaves it re-usable).           */
int64_t ds_dot_workspace_bytes(void);
int ds_dot(int64_t n, const double* x, const double* y, double* result_dev,
           void* workspace, void* stream);
/* w = alpha*x + beta*y, products rounded separately (no FMA); w may alias x or y. */
int ds_waxpby(int64_t n, double alpha, const double* x, double beta, const double* y,
              double* w, void* stream);
/* Exact sequential prefix sums (np.cumsum order); out may be NULL for reduce. */
int ds_scan(int64_t n, const double* x, double* out, double* total_dev, void* stream);

/* ---- diagonal extract / update (kernels.py:242-337) --------------------- */
/* out[i] = A(i,i) for i < min(nrows,ncols); absent -> 0.0.  COO duplicates are
 * summed in stored order (np.bincount).                                      */
int ds_extract_diag_csr(int64_t nrows, int64_t ncols, const int32_t* row_offsets,
                        const int32_t* col_indices, const double* values, double* out,
                        void* stream);
int ds_extract_diag_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                        const int32_t* cols, const double* values, double* out, void* stream);
/* Overwrite A(i,i) = d[i].  Returns DS_ERR_STRUCTURALLY_ABSENT_DIAG with
 * *first_missing set when some (i,i) is not stored (checked before writing).
 * COO duplicates: first stored occurrence takes d[i], later ones 0.0.        */
int ds_update_diag_csr(int64_t nrows, int64_t ncols, const int32_t* row_offsets,
                       const int32_t* col_indices, double* values, const double* d,
                       int64_t* first_missing, void* stream);
int ds_update_diag_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, double* values, const double* d,
                       int64_t* first_missing, void* stream);
/* DIA nnz = nonzero in-range slots (formats.py:239-255); written to host.    */
int ds_dia_count_nonzero(int64_t nrows, int64_t ncols, int32_t ndiags, const int32_t* offsets,
                         const double* values, int64_t* count, void* stream);

/* ---- conversion via the canonical COO proxy (datamove.py:208-295) -------
 * Two phases so the caller allocates outputs:  begin_* builds the canonical
 * COO (stable (row,col) sort + duplicate sums in reduceat order) on the
 * device, sizes the target and -- for DIA -- applies the fill-limit test
 * BEFORE any target allocation (datamove.py:246-252): it returns
 * DS_ERR_DIA_FILL_OVERFLOW with *out_ndiags set.  fill_limit ==
 * DS_FILL_LIMIT_DEFAULT (INT64_MIN) selects the reference default
 * 10 * max(nnz, nrows) of the source (datamove.py:55-57; for a DIA source
 * nnz = its nonzero in-range slots, counted by begin); any other value --
 * negative ones included -- is the limit itself (slots > fill_limit raises,
 * datamove.py:250-252).  An entry outside the shape returns
 * DS_ERR_INDEX_OUT_OF_RANGE (nothing is written for it).
 * finish_* writes the target arrays and frees the job; abort frees it
 * without writing.  A DIA or canonical-CSR source is read again by finish_*
 * (its entries go straight into the target): keep it alive until then.
 * DIA offsets need not ascend: unsorted or repeated diagonals are sorted and
 * summed like duplicate COO entries (datamove.py:208-235).                 */
#define DS_FILL_LIMIT_DEFAULT ((int64_t)(-9223372036854775807LL - 1))
typedef struct ds_convert_job ds_convert_job;
/* DIA source with strictly ascending offsets (1 <= ndiags <= 32) -> CSR or
 * COO in ONE pass over the slab (the canonical order is the row-major slot
 * order filtered by "column in range and value != 0", formats.py:439-479):
 * the caller sizes cols / vals by the in-range slot count (an upper bound of
 * the nonzeros) and row_idx by nrows + 1 (CSR offsets) or that count (COO
 * rows); *nnz receives the entries written (synchronises).  Other sources
 * take ds_convert_begin_dia.                                                */
int ds_dia_to_entries(int64_t nrows, int64_t ncols, int32_t ndiags, const int32_t* offsets,
                      const double* values, int target, int32_t* row_idx, int32_t* cols,
                      double* vals, int64_t* nnz, void* stream);
/* The canonicalisation's stable sort, exposed for tests: keys_in[0..n) <
 * 2^bits sorted ascending into keys_out, perm_out[i] = the input position of
 * keys_out[i]; equal keys keep their input order (np.lexsort's stability,
 * datamove.py:212).  Hand-written onesweep LSD radix sort, 8 bits a pass. */
int ds_radix_sort_pairs(const unsigned long long* keys_in, int64_t n, int bits,
                        unsigned long long* keys_out, int32_t* perm_out, void* stream);
enum { DS_FMT_COO = 0, DS_FMT_CSR = 1, DS_FMT_DIA = 2 };   /* FormatId, formats.py:33-42 */

int ds_convert_begin_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                         const int32_t* cols, const double* values, int target,
                         int64_t fill_limit, void* stream, ds_convert_job** job,
                         int64_t* out_nnz, int64_t* out_ndiags);
int ds_convert_begin_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* row_offsets,
                         const int32_t* cols, const double* values, int target,
                         int64_t fill_limit, void* stream, ds_convert_job** job,
                         int64_t* out_nnz, int64_t* out_ndiags);
int ds_convert_begin_dia(int64_t nrows, int64_t ncols, int32_t ndiags, const int32_t* offsets,
                         const double* values, int target, int64_t fill_limit, void* stream,
                         ds_convert_job** job, int64_t* out_nnz, int64_t* out_ndiags);
/* One pass for a canonical COO / CSR source ((row, col) strictly increasing,
 * every index in range) and a COO / CSR target -- the common case of the
 * reference's convert (datamove.py:261-281: the proxy's sort and duplicate
 * sums are the identity there).  src_idx = rows (COO) or row_offsets (CSR);
 * out_idx = target rows (nnz) or row_offsets (nrows + 1); out_cols /
 * out_values hold nnz.  The check and the target writes share the pass;
 * *done = 1: the target is complete.  *done = 0: not applicable (empty,
 * arrays not 16-B aligned) or not canonical -- the target arrays may have
 * been written; run begin / finish.  DS_ERR_INDEX_OUT_OF_RANGE like
 * begin_*.  Synchronises the stream.                                        */
int ds_convert_direct(int src_format, int target, int64_t nrows, int64_t ncols, int64_t nnz,
                      const int32_t* src_idx, const int32_t* cols, const double* values,
                      int32_t* out_idx, int32_t* out_cols, double* out_values, void* stream,
                      int* done);
/* Speculative CSR -> DIA (convert's DIA branch, datamove.py:238-258, whose
 * diagonal set is the COO proxy's, formats.py:439-479): the diagonal set is
 * taken from a sample of row tiles (every ntiles/256-th 128-row tile and the
 * last) and finish_dia
 * fills the slab in ONE pass that also checks the order, the index range and
 * that no entry lies outside the sampled set (the sample is a subset of the
 * true set, so no miss means equal).  DS_ERR_RETRY from begin (empty source,
 * arrays not 16-B aligned, fill limit exceeded by the sample, > 160 sampled
 * diagonals) or from finish_dia (a miss, not canonical): the target is
 * garbage -- run ds_convert_begin_csr / finish_dia.  Otherwise the result is
 * the census path's, bit for bit.                                           */
int ds_convert_begin_csr_dia_spec(int64_t nrows, int64_t ncols, int64_t nnz,
                                  const int32_t* row_offsets, const int32_t* cols,
                                  const double* values, int64_t fill_limit, void* stream,
                                  ds_convert_job** job, int64_t* out_ndiags);
/* The same for a COO source (rows, cols, values): the census of 256 evenly
 * spaced 4096-entry chunks and the last one; finish_dia clears the slab and
 * scatters with the order / range / membership checks.                    */
int ds_convert_begin_coo_dia_spec(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* rows,
                                  const int32_t* cols, const double* values, int64_t fill_limit,
                                  void* stream, ds_convert_job** job, int64_t* out_ndiags);
int ds_convert_finish_coo(ds_convert_job* job, int32_t* rows, int32_t* cols, double* values);
int ds_convert_finish_csr(ds_convert_job* job, int32_t* row_offsets, int32_t* cols,
                          double* values);
int ds_convert_finish_dia(ds_convert_job* job, int32_t* offsets, double* values);
void ds_convert_abort(ds_convert_job* job);

/* ---- on-device generate_problem for one partition (stencil.py:143-253) --
 * begin sizes the partition (nnz, ghost count); the caller allocates
 * row_offsets (n+1 int32), cols (nnz int32), vals (nnz f64), b (n f64) and
 * ghost_keys (nghosts int64: owner*n + owner_local, ascending -- the ghost
 * numbering, from which the halo plan follows); finish fills them.        */
typedef struct ds_stencil_job ds_stencil_job;
int ds_stencil_begin(int nx, int ny, int nz, int px, int py, int pz, int rank, void* stream,
                     ds_stencil_job** job, int64_t* nnz, int64_t* nghosts);
int ds_stencil_finish(ds_stencil_job* job, int32_t* row_offsets, int32_t* cols, double* vals,
                      double* b, int64_t* ghost_keys);

/* ---- split_local_remote on the device (stencil.py:256-277) ------------
 * count: loc_off (nrows+1) and the local nnz; fill: both CSR parts (remote
 * columns re-based by -n_owned; rem_off has nrows+1 entries).             */
int ds_csr_split_count(int64_t nrows, int64_t n_owned, const int32_t* row_offsets,
                       const int32_t* cols, int32_t* loc_off, int64_t* nnz_local, void* stream);
int ds_csr_split_fill(int64_t nrows, int64_t n_owned, int64_t nnz, const int32_t* row_offsets,
                      const int32_t* cols, const double* vals, const int32_t* loc_off,
                      int64_t nnz_local, int32_t* loc_cols, double* loc_vals, int32_t* rem_off,
                      int32_t* rem_cols, double* rem_vals, void* stream);

/* ---- halo exchange pieces (stencil.py:280-319) ---------------------------
 * dst[k] = src[idx[k]]: packs a neighbour's send list, or -- single process,
 * all partitions visible (peer access enabled) -- writes the ghost slice
 * x_k[n+start : n+start+count] straight from x_q (stencil.py:293-295).      */
int ds_gather(int64_t count, const int32_t* idx, const double* src, double* dst, void* stream);

/* ---- format-dispatched entry (kernels.py:166-198) -----------------------
 * One descriptor for whichever format is active, so a DynamicMatrix costs
 * one switch in C like the reference's one dict lookup (kernels.py:186).  */
typedef struct ds_matrix {
  int32_t format;            /* DS_FMT_COO / DS_FMT_CSR / DS_FMT_DIA            */
  int32_t ndiags;            /* DIA                                             */
  int64_t nrows, ncols, nnz; /* nnz: stored entries (COO/CSR)                   */
  const int32_t* idx0;       /* COO row_indices | CSR row_offsets | DIA offsets */
  const int32_t* idx1;       /* COO/CSR col_indices                             */
  const double* values;      /* COO/CSR values | DIA (nrows, ndiags) row-major  */
  const int32_t* long_rows;  /* CSR: rows > 129 entries (ds_csr_analyze); sorted
                                COO: long-run (start, end) pairs (ds_coo_long_runs);
                                or NULL                                           */
  int64_t n_long;
  int32_t rows_sorted;       /* COO: row indices nondecreasing                  */
  int32_t max_row_len;       /* CSR / sorted COO: longest row if known, else 0  */
  const int32_t* row_perm;   /* CSR: rows grouped by length bin (ds_csr_bins), or NULL */
  int64_t bins[9];           /* CSR: bin b = row_perm[bins[b] .. bins[b+1])     */
  const int32_t* tiles;      /* CSR: ds_csr_tiles plan (header, tiles, leaves, scratch), or NULL */
  int64_t ntiles;
} ds_matrix;

/* Row-length bins for irregular CSR (rows stable-sorted by bin):
 *   0: empty, 1: 1-9, 2: 10-17, 3: 18-25, 4: 26-33, 5: 34-129,
 *   6: 130-1024 (warp per row), 7: > 1024 entries (CTA per row).
 * Rows <= 33 run on the TMA pipeline (or, with a fused dot, bins 1-4 with
 * their exact number of load rounds).  perm holds nrows int32; bins[0..8]
 * are written to host memory (synchronises).                               */
int ds_csr_bins(int64_t nrows, const int32_t* row_offsets, int32_t* perm, int64_t* bins,
                void* stream);
/* SpMV tile plan for irregular CSR (csr_tile_kernel): the rows are cut into
 * "row tiles" of consecutive rows of <= 129 entries holding < 512 entries
 * (a tile boundary where row_offsets crosses a multiple of 382), and every
 * longer row into "leaf tiles": np.add.reduceat sums a row as p[first] +
 * pairwise(rest), numpy's pairwise recursion splits n > 128 addends at
 * n/2 - (n/2)%8, and its leaves (64..128 addends) are packed 4 per tile.
 * All tiles run in one grid (entry-parallel products, one lane per row or
 * leaf for the exact sums); a second small kernel replays each long row's
 * recursion over its leaf sums.  plan (int32 words, capacity >= 
 * ds_csr_tiles_capacity(nrows, nnz)): [0..7] header {tiles, leaves, long
 * rows, leaf-list offset, long-row-list offset, scratch offset, row tiles},
 * then one int4 {A, B, E0, E1} per tile (row tile: rows [A, B); leaf tile,
 * A < 0: leaves -A-1 ..; entries [E0, E1)), (start, len) per leaf, (row,
 * first leaf) per long row, and one double of SCRATCH per leaf that every
 * SpMV writes -- SpMVs sharing one plan must not run concurrently.  Writes
 * *ntiles (= the descriptor's ntiles) and *words_used (the plan may be
 * copied to a buffer of that size); synchronises.                           */
int64_t ds_csr_tiles_capacity(int64_t nrows, int64_t nnz);
int ds_csr_tiles(int64_t nrows, const int32_t* row_offsets, int32_t* plan, int64_t capacity,
                 int64_t* ntiles, int64_t* words_used, void* stream);

/* Measurement probe, not part of the path: streams col_indices + values and
 * gathers x[col] for nnz entries (no row structure), a running sum per
 * thread (sink is written only in a never-taken branch).  Timing it gives
 * the random-gather floor of an irregular SpMV on this device (bench.py,
 * BASELINE config 4).                                                      */
int ds_probe_gather(int64_t nnz, const int32_t* col_indices, const double* values,
                    const double* x, double* sink, void* stream);

int ds_spmv(const ds_matrix* a, const double* x, double* y, int accumulate, void* stream);

/* Persisting-L2 access-policy window over [base, base+bytes) for kernels
 * launched or captured on `stream` afterwards (the solver keeps its vectors
 * L2-resident while the matrix streams with evict_first); _reset clears the
 * stream attribute, the persisting lines and the carve-out.
 * DS_ERR_NOT_SUPPORTED when the window exceeds the device's persisting L2.  */
int ds_l2_persist(const void* base, int64_t bytes, void* stream);
int ds_l2_persist_reset(void* stream);

/* ---- conjugate gradient building blocks (solver.py:56-189) --------------
 * The CG scalars live on the device in a ds_cg_scalars block.  Every kernel
 * below first tests s->done and returns when set, so a chunk of iterations
 * (or a captured CUDA graph of them) can be enqueued without host round
 * trips and the iteration count / residual history stay exact.
 *
 * Global dots: each partition writes its local dot to parts[k]; the global
 * value is the rank-ordered sum parts[0] + parts[1] + ... (the reference's
 * Python sum, solver.py:140-141).  With nparts_final > 0 the kernel that
 * completes parts[k] also runs the CG stage on parts[0..nparts_final) (the
 * single-partition fast path); otherwise the caller gathers every
 * partition's part (same device, or NCCL all-gather across ranks) and calls
 * ds_cg_finalize.                                                           */
typedef struct ds_cg_scalars {
  double rr;        /* r.r of the current residual                          */
  double pap;       /* p.Ap of the current iteration                        */
  double alpha, beta;
  double scale;     /* ||b||, or 1.0 when ||b|| == 0   (solver.py:98-99)    */
  double tol;
  double bb;
  double rr_new;
  int32_t iter;     /* iterations completed                                 */
  int32_t max_iters;
  int32_t done;     /* 0 running, 1 converged, 2 breakdown (p.Ap <= 0), 3 max_iters */
  int32_t pad;
  double rr_used;   /* deferred path: the rr that produced alpha (read by the p update) */
  int32_t iter_next;/* deferred path: iteration being completed                */
  int32_t pad2;
} ds_cg_scalars;

enum { DS_CG_STAGE_NONE = 0, DS_CG_STAGE_PAP = 1, DS_CG_STAGE_RR = 2, DS_CG_STAGE_SETUP = 3 };

/* Device workspace for one stream: fused-reduction partials and tickets.
 * Must be zero-filled once before first use.                               */
int64_t ds_cg_workspace_bytes(void);

/* y = A x (accumulate: y += A x); if dot_with != NULL also
 * *dot_out = dot_with[0:nrows] . y  (fused into the SpMV epilogue when the
 * kernel supports it), then the CG stage when nparts_final > 0.  s may be
 * NULL (no guard).                                                          */
int ds_cg_spmv_dot(const ds_matrix* a, const double* x, double* y, int accumulate,
                   const double* dot_with, double* dot_out, int stage, ds_cg_scalars* s,
                   double* history, const double* parts, int nparts_final, void* workspace,
                   void* stream);
/* r = 1*b + (-1)*ap; p = 1*r + 0*r (solver.py:89,101 / 155-167);
 * bb_out = b.b, rr_out = r.r (partition-local).                            */
int ds_cg_setup_residual(int64_t n, const double* b, const double* ap, double* r, double* p,
                         double* bb_out, double* rr_out, void* workspace, void* stream);
/* s <- tol/max_iters, scale from sum(bb_parts), rr from sum(rr_parts),
 * history[0], done (0 or 1 converged at x0, 3 when max_iters <= 0).        */
int ds_cg_setup_finalize(ds_cg_scalars* s, const double* bb_parts, const double* rr_parts,
                         int nparts, double tol, int32_t max_iters, double* history,
                         void* stream);
/* x = 1*x + alpha*p; r = 1*r + (-alpha)*ap; *rr_out = r.r, then stage RR
 * when nparts_final > 0 (solver.py:177-184).                               */
int ds_cg_update(int64_t n, double* x, double* r, const double* p, const double* ap,
                 ds_cg_scalars* s, double* rr_out, double* history, const double* parts,
                 int nparts_final, void* workspace, void* stream);
/* p = 1*r + beta*p  (solver.py:185-188) */
int ds_cg_direction(int64_t n, const double* r, double* p, const ds_cg_scalars* s, void* stream);
/* Stage PAP or RR over parts[0..nparts) (after an all-gather).             */
int ds_cg_finalize(int stage, ds_cg_scalars* s, double* history, const double* parts,
                   int nparts, void* stream);
/* Deferred-reduction iteration for ONE partition (no all-gather needed):
 * the SpMV (stage DS_CG_STAGE_DEFERRED in ds_cg_spmv_dot) and the update
 * only write fixed-order block partials; the NEXT kernel reduces them in its
 * prologue (every block identically) and derives alpha / breakdown, resp.
 * history / convergence / beta.  No completion tickets, no tail block: each
 * scalar is written by one kernel and read only by later ones.            */
enum { DS_CG_STAGE_DEFERRED = 4 };
int ds_cg_update_deferred(int64_t n, double* x, double* r, const double* p, const double* ap,
                          ds_cg_scalars* s, void* workspace, void* stream);
int ds_cg_direction_deferred(int64_t n, const double* r, double* p, ds_cg_scalars* s,
                             double* history, void* workspace, void* stream);
/* Both in one launch: update, a grid-wide barrier (co-resident grid,
 * cooperative launch when available), then every block reduces the r.r
 * partials and applies the direction.  DS_ERR_NOT_SUPPORTED (nothing
 * launched) for n < 2 or vectors not 16-byte aligned.                      */
int ds_cg_update_direction_deferred(int64_t n, double* x, double* r, double* p,
                                    const double* ap, ds_cg_scalars* s, double* history,
                                    void* workspace, void* stream);
/* The same two kernels for one partition per process: the prologue sums the
 * all-gathered partition dots pap_all[0..nparts) / rr_all[0..nparts)
 * sequentially in rank order (solver.py:140-141); the update's partition
 * r.r goes to *rr_mine (completion ticket) for the next all-gather.        */
int ds_cg_update_gathered(int64_t n, double* x, double* r, const double* p, const double* ap,
                          ds_cg_scalars* s, const double* pap_all, int nparts, double* rr_mine,
                          void* workspace, void* stream);
int ds_cg_direction_gathered(int64_t n, const double* r, double* p, ds_cg_scalars* s,
                             double* history, const double* rr_all, int nparts, void* workspace,
                             void* stream);
/* halo gather guarded by s->done (dst[k] = src[idx[k]])                    */
int ds_cg_gather(int64_t count, const int32_t* idx, const double* src, double* dst,
                 const ds_cg_scalars* s, void* stream);

/* ---- the solve loop on the device ---------------------------------------
 * begin: a graph with one WHILE conditional node (condition default 1 at
 * every launch) and `stream` capturing into its body; enqueue K iterations
 * and ds_cg_while_continue (condition = s->done == 0) on `stream`; end:
 * stop capturing, instantiate.  One ds_graph_exec_launch then iterates until
 * convergence / breakdown / max_iters without host round trips.            */
int ds_while_graph_begin(void* stream, void** graph, unsigned long long* handle);
int ds_cg_while_continue(unsigned long long handle, const ds_cg_scalars* s, void* stream);
int ds_while_graph_end(void* stream, void* graph, void** exec);
int ds_graph_exec_launch(void* exec, void* stream);
int ds_graph_destroy(void* graph, void* exec);

/* ---- one partition per process: NCCL halo exchange + global dots --------
 * (stencil.py:280-295 / solver.py:140-141 across processes).  NCCL is
 * resolved at run time from the libnccl.so.2 already loaded in the process.
 * The unique id is created on rank 0 and broadcast by the caller.          */
int ds_nccl_unique_id_bytes(void);
int ds_nccl_unique_id(char* out, int nbytes);
int ds_nccl_comm_init(const char* id_bytes, int nranks, int rank, void** comm);
int ds_nccl_comm_destroy(void* comm);
/* For each neighbour q (ascending rank): gather x_full[send_idx[q][k]] into
 * send_bufs[q] (the gathers are skipped once s->done != 0: p no longer
 * changes; s may be NULL = never skipped), then in one NCCL group send it to
 * peers[q] and receive recv_counts[q] doubles into x_full + recv_starts[q].
 * The sends and receives themselves are unconditional, so every rank posts
 * the same operations.                                                      */
int ds_halo_exchange(int nnbr, const int32_t* peers, const int64_t* send_counts,
                     const int32_t* const* send_idx, double* const* send_bufs,
                     const int64_t* recv_counts, const int64_t* recv_starts, double* x_full,
                     const ds_cg_scalars* s, void* comm, void* stream);
/* recv[r*count : (r+1)*count] = rank r's send (ncclAllGather, float64).   */
int ds_allgather_f64(const double* send, double* recv, int64_t count, void* comm, void* stream);

/* ---- one partition per process: peer-memory transport (CUDA IPC over
 * NVLink / NVSwitch; several ranks may also share one GPU) -----------------
 * The same exchanges as above with plain loads / stores on mapped peer
 * memory instead of NCCL.  Flags are uint32 words, raised (1) by their
 * producer and cleared (0) by their consumer.  wait_mode: DS_PEER_WAIT_SPIN
 * polls inside a kernel (traps after 30 s), DS_PEER_WAIT_MEMOP blocks the
 * stream with cuStreamWaitValue32 and clears with cuStreamWriteValue32.    */
#define DS_PEER_MAX_RANKS 64
#define DS_PEER_MAX_NBR 26
enum { DS_PEER_WAIT_SPIN = 0, DS_PEER_WAIT_MEMOP = 1 };
/* export: CUDA IPC handle of ptr's allocation + ptr's byte offset in it
 * (ds_ipc_handle_bytes() bytes); import maps it (lazy peer access) and
 * returns the address of ptr in this process; close unmaps.               */
int ds_ipc_handle_bytes(void);
int ds_ipc_export(const void* ptr, char* out);
int ds_ipc_import(const char* in, void** ptr);
int ds_ipc_close(void* ptr);
/* all_ptrs[r][stage*nranks + rank] = *mine and flag_ptrs[r][same] = 1 for
 * every rank r (r == rank: this rank's own, unmapped block), then wait until
 * my_flags[stage*nranks + r] is raised for every r and clear them: after it,
 * all_ptrs[rank][stage*nranks + 0..nranks) holds every partition's dot.    */
int ds_peer_allgather_f64(const double* mine, int stage, int rank, int nranks,
                          double* const* all_ptrs, unsigned* const* flag_ptrs,
                          unsigned* my_flags, int wait_mode, void* stream);
/* dst[q][j] = p[idx[q][j]] for j < counts[q] (remote stores into neighbour
 * q's ghost slots), then -- every store fenced at system scope -- raise
 * flags[q] (neighbour q's flag for this rank).  ticket: a zeroed device word
 * owned by this call site.                                                 */
int ds_peer_halo_push(int nnbr, const int64_t* counts, const int32_t* const* idx,
                      const double* p, double* const* dst, unsigned* const* flags,
                      unsigned* ticket, void* stream);
/* wait until each of flags[0..n) is raised, then clear it                   */
int ds_peer_wait_flags(int n, unsigned* const* flags, int wait_mode, void* stream);

/* ---- HPCG smoother and multigrid transfers (NOT in the
 * reference -- parity pinned to the oracle's restatement of HPCG's
 * ComputeSYMGS_ref / ComputeMG_ref with the 8-colour stencil ordering) -----
 * ds_symgs: one symmetric sweep in place, colours 0..n-1 then n-1..0 (the
 * second, identical visit of colour n-1 is skipped); rows of
 * colour c are color_rows[color_start[c] .. color_start[c+1]).  Per row:
 * s = r[i]; s -= a_ij*x[j] (j != i, stored order, no FMA); x[i] = s / a_ii. */
int ds_symgs(int64_t nrows, const int32_t* row_offsets, const int32_t* cols,
             const double* values, const int32_t* color_rows, const int64_t* color_start,
             int ncolors, const double* r, double* x, void* stream);
/* Colour-ordered ELL layout of the same sweep (coalesced slot loads):
 * ds_symgs_ell_width -> max off-diagonal count per row (synchronises stream);
 * round it up to a supported width (8, 16, 26, 32); ds_symgs_ell_fill writes
 * ell_cols/ell_vals [width][nrows] (slot-major over colour position),
 * ell_len[nrows] and diag[nrows]; ds_symgs_ell sweeps bitwise like ds_symgs. */
int ds_symgs_ell_width(int64_t nrows, const int32_t* row_offsets, const int32_t* cols,
                       int32_t* width_out, void* stream);
int ds_symgs_ell_fill(int64_t nrows, int32_t width, const int32_t* row_offsets,
                      const int32_t* cols, const double* values, const int32_t* color_rows,
                      int32_t* ell_cols, double* ell_vals, int32_t* ell_len, double* diag,
                      void* stream);
int ds_symgs_ell(int64_t nrows, int32_t width, const int32_t* color_rows,
                 const int64_t* color_start, int ncolors, const int32_t* ell_cols,
                 const double* ell_vals, const int32_t* ell_len, const double* diag,
                 const double* r, double* x, void* stream);
/* Offset ELL (the sweep without column indices): for an operator whose
 * off-diagonals fall on <= 32 distinct offsets (col - row, ascending in
 * `offsets`, padded with 0 to `width` = 26 or 32), slot q of colour-ordered
 * position k is offset q: oell_vals[q * nrows + k] (0.0 where absent), mask[k]
 * bit q = present, diag[k].  Same arithmetic as ds_symgs_ell, operation for
 * operation; 8 B per slot streamed instead of 12.  The fill returns
 * DS_ERR_NOT_SUPPORTED if a row holds an offset outside the list.  The fill
 * takes the offsets in DEVICE memory, the sweep in HOST memory (they travel
 * as a kernel parameter).                                                  */
int ds_symgs_oell_fill(int64_t nrows, int32_t width, const int32_t* offsets,
                       const int32_t* row_offsets, const int32_t* cols, const double* values,
                       const int32_t* color_rows, double* oell_vals, uint32_t* mask,
                       double* diag, void* stream);
int ds_symgs_oell(int64_t nrows, int32_t width, const int32_t* offsets_host,
                  const int32_t* color_rows, const int64_t* color_start, int ncolors,
                  const double* oell_vals, const uint32_t* mask, const double* diag,
                  const double* r, double* x, void* stream);
/* Device-resident PCG (ComputeCG_ref with z = M r): the host writes the block
 * after setup; each iteration is spmv(p) -> ds_dot(p,Ap -> &pap) ->
 * ds_pcg_alpha -> ds_pcg_axpy(x += alpha p) -> ds_pcg_axpy(r -= alpha Ap) ->
 * ds_dot(r,r -> &rr) -> ds_pcg_check -> V-cycle(r -> z) ->
 * ds_dot(r,z -> &rtz_new) -> ds_pcg_beta -> ds_pcg_axpy(p = z + beta p).
 * Vector updates are no-ops once done != 0 (graph replays may overshoot).  */
typedef struct ds_pcg_scalars {
  double rtz, pap, rr, rtz_new, alpha, beta, scale, tol;
  int32_t iter, max_iters;
  int32_t done;     /* 0 running, 1 converged, 2 breakdown, 3 max_iters     */
  int32_t pad;
} ds_pcg_scalars;
int ds_pcg_alpha(ds_pcg_scalars* s, void* stream);
int ds_pcg_check(ds_pcg_scalars* s, double* history, void* stream);
int ds_pcg_beta(ds_pcg_scalars* s, void* stream);
/* w = 1.0*x + c*y, c = *coef_dev (negated when negate != 0); guarded by s->done */
int ds_pcg_axpy(int64_t n, double* w, const double* x, const double* coef_dev, int negate,
                const double* y, const ds_pcg_scalars* s, void* stream);
/* rc[i] = r[f2c[i]] - axf[f2c[i]]  /  x[f2c[i]] += xc[i]                   */
/* Fused residual + restriction on a DIA operator: rc[i] = r[f] - (A z)[f],
 * f = f2c[i], forming only the coarse rows of A z (bitwise equal to
 * ds_spmv + ds_mg_restrict).  DS_ERR_NOT_SUPPORTED for other formats.      */
int ds_mg_restrict_residual(const ds_matrix* a, int64_t ncoarse, const int32_t* f2c,
                            const double* z, const double* r, double* rc, void* stream);
int ds_mg_restrict(int64_t ncoarse, const int32_t* f2c, const double* r, const double* axf,
                   double* rc, void* stream);
int ds_mg_prolong(int64_t ncoarse, const int32_t* f2c, const double* xc, double* x,
                  void* stream);

/* ---- DIA diagonal column helpers (kernels.py:258-262, 325-330) --------- */
/* direction 0: out[i] = values[i*ndiags + j0] (i < n); 1: values[...] = d[i] */
int ds_dia_diag_column(int64_t n, int32_t ndiags, int32_t j0, double* values, double* vec,
                       int direction, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DYNSPARSE_B200_H */
