/*
 * skx.h -- C ABI of libskx, the B200 (sm_100a) implementation of the hot path
 * of the sketched Tucker-ALS algorithm (arXiv 2104.01101) whose reference is
 * the pure-Python package `sketchals` (/root/reference/pkg/src/sketchals,
 * cited as src/<file>:<line>).
 *
 * The reference has no FFI: its boundary is the Python function API re-exported
 * by src/__init__.py:3-69.  The Python package paper_2104_01101_b200 keeps that
 * API verbatim and binds these entry points with ctypes (INTEGRATION.md shows
 * the binding).  Each entry cites the reference function it replaces.
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless its name ends in _h;
 *  - every call takes the cudaStream_t `stream` (as void*) and is asynchronous;
 *  - no hidden allocations: calls that need scratch take (ws, ws_bytes); pass
 *    ws = NULL to query the required size, returned in *ws_bytes;
 *  - return codes: 0 ok, 1 invalid argument (-> ValueError), 2 rank deficient
 *    (-> RankDeficientError), 3 CUDA error; skx_last_error() has the message;
 *  - matrices are row-major float64; index arrays int32 unless stated;
 *  - "packed table": uint32 per index, low 31 bits = bucket, bit 31 = sign -1.
 *
 * Random streams follow numpy 2.3.5 Generator(Philox) exactly: raw u64 number p
 * of a stream with key (k0,k1) is word p%4 of Philox4x64-10 at counter
 * (p/4+1,0,0,0).  The host keeps numpy's Generator state and hands the device
 * (key, raw position, buffered-uint32 flag and value).
 */
#ifndef SKX_H_
#define SKX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKX_OK 0
#define SKX_EINVAL 1
#define SKX_ERANK 2
#define SKX_ECUDA 3

const char* skx_last_error(void);
/* number of kernels libskx has launched since load (all threads) */
long long skx_launch_count(void);
int skx_version(void);

/* ---------------------------------------------------------------- K0: RNG */

/* Generator.random(n) from raw position p0 (numpy next_double).
 * Replaces the draws inside rng.choice at src/sketching.py:211. */
int skx_philox_uniform(uint64_t k0, uint64_t k1, uint64_t p0, int64_t n, double* out,
                       void* stream);

/* Generator.standard_normal(n) (numpy 256-level ziggurat, bit-exact) starting
 * at the raw position *p0 (device u64); writes the position after the last
 * consumed draw to *p_end (device u64; may alias p0).
 * Replaces rng.standard_normal at src/linalg.py:107 and src/sketching.py:323. */
int skx_philox_normal(uint64_t k0, uint64_t k1, const uint64_t* p0, int64_t n, double* out,
                      uint64_t* p_end, void* ws, size_t* ws_bytes, void* stream);

/* Lemire rejection scan for Generator.integers(0, k, .): lists (unordered)
 * the absolute 32-bit positions A = 2*raw + half of every draw in raw words
 * [raw_lo, raw_hi) that numpy would reject (rejection depends only on the
 * drawn value, so the scan may start before the call's exact start is known).
 * Count written to *count; positions beyond cap are counted, not stored.
 * Used to place RRF CountSketch tables (src/sketching.py:54-56). */
int skx_lemire_scan(uint64_t k0, uint64_t k1, uint64_t raw_lo, uint64_t raw_hi, uint32_t k,
                    uint64_t* rej, int64_t cap, unsigned long long* count, void* stream);

/* ------------------------------------------------- K1/K2: TensorSketch */

/* Packed per-mode tables from the polynomial-hash coefficients drawn on the
 * host (4 hash then 5 sign coefficients per mode, coeffs_h = nmodes x 9).
 * Replaces _poly_hash/_hash_family/_sign_family, src/sketching.py:25-43,80-86.
 * tab receives sum(extents) entries, mode after mode. */
int skx_ts_tables(int nmodes, const int64_t* extents_h, const int64_t* coeffs_h, int64_t m,
                  uint32_t* tab, void* stream);

/* ------------------------------------------------------ COO layouts */

/* Record stride (8-byte words) of the fibre-major layout for a sparse order
 * ndim: 2 (16-byte records) for ndim <= 3, 3 for ndim 4..5, -1 otherwise. */
int skx_coo_rec_words(int ndim);

/* Fibre-major layout of `mode` for a lexsorted COO tensor (coords = ndim x nnz
 * SoA int32, vals f64): records {int32 other coords (ascending modes),
 * f64 value} ordered by (i_mode, others) -- a stable radix sort by i_mode --
 * and colptr (s_mode + 1 offsets).  The device counterpart of the cached
 * unfoldings matricize_t / mode_sort (src/tensors.py:151-194, 89-95). */
int skx_coo_fibre(int ndim, const int64_t* shape_h, int mode, int64_t nnz, const int32_t* coords,
                  const double* vals, void* rec_out, int64_t* colptr, void* ws, size_t* ws_bytes,
                  void* stream);

/* Same layout for an order-3 tensor, with mode `mode`'s TensorSketch bucket
 * and sign folded into each record (tab/tab_off_h/m as skx_ts_rhs_coo): the
 * second coordinate word holds c1 | bucket << bb | neg << 31 with
 * bb = ceil(log2 s_b) of the second other mode.  *c1_mask (host) receives
 * (1 << bb) - 1, the mask every consumer applies to recover c1.  Fails with 1
 * (invalid argument) when bb + ceil(log2 m) > 31. */
int skx_coo_fibre_ts(const int64_t* shape_h, int mode, int64_t nnz, const int32_t* coords,
                     const double* vals, const uint32_t* tab, const int64_t* tab_off_h,
                     int64_t m, void* rec_out, int64_t* colptr, uint32_t* c1_mask, void* ws,
                     size_t* ws_bytes, void* stream);
/* Records [lo, hi) of the mode-0 fibre layout of a lexsorted COO (input order,
 * the layout skx_coo_fibre builds for mode 0; its colptr is the mode-0 slice
 * pointer array), coordinate rows of stride ld: the layout built chunk by
 * chunk while a host COO is uploaded (src/tensors.py:89-95 mode_sort(0)). */
int skx_coo_pack0_range(int ndim, int64_t ld, int64_t lo, int64_t hi, const int32_t* coords,
                        const double* vals, void* rec_out, void* stream);

/* Y^T = (S . T_(n)^T)^T for a COO tensor in the fibre-major layout of mode n
 * (skx_coo_fibre); tab = packed tables of the other modes concatenated,
 * tab_off_h offsets; c1_mask recovers the last other coordinate (0xffffffff
 * for skx_coo_fibre layouts).  packed_bb >= 0: the layout came from
 * skx_coo_fibre_ts with THIS operator's tables and carries bucket/sign above
 * bit packed_bb (tab unused).  yt is s_n x m (row i_n = column i_n of the
 * reference's m x s_n output).  Replaces ts_apply_rhs sparse branch,
 * src/sketching.py:150-167. */
int skx_ts_rhs_coo(int n_other, int64_t s_n, const int64_t* colptr, const void* rec,
                   const uint32_t* tab, const int64_t* tab_off_h, int64_t m, uint32_t c1_mask,
                   int packed_bb, double* yt, void* stream);

/* Same for a dense C-order tensor (ndim, shape_h) and target mode.
 * Replaces ts_apply_rhs dense branch, src/sketching.py:168-175. */
int skx_ts_rhs_dense(const double* t, int ndim, const int64_t* shape_h, int mode,
                     const uint32_t* tab, const int64_t* tab_off_h, int64_t m, double* yt,
                     void* ws, size_t* ws_bytes, void* stream);

/* Composed packed table over all P = prod(ext) rows of the chain (first mode
 * slowest): bucket = sum of per-mode buckets mod m, sign = product
 * (src/sketching.py:92-102).  Lets a dense (P x c) right-hand side be
 * sketched by skx_rrf_stage1_dense. */
int skx_ts_combine(int n, const int64_t* ext_h, const uint32_t* tab, const int64_t* tab_off_h,
                   int64_t m, int64_t P, uint32_t* out, void* stream);

/* Kronecker-sketch plan of a TensorSketch operator: per-mode bucket-sorted,
 * run-length-encoded row lists (depends only on the tables, so it is built once
 * per operator and reused by every sub-problem).  plan = NULL or ws = NULL
 * queries *plan_bytes / *ws_bytes. */
int skx_ts_kron_plan(int n_other, const int64_t* ext_h, const uint32_t* tab,
                     const int64_t* tab_off_h, int64_t m, void* plan, size_t* plan_bytes,
                     void* ws, size_t* ws_bytes, void* stream);

/* Z = S . kron(A_1, ..., A_k) (first factor slowest), m x prod(R), written
 * COLUMN-major (z[col*m + row]) -- the layout cuSOLVER's QR consumes.
 * factors_h: host array of device pointers to s_k x R_k row-major factors.
 * Replaces ts_apply_kron, src/sketching.py:113-147 (exact circular convolution
 * instead of FFT; equal up to rounding). */
int skx_ts_kron_apply(int n_other, const int64_t* ext_h, const int64_t* ranks_h,
                      const double* const* factors_h, const void* plan, int64_t m, double* z,
                      void* ws, size_t* ws_bytes, void* stream);

/* ------------------------------------------------------ K3: leverage */

/* Leverage gather of an order-3 COO tensor for a mode-1 or mode-2
 * sub-problem straight from its mode-0 fibre layout (skx_coo_fibre mode 0;
 * c1_mask as skx_ts_rhs_coo): sample j's fibre (idx[2j] = i0, idx[2j+1] =
 * the other index) lies in slice i0.  Call twice: with hit_col == NULL to
 * write hit_off (m + 1 offsets, hit_off[m] = total), then with outputs of
 * `cap` entries: per sample, ascending column, value scaled by w[j].
 * Replaces _fetch_rows on the CSR of T_(n)^T (src/sketching.py:262-267). */
int skx_slice_hits(int mode, int64_t s0, const int64_t* colptr0, const void* rec0,
                   uint32_t c1_mask, const int64_t* idx, const double* w, int64_t m,
                   int64_t* hit_off, int64_t* hit_col, double* hit_val, int64_t cap, void* ws,
                   size_t* ws_bytes, void* stream);

/* p = max(scores,0)/sum, cdf = cumsum(p)/cdf[-1] (src/sketching.py:207-210 and
 * numpy Generator.choice).  */
int skx_lev_prepare(const double* scores, int64_t s, double* p, double* cdf, void* ws,
                    size_t* ws_bytes, void* stream);

/* Leverage scores l_i = ||a_i R^-1||^2 of a tall s x R factor (R <= 32),
 * R from a Cholesky of the Gram A^T A (src/linalg.py:73-84 leverage_scores;
 * any R of a QR of A gives the same Q = A R^-1).  *bad (device int) = 1
 * when the Gram route cannot reproduce the reference's Householder rank test
 * (|R_ii| < 1e-12 ||A||_F, src/linalg.py:44-52) or loses score bits: failed
 * pivot or min R_jj < 1e-2 max R_jj; the caller then decides on a Householder
 * (TSQR) factorisation.  Orthonormal factors (the driver's) never flag. */
int skx_lev_scores(const double* a, int64_t s, int R, double* scores, int* bad, void* ws,
                   size_t* ws_bytes, void* stream);

/* Draw m samples per mode: for mode k, uniforms at raw positions
 * p0 + k*m + j; idx[j*n_other+k] = searchsorted(cdf_k, u, 'right');
 * w[j] = 1/sqrt(m * prod_k p_k[idx]).  src/sketching.py:211-216. */
int skx_lev_sample(int n_other, const int64_t* ext_h, const double* const* p_h,
                   const double* const* cdf_h, int64_t m, uint64_t k0, uint64_t k1, uint64_t p0,
                   int64_t* idx, double* w, void* stream);

/* Deterministic leverage sampling: idx (m x k, int64) = the original
 * multi-indices of the m largest products of one score per list, in the pop
 * order of the reference's best-first heap (products descending, ties by
 * lexicographic multi-index, a tuple entering the frontier only once a
 * predecessor was popped) -- src/sketching.py:224-259 `_top_m_products`,
 * used by lev_build(variant="deterministic") at :218-220. scores_h: host
 * array of k device pointers (len_h[j] doubles each). */
int skx_top_m_products(int k, const int64_t* len_h, const double* const* scores_h, int64_t m,
                       int64_t* idx, void* ws, size_t* ws_bytes, void* stream);

/* Z[j,:] = w_j kron_k A_k[idx_jk,:], column-major m x prod(R)
 * (src/sketching.py:280-285). */
int skx_kron_rows(int n_other, const int64_t* ranks_h, const double* const* factors_h,
                  const int64_t* idx, const double* w, int64_t m, double* z, void* stream);

/* Y[j,:] = w_j * T_(n)^T[flat_j,:] for a dense tensor (src/sketching.py:262-266). */
int skx_gather_fibers_dense(const double* t, int ndim, const int64_t* shape_h, int mode,
                            const int64_t* idx, const double* w, int64_t m, double* y,
                            void* stream);

/* Sparse fibre gather.  keys: per-mode "other-major" layout sorted by
 * key = flat_other * s_n + i_n (int64), vals matching.  Sample j's hits are
 * hit_col/hit_val[hit_off[j] .. hit_off[j+1]) (i_n ascending, value w_j*v);
 * hit_off has m+1 entries, hit_off[m] = total (entries past cap dropped).
 * Deterministic (count, scan, write).  src/sketching.py:262-264. */
int skx_gather_fibers_coo(int n_other, const int64_t* ext_h, int64_t s_n, int64_t nnz,
                          const int64_t* keys, const double* vals, const int64_t* idx,
                          const double* w, int64_t m, int64_t* hit_off, int64_t* hit_col,
                          double* hit_val, int64_t cap, void* ws, size_t* ws_bytes, void* stream);

/* The nonzeros of a lexsorted COO tensor (coords_h[k]: int32 coordinates of
 * mode k, extents shape_h) whose other-mode flat index is in sflat (m values,
 * sorted ascending, unique): their keys flat * s_mode + i_mode and values, in
 * no particular order (the caller sorts the few hits), at most cap of them;
 * *count (device) = the number found.  One pass over the coordinates replaces
 * the sorted key array of skx_gather_fibers_coo (src/sketching.py:262-264). */
int skx_filter_fibers_coo(int ndim, const int64_t* shape_h, int mode, int64_t nnz,
                          const int32_t* const* coords_h, const double* vals, const int64_t* sflat,
                          int64_t m, int64_t* out_key, double* out_val, int64_t cap,
                          uint64_t* count, void* stream);

/* ------------------------------------------------- K4: range finder */

/* Chunk-wise skx_rrf_stage1_fx for a tensor arriving in pieces: the caller
 * zeroes `acc` (s_mode * k2 cells of 32 bytes), calls _acc per chunk (coords
 * = the chunk's first entry of SoA row 0, rows ld apart) and _convert once.
 * Same exact sums.  max_per_cell: a bound on the nonzeros in any block of
 * 2^CB mode-n rows (skx_stage_compact3's rowmax; CB as skx_rrf_stage1_fx
 * chooses it), or -1 if unknown; *limb_flag records the limb count used. */
int skx_rrf_stage1_fx_acc(int ndim, const int64_t* shape_h, int mode, int64_t n,
                          const int32_t* coords, int64_t ld, const double* vals, int emax,
                          uint64_t k0, uint64_t k1, uint64_t p0, uint32_t has_pending,
                          uint32_t pending, uint64_t sign_q0, const uint64_t* rej, int64_t nrej,
                          int64_t k2, unsigned long long* acc, unsigned int* limb_flag,
                          int64_t max_per_cell, void* stream);
int skx_rrf_stage1_fx_convert(const unsigned long long* acc, int64_t cells, int emax,
                              const unsigned int* limb_flag, double* stage1, void* stream);

/* Range of the nonzero values: out3[0] = max, out3[1] = min unbiased binary
 * exponent of the nonzero |v|, out3[2] = 1 if any value is inf/NaN or
 * subnormal.  Decides whether skx_rrf_stage1_fx can sum exactly. */
int skx_value_range(const double* vals, int64_t nnz, int* out3, void* stream);

/* RRF stage 1 (CountSketch of T_(mode), s_mode x k2) straight from the
 * lexsorted SoA COO, without a fibre layout: every nonzero adds
 * sign(j) * v * 2^S (S = 93 - emax) into an exact fixed-point accumulator
 * (three 32-bit limbs summed by 64-bit atomic reductions; integer sums are
 * order independent, so the result is deterministic) which is rounded once
 * to double.  Requires the
 * skx_value_range result: no non-finite values and emin >= emax - 41
 * (every contribution then is an exact integer).  Same tables and stream
 * positions as skx_rrf_stage1_coo (src/sketching.py:54-56, 327-341).
 * Workspace: 32 * s_mode * k2 bytes. */
int skx_rrf_stage1_fx(int ndim, const int64_t* shape_h, int mode, int64_t nnz,
                      const int32_t* coords, const double* vals, int emax, uint64_t k0,
                      uint64_t k1, uint64_t p0, uint32_t has_pending, uint32_t pending,
                      uint64_t sign_q0, const uint64_t* rej, int64_t nrej, int64_t k2,
                      double* stage1, void* ws, size_t* ws_bytes, void* stream);

/* stage1[i_n, c] = sum_j T_(n)[i_n, j] sign_j [hash_j == c] where hash/sign are
 * the numpy draws integers(0,k2,P) then integers(0,2,P) of the u32 run
 * (p0, has_pending, pending), hash draws shifted past the sorted rejection
 * list rej (nrej entries).  COO input in fibre-major layout (skx_coo_fibre).
 * Replaces CountSketchOp.build + composite_apply stage 1, src/sketching.py:
 * 54-56, 327-340. */
int skx_rrf_stage1_coo(int n_other, const int64_t* ext_h, int64_t s_n, const int64_t* colptr,
                       const void* rec, uint64_t k0, uint64_t k1, uint64_t p0,
                       uint32_t has_pending, uint32_t pending, uint64_t sign_q0,
                       const uint64_t* rej, int64_t nrej, int64_t k2, uint32_t c1_mask,
                       double* stage1, void* stream);

/* Fill n u64 with UINT64_MAX (pre-fill of a rejection buffer). */
int skx_fill_u64max(uint64_t* a, int64_t n, void* stream);

/* Sort the rejection list of skx_lemire_scan (cap entries, pre-filled with
 * UINT64_MAX), map it onto the run indices r_i of an integers() call starting
 * at raw word p0 (preceded by the buffered high half of raw word pend_raw when
 * has = 1), and write the d-array d_i = r_i - i (padded with UINT64_MAX) and
 * #{d_i <= P-1} -- the rejections among the first P accepted draws -- to
 * *n_le.  The sign run then starts at run index P + *n_le. */
int skx_lemire_finish(uint64_t* rej, const unsigned long long* count, int64_t cap, uint64_t p0,
                      uint32_t has, uint64_t pend_raw, uint64_t P, uint64_t* d,
                      unsigned long long* n_le, void* ws, size_t* ws_bytes, void* stream);

/* Materialise the packed (hash|sign) table for columns [0, P) (dense inputs). */
int skx_rrf_table(uint64_t k0, uint64_t k1, uint64_t p0, uint32_t has_pending,
                  uint32_t pending, uint64_t sign_q0, const uint64_t* rej, int64_t nrej,
                  int64_t P, int64_t k2, uint32_t* tab, void* stream);

/* Dense stage 1 given a full packed table over the P_n columns (s_n x k2 out). */
int skx_rrf_stage1_dense(const double* t, int ndim, const int64_t* shape_h, int mode,
                         const uint32_t* tab, int64_t k2, double* stage1, void* ws,
                         size_t* ws_bytes, void* stream);

/* --------------------------------------- K5/K7: residual and fitness */

/* out[0] = sum_{o,x} (sum_r U[o,r] Vt[r,x] - Y[o*ld + x])^2: the squared
 * residual || Z core_t a^T - Y ||_F^2 of a sub-problem (src/tucker.py:274) with
 * P = Z core_t, in whichever orientation makes Y's unit-stride index inner
 * (U = a, Vt = P^T for Y^T storage; U = P, Vt = a^T for row-major Y). */
int skx_resid_sq(const double* u, const double* vt, int64_t n_out, int64_t n_in, int64_t R,
                 const double* y, int64_t ld, double* out, void* ws, size_t* ws_bytes,
                 void* stream);

/* R factor (w x w, row-major, upper) of the n x w matrix A[i,j] = a[i*rs + j*cs]
 * by TSQR with Householder blocks (LAPACK dlarfg signs), w <= 96.  Replaces the
 * LAPACK QRs of tall-skinny operands: np.linalg.qr in src/linalg.py:45 (factor
 * leverage scores) and the SVDs of src/linalg.py:59 / src/tucker.py:141, which
 * are taken as SVD(R). */
int skx_tsqr_r(const double* a, int64_t n, int w, int64_t rs, int64_t cs, double* r, void* ws,
               size_t* ws_bytes, void* stream);

/* Upper Cholesky factor (R^T R = g, row-major n x n, n <= 128) in one CTA;
 * *info = 0, or k+1 when pivot k is not positive.  Used by the CholeskyQR2
 * factorisation of the sketched system (src/linalg.py:103). */
int skx_chol_upper(const double* g, int n, double* r, int* info, void* stream);

/* One-sided Jacobi SVD of the n x n matrix A[i,j] = a[i*rs + j*cs] (n <= 112):
 * A = U diag(s) V^T with s descending, U and V row-major.  Replaces the LAPACK
 * SVD of small R factors (src/linalg.py:59, src/tucker.py:141). */
int skx_jacobi_svd(const double* a, int n, int64_t rs, int64_t cs, double* u, double* s,
                   double* v, void* stream);

/* Middle step of the associated rsvd_lrls (src/linalg.py:105-110) for a test
 * width w < r: with B = Q_z^T (Y G) (r x w, row-major) and the upper R_z
 * (r x r, row-major), q = thin-Q of R_z^-1 B (Householder, LAPACK sign
 * convention) and x = R_z^-T q, both r x w row-major.  One CTA; r <= 128,
 * w <= 32.  Replaces np.linalg.solve / np.linalg.qr on the small operands. */
int skx_lrls_mid(const double* rz, const double* b, int r, int w, double* q, double* x,
                 void* stream);

/* Upper Cholesky factor R (R^T R = g) AND its inverse R^-1 of an SPD n x n
 * Gram (row-major; n <= 512) in one CTA: blocked left-looking Cholesky and
 * blocked bottom-up inverse on FP64 tensor cores.  *info = 0, or k+1 when
 * pivot k is not positive (r and rinv are then zero).  The wide-system
 * (r = prod of the other ranks > 128: configs 3 and 5) step of the Cholesky
 * QR that stands in for reduced_qr(z) (src/linalg.py:38-52, called at
 * src/linalg.py:103); replaces cuSOLVER potrf + a TRSM against I. */
int skx_chol_inv_upper(const double* g, int n, double* r, double* rinv, int* info, void* stream);

/* Thin Q (r x w row-major, w <= 32, w <= r) of the r x w row-major matrix c by
 * Householder reflections with LAPACK's geqr2/org2r conventions, one CTA
 * (2 r w doubles of shared memory).  The QR of X_ls G in rsvd_lrls
 * (src/linalg.py:109) for wide systems (r > 128). */
int skx_house_q(const double* c, int r, int w, double* q, void* stream);

/* RRF stage 1 with L2-resident accumulators (leverage runs, config 5): the
 * nonzeros of the lexsorted order-ndim COO (int32 SoA coords, ndim rows of
 * nnz) partitioned by output row block for up to two RRF modes (modes_h[0..
 * nmode-1]) into records key = i_n << 40 | j (j = flat other-mode index,
 * others ascending, first slowest -- the unfolding column of
 * src/tensors.py:151-166), value.  RNG-independent: runs while the rejection
 * scans occupy the SMs.  Workspace queried with ws = NULL. */
int skx_rrf_partition(int ndim, const int64_t* shape_h, int64_t nnz, const int32_t* coords,
                      const double* vals, int nmode, const int* modes_h, uint64_t* key0,
                      double* val0, uint64_t* key1, double* val1, void* ws, size_t* ws_bytes,
                      void* stream);

/* Stage 1 of the RRF composite sketch (src/sketching.py:327-341 with the
 * tables of :305-324) of one mode from its partitioned records: exact
 * fixed-point sums as skx_rrf_stage1_fx (bitwise the same result), with the
 * accumulator rows of the current row block resident in L2.  rows = the
 * mode's coordinate row of the COO (row-count bound for the limb count). */
int skx_rrf_stage1_rec(int64_t s_n, uint64_t P, int64_t nnz, const int32_t* rows,
                       const uint64_t* keys, const double* vals, int emax, uint64_t k0,
                       uint64_t k1, uint64_t p0, uint32_t has_pending, uint32_t pending,
                       uint64_t sign_q0, const uint64_t* rej, int64_t nrej, int64_t k2,
                       double* stage1, void* ws, size_t* ws_bytes, void* stream);

/* Host function (no GPU): the compact order-3 staging of an int64 (nnz, 3)
 * COO, built once at SparseTensor.from_sorted -- validated on the way
 * (*status: 0 ok, 1 coordinate out of range, 2 not strictly lexsorted;
 * src/tensors.py:35-60) -- slice pointers ptr0[s0 + 1], packed[e] = (d << b2)
 * | i2 (d = i1 increment inside the slice, absolute at a slice start; d >=
 * 2^(32-b2) - 1 escapes to exc_idx/exc_val of capacity cap, *n_exc = the
 * number needed). */
int skx_stage_compact3(const int64_t* coords, int64_t nnz, int64_t s0, int64_t s1, int64_t s2,
                       int b2, int64_t* ptr0, uint32_t* packed, int64_t* exc_idx,
                       int32_t* exc_val, int64_t cap, int64_t* n_exc, int* status);

/* Host function (no GPU), also at staging: what the device would otherwise
 * compute with a full pass and a host round trip before any RRF stage-1 sum
 * can start -- the value range as skx_value_range (vrange3) and, for modes 1
 * and 2, the largest nonzero count of any block of 2^CB rows, CB the smallest
 * with ceil(s_n / 2^CB) <= 32768 (rowmax2: the limb bound of skx_rrf_stage1_*). */
int skx_stage_stats3(const int64_t* coords, const double* vals, int64_t nnz, int64_t s1, int64_t s2,
                     int* vrange3, int64_t* rowmax2);

/* Restore the int32 SoA device layout (3 rows of ld) of the lexsorted
 * order-3 COO for slices [s_lo, s_hi) from its compact host staging (the
 * tensor object's pinned upload form, SparseTensor.from_sorted): ptr0 = the
 * mode-0 slice pointers (device, s_0 + 1), packed[e] = (d << b2) | i2 with d
 * the i1 increment inside the slice (absolute for a slice's first nonzero;
 * d = 2^(32-b2) - 1 escapes to exc_val at the sorted index exc_idx).  The
 * layout the reference keeps in SparseTensor.coords (src/tensors.py:26-60). */
int skx_coo_unpack3(const int64_t* ptr0, int64_t s_lo, int64_t s_hi, const uint32_t* packed,
                    int b2, const int64_t* exc_idx, const int32_t* exc_val, int64_t n_exc,
                    int32_t* coords, int64_t ld, void* stream);

/* Skip-mode sparse TTMc of an order-3 COO tensor (ttmc(t, factors, skip=n),
 * src/tensors.py:261-277): from mode n's fibre-major layout (skx_coo_fibre /
 * skx_coo_fibre_ts with c1_mask), out (s_n x R1*R2, row-major; column
 * k1*R2 + k2) = sum over each column's nonzeros of v * A1[i1,k1] * A2[i2,k2]
 * in layout order, products and sums unfused (numpy's rounding).  A1 (s_1 x
 * R1) and A2 (s_2 x R2) are the first and second other modes' factors,
 * row-major; R1*R2 <= 1024. */
int skx_ttmc3_skip_coo(int64_t s_n, const int64_t* colptr, const void* rec, uint32_t c1_mask,
                       const double* a1, int r1, const double* a2, int r2, double* out,
                       void* stream);

/* Decision flags of the sketched Cholesky QR (src/linalg.py:44-52 and the
 * orthogonality check of the one-pass factor), all r x r row-major: G1 = Z^T Z,
 * its Cholesky factor R1 (+ info), G2 = Q1^T Q1.  out[0] unsafe, out[1] one
 * pass suffices, out[2] rank-deficient, out[3] = out[0] | !out[1] | out[2]. */
int skx_cholqr_flags(const double* g1, const double* r1, const int* info, const double* g2, int r,
                     int* out, void* stream);

/* Mode-last copy of a dense C-order tensor: out has mode `mode` moved to the
 * fastest-varying position, the other modes in their order (the layout in
 * which every dense sketch of that mode takes the gather form). */
int skx_mode_last(const double* t, int ndim, const int64_t* shape_h, int mode, double* out,
                  void* stream);

/* out[0] = sum(x^2) with a fixed-order reduction. */
int skx_sumsq(const double* x, int64_t n, double* out, void* ws, size_t* ws_bytes,
              void* stream);

/* Tucker cross term <ttmc(T,{A}), C> over a lexsorted COO tensor (coords =
 * ndim x nnz SoA int32), factors_h device pointers (s_k x R_k), core C
 * (C-order R_0 x ... x R_{N-1}); colptr0/rec0 (the mode-0 fibre-major layout,
 * may be NULL; c1_mask as skx_ts_rhs_coo) enable the order-3 sliced kernel.
 * out[0] = cross.
 * Replaces the sparse ttmc + vdot at src/tensors.py:249-258, 351-352. */
int skx_tucker_cross_coo(int ndim, const int64_t* shape_h, const int64_t* ranks_h,
                         int64_t nnz, const int32_t* coords, const double* vals,
                         const double* const* factors_h, const double* core,
                         const int64_t* colptr0, const void* rec0, uint32_t c1_mask, double* out,
                         void* ws, size_t* ws_bytes, void* stream);

/* Full TTMc P = X x_0 A0^T x_1 A1^T x_2 A2^T (400 x R0 row-major: P[(b*20+c),
 * a]) of an order-3 COO at ranks (R0 <= 32, 20, 20) from its mode-0 fibre
 * layout (colptr0, rec0, c1_mask as skx_tucker_cross_coo): per-slice sums
 * v a1 a2^T on FP64 tensor cores with both factor rows by TMA gather4, then
 * one GEMM with A0.  <P, C> is the cross term of any core C on these factors
 * (src/tensors.py:217-258, 339-353): Algorithm 6's last Tucker fitness and
 * its final CP fitness (CP model = Tucker model with core [[w; B_0, B_1,
 * B_2]], src/cp.py:214-224) from one pass over the nonzeros. */
int skx_tucker_ttmc3_r20(const int64_t* shape_h, int R0, const int64_t* colptr0, const void* rec0,
                         uint32_t c1_mask, const double* A0, const double* A1, const double* A2,
                         double* P, void* ws, size_t* ws_bytes, void* stream);

/* CP cross term sum(weights * A_0 .* mttkrp(T, A, 0)) over lexsorted COO.
 * Replaces src/tensors.py:354-357 (+ mttkrp :322-323). */
int skx_cp_cross_coo(int ndim, const int64_t* shape_h, int64_t R, int64_t nnz,
                     const int32_t* coords, const double* vals, const double* const* factors_h,
                     const double* weights, double* out, void* ws, size_t* ws_bytes,
                     void* stream);

/* Same cross term for an order-3 tensor over its mode-0 fibre layout
 * (skx_coo_fibre mode 0: colptr0 = s0 + 1 offsets, 16-byte records, c1_mask
 * as skx_ts_rhs_coo): warp per slice, the two random factor rows of every
 * nonzero loaded as 16-byte chunks by 2*ceil(R/2) lanes.  R <= 32. */
int skx_cp_cross_fibre3(int64_t s0, const int64_t* colptr0, const void* rec0, uint32_t c1_mask,
                        int R, const double* const* factors_h, const double* weights, double* out,
                        void* ws, size_t* ws_bytes, void* stream);

/* Dense mode product with a factor's transpose, the building block of the
 * dense Tucker fitness (src/tensors.py:217-247, 349-353): for T viewed as
 * (B, s, P) in C order, out[b, r, p] = sum_i a[i*R + r] T[b, i, p]
 * (out is B x R x P).  R <= 32. */
int skx_ttm_lead(const double* t, int64_t B, int64_t s, int64_t P, const double* a, int R,
                 double* out, void* stream);

/* K5: the passes over the sketched right-hand side Y in rsvd_lrls
 * (src/linalg.py:103-112, associated form: Y G and W^T Y with w <= 32
 * columns), on FP64 tensor cores.  Row-major operands with leading
 * dimensions; N <= 32.
 *   skx_gemm_ab:  C (M x N) = A (M x K) B (K x N), A streamed by rows (K
 *                 split over CTAs when the row blocks alone fill the GPU's
 *                 waves badly; workspace query with ws = NULL);
 *   skx_gemm_atb: C (M x N) = A^T B with A (K x M), B (K x N): split-K over
 *                 CTAs, partials summed in a fixed order (workspace query
 *                 with ws = NULL).  Deterministic. */
int skx_gemm_ab(int64_t M, int N, int64_t K, const double* A, int64_t lda, const double* B,
                int64_t ldb, double* C, int64_t ldc, void* ws, size_t* ws_bytes, void* stream);
int skx_gemm_atb(int64_t M, int N, int64_t K, const double* A, int64_t lda, const double* B,
                 int64_t ldb, double* C, int64_t ldc, void* ws, size_t* ws_bytes, void* stream);

/* ------------------------------------------------ K8: CP-ALS on the core */

/* CP-ALS of a dense order-3 core (dims_h = I, J, K; C-order) in one CTA:
 * hosvd-of-core init (leading eigenvectors of the unfolding Grams,
 * src/tucker.py:112-126), `sweeps` sweeps of the normal-equations update
 * A_n = mttkrp(C, A, n) pinv(hadamard of the other Grams, rcond=1e-12) with
 * column normalisation into weights (src/cp.py:119-174 with on_core=True),
 * the sub-problem residuals (src/cp.py:96-99; residuals = 3*sweeps) and the
 * CP fitness after each sweep (src/tensors.py:339-368; fitness = sweeps).
 * factors receives I*R + J*R + K*R doubles (row-major, mode after mode),
 * weights R; *info = 0 ok, 1 zero-norm core.  Needs rank <= min(I,J,K) <= 32
 * and skx_cp_core_smem_bytes(dims_h, rank) within the shared-memory limit. */
int skx_cp_core_als(const int64_t* dims_h, int rank, int sweeps, const double* core,
                    double* factors, double* weights, double* residuals, double* fitness,
                    int* info, void* stream);
size_t skx_cp_core_smem_bytes(const int64_t* dims_h, int rank);

/* ------------------------------------------- K7: model fitness, one call each
 * fitness(t, model) = 1 - ||T - model||_F / ||T||_F assembled from
 * ||T||^2 - 2 <T, model> + ||model||^2, clamped at 0 (src/tensors.py:339-368);
 * *fit (device scalar) receives it.  norm2: device scalar ||T||^2 if the
 * caller has it, else NULL (computed).  No host synchronisation. */

/* Tucker model, sparse: cross term by skx_tucker_cross_coo (same arguments:
 * colptr0 / rec0 = the mode-0 fibre layout for the order-3 kernels, or NULL),
 * ||model||^2 = ||C||^2 (orthonormal factors, src/tensors.py:351-353). */
int skx_fitness_tucker_coo(int ndim, const int64_t* shape_h, const int64_t* ranks_h, int64_t nnz,
                           const int32_t* coords, const double* vals,
                           const double* const* factors_h, const double* core,
                           const int64_t* colptr0, const void* rec0, uint32_t c1_mask,
                           const double* norm2, double* fit, void* ws, size_t* ws_bytes,
                           void* stream);
/* Tucker model, dense C-order tensor t: ttmc(t, A) by skx_ttm_lead mode
 * products in ascending mode order (src/tensors.py:217-247), ranks <= 32. */
int skx_fitness_tucker_dense(int ndim, const int64_t* shape_h, const double* t,
                             const int64_t* ranks_h, const double* const* factors_h,
                             const double* core, const double* norm2, double* fit, void* ws,
                             size_t* ws_bytes, void* stream);
/* CP model (factors s_k x R, weights R, R <= 32), sparse: cross term by
 * skx_cp_cross_fibre3 (order 3 with the mode-0 layout) or skx_cp_cross_coo;
 * ||model||^2 from the Hadamard product of the factor Grams
 * (src/tensors.py:354-361). */
int skx_fitness_cp_coo(int ndim, const int64_t* shape_h, int R, int64_t nnz,
                       const int32_t* coords, const double* vals, const double* const* factors_h,
                       const double* weights, const int64_t* colptr0, const void* rec0,
                       uint32_t c1_mask, const double* norm2, double* fit, void* ws,
                       size_t* ws_bytes, void* stream);

/* ---------------------------------- multi-GPU reductions, NCCL
 * The data-path collectives of the nnz-sharded solve (dist.py: Y_n
 * reduce-scattered by columns, fitness cross terms all-reduced, the sampled
 * fibres all-gathered), for callers that drive libskx without
 * torch.distributed.  libnccl.so.2 is opened at first use (no link
 * dependency).  unique_id / id_out: 128-byte ncclUniqueId in HOST memory
 * (rank 0 creates it, the caller broadcasts it); comm: opaque handle.  Sums
 * are float64; counts are elements; recv of reduce-scatter holds recv_count
 * elements per rank, of all-gather nranks * send_count. */
int skx_nccl_unique_id(void* id_out);
int skx_nccl_init(const void* unique_id, int rank, int nranks, void** comm_out);
int skx_nccl_destroy(void* comm);
int skx_allreduce_sum(void* comm, const double* send, double* recv, int64_t count, void* stream);
int skx_reduce_scatter_sum(void* comm, const double* send, double* recv, int64_t recv_count,
                           void* stream);
int skx_allgather(void* comm, const double* send, double* recv, int64_t send_count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKX_H_ */
