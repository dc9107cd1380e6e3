/*
 * urv_b200.h -- C ABI of liburv_b200.so, the B200-native (sm_100a, FP64)
 * implementation of the PowerURV hot path of arXiv 1812.06007.
 *
 * The reference (`/root/reference/pkg/src/urv`, pure Python + NumPy) has no
 * native FFI: its boundary for this path is the Python function
 *     urv.power_urv(a, q=1, reorth=True, seed=0) -> UrvFactorization
 * (factorizations.py:104-145), plus the kernels it calls.  Each entry point
 * below replaces one reference interface; the Python package
 * `paper_1812_06007_b200` binds them with ctypes and re-exposes the reference's
 * Python signatures, return types and exceptions.
 *
 * Conventions: all matrices are float64, column-major with an explicit leading
 * dimension (element count).  `*_on_device` flags say whether a pointer is a
 * CUDA device pointer (1) or host memory (0).  `stream` may be NULL (the library
 * then uses a private stream and synchronises before returning); with a non-NULL
 * stream the call is still synchronous on return.  Every call is reentrant and
 * bitwise deterministic for a given input and GPU; factorisations on one device
 * are serialised internally (the panel kernel uses a grid-wide barrier).
 *
 * Return codes:
 *   0 URV_OK, 1 URV_INVALID (-> ValueError), 2 URV_COLLAPSE (-> RankCollapseError),
 *   3 URV_CUDA_ERROR, 4 URV_NCCL_ERROR (-> RuntimeError), 5 URV_OOM (-> MemoryError),
 *   6 URV_UNSUPPORTED (a size the device path does not handle -> NotImplementedError).
 * urv_last_error() returns a thread-local message for the last failure.
 */
#ifndef URV_B200_H_
#define URV_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define URV_OK 0
#define URV_INVALID 1
#define URV_COLLAPSE 2
#define URV_CUDA_ERROR 3
#define URV_NCCL_ERROR 4
#define URV_OOM 5
#define URV_UNSUPPORTED 6

/* Per-stage diagnostics written by urv_power_urv_f64, 4 doubles per stage:
 *   [0] sum of squares of the stage's input matrix (||Y||_F^2, factorizations.py:76)
 *   [1] number of non-finite entries                (core.py:52)
 *   [2] number of nonzero entries                   (factorizations.py:96, `y.any()`)
 *   [3] #{j : R(j,j) < EPS * ||Y||_F}               (factorizations.py:80)
 * Stage layout (n_stages = 2q + 3):
 *   0         : the input A (validated_matrix, core.py:47-54)
 *   1 .. 2q   : reorth: power step i after A (odd) / after A^T (even), factorizations.py:91-92
 *               no reorth: stage 1 holds the final powered sample (factorizations.py:93-100)
 *   2q + 1    : "right-factor QR" (factorizations.py:142)
 *   2q + 2    : A V before the final QR (factorizations.py:143; only [1] is meaningful)
 * The Python wrapper turns these into RankCollapseError / ValueError / the
 * Provenance.warnings strings in the reference's exact order and wording.
 */
#define URV_STAGE_FIELDS 4

/* Replaces urv.power_urv / urv.ddh_urv (factorizations.py:104-155).
 * A: m x n (m >= n >= 1).  If a_rowmajor, A points at a C-order m x n array,
 *    i.e. a column-major n x m buffer with leading dimension lda (no host transpose).
 * G: the n x n Gaussian test matrix (random.py:52-61), column-major, ldg; or NULL, in
 *    which case it is drawn on the device from (seed, rng_stream) -- see urv_gaussian_f64.
 * q >= 0 power steps; reorth as in the reference.  skip_redundant_qr = 1 drops
 *    the final V = Q(Y) when q >= 1 and reorth (Y is already orthonormal; outputs
 *    change at the 1e-15 level only); 0 reproduces the reference sequence.
 * U (m x n), R (n x n, exact zeros below the diagonal), V (n x n) are written
 *    on the host or the device per out_on_device.
 * stage_info: host array of URV_STAGE_FIELDS * n_stages doubles (may be NULL). */
int urv_power_urv_f64(const double* A, int64_t m, int64_t n, int64_t lda, int a_rowmajor, int a_on_device,
                      const double* G, int64_t ldg, int g_on_device, uint64_t seed, uint64_t rng_stream,
                      int q, int reorth, int skip_redundant_qr,
                      double* U, int64_t ldu, double* R, int64_t ldr, double* V, int64_t ldv,
                      int out_on_device, double* stage_info, int64_t n_stages, void* stream);

/* Replaces urv.rsvd (factorizations.py:180-207): randomized SVD of rank ell.
 * A: m x n (any shape, 1 <= ell < min(m, n)), layout as for urv_power_urv_f64.
 * G: the n x ell Gaussian sample (= the first ell columns of the n x n draw), or NULL
 *    to draw it on the device from (seed, rng_stream).
 * U (m x ell), sigma (ell, nonincreasing), V (n x ell): a ~= U diag(sigma) V^T.
 *    Singular-vector signs follow the device SVD, not LAPACK's (any sign pair is valid).
 * stage_info (n_stages = 2q + 2): 0 = A, 1 .. 2q = power steps as for power_urv,
 *    2q + 1 = "range-finder QR" (factorizations.py:201).  When a stage shows a
 *    collapse or non-finite values the call returns URV_OK without writing U, sigma,
 *    V; the caller raises from stage_info (the reference raises at that point). */
int urv_rsvd_f64(const double* A, int64_t m, int64_t n, int64_t lda, int a_rowmajor, int a_on_device, int64_t ell,
                 const double* G, int64_t ldg, int g_on_device, uint64_t seed, uint64_t rng_stream, int q, int reorth,
                 double* U, int64_t ldu, double* sigma, double* V, int64_t ldv, int out_on_device,
                 double* stage_info, int64_t n_stages, void* stream);

/* URVK1 payload streaming (io.py:42-71).  The caller parses the
 * 21-byte header (magic "URVK1" + two little-endian u64 dims); these move the
 * column-major little-endian float64 payload between the file at byte `offset` and
 * device memory in column blocks through pinned staging buffers (pread/pwrite
 * overlapped with the copies), so the matrix never has to fit in host RAM.
 * urv_read_f64_file: file -> dst (device, rows x cols, ld ldd); fails with
 *   URV_INVALID if the file is shorter than offset + 8 rows cols bytes.
 * urv_write_f64_file: src (device) -> existing file, extended as needed. */
int urv_read_f64_file(const char* path, int64_t offset, int64_t rows, int64_t cols, double* dst, int64_t ldd,
                      void* stream);
int urv_write_f64_file(const char* path, int64_t offset, const double* src, int64_t rows, int64_t cols, int64_t lds,
                       void* stream);

/* Device generator of the reference's Gaussian test matrix (random.py:47-61):
 * NumPy's Generator(Philox(key=[seed, stream])).standard_normal(rows*cols) in
 * column-major order, bit-identical.  urv_rng_set_tables installs NumPy's
 * 256-layer ziggurat tables (wi, fi: 256 doubles; ki: 256 uint64; r, 1/r), which
 * the Python layer locates in the installed NumPy and verifies against NumPy's
 * own stream.  urv_gaussian_f64 returns URV_INVALID when the tables are not set
 * or the draw chain could not be resolved (the caller then draws on the host). */
int urv_rng_set_tables(const double* wi, const double* fi, const uint64_t* ki, double r, double inv_r);
int urv_gaussian_f64(uint64_t seed, uint64_t stream, int64_t rows, int64_t cols, double* out, int64_t ldo,
                     int out_on_device, void* cuda_stream);

/* Replaces urv.householder_qr (core.py:112-158): thin QR, diag(R) >= 0, explicit Q.
 * Q: m x n, R: n x n.  stage_info (may be NULL): 4 doubles as above for A. */
int urv_householder_qr_f64(const double* A, int64_t m, int64_t n, int64_t lda, int a_rowmajor,
                           int a_on_device, double* Q, int64_t ldq, double* R, int64_t ldr, int out_on_device,
                           double* stage_info, void* stream);

/* Householder QR of the device m x n W (m >= n) in place, LAPACK's compact form:
 * R on/above the diagonal, the unit-lower reflectors below it, tau[j] (device, n
 * doubles) with H_j = I - tau_j v_j v_j^T and diag(R) >= 0 -- the factorisation
 * half of householder_qr (core.py:143-152) without forming Q, for callers that apply
 * or form Q themselves (e.g. LAPACK/cuSOLVER orgqr as a cross-check).  ldw even,
 * W 16-byte aligned. */
int urv_qr_factor_f64(double* W, int64_t m, int64_t n, int64_t ldw, double* tau, void* stream);

/* Building blocks of the multi-GPU column-block-cyclic Householder QR (distributed.py,
 * SURVEY 8(e)); together they restate householder_qr's blocked loop (core.py:143-157)
 * one 256-column block at a time.  Device pointers only.
 * urv_geqrt_f64: factor the m x k panel W in place (k <= 256, m >= k): R on and above the
 *   diagonal (diag(R) >= 0, core.py:57-98), the reflectors V below it (unit diagonal implied);
 *   T (k x k, upper triangular, core.py:101-109) with H = I - V T V^T.  ldw even, W 16-byte aligned.
 * urv_larfb_f64: C (m x ncols) <- H^T C (trans = 1, the trailing update core.py:149-151) or
 *   H C (trans = 0, the explicit-Q step core.py:154-157), V taken from the factored panel P.
 * Both (and urv_dgemm_f64) are asynchronous on a caller-supplied stream (like cuBLAS) and
 * synchronous on the private stream (NULL).  Every call whose work contains cooperative
 * panel kernels (geqrt, the QR / power_urv / rsvd entry points) is chained after the
 * previous one on the device by an internal event, so two panels never co-reside. */
int urv_geqrt_f64(double* W, int64_t m, int64_t k, int64_t ldw, double* T, int64_t ldt, void* stream);
int urv_larfb_f64(const double* P, int64_t ldp, int64_t m, int64_t k, const double* T, int64_t ldt, int trans,
                  double* C, int64_t ldc, int64_t ncols, void* stream);

/* Rank-revealing profiles on the device (diagnostics.py:86-169).  For a
 * URV factorization the rank-k residual is U(:, k:) R(k:, k:) V^T up to the reconstruction
 * error, so the profiles are functions of R alone.  Device pointers only, R upper triangular.
 * urv_tail_sumsq_f64: out[i] = sum_{j >= i} R(i, j)^2 (i < n); suffix sums give every
 *   ||R(k:, k:)||_F = abs_frobenius[k] (diagnostics.py:98, :132).
 * urv_trmv_upper_f64: y = B x (trans = 0) or B^T x (trans = 1), B = R(k0:k0+N, k0:k0+N): the
 *   products of the Lanczos iteration for smax(R22) (abs_spectral, smax_r22; :117-169).
 * urv_tri_inv_f64: X = R^{-1}; smin(R(:k, :k)) = 1 / smax(X(:k, :k)) (smin_r11, :163-166).
 *   R, X 16-byte aligned with even leading dimensions. */
int urv_tail_sumsq_f64(const double* R, int64_t n, int64_t ldr, double* out, void* stream);
int urv_trmv_upper_f64(const double* R, int64_t ldr, int64_t k0, int64_t N, int trans, const double* x, double* y,
                       void* stream);
int urv_tri_inv_f64(const double* R, int64_t n, int64_t ldr, double* X, int64_t ldx, void* stream);

/* The FP64 GEMM engine behind the reference's `@` on the hot path
 * (factorizations.py:91, :92, :143; core.py:151, :157).  Device pointers only:
 * C = alpha op(A) op(B) + beta C, ta/tb in {'N','T'}.  Leading dimensions must be even. */
int urv_dgemm_f64(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream);

/* Fixed-order device reduction behind `np.linalg.norm(y)`, `np.isfinite(a).all()`
 * and `y.any()` (factorizations.py:76, core.py:52, factorizations.py:96):
 * out[0] = sum of squares, out[1] = #non-finite, out[2] = #nonzero of the
 * rows x cols column-major matrix A (host or device).  Used by the sharded path. */
int urv_matrix_stats_f64(const double* A, int64_t rows, int64_t cols, int64_t lda, int a_on_device, double* out,
                         void* stream);

/* Per-kernel timing registry (CUDA events around every launch while enabled).
 * Classes: 0 dgemm_tma_dmma (128x128 tiles), 1 panel_geqr2, 2 apply_t / T products,
 * 3 auxiliary kernels, 4 dgemm_tma_dmma 128x64 (rank-k updates), 5 dgemm_tma_dmma 64x128 (M <= 64).
 * urv_stats_read fills out[4*c + {0,1,2,3}] = {launches, algorithmic flops,
 * algorithmic bytes, summed milliseconds} for c < n_classes and resets. */
void urv_stats_enable(int on);
int urv_stats_read(double* out, int n_classes);
/* Debug timeline of the recorded scopes (call before urv_stats_read, which clears
 * them): out[5*i + {0..4}] = {kernel class, stream index (order of first use),
 * start ms, end ms, algorithmic flops}, times relative to the first scope.
 * Returns the number of records written, or -1 on a CUDA error. */
int urv_stats_timeline(double* out, int max_records);

/* ---- One-process multi-GPU collectives (power_urv(..., ngpus=N)) ----
 * one process drives every GPU (one host thread per GPU) over NCCL
 * communicators made by ncclCommInitAll; these wrap the collectives the row-sharded
 * PowerURV needs (distributed.py) for that mode.  The reference has no multi-GPU
 * path.  NCCL is resolved at run time (libnccl.so.2); when it is absent,
 * urv_nccl_available() returns 0 and the others return URV_NCCL_ERROR.  All
 * buffers are device pointers on the communicator's device, counts in doubles;
 * every call is enqueued on `stream` (stream-ordered, asynchronous). */
int urv_nccl_available(void);
/* Packing for the layout changes of the sharded path (distributed.py: row blocks <->
 * column-cyclic blocks, the transposing all-to-alls of the implicit-Q power steps):
 * dst(:, j) = src(:, idx[j]) (by_rows = 0) or dst(i, :) = src(idx[i], :) (by_rows = 1), dst
 * rows x cols, all column-major device buffers, idx a device int64 array. */
int urv_gather_f64(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx, int by_rows,
                   double* dst, int64_t ldd, void* stream);
int urv_nccl_init_all(int ndev, const int* devices, void** comms);
int urv_nccl_destroy(void* comm);
int urv_nccl_all_reduce_f64(void* comm, const double* send, double* recv, int64_t count, void* stream);
int urv_nccl_broadcast_f64(void* comm, double* buf, int64_t count, int root, void* stream);
int urv_nccl_all_gather_f64(void* comm, const double* send, double* recv, int64_t count, void* stream);
int urv_nccl_reduce_scatter_f64(void* comm, const double* send, double* recv, int64_t count, void* stream);
int urv_nccl_all_to_all_f64(void* comm, int nranks, const double* send, const int64_t* send_counts,
                            const int64_t* send_displs, double* recv, const int64_t* recv_counts,
                            const int64_t* recv_displs, void* stream);

/* Selects the CUDA device used by subsequent calls from this host thread
 * (the library links its own static CUDA runtime). */
int urv_set_device(int device);
/* Debug hook (only active with URV_PANEL_PROF set in the environment): per-phase
 * clock64 cycles accumulated by the cooperative panel kernel since the last read,
 * out[0..5] CTA 0, out[6] columns, out[7] grid size, out[8..15] the same for the
 * last CTA.  Returns the number of values written (0 when disabled). */
int urv_debug_panel_cycles(double* out, int n);

/* Returns every cached byte of the library's device memory pool (current device)
 * to the driver; waits for the device first.  The pool otherwise keeps up to
 * URV_POOL_KEEP_MB (default: a fifth of the device memory) of freed scratch between
 * calls, which spares repeated calls re-mapping it. */
int urv_release_memory(void);

/* Number of kernels this library has launched so far (all threads). */
long long urv_launch_count(void);
int urv_device_count(void);

const char* urv_last_error(void);
const char* urv_version(void);

#ifdef __cplusplus
}
#endif

#endif /* URV_B200_H_ */
