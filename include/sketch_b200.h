/*
 * sketch_b200.h — C ABI of the B200-native structured-sketch library (libsketch_b200.so).
 *
 * Drop-in boundary for the reference `sketchkit` apply path.  The reference has no FFI: its
 * boundary is Python method dispatch on TestMatrix subclasses (pkg/src/sketchkit/sketch/
 * base.py:48-113).  Each entry point below replaces the compiled third-party routine that
 * executes one reference apply path and is what a ctypes binding of that path
 * would call (INTEGRATION.md shows the binding this repo ships).
 *
 * Conventions (all entry points):
 *   - A, Y, SA, workspaces and every Omega array are DEVICE pointers owned by the caller.
 *   - Matrices are row-major with a leading dimension (row stride, in elements); columns are
 *     unit-stride.  The reference accepts any memory order; the host layer makes rows contiguous.
 *   - Every call is asynchronous on the given cudaStream_t (passed as void*; NULL = legacy
 *     default stream).  Nothing is allocated; workspaces are caller-provided.
 *   - Return value: SK_OK (0) or a negative status; sk_last_error() gives a thread-local
 *     message.  Nothing throws across the ABI.
 *   - dtype: SK_F32 or SK_F64, the element type of A and of the output.
 *   - Device: the calling thread's current CUDA device (cudaSetDevice), which must own the buffers.
 *     Any host thread may call any entry point concurrently (the reference runs trials on a thread
 *     pool); launch state cached inside the library is per device and guarded.
 *
 * Omega encodings (built by the host layer from the bit-exact test-matrix arrays):
 *   bcsc ("blocked column lists") for exactly-zeta-per-row sparse Omega (SparseUniform /
 *   SparseStack, src/sketch/sparse.py:118-194): the d rows of Omega are cut into chunks of
 *   `chunk_rows` (a power of two <= 32768).  For chunk h and column c the entries
 *   ent[ptr[h*k + c] .. ptr[h*k + c + 1]) are uint16 values (local_row << 1) | negative,
 *   ascending in local_row.  Values are +-1; the 1/sqrt(zeta) magnitude is `scale`.
 *   srtt sampler (SparseColTM, src/sketch/sparse.py:308-320): samp[c*xi + x] = row | (neg << 31).
 *   Khatri-Rao (src/sketch/khatri_rao.py:101-164) is passed as its factors, never as Omega: with
 *   d = P * dl (the trailing factors span q < dl, the leading ones P), F = the Khatri-Rao product of
 *   the trailing factors (dl x k) and W = that of the leading ones (P x k, all ones for one factor),
 *   Omega[P*dl + q, j] = W[P, j] * F[q, j].  Config 5: F = factor 1 (256 x 512), W = factor 0.
 */
#ifndef SKETCH_B200_H
#define SKETCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 2

#if defined(__GNUC__)
#define SK_API __attribute__((visibility("default")))
#else
#define SK_API
#endif

enum sk_status {
  SK_OK = 0,
  SK_EINVAL = -1,       /* bad shape / leading dimension / dtype / pointer */
  SK_EUNSUPPORTED = -2, /* valid request this build has no kernel for */
  SK_ECUDA = -3         /* a CUDA runtime error (message in sk_last_error) */
};

enum sk_dtype { SK_F32 = 0, SK_F64 = 1 };

enum sk_transform { SK_WHT = 0, SK_DCT3 = 1 };

/* OR-ed into `transform`: every dvals[j] is exactly +1 or -1 (the kernel may use sign bits). */
#define SK_DIAG_PM1 0x100

/* Library identity and errors. */
SK_API int sk_abi_version(void);
SK_API const char* sk_last_error(void);
/* Number of streaming multiprocessors of `device` (grid sizing), or a negative status. */
SK_API int sk_device_sm_count(int device);

/*
 * K1 — Y[n,k] = scale * A[n,d] * Omega[d,k] for a bcsc-encoded sparse Omega.
 * Replaces `_SparseTM.apply_right` = `a @ self.matrix` (src/sketch/sparse.py:63-66), executed by
 * scipy sparsetools csc_matvecs.  `chunk_rows` must equal sk_sparse_right_chunk_rows(dtype, d, k).
 * `nnz` = number of entries (ptr[last]); when the encoding is small the kernel stages it in
 * shared memory (pass 0 if unknown).
 */
SK_API int sk_sparse_right_chunk_rows(int dtype, int64_t d, int64_t k);
SK_API int sk_sparse_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda,
                           const int32_t* ptr, const uint16_t* ent, int32_t chunk_rows, int64_t nnz,
                           int64_t k, double scale, void* Y, int64_t ldy, void* stream);

/*
 * K1r — float64 Y[n,k] = scale * A * Omega (k <= 256) on a warp-specialised ring: producer warps
 * copy 64 x 64 chunks of A into a 4-stage shared-memory ring with cp.async (8-byte XOR swizzle,
 * conflict-free column gathers), 16 consumer warps accumulate 16 columns each in registers, and
 * the chunk stream is split evenly over the SMs (stream-K; tiles cut between two CTAs are combined
 * in a fixed order).  Replaces `_SparseTM.apply_right` (src/sketch/sparse.py:63-66) for float64
 * (BASELINE config 1).  Omega in the ring encoding: for unit h (rows 128h ..) and warp w (columns
 * 16w ..), lists[16*seg[16h + w] ..] = 16 uint8 column counts, then uint16 entries ((row / 64) % 2) << 15 |
 * (row % 64) << 3 | neg (sketch/encode.py ring_encode); seg has ceil(d/128)*16 + 1 entries.
 * Workspace: sk_sparse_right_ring_workspace_bytes(n, d).  A 8-byte, lists 16-byte aligned.
 * sk_sparse_right_ring_slab: the same on a row slab of Omega (A pointing at the slab's first column,
 * d = the slab's width, lists encoded with slab-local rows) with Y += when `accumulate` is set, so an
 * Omega whose lists exceed shared memory runs as a fixed sequence of slabs (deterministic sums).
 */
SK_API int sk_sparse_right_ring_supported(int dtype, int64_t d, int64_t k, int64_t seg_bytes);
SK_API size_t sk_sparse_right_ring_workspace_bytes(int64_t n, int64_t d);
SK_API int sk_sparse_right_ring(const double* A, int64_t n, int64_t d, int64_t lda, const uint8_t* lists,
                                const uint32_t* seg, int64_t seg_bytes, int64_t k, double scale, double* Y,
                                int64_t ldy, void* ws, size_t ws_bytes, void* stream);
SK_API int sk_sparse_right_ring_slab(const double* A, int64_t n, int64_t d, int64_t lda, const uint8_t* lists,
                                     const uint32_t* seg, int64_t seg_bytes, int64_t k, double scale, double* Y,
                                     int64_t ldy, int accumulate, void* ws, size_t ws_bytes, void* stream);

/*
 * K1c — Y[n,k] (=, or += with `accumulate`) scale * A * Omega for a sparse-sign Omega with lanes =
 * output columns: each lane holds its column's whole list of Omega entries in registers (half byte
 * offsets into a row of A, sign in bit 31) and one thread streams pairs of whole rows of A into a
 * shared-memory ring (cp.async.bulk).  Replaces `_SparseTM.apply_right` (src/sketch/sparse.py:63-66)
 * for float32 / float64 A (BASELINE config 1).  Columns go 256 per CTA group (groups =
 * sk_sparse_right_cols_groups(k)); colmap [groups*256] (lane -> column, -1 none), tw [groups*8]
 * (positions per warp, multiples of 8) and ent [groups*8][maxp][32] come from
 * sk_sparse_right_cols_encode over the (row, column, neg) triplets of Omega (host arrays): call it
 * with ent = NULL to get `need` (the longest warp's positions), pick maxp in {32, 64, 96, 128} >=
 * need, then call again with ent.  The encoder orders each lane's list so that the lanes of one
 * 128-byte wavefront read distinct bank slots where possible (Omega is fixed, so this is paid once).
 * A 16-byte aligned with 16-byte aligned rows, d * sizeof(T) a multiple of 16; an Omega whose
 * lists exceed maxp = 128 runs as row slabs of Omega (A offset to the slab, accumulate = 1 after
 * the first).
 */
SK_API int sk_sparse_right_cols_groups(int64_t k);
SK_API int sk_sparse_right_cols_supported(int dtype, int64_t d, int64_t k, int32_t maxp);
SK_API int sk_sparse_right_cols_encode(int dtype, int64_t d, int64_t k, int64_t nnz, const int64_t* rows,
                                       const int64_t* cols, const uint8_t* neg, int32_t maxp, uint32_t* ent,
                                       int32_t* colmap, int32_t* tw, int32_t* need);
SK_API int sk_sparse_right_cols(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const uint32_t* ent,
                                const int32_t* colmap, const int32_t* tw, int64_t k, int32_t maxp, double scale,
                                void* Y, int64_t ldy, int accumulate, void* stream);

/*
 * K1s — Y[n,k] = scale * A * Omega for a sparse A in CSR (int64 indptr[n+1], int32 indices, values
 * of `dtype`) and a sparse-sign Omega given by rows: int32 indptr[d+1] and int32 entries
 * `c | neg << 31` (magnitude folded into `scale`). A is never densified. Replaces
 * `_SparseTM.apply_right` for SciPy-sparse A (src/sketch/sparse.py:63-66); the adjoint of a sparse
 * B (sparse.py:68-71) is this on B^T. Sums are accumulated with atomics (order not reproducible).
 */
SK_API int sk_sparse_right_csr(int dtype, int64_t n, int64_t d, const int64_t* a_indptr, const int32_t* a_indices,
                               const void* a_values, const int32_t* omega_indptr, const int32_t* omega_entries,
                               int64_t k, double scale, void* Y, int64_t ldy, void* stream);

/*
 * Device NumPy Philox stream: out[i] = 32-bit output number (first + i) of a fresh
 * numpy.random.Philox generator with 256-bit counter `counter4` and 128-bit key `key2` (HOST
 * arrays, from `bit_generator.state`); `first` a multiple of 8, `out` 16-byte aligned device memory.
 * Lets test matrices be drawn on the GPU bit-identically to the reference (src/core/rng.py:18-70).
 */
SK_API int sk_philox_u32(const uint64_t* key2, const uint64_t* counter4, uint64_t first, int64_t count,
                         uint32_t* out, void* stream);

/*
 * K2 — SA[k,m] = scale * Omega[d,k]^T * A[d,m] (accumulate != 0: SA += ...).
 * Replaces `_SparseTM.apply_adjoint` = `self.matrix.conj().T @ b` (src/sketch/sparse.py:68-78).
 * Workspace of sk_sparse_adjoint_workspace_bytes(...) bytes (may be 0 -> pass NULL).
 * `chunk_rows` must equal sk_sparse_adjoint_chunk_rows(dtype, d, k).
 * Optional fast-path segment table `seg` (NULL to skip): for every chunk h and group g of 1024
 * output rows, seg[2*(h*G + g)] = the group's first entry offset rounded down to a multiple of 8
 * and seg[2*(h*G + g) + 1] = its entry count rounded up to a multiple of 8 (G = ceil(k/1024));
 * `ent_cap` = the maximum such count.  With `seg`, `ptr` must stay readable for 1028 ints past
 * its end and `ent` for 8 uint16 past its end (zero padding).
 */
SK_API int sk_sparse_adjoint_chunk_rows(int dtype, int64_t d, int64_t k);
SK_API size_t sk_sparse_adjoint_workspace_bytes(int dtype, int64_t d, int64_t m, int64_t k);
SK_API int sk_sparse_adjoint(int dtype, const void* A, int64_t d, int64_t m, int64_t lda,
                             const int32_t* ptr, const uint16_t* ent, int32_t chunk_rows,
                             const int32_t* seg, int32_t ent_cap, int64_t k, double scale, void* SA,
                             int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream);

/*
 * K2w — float32 SA[k,m] = scale * Omega^T * A with register accumulators (BASELINE config 4).
 * Same result contract as sk_sparse_adjoint (deterministic float64 reduction of row pieces).
 * Omega is given as its nonzero pattern (rows, cols, neg flags; any number per row, magnitude in
 * `scale`) and encoded once on the host by sk_sparse_adjoint_wide_encode into `enc` (uint16) with
 * segment offsets `seg_off` (sk_sparse_adjoint_wide_segments(d, k) int64) and capacity `seg_cap`;
 * call it first with enc = NULL to get the required length. A must be 16-byte aligned, lda % 4 == 0.
 * Replaces `_SparseTM.apply_adjoint` (src/sketch/sparse.py:68-78).
 */
SK_API int64_t sk_sparse_adjoint_wide_encode(int64_t d, int64_t k, int64_t nnz, const int64_t* rows,
                                             const int64_t* cols, const uint8_t* neg, uint16_t* enc,
                                             int64_t enc_cap, int64_t* seg_off, int32_t* seg_cap);
SK_API int64_t sk_sparse_adjoint_wide_segments(int64_t d, int64_t k);
SK_API size_t sk_sparse_adjoint_wide_workspace_bytes(int64_t d, int64_t m, int64_t k);
SK_API int sk_sparse_adjoint_wide(const float* A, int64_t d, int64_t m, int64_t lda, const uint16_t* enc,
                                  const int64_t* seg_off, int32_t seg_cap, int64_t k, double scale, float* SA,
                                  int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream);

/* float64 K2w (the reference's dtype): the same encoding and layout with 64-column slices (two
 * float64 columns per lane, 16-byte loads) and float64 accumulation. A 16-byte aligned, lda even. */
SK_API size_t sk_sparse_adjoint_wide_workspace_bytes_f64(int64_t d, int64_t m, int64_t k);
SK_API int sk_sparse_adjoint_wide_f64(const double* A, int64_t d, int64_t m, int64_t lda, const uint16_t* enc,
                                      const int64_t* seg_off, int32_t seg_cap, int64_t k, double scale, double* SA,
                                      int64_t ldsa, int accumulate, void* ws, size_t ws_bytes, void* stream);
SK_API int sk_sparse_adjoint_wide_rows_f64(const double* A, int64_t d, int64_t r0, int64_t r1, int64_t m,
                                           int64_t lda, const uint16_t* enc, const int64_t* seg_off, int32_t seg_cap,
                                           int64_t k, double scale, double* SA, int64_t ldsa, int accumulate, void* ws,
                                           size_t ws_bytes, void* stream);

/*
 * K2g — the same adjoint by row gathers (float32 / float64): S = Omega^T given in CSR by target row
 * (ent: for output row q the A rows j it sums, ascending, as j | neg << 31; off[q][p]: start of
 * row piece p in q's list, npieces + 1 per row, pieces of sk_sparse_adjoint_gather_pieces() rows).
 * One warp per (piece, output row, 1 KB column block) sums its rows fetched with TMA row gathers;
 * pieces are handed out in order so A streams from DRAM once. A 16-byte aligned with 16-byte rows.
 */
SK_API int64_t sk_sparse_adjoint_gather_pieces(int dtype, int64_t d, int64_t m, int64_t k, int64_t* piece_rows);
SK_API size_t sk_sparse_adjoint_gather_workspace_bytes(int dtype, int64_t d, int64_t m, int64_t k);
SK_API int sk_sparse_adjoint_gather(int dtype, const void* A, int64_t d, int64_t m, int64_t lda, const int32_t* ent,
                                    const int64_t* off, int64_t k, double scale, void* SA, int64_t ldsa,
                                    int accumulate, void* ws, size_t ws_bytes, void* stream);
/* Narrow operands of the same adjoint (m <= 8 columns, any row stride ldb, e.g. a right-hand side
 * vector): one warp per target row over the K2g encoding, float64 sums in a fixed order. */
SK_API int sk_sparse_adjoint_narrow(int dtype, const void* B, int64_t d, int64_t m, int64_t ldb, const int32_t* ent,
                                    const int64_t* off, int npieces, int64_t k, double scale, void* SA, int64_t ldsa,
                                    void* stream);
/* The same for the row block [r0, r1) of Omega (r0 % 128 == 0): A points at row r0 of the operand
 * and holds r1 - r0 rows; SA (+)= scale * Omega[r0:r1]^T * A. Lets a caller stream A through L2 in
 * row blocks and chain other kernels on each block (two-sided sketches). Workspace:
 * sk_sparse_adjoint_wide_workspace_bytes(r1 - r0, m, k). */
SK_API int sk_sparse_adjoint_wide_rows(const float* A, int64_t d, int64_t r0, int64_t r1, int64_t m, int64_t lda,
                                       const uint16_t* enc, const int64_t* seg_off, int32_t seg_cap, int64_t k,
                                       double scale, float* SA, int64_t ldsa, int accumulate, void* ws,
                                       size_t ws_bytes, void* stream);

/*
 * K3 — Y[n,k] = A[n,d] * D * F * S for the sparse randomized trigonometric transform,
 * F = unnormalised Walsh-Hadamard (transform SK_WHT, d a power of two); `scale` carries
 * 1/sqrt(d) * sqrt(d/xi)/sqrt(k).  dvals: d elements of `dtype` (the diagonal D).
 * Replaces `SparseRttTM.apply_right` (src/sketch/rtt.py:129-140) with wht (rtt.py:28-44).
 */
SK_API int sk_srtt_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const void* dvals,
                  int transform, const int32_t* samp, int32_t xi, int64_t k, double scale, void* Y,
                  int64_t ldy, void* stream);

/*
 * Long SRTT rows: Z[r, 8192a : 8192(a+1)] = H_8192 (D[8192a : ...] o A[r, same]), unnormalised,
 * for every segment a < d / 8192 (float32, d a multiple of 8192, D exactly +-1, 16-byte aligned).
 * The tcgen05 SRTT kernel in segment mode; the caller finishes H_d = H_{d/8192} (x) H_8192 on the
 * outputs it needs.
 */
SK_API int sk_wht_segments_f32(const float* A, int64_t n, int64_t d, int64_t lda, const float* dvals, float* Z,
                               int64_t ldz, void* stream);
/* ... and the sampled outputs of the outer transform: Y[r, c] = scale * sum_x sign * (H_d x)_j with
 * H_d = H_{d/8192} (x) H_8192 applied to the segment transforms Z (sampler as in sk_srtt_right). */
SK_API int sk_srtt_outer_f32(const float* Z, int64_t n, int64_t d, int64_t ldz, const int32_t* samp, int32_t xi,
                             int64_t k, double scale, float* Y, int64_t ldy, void* stream);

/*
 * DCT-III rows via one real inverse FFT: V[r, k] = tw_k (A[r, k] w_k - i A[r, N-k] w_{N-k}) for
 * k <= N/2 (A[r, N] = 0), interleaved complex of `dtype` with row stride ldv (in reals, >= N + 2);
 * tw = exp(i pi k / 2N) interleaved. irfft(V, N) then gives x_{2n} = v_n, x_{2n+1} = v_{N-1-n}.
 * Serves SparseRttTM with the DCT transform (src/sketch/rtt.py:129-140). N even.
 */
SK_API int sk_dct3_prep(int dtype, const void* A, int64_t n, int64_t N, int64_t lda, const void* w, const void* tw,
                        void* V, int64_t ldv, void* stream);

/*
 * Mixed-precision matrix-vector products for sketch-and-precondition LSQR: float32 A read once,
 * float64 vectors and accumulation. y = A v; z = A^T u (deterministic ordered reduction; workspace
 * of sk_gemv_t_f32_f64_workspace_bytes(n, d) bytes).
 */
SK_API int sk_gemv_f32_f64(const float* A, int64_t n, int64_t d, int64_t lda, const double* v, double* y,
                           void* stream);
SK_API size_t sk_gemv_t_f32_f64_workspace_bytes(int64_t n, int64_t d);
SK_API int sk_gemv_t_f32_f64(const float* A, int64_t n, int64_t d, int64_t lda, const double* u, double* z,
                             double* ws, size_t ws_bytes, void* stream);
/*
 * One LSQR bidiagonalisation step in a single pass over float32 A (d = 128 q <= 512, 16-byte
 * aligned, lda % 4 == 0): u <- A v - alpha u in place, zb[0:d] = A^T u_new and zb[d] = ||u_new||^2
 * (float64, deterministic). The LSQR iteration of sketch-and-precondition (new in this repository:
 * the reference has only sketch_and_solve, rand_nla.py:278-297) otherwise reads A twice.
 * Workspace: sk_lsqr_step_f32_f64_workspace_bytes(n, d) bytes.
 */
SK_API size_t sk_lsqr_step_f32_f64_workspace_bytes(int64_t n, int64_t d);
/*
 * LSQR recurrences on the device after sk_lsqr_step_f32_f64 (called with alpha = 1, the scale carried
 * by v''): from zb = [A^T u_dev, ||u_dev||^2] updates v, w, x (d <= 512, float64), the Paige & Saunders
 * state [alpha, c, phibar, rhobar, anorm2, ddnorm, bnorm, atol, btol, istop, itn] and writes the next
 * step's v'' = (c'/alpha') R^-1 v' and scal = [itn, istop, r1norm, arnorm, test2, acond, test1, beta].
 * One CTA; a no-op once istop != 0.  Rinv / RinvT: R^-1 and its transpose, d x d row-major.
 */
SK_API int sk_lsqr_recur_f64(int64_t d, const double* Rinv, const double* RinvT, const double* zb, double* v,
                             double* w, double* x, double* vnext, double* state, double* scal, void* stream);

SK_API int sk_lsqr_step_f32_f64(const float* A, int64_t n, int64_t d, int64_t lda, const double* v, double alpha,
                                double* u, double* zb, double* ws, size_t ws_bytes, void* stream);

/*
 * K-TC — Y[n,k] = scale * A[n,d] * B[d,k] on the tcgen05 tensor cores, float32 A split in-kernel
 * into bf16 hi + lo, fp32 accumulation in TMEM.  B is given transposed and pre-converted: Bt_hi
 * (k x d bf16, row stride ldb) and optionally Bt_lo (the bf16 residual of B; NULL when B is exact in
 * bf16, e.g. the +-1 sparse-sign and Khatri-Rao matrices).  A 16-byte aligned with
 * lda and d multiples of 4; ldb a multiple of 8.  Serves the dense form of SparseUniform/SparseStack
 * (src/sketch/sparse.py:63-66, config 3), KhatriRaoTM.apply_right (src/sketch/khatri_rao.py:158-164,
 * config 5) and GaussianTM (src/sketch/gaussian.py + base.py:75-79).  A workspace of
 * sk_dense_tc_workspace_bytes(...) bytes is needed when the launch splits K (few row tiles).
 */
SK_API int sk_dense_tc_supported(int64_t k);
SK_API size_t sk_dense_tc_workspace_bytes(int64_t n, int64_t d, int64_t k, int split_b);
SK_API int sk_dense_right_tc(const float* A, int64_t n, int64_t d, int64_t lda, const uint16_t* Bt_hi,
                             const uint16_t* Bt_lo, int64_t ldb, int64_t k, double scale, float* Y,
                             int64_t ldy, void* ws, size_t ws_bytes, void* stream);

/*
 * K-TC, transposed operand — Y[d,k] = scale * A^T W for A [n rows][d cols] float32 (as stored) and
 * W [n][k] given transposed as Wt_hi / Wt_lo (k x n bf16 hi + residual, row stride ldw): the second
 * rsvd pass B = Q^* A (reference src/rand_nla.py:104, `q.conj().T @ a`), returned as B^T, with
 * BF16x3 (A hi, A lo) x W hi + A hi x W lo.  The TMA lands 64 x 128 fp32 boxes of A and the
 * converter warps transpose while splitting.  A 16-byte aligned with lda, d multiples of 4; ldw a
 * multiple of 8.  Workspace: sk_dense_tn_tc_workspace_bytes(n, d, k) (split-K partials).
 */
SK_API size_t sk_dense_tn_tc_workspace_bytes(int64_t n, int64_t d, int64_t k);
SK_API int sk_dense_tn_tc(const float* A, int64_t n, int64_t d, int64_t lda, const uint16_t* Wt_hi,
                          const uint16_t* Wt_lo, int64_t ldw, int64_t k, double scale, float* Y, int64_t ldy,
                          void* ws, size_t ws_bytes, void* stream);

/*
 * K4 — Khatri-Rao sketch without forming Omega: Y[n,k] = scale * sum_{P,q} A[i, P*dl+q] W[P,j] F[q,j].
 * Replaces `KhatriRaoTM.apply_right` (src/sketch/khatri_rao.py:158-164, mode contractions of
 * `_contract` :62-74; BASELINE config 5).  tcgen05 on CTA pairs: each pair keeps its N block of F^T
 * resident in shared memory (Ft_hi: k x dl bf16, row stride ldf; Ft_lo its bf16 residual, NULL when F
 * is exact, e.g. Rademacher), streams A once (float32 split to bf16 hi + lo), accumulates one P at a
 * time in TMEM and folds it into registers scaled by W[P, :] (float32, row stride ldw).  A 16-byte
 * aligned with lda, dl multiples of 4; q >= dl in a 64-wide k-block is zero-filled by the TMA.
 * Workspace: sk_kr_workspace_bytes(n, P, dl, k, Ft_lo != NULL, 0).
 */
SK_API size_t sk_kr_workspace_bytes(int64_t n, int64_t P, int64_t dl, int64_t k, int split_f, int trans);
SK_API int sk_kr_right(const float* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const uint16_t* Ft_hi,
                       const uint16_t* Ft_lo, int64_t ldf, const float* W, int64_t ldw, int64_t k, double scale,
                       float* Y, int64_t ldy, void* ws, size_t ws_bytes, void* stream);
/* sk_kr_right with +-1 column weights (W[P,j] = wabs * (1 - 2 bit), bit j % 32 of
 * Wbits[P * ldwb + j / 32]; e.g. BASELINE config 5's Rademacher factors): the reducer warps prefetch a
 * chunk's 128 sign bits one chunk ahead instead of loading 128 float weights per chunk.  W (the same
 * weights as float32) is still required; N blocks not starting on 32-column boundaries use it. */
SK_API int sk_kr_right_signs(const float* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const uint16_t* Ft_hi,
                             const uint16_t* Ft_lo, int64_t ldf, const float* W, int64_t ldw, const uint32_t* Wbits,
                             int64_t ldwb, double wabs, int64_t k, double scale, float* Y, int64_t ldy, void* ws,
                             size_t ws_bytes, void* stream);
/*
 * K4 adjoint — X[k,m] = scale * Omega^T B for B [P*dl rows][m] float32 (row stride ldb), read in
 * place (no transposed copy).  Replaces `KhatriRaoTM.apply_adjoint` (src/sketch/khatri_rao.py:147-156).
 * Workspace: sk_kr_workspace_bytes(m, P, dl, k, Ft_lo != NULL, 1).
 */
SK_API int sk_kr_adjoint(const float* B, int64_t m, int64_t P, int64_t dl, int64_t ldb, const uint16_t* Ft_hi,
                         const uint16_t* Ft_lo, int64_t ldf, const float* W, int64_t ldw, int64_t k, double scale,
                         float* X, int64_t ldx, void* ws, size_t ws_bytes, void* stream);
/*
 * K3b — SRTT with the DCT transform (the reference's real-field default, src/sketch/rtt.py:92-93,
 * 129-140) in ONE kernel for power-of-two d: per row, Makhoul's real-IFFT form of the DCT-III folded
 * into a length-d/2 complex IDFT (Stockham radix-16 passes in shared memory), then the sampled
 * outputs.  w = D / s (s the orthonormal DCT weights, d values of `dtype`); samp[c*xi + x] = t | neg << 31,
 * t the index of the sampled output in the transformed row's IDFT order; scale = sampler magnitude / d
 * (sketch/trig.py _dct_fft_tables); the trig tables are formed on the device.  Rows 16-byte aligned;
 * float32 d <= 16384, float64 d <= 8192 (sk_srtt_dct_supported).
 */
SK_API int sk_srtt_dct_supported(int dtype, int64_t d);
SK_API int sk_srtt_dct_right(int dtype, const void* A, int64_t n, int64_t d, int64_t lda, const void* w,
                             const int32_t* samp, int32_t xi, int64_t k, double scale, void* Y, int64_t ldy,
                             void* stream);

/*
 * K6 — fused two-sided sketch: Y[n,k] = sy * A Omega and XT[p,d] = sx * Psi^T A from ONE
 * read of float32 A, both on tcgen05 (BF16x2 on A).  Replaces the pair `_sketch_right(a, omega)` /
 * `_sketch_left_adjoint(a, psi)` of the generalized-Nystrom drivers (src/rand_nla.py:191-202,
 * 230-245).  Omega^T: k x d bf16 (row stride ldb) + residual or NULL; Psi: a sparse-sign matrix with
 * zeta targets per row of A, given as psi[n][zeta] uint8 = q | neg << 7 (q < p <= 128); k <= 128.
 * A 16-byte aligned, lda % 4 == 0, ldb % 8 == 0.  Workspace: sk_two_sided_workspace_bytes(n, d, k,
 * Bt_lo != NULL) (per-CTA partials of XT, reduced in a fixed order).
 */
SK_API size_t sk_two_sided_workspace_bytes(int64_t n, int64_t d, int64_t k, int split_omega);
SK_API int sk_two_sided_sketch(const float* A, int64_t n, int64_t d, int64_t lda, const uint16_t* Bt_hi,
                               const uint16_t* Bt_lo, int64_t ldb, int64_t k, double sy, const uint8_t* psi,
                               int32_t zeta, int64_t p, double sx, float* Y, int64_t ldy, float* XT, int64_t ldx,
                               void* ws, size_t ws_bytes, void* stream);

/*
 * K5d / K4c — the same contractions for float64 (the reference's dtype) and for float32 shapes the
 * tcgen05 form does not take.  F is dl x k (row stride ldf) and W is P x k (row stride ldw), both of
 * `dtype`; W may be NULL when P == 1 (a dense Omega = F: the Gaussian family and the adjoints of
 * materialised operators).  Adjoint: X[k,m] from B [P*dl][m], read in place.  float64 runs on the
 * FP64 tensor cores (K5d: DMMA, the Khatri-Rao tile W[P,:] * F synthesised in shared memory) when
 * n (m) >= 64, k >= 8, the pointers are 16-byte aligned and the row strides even; otherwise, and for
 * float32, on the CUDA cores (K4c, float64 accumulation).  Parity 1e-12 (float64).
 */
SK_API int sk_kr_right_cc(int dtype, const void* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const void* F,
                          int64_t ldf, const void* W, int64_t ldw, int64_t k, double scale, void* Y, int64_t ldy,
                          void* stream);
SK_API int sk_kr_adjoint_cc(int dtype, const void* B, int64_t m, int64_t P, int64_t dl, int64_t ldb, const void* F,
                            int64_t ldf, const void* W, int64_t ldw, int64_t k, double scale, void* X, int64_t ldx,
                            void* stream);

/*
 * Complex fields (the reference's default Khatri-Rao base is complex_spherical; Gaussian and SRTT
 * have complex variants) on the same float64 DMMA engine, one real product per call over planar
 * data: Y (+)= scale * A * Re(Omega) (part 0) or Im(Omega) (part 1), A a real plane (n x P*dl);
 * Omega = W (x) F given as the real / imaginary planes of F (dl x k) and W (P x k), or W = NULL with
 * Fi = NULL for a dense plane Omega_part = Fr (P = 1).  accumulate != 0 adds into Y.  A complex
 * product is the caller's sum of such calls, e.g. Re(A Omega) = Ar Re(Omega) - Ai Im(Omega).  The
 * adjoint form reads B (P*dl x m) in place and writes X (k x m).  16-byte aligned planes, even row
 * strides.
 */
SK_API int sk_kr_right_z(const double* A, int64_t n, int64_t P, int64_t dl, int64_t lda, const double* Fr,
                         const double* Fi, int64_t ldf, const double* Wr, const double* Wi, int64_t ldw, int64_t k,
                         int part, double scale, int accumulate, double* Y, int64_t ldy, void* stream);
SK_API int sk_kr_adjoint_z(const double* B, int64_t m, int64_t P, int64_t dl, int64_t ldb, const double* Fr,
                           const double* Fi, int64_t ldf, const double* Wr, const double* Wi, int64_t ldw, int64_t k,
                           int part, double scale, int accumulate, double* X, int64_t ldx, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SKETCH_B200_H */
