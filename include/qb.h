/*
 * qb.h — C ABI of the B200-native blocked randomized QB factorization
 *        ("randQB_b" / "randQB_pb") of P.-G. Martinsson and S. Voronin,
 *        "A randomized blocked algorithm for efficiently computing rank-revealing
 *        factorizations of matrices", arXiv 1503.07157.
 *
 * Citations "P:n" are line numbers of the paper text (reference PAPER.md); readings Rn are
 * the interpretations listed in DESIGN.md §3.
 *
 * Problem: given an m x n matrix A and a tolerance eps, find a
 * rank k, an m x k matrix Q with orthonormal columns and a k x n matrix B = Q^* A with
 * ||A - QB||_F <= eps; k is an OUTPUT.  The library runs Fig. 2 (randQB_b) for
 * q = 0 and Fig. 4 (randQB_pb) with P = q power steps for q >= 1, block by block:
 *   Omega_i = randn(n, b)                       (counter-based)
 *   Q_i = orth(A Omega_i); q x {Q_i = orth(A^* Q_i); Q_i = orth(A Q_i)}
 *   Q_i = orth(Q_i - Qbar Qbar^* Q_i)           (re-projection, line (3') / (8))
 *   B_i = Q_i^* A;  A = A - Q_i B_i;  stop once ||A||_F <= eps   (R1, R4)
 *
 * Conventions for every entry point:
 *   - All matrices are dense, FP64 (QB_F64) or FP32 (QB_F32) as chosen at qb_create.  An FP32
 *     context takes float A and returns float Q, B: the residual A^(i) is kept in FP32 and its
 *     products run on the tensor cores as 3xTF32 with FP32 accumulation (reading R18b), with
 *     Omega = RN32(Omega); orth, re-projection and all norms are FP64.  Its
 *     results meet FP32 tolerances.
 *   - "device" pointers are CUDA device pointers on the context's device; the caller owns
 *     everything it passes in; the context owns everything it hands out.
 *   - Column-major means element (i, j) at ptr[i + j*ld]; row-major means ptr[i*ld + j].
 *   - Calls are blocking with respect to the context stream unless stated otherwise and
 *     return a qb_status; nothing is thrown across the ABI.  After QB_ERR_CUDA the context
 *     must be destroyed.  qb_last_error() describes the last failure.
 *   - A context is not thread-safe; use one per host thread.
 */
#ifndef QB_H_
#define QB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qb_ctx_s* qb_ctx;

typedef enum {
  QB_OK = 0,                  /* converged: ||A - QB||_F <= eps (or k = 0)                    */
  QB_NOT_CONVERGED = 1,       /* reached kmax with ||A - QB||_F > eps; outputs valid (R5)     */
  QB_ERR_INVALID_ARG = 2,     /* bad dims / ld / b < 1 / q < 0 / eps < 0 or NaN / NaN-Inf in A */
  QB_ERR_OOM = 3,             /* device allocation failed                                      */
  QB_ERR_CUDA = 4,            /* CUDA runtime error (sticky; destroy the context)              */
  QB_ERR_NCCL = 5,            /* NCCL error (distributed contexts)                             */
  QB_ERR_ORTH_BREAKDOWN = 6,  /* CholeskyQR failed even after the shifted fallback (R8)        */
  QB_ERR_UNSUPPORTED = 7      /* valid request this build does not implement (see message)     */
} qb_status;

typedef enum { QB_F64 = 0, QB_F32 = 1 } qb_dtype;

/* qb_factor flags */
enum {
  QB_OVERWRITE_A = 1u,  /* A may be used as the residual workspace and is destroyed (P:112:
                           "A^(j) can overwrite A^(j-1)"); requires lda even and A 16-byte
                           aligned, otherwise an internal copy is made anyway.              */
  QB_NO_REPROJ = 2u,    /* skip line (3')/(8) — for demonstrating P:684-696 only            */
  QB_SKIP_POWER_ORTH = 4u, /* q >= 1: Y = A (A^* Y) q times, one orth per block (P:915-931,
                             the blocked "skip re-orthonormalization" variant, NEXT-3)     */
  QB_FORCE_GENERAL = 8u   /* diagnostics/tests: never take the one-launch small-problem path
                             (FP64 A of at most 262144 entries that fits one cluster's shared
                             memory, b <= 64); the result is the same loop either way       */
};

/* Per-block record (qb_stats).  r2 is the directly computed ||A^(i)||_F^2 (the stop test,
 * R1); ei is the error indicator ||A||_F^2 - sum_j ||B_j||_F^2 (the Frobenius
 * identity) recorded beside it.  fallback counts shifted-CholeskyQR retries in the block.  */
typedef struct {
  int64_t ell;        /* columns accepted after this block (= k so far)                     */
  int64_t w;          /* width of this block (b, or less for the last block when capped)   */
  double r2;          /* ||A^(i)||_F^2                                                      */
  double ei;          /* ||A||_F^2 - sum_{j<=i} ||B_j||_F^2                                 */
  double ms;          /* device time of the whole block (CUDA events), milliseconds         */
  double ms_sketch;   /* Omega_i + Y_i = A Omega_i (line (3) product)                       */
  double ms_bmat;     /* B_i = Q_i^* A (line (9)) incl. its split-K reduction               */
  double ms_down;     /* A -= Q_i B_i with the fused ||A^(i)||_F^2 epilogue (line (10))     */
  int32_t fallback;   /* number of shifted-CholeskyQR fallbacks taken in this block         */
  int32_t reserved;
  double ms_orth;     /* CholeskyQR of m-row panels (lines (3), (6), (8)): replicated on column shards */
  double ms_orth_z;   /* CholeskyQR of the power steps' n-row Z (line (5))                   */
  double ms_reproj;   /* re-projection products W = Qbar^* Q_i, Q_i -= Qbar W (line (8))     */
  double ms_power;    /* power-step products Z = A^* Q_i, Y = A Z (lines (5), (6)) + their sums */
  double kappa_r;     /* kappa-proxy: max R_jj / min R_jj of the block's first CholeskyQR
                         factorization (= the conditioning of the sketch Y_i; 0 if none ran)      */
} qb_block_stats;

/* Create a context on CUDA device `device` computing in `dtype`.  `cuda_stream` is a
 * cudaStream_t to run on (cudaStreamLegacy = (void*)1 for the legacy default stream), or
 * NULL for a context-owned blocking stream (ordered after legacy-default-stream work).
 * Errors: QB_ERR_INVALID_ARG (bad device / dtype), QB_ERR_CUDA.                           */
qb_status qb_create(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream);

/* Distributed context (column sharding; = qb_create_sharded with QB_SHARD_COLS,
 * QB_COMM_NCCL): this process is rank `rank` of
 * `nranks`, one GPU each; `nccl_unique_id` points to the 128-byte ncclUniqueId that rank 0
 * created (qb_nccl_unique_id) and the caller broadcast.  Each rank passes its column shard
 * A(:, col_offset : col_offset + n_local) to qb_factor with n = n_local and the global
 * column count in `n_global`; Omega rows are drawn for the same global indices, so every P
 * sees the same Omega.  Collective: all ranks call it.  Errors: QB_ERR_NCCL when NCCL is
 * unavailable or fails, plus those of qb_create.                                           */
qb_status qb_create_dist(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream,
                         int rank, int nranks, const void* nccl_unique_id,
                         int64_t col_offset, int64_t n_global);

/* Row-sharded distributed context (NEXT-2, tall-skinny A; = qb_create_sharded with
 * QB_SHARD_ROWS, QB_COMM_NCCL): this rank holds rows
 * row_offset .. row_offset + m_local - 1 of an m_global x n matrix and passes that block to
 * qb_factor with m = m_local.  Omega is replicated (all n rows), Y_i and Q_i stay local; the
 * CholeskyQR Grams, the re-projection coefficients W, the power step's Z and B_i are summed
 * with NCCL, so B is REPLICATED and Q is this rank's rows of Q.  rqb_svd works on it (U is
 * this rank's rows).  Collective.  Errors as for qb_create_dist.                            */
qb_status qb_create_dist_rows(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream,
                              int rank, int nranks, const void* nccl_unique_id,
                              int64_t row_offset, int64_t m_global);

/* ---- One descriptor for every sharded context (SURVEY.md §8(b) "qb_dist").
 * The paper designs the method for "shared and distributed memory machines"; the
 * sharded loop is the same Fig. 2 / Fig. 4 loop with one exchange per application of A.
 *   shard   QB_SHARD_COLS: this rank holds columns offset .. offset + n_local - 1 of an
 *           m x global matrix (square A; Y_i and the scalars are summed, Q replicated, B local).
 *           QB_SHARD_ROWS: rows offset .. offset + m_local - 1 of a global x n matrix
 *           (tall-skinny A; Grams, W, Z, B_i are summed, Q row-distributed, B replicated).
 *   comm    QB_COMM_NCCL: one process (or thread) per GPU, an NCCL communicator built from the
 *           128-byte `nccl_id` rank 0 created (qb_nccl_unique_id) and the caller broadcast.
 *           QB_COMM_LOOPBACK: `nranks` contexts of ONE process on ONE device, each driven by its
 *           own host thread, exchanging through `loopback` (qb_loopback_create): each collective
 *           waits for every rank's stream on the host, sums all ranks' buffers in rank order
 *           with one kernel, and copies the sum back.  No kernel waits on another rank, so the
 *           sharded code path runs on one GPU for testing (it is not a performance path).
 * The sums are identical on every rank, so the replicated orth is too.  Collective: all ranks
 * call qb_create_sharded and then every qb_factor together.  Errors: QB_ERR_INVALID_ARG for an
 * inconsistent descriptor (or loopback ranks on different devices), QB_ERR_NCCL when NCCL is
 * unavailable or fails.  A failing rank aborts a loopback group, so its peers return
 * QB_ERR_NCCL instead of waiting; NCCL waits poll ncclCommGetAsyncError and give up after
 * QB_COMM_TIMEOUT_S seconds (default 600), aborting the communicator.                     */
#define QB_LOOPBACK_MAX_RANKS 8
typedef struct qb_loopback_s* qb_loopback;
enum { QB_SHARD_COLS = 0, QB_SHARD_ROWS = 1 };
enum { QB_COMM_NCCL = 0, QB_COMM_LOOPBACK = 1 };
typedef struct {
  int rank, nranks;        /* 0 <= rank < nranks                                             */
  int shard;               /* QB_SHARD_COLS | QB_SHARD_ROWS                                  */
  int comm;                /* QB_COMM_NCCL | QB_COMM_LOOPBACK                                */
  const void* nccl_id;     /* QB_COMM_NCCL: 128-byte ncclUniqueId                            */
  qb_loopback loopback;    /* QB_COMM_LOOPBACK: the group (outlives its contexts)            */
  int64_t offset;          /* first global column (COLS) / row (ROWS) of this rank's shard   */
  int64_t global;          /* n_global (COLS) / m_global (ROWS)                              */
} qb_dist;

qb_status qb_create_sharded(qb_ctx* out, int device, qb_dtype dtype, void* cuda_stream, const qb_dist* dist);

/* A loopback group of `nranks` (1 .. QB_LOOPBACK_MAX_RANKS) in-process ranks; destroy it after
 * its contexts.  QB_ERR_INVALID_ARG for a bad count.                                        */
qb_status qb_loopback_create(qb_loopback* out, int nranks);
void qb_loopback_destroy(qb_loopback group);

/* Write a fresh ncclUniqueId (128 bytes) to `out128`.  QB_ERR_NCCL if NCCL is absent.      */
qb_status qb_nccl_unique_id(void* out128);

/* The factorization (Fig. 2 / Fig. 4).
 *   A      device, column-major m x n, leading dimension lda >= m (the local column shard
 *          for a distributed context).  Read-only unless QB_OVERWRITE_A.
 *   eps    absolute Frobenius tolerance (R2), eps >= 0.  The loop stops after the first
 *          block with ||A^(i)||_F^2 <= eps^2 (R4); ||A||_F <= eps returns k = 0 (R3).
 *   b      block size, 1 <= b <= 256 in this build; q >= 0 power steps; seed selects Omega.
 *   kmax   rank cap; <= 0 means min(m, n_global).  The last block is narrowed to hit it (R5).
 * Outputs (all optional except k):
 *   *k     rank found.   *resid = ||A^(k)||_F (direct, R1).
 *   *Q     device, column-major m x k, leading dimension *ldq (context-owned, replicated on
 *          every rank).  *B: device, ROW-major k x n (row i = B(i, :)), leading dimension
 *          *ldb (context-owned; the local column shard on a distributed context).  Both stay
 *          valid until the next qb_factor or qb_destroy.
 * Empty A (m = 0 or n = 0, single-rank context; A may be NULL, lda >= max(m, 1)): ||A||_F = 0
 * <= eps, so QB_OK with k = 0, *resid = 0 and NULL Q / B (reading R3).
 * Returns QB_OK, QB_NOT_CONVERGED (outputs valid), or an error.                           */
qb_status qb_factor(qb_ctx ctx, void* A, int64_t m, int64_t n, int64_t lda, double eps,
                    int64_t b, int q, uint64_t seed, int64_t kmax, unsigned flags,
                    int64_t* k, const void** Q, int64_t* ldq, const void** B, int64_t* ldb,
                    double* resid);

/* Fixed-rank schemes (NEXT-4): randQB (Fig. 1) for P = 0 and randQB_p (Fig. 3,
 * P:826-849) for P >= 1, unblocked: Omega = randn(n, l) (columns 0..l-1 of the same generator
 * as qb_factor, so its Omega_i are slices of this one, eq. (OmegaBlock));
 * Q = orth(A Omega); P times { Q = orth(A^* Q); Q = orth(A Q) }; B = Q^* A.  With
 * QB_SKIP_POWER_ORTH: Y = A Omega; P times Y = A (A^* Y); Q = orth(Y).
 * orth of the m x l panel: 256 columns at a time, two block Gram-Schmidt projections against the
 * finished columns and CholeskyQR2 (shifted fallback, R8).
 *   A     device, column-major m x n (lda); read-only unless QB_OVERWRITE_A.  1 <= l <= min(m, n).
 *   *resid (optional) = ||A - QB||_F, computed directly (one more rank-l update, of A itself
 *          under QB_OVERWRITE_A, else of a context-owned copy).
 * Outputs Q (column-major m x l, *ldq) and B (ROW-major l x n, *ldb) are context-owned as for
 * qb_factor; rqb_svd afterwards converts this factorization.  Distributed contexts:
 * QB_ERR_UNSUPPORTED.  Blocking.                                                            */
qb_status qb_fixed_rank(qb_ctx ctx, void* A, int64_t m, int64_t n, int64_t lda, int64_t l, int P,
                        uint64_t seed, unsigned flags, const void** Q, int64_t* ldq, const void** B,
                        int64_t* ldb, double* resid);

/* qb_factor with HOST buffers (end-to-end entry point): A_host (column-major, lda_host) is
 * copied to the device on the context stream (pinned memory makes this a DMA at full PCIe /
 * C2C rate), factored with the device path, and Q (column-major m x k, ldq_host) and B
 * (row-major k x n, ldb_host) are copied back into caller buffers with room for kcap_host
 * columns / rows (only min(k, kcap_host) are written; *k is the true rank).               */
qb_status qb_factor_host(qb_ctx ctx, const void* A_host, int64_t m, int64_t n, int64_t lda_host,
                         double eps, int64_t b, int q, uint64_t seed, int64_t kmax, int64_t* k,
                         void* Q_host, int64_t ldq_host, void* B_host, int64_t ldb_host,
                         int64_t kcap_host, double* resid);

/* Per-block records of the last qb_factor: copies min(cap, nblocks) records to `out`
 * (may be NULL when cap = 0) and the total count to *nblocks.                              */
qb_status qb_stats(qb_ctx ctx, qb_block_stats* out, int64_t cap, int64_t* nblocks);

/* Omega(row0:row1, col0:col0+w) of the generator of DESIGN.md §3.3 ("randn(n,b)",
 * eq. (OmegaBlock)) written ROW-major to device memory `out` (element (r, c) at
 * out[(r - row0)*ldo + (c - col0)], ldo >= w), in the context dtype (FP32 = RN32 of the
 * FP64 draw).  Asynchronous on the context stream.                                        */
qb_status qb_omega(qb_ctx ctx, uint64_t seed, int64_t row0, int64_t row1, int64_t col0,
                   int64_t w, void* out, int64_t ldo);

/* orth(X) by CholeskyQR2 with the shifted-CholeskyQR3 fallback (R8): X is
 * device, column-major m x w (ldx), in the context's dtype, overwritten by Q with orthonormal
 * columns spanning ran(X); diag(R) > 0.  w <= 256.  FP32 contexts orthonormalise the exactly
 * widened panel in FP64 and round the result.  Returns QB_ERR_ORTH_BREAKDOWN if even the
 * shifted variant fails.  Blocking.                                                       */
qb_status qb_orth(qb_ctx ctx, void* X, int64_t m, int64_t w, int64_t ldx);

/* Test hook: one product with the library's FP64 GEMM (the kernel behind every contraction of
 * the loop).  layout 0 (NN): C = A B with A[i + k*lda] (m x k) and B[j + k*ldb] (k x n, i.e.
 * B row-major); layout 1 (TN): C = A^T B with A[k + i*lda] and B[k + j*ldb].  epi 0: C
 * column-major = result; 1: C row-major (C[i*ldc + j]) = result; 2: C column-major -= result
 * (then *sumsq = ||C||_F^2 of the updated C, else *sumsq = ||result||_F^2 when sumsq != NULL).
 * split != 0 lets the library split K (fixed-order reduction).  Blocking.  FP64 context: A, B,
 * C double.  FP32 context: the 3xTF32 tensor-core GEMM — A, B float; C double for epi 0/1,
 * float for epi 2.  Pointers must be 16-byte aligned, leading dimensions multiples of 16 bytes
 * (TMA).                                                                                       */
qb_status qb_gemm(qb_ctx ctx, int layout, int epi, int64_t M, int64_t N, int64_t K,
                  const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                  int split, double* sumsq);

/* Test hook: the CholeskyQR core on a w x w Gram matrix G (device, column-major, ldg):
 * Rinv (device, ROW-major, ldr) = R^-1 with R^T R = G (+ the shifted-CholeskyQR shift of
 * reading R8 on breakdown, computed for an m_rows-row X); *shifted = 0 / 1.  w <= 256.
 * Returns QB_ERR_ORTH_BREAKDOWN if the shifted factorization fails too.  Blocking.          */
qb_status qb_chol_rinv(qb_ctx ctx, const void* G, int64_t ldg, int64_t w, int64_t m_rows,
                       void* Rinv, int64_t ldr, int* shifted);

/* Partial SVD from the context's last qb_factor / qb_fixed_rank (NEXT-1):
 * B = Uhat D V^*, U = Q Uhat, so that A ~ U diag(S) V^* with U^*U = V^*V = I and S descending.
 * B^T = Q_B R by block Gram-Schmidt + CholeskyQR2; the k x k SVD of R^T by this library's block
 * one-sided Jacobi (relatively accurate, DESIGN.md §5 "rqb_svd"; no solver library); U = Q Uhat,
 * V = Q_B J on the library's GEMMs; FP64 internally on every context.
 * The rank kept, k' (*kk), is chosen from the decaying singular values ("choose a rank k ...
 * based on the decaying singular values"; truncation undoes the over-sampling,
 * P:405-406):
 *   eps_or_0 > 0: the smallest k' with ||A - U_k' D_k' V_k'^*||_F^2 = r_k^2 + sum_{j > k'} D_j^2
 *                 <= eps^2, where r_k = ||A - QB||_F of the factorization (0 for a qb_fixed_rank
 *                 call without its residual) — the tail rule;
 *   kkeep_or_0 > 0: at most kkeep triplets; with both, the smaller k'; with neither, k' = k.
 * Outputs (context-owned, valid until the next call): U column-major m x k' (ld *ldu), S k'
 * values, V column-major n x k' (ld *ldv), in the context's dtype.  k' = 0 gives NULL pointers.
 * Errors: QB_ERR_INVALID_ARG without a prior factorization or with eps < 0 / NaN;
 * QB_ERR_UNSUPPORTED on column-sharded contexts, or if the Jacobi sweeps do not converge
 * (40 sweeps).  Blocking.                                                                   */
qb_status rqb_svd(qb_ctx ctx, double eps_or_0, int64_t kkeep_or_0, int64_t* kk, const void** U, int64_t* ldu,
                  const void** S, const void** V, int64_t* ldv);

/* Number of Jacobi sweeps the last rqb_svd took (diagnostics).                              */
int qb_svd_sweeps(qb_ctx ctx);

/* Partial pivoted QR from the context's last factorization (NEXT-4):
 * B P = Q~ R by Householder QR with column pivoting of the k x n factor B (LAPACK dlaqp2
 * order: first column of largest partial norm, norms downdated and recomputed on cancellation),
 * Q^ = Q Q~, so that A P ~ Q^ R.  FP64 internally; computed by panels of 32 pivots (LAPACK
 * dlaqps: the trailing update deferred to one GEMM per panel), which leaves the pivots of the
 * unblocked order unchanged.
 * Outputs: perm (HOST, n entries, caller-owned): column j of A P is column perm[j] of A;
 * Q^ device column-major m x k (*ldqh); R device ROW-major k x n upper trapezoidal (*ldr);
 * both context-owned, in the context's dtype, valid until the next call.  k = 0 gives the
 * identity permutation and NULL factors.  Errors: QB_ERR_INVALID_ARG without a factorization,
 * QB_ERR_UNSUPPORTED on column-sharded contexts.  Blocking.                                */
qb_status qb_pivoted_qr(qb_ctx ctx, int64_t* perm, const void** Qh, int64_t* ldqh, const void** R,
                        int64_t* ldr);

/* Number of the library's own kernel launches since the context was created.              */
int64_t qb_kernel_launches(qb_ctx ctx);

void qb_destroy(qb_ctx ctx);
const char* qb_status_string(qb_status s);
const char* qb_last_error(qb_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* QB_H_ */
