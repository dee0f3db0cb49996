/*
 * ks.h -- C ABI of the B200-native Odd-Even parallel-in-time Kalman smoother
 * (Gargir & Toledo, "Parallel-in-Time Kalman Smoothing Using Orthogonal
 * Transformations", arXiv 2502.11686; P:n = line n of the paper text).
 *
 * All arithmetic is fp64 and runs in sm_100a kernels on the caller's CUDA
 * stream.  No function allocates device memory: the caller (PyTorch) owns the
 * workspace and all buffers.  Blocks are row-major.
 *
 * Problem (Eq. (1)-(6)), with the paper's evolution matrix
 * H_i = I (the *observation* matrix, paper G_i, is called H here
 * as in BASELINE.json):
 *     x_i = F_i x_{i-1} + c_i + eps_i,  cov(eps_i) = K_i      (i >= 1)
 *     o_i = H_i x_i + delta_i,          cov(delta_i) = L_i    (m_i >= 0 rows)
 *     x_hat = argmin sum_i |V_i(x_i - F_i x_{i-1} - c_i)|^2 + |W_i(o_i - H_i x_i)|^2
 * with V_i^T V_i = K_i^{-1}, W_i^T W_i = L_i^{-1}.  The outputs are
 * the smoothed states x_hat_i and their covariances cov(x_hat_i), the diagonal
 * blocks of (R^T R)^{-1}.  There is no prior on x_0:
 * the stacked matrix UA must have full column rank.
 *
 * Call order (each returns KS_ERR_ORDER when called out of order):
 *     ks_create -> ks_whiten -> ks_factor -> ks_solve [-> ks_selinv] -> ks_get
 *                                          or ks_solve_selinv        -> ks_get
 * ks_selinv is optional (the paper's "NC" variant);
 * ks_solve_selinv does both backward phases in one pass over the factor.  All calls only
 * ENQUEUE work on the stream given to ks_create; only ks_sync_status and
 * ks_get with host destination buffers synchronise.
 */
#ifndef KS_H
#define KS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ks_ctx ks_ctx;

/* Status codes.  Argument/launch errors are returned synchronously; numerical
 * failures (NOT_SPD, RANK) are recorded on the device and reported by
 * ks_sync_status (after which outputs are undefined). */
enum {
    KS_OK = 0,
    KS_ERR_ARG = 1,       /* bad argument (null pointer, size, stride, flags)   */
    KS_ERR_ORDER = 2,     /* call out of order                                  */
    KS_ERR_CUDA = 3,      /* a CUDA launch/runtime call failed                  */
    KS_ERR_NCCL = 4,      /* NCCL missing or an NCCL call failed (multi-GPU)    */
    KS_ERR_NOT_SPD = 5,   /* K_i or L_i not SPD: Cholesky pivot <= 0     */
    KS_ERR_RANK = 6,      /* UA rank deficient: |R_jj[d][d]| <= 1e-12*|stack|_F */
    KS_ERR_WORKSPACE = 7  /* workspace too small or misaligned                  */
};

/* ks_problem.flags */
enum {
    KS_HOST_INPUTS = 1u,  /* F,H,c,o,K,L,m are HOST pointers (pinned recommended);
                             ks_whiten copies them into the workspace first      */
    KS_OUTPUTS_BOUND = 2u,/* the caller binds states_out (and cov_out, unless it
                             never calls ks_selinv) in ks_create, so the
                             workspace holds no output buffers                   */
    KS_GENERIC_PATH = 4u, /* force the CTA-per-pair shared-memory kernels even
                             when n, m_max <= 8 (default there: one thread per
                             pair, registers + Givens; used to cross-check)     */
    KS_NO_FUSED_TAIL = 8u,/* small path: launch every factor level separately
                             instead of running the recursion's tail (levels
                             with few columns) in one on-chip kernel (cross-check) */
    KS_BIG_PATH = 64u,    /* force the large-n path (batched HBM-resident block
                             kernels, the default when the CTA path's shared
                             memory does not fit, e.g. n = m = 500; one GPU,
                             uniform model; used to cross-check at small n)      */
    KS_KEEP_WHITENING = 32u, /* keep the observation whitening factors M_i in the
                             workspace so that ks_update_obs can re-whiten new
                             observations o without redoing the model */
    KS_COV_IS_CHOL = 16u  /* K and L hold lower-triangular Cholesky factors
                             Lam_i (K_i = Lam Lam^T) and M_i (L_i = M M^T) instead
                             of the covariances ("whitening factors K_i, L_i",
                             BASELINE north_star; any V with V^T V = K^{-1} is a
                             valid whitening).  Only the lower
                             triangle is read; a zero diagonal entry is recorded
                             as KS_ERR_NOT_SPD                                   */
};

/* One problem (or, multi-GPU, one rank's contiguous shard of steps).
 * Per-step arrays have their own stride in doubles; stride 0 = the same block
 * at every step (a constant model).  Rows of H, o, L beyond m_i are ignored.
 * F, K, c of the first GLOBAL step are ignored (x_0 has no evolution equation,
 * P:153-154); on a shard that does not start at global step 0, the first local
 * step's F, K, c couple it to the previous shard's last step (no halo). */
typedef struct ks_problem {
    int64_t nsteps;          /* N >= 1 states in this context (paper k+1)          */
    int32_t n;               /* state dimension, 1 <= n <= KS_MAX_N                */
    int32_t m_max;           /* max observation dimension, 0 <= m_max <= KS_MAX_M  */
    const int32_t *m;        /* [N] observation dims in [0, m_max]; NULL = all m_max */
    const double *F;         /* [N][n][n]      evolution F_i                        */
    const double *H;         /* [N][m_max][n]  observation H_i (paper G_i)          */
    const double *c;         /* [N][n]         forcing c_i; NULL = 0                */
    const double *o;         /* [N][m_max]     observations o_i                     */
    const double *K;         /* [N][n][n]      evolution-noise covariance (SPD)     */
    const double *L;         /* [N][m_max][m_max] observation-noise covariance (SPD) */
    int64_t sF, sH, sc, so, sK, sL;   /* per-step strides in doubles, 0 = constant */
    uint32_t flags;          /* KS_HOST_INPUTS | KS_OUTPUTS_BOUND | KS_GENERIC_PATH | KS_NO_FUSED_TAIL |
                                KS_COV_IS_CHOL | KS_KEEP_WHITENING */
    /* Batched independent problems (P:301-316, P:608-615:
     * many small linear smoothing problems of one structure, e.g. the inner
     * solves of a Gauss-Newton / Levenberg-Marquardt smoother).  batch = B >= 1
     * (0 means 1): the N steps are B independent problems of N / B steps each
     * (N % B == 0); problem b is steps [b N/B, (b+1) N/B) and, like step 0,
     * the first step of every problem has no evolution equation (its F, K, c
     * are ignored).  The least-squares problem is then block diagonal over
     * the problems and every output equals that problem's own solution; all
     * problems go through the same launches.  Multi-GPU: segments are counted
     * in global steps (nsteps_global / B each). */
    int64_t batch;
    /* General model: evolution
     * H_i x_i = F_i x_{i-1} + c_i + eps_i with H_i of size l_i x n_i,
     * F_i l_i x n_{i-1}, K_i l_i x l_i, and state dimensions n_i <= n.
     * Arrays keep their uniform [n][n] / [m_max][n] / [n] shapes; rows >= l_i
     * and columns >= n_i (F: >= n_{i-1}) are ignored.  All NULL = the
     * uniform model above (H_i = I, l_i = n_i = n).  Multi-GPU shards: the
     * first step of a shard on rank > 0 has no n_{i-1} (it lives on the
     * previous rank), so the library cannot mask its F_i -- that block's
     * columns >= n_{i-1} must be ZERO (dist.pad_shard zeroes them). */
    const double *Hev;       /* [N][n][n] evolution matrix H_i (the paper's H); NULL = I */
    int64_t sHev;            /* per-step stride in doubles, 0 = constant                 */
    const int32_t *l;        /* [N] evolution rows l_i in [1, n]; NULL = n_i             */
    const int32_t *nstate;   /* [N] state dimensions n_i in [1, n]; NULL = all n         */
    int32_t nstate_min;      /* min_i n_i (sizes the padding rows), if nstate != NULL    */
} ks_problem;

#define KS_MAX_N 512   /* n > ~48: the large-n path (batched HBM-resident kernels) */
#define KS_MAX_M 512

/* Multi-GPU time sharding.  One process per GPU.
 * Rank r owns the contiguous global steps [first_global_step,
 * first_global_step + nsteps) with nsteps = nsteps_global / nranks a power of
 * two >= 2 and first_global_step = r * nsteps.  Every rank reduces its steps
 * to one boundary column with no communication (the coupling row of a shard's
 * first step is stored with that step, so there is no halo); the P boundary
 * columns are exchanged with ONE allgather of (3n^2+2n+1) doubles per rank,
 * factored, solved and inverted redundantly on every rank, and each rank then
 * runs its local backward levels.
 *
 * ks_dist_unique_id (rank 0 only; broadcast the 128 bytes through
 * torch.distributed or any other channel) and ks_dist_create (collective over
 * the ranks, with the rank's CUDA device current) create a library-owned NCCL
 * communicator (libnccl.so.2 is dlopen'ed: no link-time dependency); ks_factor
 * then performs the allgather itself on the context's stream (capturable in a
 * CUDA graph).  With id == NULL there is no communicator and the caller drives
 * the exchange: ks_factor returns after the local levels, the caller
 * allgathers the ks_boundary_buffers `send` buffers into `recv` (rank order)
 * on the context's stream and calls ks_factor_boundary.  A ks_dist is
 * borrowed by every context created with it and must outlive them. */
typedef struct ks_dist ks_dist;
int ks_dist_unique_id(unsigned char id[128]);                   /* KS_ERR_NCCL: no NCCL */
int ks_dist_create(ks_dist **out, int rank, int nranks, const unsigned char *id /* 128 bytes or NULL */,
                   int64_t first_global_step, int64_t nsteps_global);
/* rank, nranks, and the NCCL communicator's own rank count (ncclCommCount;
 * 0 without a communicator). */
int ks_dist_info(const ks_dist *d, int *rank, int *nranks, int *nccl_nranks);
void ks_dist_destroy(ks_dist *d);

/* Bytes of device workspace a context needs (0 on bad arguments). */
size_t ks_workspace_bytes(const ks_problem *p, const ks_dist *dist /* NULL = one GPU */);

/* Create a context.  `workspace` is a device buffer of >= ks_workspace_bytes
 * bytes, 256-byte aligned, borrowed for the context's lifetime.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Input arrays are borrowed until
 * the work enqueued by ks_whiten has completed.  `states_out` ([N][n]) and
 * `cov_out` ([N][n][n]) are optional DEVICE buffers that ks_solve / ks_selinv
 * write directly (zero-copy); when NULL, results live in the workspace and
 * ks_get copies them out.  `dist` (NULL = one GPU) is borrowed. */
int ks_create(ks_ctx **out, const ks_problem *p, void *workspace, size_t ws_bytes,
              void *stream, const ks_dist *dist, double *states_out, double *cov_out);

/* Phase 1: Cholesky K_i = Lam Lam^T, L_i = M M^T and
 * triangular solves: C_i = M^{-1}H_i, y_i = M^{-1}o_i, -B_i = -Lam^{-1}F_i,
 * D_i = Lam^{-1}, e_i = Lam^{-1}c_i.  A non-SPD K_i/L_i is recorded. */
int ks_whiten(ks_ctx *ctx);

/* Phase 2: recursive odd-even block QR of U A P with
 * Q^T U b, level by level; each level is one launch over all (even, odd)
 * column pairs.  Stores per eliminated column T = R_jj^{-1}[R_{j,l} R_{j,r}],
 * w = R_jj^{-1} z_j and P = R_jj^{-1} R_jj^{-T} for the backward phases.
 * Multi-GPU: local levels, boundary allgather, replicated boundary levels. */
int ks_factor(ks_ctx *ctx);

/* Phase 3: block back-substitution over the levels in reverse:
 * x_j = w_j - T_l x_l - T_r x_r. */
int ks_solve(ks_ctx *ctx);

/* Phase 4 (Alg. 2): odd-even block SelInv over the levels in
 * reverse: S_{j,I} = -T S_{I,I}, S_jj = P - S_{j,I} T^T, symmetrised. */
int ks_selinv(ks_ctx *ctx);

/* Phases 3 + 4 fused: the same results as ks_solve followed by ks_selinv
 * (bitwise), computed in one backward sweep over the levels that reads each
 * stored R record once (P:592-600 and Alg. 2, P:792-824 share the loop over
 * the levels in reverse and the operand T = R_jj^{-1}[R_{j,l} R_{j,r}]).
 * Requires a covariance buffer (cov_out bound, or KS_OUTPUTS_BOUND unset);
 * KS_ERR_ARG otherwise. */
int ks_solve_selinv(ks_ctx *ctx);

/* Repeated solves with new observations (P:301-316:
 * each Gauss-Newton step re-solves one structure; the NC variant
 * for exactly that use).  Replaces the observation array o (same layout,
 * stride and memory kind as at ks_create; borrowed until the enqueued work
 * completes) and re-whitens only y_i = M_i^{-1} o_i, keeping every other
 * whitened block; the context returns to the whitened stage, so the caller
 * continues with ks_factor -> ks_solve.  The covariances do not depend on o:
 * those of a previous ks_selinv stay valid (ks_get may still return them).
 * Needs KS_KEEP_WHITENING unless the observation model is constant (H, L
 * stride 0, m == NULL), where the factor whitens o itself (KS_ERR_ARG otherwise);
 * KS_ERR_ORDER before ks_whiten. */
int ks_update_obs(ks_ctx *ctx, const double *o);

/* Copy results into caller buffers (device or host; NULL = skip).  A pointer
 * equal to the bound output buffer is a no-op.  Host destinations synchronise
 * the stream.  cov requires a prior ks_selinv. */
int ks_get(ks_ctx *ctx, double *states, double *cov);

/* ks_get without the synchronisation for host destinations: the copies are
 * only enqueued on the context's stream (pinned host buffers make them
 * asynchronous DMA), so a caller streaming many problems can overlap the
 * device-to-host copy of one context with the work of another; the results
 * are valid once the stream has been synchronised. */
int ks_get_async(ks_ctx *ctx, double *states, double *cov);

/* ks_get with the covariance blocks in PACKED symmetric form: S_ii is
 * symmetric (reading R13: every path stores it exactly symmetric), so
 * only its upper triangle is returned, row by row -- cov_packed[i * P + k],
 * P = n (n + 1) / 2, k enumerating (r, c) with r <= c for r = 0 .. n-1 and
 * c = r .. n-1 -- which carries the whole result in P / n^2 of the bytes
 * (21 of 36 doubles at n = 6; the host-copy volume of an end-to-end solve).
 * cov_packed (N * P doubles) is device memory or PAGE-LOCKED host memory
 * (pinned / registered): a kernel on the context's stream writes it
 * directly (host destinations over PCIe, no staging buffer).  Pageable host
 * memory is KS_ERR_ARG.  states as in ks_get.  sync != 0 synchronises the
 * stream when a destination is on the host (ks_get), sync == 0 only enqueues
 * (ks_get_async).  Needs a prior ks_selinv (KS_ERR_ORDER otherwise). */
int ks_get_packed(ks_ctx *ctx, double *states, double *cov_packed, int sync);

/* Synchronise the stream and report the first numerical failure:
 * KS_OK, KS_ERR_NOT_SPD (bad_kind 1 = K, 2 = L), KS_ERR_RANK, or (small path,
 * n, m_max <= 8) KS_ERR_ARG with bad_kind 3 when a whitened block column's
 * norm lies outside [1e-80, 1e60] (the Givens kernels' exponent range); bad_step
 * is the local step index (or -1).  Also surfaces asynchronous CUDA errors. */
int ks_sync_status(ks_ctx *ctx, int64_t *bad_step, int *bad_kind);

/* Multi-GPU without a communicator (ks_dist_create with id == NULL): after ks_factor returns KS_OK on every
 * rank, the caller allgathers `send` (bytes each) from every rank into
 * `recv` (nranks * bytes, rank order) on the context's stream, then calls
 * ks_factor_boundary.  Device pointers inside the workspace. */
int ks_boundary_buffers(ks_ctx *ctx, void **send, void **recv, size_t *bytes);
int ks_factor_boundary(ks_ctx *ctx);

/* Per-kernel-family device timing with CUDA events recorded around every
 * launch on the context's stream (0 = off; ks_set_timing synchronises and
 * resets).  Families: 0 whiten, 1 factor levels, 2 solve levels, 3 selinv
 * levels, 4 multi-GPU boundary system, 5 fused solve+selinv levels.
 * ms[f] = summed event time, launches[f] = timed launches (synchronises). */
#define KS_NFAMILIES 6
int ks_set_timing(ks_ctx *ctx, int on);
int ks_get_timing(ks_ctx *ctx, double ms[KS_NFAMILIES], int64_t launches[KS_NFAMILIES]);

/* The individual timed launches since ks_set_timing (synchronises): returns
 * their count (negative = -error code) and fills up to `cap` entries of
 * family[], level[] (recursion level L) and ms[]. */
int64_t ks_get_launch_times(ks_ctx *ctx, int64_t cap, int32_t *family, int32_t *level, float *ms);

/* Number of factor levels (floor(log2 N) + 1 on one GPU, plus the boundary
 * levels when sharded) and the number of kernels launched by this context so
 * far (cumulative). */
int ks_info(ks_ctx *ctx, int64_t *levels, int64_t *launches);

/* Diagnostics: measured fp64 FMA throughput of the current device in
 * TFLOP/s (a DFMA-chain kernel over all SMs, best of 3, on `stream`), the
 * FP64 roofline denominator (MEASURED_PEAKS.json has none).  <= 0 on error. */
double ks_peak_fp64_tflops(void *stream);

/* Debug export of the host level plan every context uses (SURVEY §8(a) a2,
 * P:381-422): level[j] = the recursion level at which step
 * j < N is eliminated (the number of trailing one bits of j, the last
 * surviving column at the top level).  Returns the number of levels
 * (floor(log2 N) + 1), or -KS_ERR_ARG; level may be NULL. */
int ks_level_of_steps(int64_t N, int32_t *level);

const char *ks_strerror(int code);
void ks_destroy(ks_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* KS_H */
