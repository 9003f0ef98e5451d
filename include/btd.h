/*
 * btd.h -- C ABI of the B200 (sm_100a) nested-dissection block-tridiagonal Cholesky library.
 *
 * Problem (§3): Psi is symmetric positive definite block
 * tridiagonal with N diagonal blocks D_i (n x n, symmetric) and N-1 coupling
 * blocks E_i at block position (i+1, i). The library computes the multi-stage
 * (nested-dissection) factorization P Psi P^T = L^ L^^T (PAPER.md:486-560,
 * Algorithm 4; permutation P_inf of PAPER.md:488-508) and solves Psi x = b
 * with the level sweeps of Algorithm 6, for one system or a
 * batch of independent systems. Every step runs in hand-written CUDA kernels.
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by all calls
 * ---------------------------------------------------------------------------
 * Indices. Original block indices are 1-based, i = 1..N. Level l = 1..L with
 * L = floor(log2 N) + 1 and stride s = 2^(l-1); the columns
 * eliminated at level l are i = s, 3s, 5s, ... <= N.
 *
 * Layouts (all arrays contiguous, batch outermost, blocks row-major):
 *   D    [batch][N][n][n]     only the lower triangle of each block is read
 *   E    [batch][N-1][n][n]   E[k-1] is block (k+1, k) of Psi
 *   Dhat [batch][N][n][n]     Dhat[i-1] = diagonal block of L^ for original block i;
 *                             lower triangular, strict upper written as exact zeros
 *   C    [batch][nC][n][n]    coupling blocks, nC = btd_num_coupling_blocks()
 *   b, x [batch][N][n][m]
 * Coupling slot (l, k), k = 1 .. floor(N/s) - 1, lives at index
 * off(l) + k - 1 with off(l) = sum_{l' < l} (floor(N / 2^(l'-1)) - 1)
 * (level-major, k ascending). It couples original blocks a = k s and
 * b = (k+1) s and holds block (b, a) of M + M^T, where M is L^ with rows and
 * columns relabelled by original block index ("Psi-lower orientation",
 * SURVEY.md §8(c) A2). For odd k the column a is eliminated at level l and the
 * slot holds the L^ block (b, a) = E^_{l,k} D^_a^{-T}-form of Alg. 4 l.10; for
 * even k the column b is eliminated at level l and the slot holds the
 * transpose of L^ block (a, b), i.e. D^_b^{-1} E^_{l,k} of Alg. 4 l.12. Slots
 * of level l >= 2 are the fill blocks of Alg. 4 l.13 (the paper's E^ first
 * subscript is read as the level). Level 1 slots
 * correspond one to one to E.
 *
 * Precision. BTD_F32 computes in binary32, BTD_F64 in binary64, end to end
 * (FMA contraction allowed, no TF32). Block sizes n that
 * are not a compiled size are padded internally with an identity diagonal,
 * which changes no output value.
 *
 * Memory and streams. The caller allocates every buffer (device memory unless
 * a name says host). The library never allocates device memory. Every call
 * taking a stream is asynchronous on that stream (a cudaStream_t passed as
 * void*, NULL = legacy default stream) and never synchronises it. In-place use
 * is allowed: Dhat may alias D, and the first N-1 blocks of C may alias E.
 *
 * Errors. Return values report argument and launch errors only. Numerical
 * failure is reported per system in device memory, LAPACK style: info[j] = 0
 * on success, otherwise the 1-based original index of the failing pivot block
 * (pivot <= 0 or NaN); if several blocks fail
 * the one with the smallest (level, index) is reported. Outputs of a failed
 * system are unspecified.
 */
#ifndef BTD_H
#define BTD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct btd_plan btd_plan; /* host-only, immutable after create, thread-safe to share */

typedef enum { BTD_F32 = 0, BTD_F64 = 1 } btd_dtype;

typedef enum {
    BTD_OK = 0,
    BTD_EINVAL = 1,      /* bad argument (null pointer, size out of range, misaligned buffer) */
    BTD_ECUDA = 2,       /* a CUDA runtime call or kernel launch failed */
    BTD_ENOMEM = 3,      /* host allocation for the plan failed */
    BTD_EUNSUPPORTED = 4 /* size/variant outside what this build supports (n > 128; FUSED/LEVEL need n <= 32) */
} btd_status;

/* Variant selector (btd_plan_create_ex). AUTO picks by size. */
typedef enum {
    BTD_VARIANT_AUTO = 0,
    BTD_VARIANT_FUSED = 1, /* one CTA per system, all levels + both sweeps in one launch, state in smem */
    BTD_VARIANT_LEVEL = 2, /* one launch per level (Alg. 4 deferred form), state in the output buffers */
    BTD_VARIANT_PERSIST = 3, /* one cooperative launch, all levels as grid-wide phases; any n <= 128 */
    BTD_VARIANT_WIDE = 4,    /* one cooperative launch, one CTA per column op (single systems, n <= 32) */
    BTD_VARIANT_ATOMIC = 5   /* WIDE with Algorithm 5's schedule: fully right-looking,
                                both Schur updates of a column pushed with atomic adds (contention <= 2,
                                P:660), per-level chain potrf -> trsm -> syrk; n <= 32. The summation
                                order at a separator is not deterministic: results agree with the other
                                variants to rounding, not bitwise. */
} btd_variant;

/* Create a plan for `batch` systems of N blocks of size n with m right-hand sides.
 * Requires N >= 1, 1 <= n <= 128, batch >= 1, m >= 1. The plan is the symbolic
 * analysis of a0: levels, slot offsets and kernel choice,
 * all derived from (N, n, batch, m, dtype) alone. */
btd_status btd_plan_create(btd_plan **out, int64_t N, int64_t n, int64_t batch, int64_t m,
                           btd_dtype dtype);
btd_status btd_plan_create_ex(btd_plan **out, int64_t N, int64_t n, int64_t batch, int64_t m,
                              btd_dtype dtype, btd_variant variant);
void btd_plan_destroy(btd_plan *plan);

/* floor(log2 N) + 1. */
int32_t btd_num_levels(const btd_plan *plan);
/* Coupling blocks per system: sum_l (floor(N/2^(l-1)) - 1) = (N-1) + (#interior eliminations). */
int64_t btd_num_coupling_blocks(const btd_plan *plan);
/* Offset of level l's first slot (1 <= l <= L+1; l = L+1 returns the total). -1 if out of range. */
int64_t btd_level_offset(const btd_plan *plan, int32_t level);
/* P_inf as host array perm[new position] = original index, both 0-based. */
btd_status btd_permutation(const btd_plan *plan, int64_t *host_perm);
/* The variant the plan will launch (BTD_VARIANT_FUSED, _LEVEL, _PERSIST, _WIDE or _ATOMIC). */
int32_t btd_plan_variant(const btd_plan *plan);
/* Number of kernel launches one call of factor / solve / factor_solve makes (op = 0 / 1 / 2). */
int32_t btd_plan_launches(const btd_plan *plan, int32_t op);
/* Bytes of dynamic shared memory per CTA of the fused kernel (0 for the level variant). */
int64_t btd_plan_smem_bytes(const btd_plan *plan);

/* Factorization P Psi P^T = L^ L^^T (Algorithm 4). Device pointers D, E (E may be
 * NULL when N = 1), Dhat, C, info[batch]. */
btd_status btd_factor(const btd_plan *plan, const void *D, const void *E, void *Dhat, void *C,
                      int32_t *info, void *stream);

/* Solve Psi x = b with a factor from btd_factor (Algorithm 6). b may alias x. */
btd_status btd_solve(const btd_plan *plan, const void *Dhat, const void *C, const void *b, void *x,
                     void *stream);

/* Factor and solve in one call; the forward sweep is interlaced with the factorization
 * (PAPER.md:672-676, 755). Writes Dhat, C, x and info. */
btd_status btd_factor_solve(const btd_plan *plan, const void *D, const void *E, const void *b,
                            void *Dhat, void *C, void *x, int32_t *info, void *stream);

/* End-to-end variant with HOST inputs and outputs: copies host_D/host_E/host_b
 * (page-locked recommended) to the caller's device buffers dev_D/dev_E/dev_b,
 * runs btd_factor_solve, and copies Dhat, C, x and info back to the host
 * arrays, all on `stream`. The batch is processed in `chunks` slices so that
 * copies of one slice overlap compute of another (chunks >= 1; the device
 * buffers must hold the whole batch). Asynchronous like every other call. */
btd_status btd_factor_solve_host(const btd_plan *plan, const void *host_D, const void *host_E,
                                 const void *host_b, void *host_Dhat, void *host_C, void *host_x,
                                 int32_t *host_info, void *dev_D, void *dev_E, void *dev_b,
                                 void *dev_Dhat, void *dev_C, void *dev_x, int32_t *dev_info,
                                 int32_t chunks, void *stream);

/* ---------------------------------------------------------------------------
 * Extensions (csrc/btd_ext.cu). Each one reuses the core
 * factor/solve above for its O(N n^3) work; its own kernels are the packing,
 * residual and border steps named below.
 * ------------------------------------------------------------------------- */

/* f4a mixed precision ("mixed-precision strategies"; R8):
 * classical iterative refinement on a binary32 factorization. `plan` must be a
 * BTD_F32 plan of the system's (N, n, batch, m). Inputs D, E, b are binary64
 * device arrays in the layouts above; Dhat, C receive the binary32 factor of
 * fl32(Psi); x [batch][N][n][m] (binary64) receives x_iters, where
 *   x_0 = solve32(fl32(b)),  x_k = x_{k-1} + solve32(fl32(b - Psi x_{k-1}))
 * with the residual formed in binary64. resid (optional, binary64 [batch]):
 * ||b - Psi x_iters||_2 / ||b||_2 per system (summation order not deterministic).
 * work: device workspace of btd_mixed_workspace_bytes() bytes, 16-byte aligned,
 * owned by the caller, not read across calls. Launches: 3 + 1 + 2*iters + 1
 * (+1 with resid). info as btd_factor (the binary32 pivots). */
btd_status btd_mixed_workspace_bytes(const btd_plan *plan, size_t *bytes);
btd_status btd_mixed_factor_solve(const btd_plan *plan, const double *D, const double *E, const double *b,
                                  float *Dhat, float *C, double *x, int32_t *info, int32_t iters, double *resid,
                                  void *work, void *stream);
/* The same refinement for a new right-hand side with a binary32 factor (Dhat, C) from
 * btd_mixed_factor_solve (or btd_factor on fl32(D, E)): x_0 = solve32(fl32(b)), then iters
 * steps with the binary64 residual of (D, E). Same workspace. Launches: 2 + 2*iters + 1. */
btd_status btd_mixed_solve(const btd_plan *plan, const double *D, const double *E, const double *b,
                           const float *Dhat, const float *C, double *x, int32_t iters, double *resid, void *work,
                           void *stream);

/* f4b arrowhead ("arrow structures"; R9): solves
 *   [[Psi, G^T], [G, Z]] [x; x_a] = [b; b_a]
 * with the border eliminated last (ordering diag(P_inf, I)). `plan` is the plan
 * of Psi with m = na + mb (the border columns ride as extra right-hand sides).
 * G [batch][N][na][n] (G[i-1] = border block of original block i), Z [batch][na][na]
 * (lower triangle read), b [batch][N][n][mb], b_a [batch][na][mb].
 * Outputs: Dhat, C (factor of Psi, layout above); Y [batch][N][n][na+mb] =
 * Psi^{-1} [G^T | b] (its first na columns are V = Psi^{-1} G^T); LZ [batch][na][na]
 * = chol(Z - G V) (strict upper zero); x [batch][N][n][mb]; x_a [batch][na][mb].
 * R [batch][N][n][na+mb] is caller workspace. info[j] = N + 1 if the border
 * Schur complement is not positive definite (and Psi was). Needs na*(na+mb)+256
 * elements of shared memory (<= 227 KB). Runs btd_factor, then btd_solve with
 * the na+mb right-hand sides. Launches: 5 (+ the core calls' own). */
btd_status btd_arrow_factor_solve(const btd_plan *plan, int64_t na, const void *D, const void *E, const void *G,
                                  const void *Z, const void *b, const void *ba, void *Dhat, void *C, void *R, void *Y,
                                  void *LZ, void *x, void *xa, int32_t *info, void *stream);

/* f4c block banded, bandwidth w ("block banded matrices with larger
 * bandwidth"; R11): D [batch][N][n][n], A [batch][w][N][n][n] with
 * A[k-1][i-1] = block (i+k, i) of Psi_w, b, x [batch][N][n][m]. The system is
 * solved as the block-tridiagonal matrix of super-blocks of w consecutive blocks
 * (N' = ceil(N/w) super-blocks of size w n, identity padding). `plan` is the plan
 * of (N', w n, batch, m). Caller workspace: Dp [batch][N'][wn][wn], Ep
 * [batch][N'-1][wn][wn], bp, xp [batch][N'][wn][m]. Outputs: Dhat, C (factor of
 * the super-block system, layout above), x, info (super-block pivot index).
 * Launches: 3. */
btd_status btd_banded_factor_solve(const btd_plan *plan, int64_t N, int64_t n, int64_t w, const void *D,
                                   const void *A, const void *b, void *Dp, void *Ep, void *bp, void *Dhat, void *C,
                                   void *xp, void *x, int32_t *info, void *stream);

/* f3 partition permutation (Algorithm 2; R10), one
 * chunk per call so that each rank of a multi-GPU job runs its own chunk:
 * chunk k holds N_k consecutive blocks (D [N_k][n][n], E [N_k-1][n][n], b
 * [N_k][n][m]); its left pivot A_k sits before it, its right pivot A_{k+1}
 * after it. Bk = Psi[D_1k, A_k] and Ak, ak (pivot diagonal block and rhs
 * [n][m]) are NULL for the first chunk; Fk = Psi[A_{k+1}, D_{N_k k}] is NULL
 * for the last. `plan` is the chunk's plan with batch 1 and m = nb + nf + m_b
 * (nb = n if Bk, nf = n if Fk).
 * btd_partition_local: R (workspace) = [B_k e_1 | F_k^T e_N | b], factor and
 *   solve the chunk (Dhat, C, Y = Psi_k^{-1} R), and write the chunk's packet
 *   (3 n^2 + 2 n m_b elements): A_k - B_k^T Psi_k^{-1} B_k | F_k Psi_k^{-1} F_k^T |
 *   -F_k Psi_k^{-1} B_k | a_k - B_k^T Psi_k^{-1} b | F_k Psi_k^{-1} b.
 * btd_partition_reduce: from the p packets (chunk order, contiguous) assemble the
 *   block-tridiagonal pivot system (p-1 blocks: DS, ES, bS) and factor/solve it
 *   (plan ps: N = p-1, batch 1, m = m_b) -> xS = pivot solutions.
 * btd_partition_finish: x = Y[:, b] - Y[:, B] xL - Y[:, F] xR with xL = xS[k-2]
 *   (NULL for the first chunk) and xR = xS[k-1] (NULL for the last).
 * Launches: local 3, reduce 2, finish 1. */
btd_status btd_partition_local(const btd_plan *plan, const void *D, const void *E, const void *Bk, const void *Fk,
                               const void *Ak, const void *ak, const void *b, void *R, void *Dhat, void *C, void *Y,
                               void *packet, int32_t *info, void *stream);
btd_status btd_partition_reduce(const btd_plan *ps, int32_t p, const void *packets, void *DS, void *ES, void *bS,
                                void *DhatS, void *CS, void *xS, int32_t *infoS, void *stream);
btd_status btd_partition_finish(const btd_plan *plan, const void *Y, const void *xL, const void *xR, void *x,
                                void *stream);

const char *btd_status_string(btd_status status);
/* Last CUDA error string observed by this thread inside the library (or ""). */
const char *btd_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BTD_H */
