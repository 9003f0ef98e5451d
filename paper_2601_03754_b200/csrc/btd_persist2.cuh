// btd_persist2.cuh -- PERSIST2: single systems (and small batches) with large blocks, 32 < n <= 128
// (BASELINE config c4: fp64, n = 128, N = 256), one cooperative launch per call.
//
// Algorithm 4 level by level, with the paper's blocked kernels for n >= 32
// ("the blocked variant tiles the operations", P:744-746 tile size 32 when 32 divides
// n): every n x n block op is split into 32-wide panels and 8 x 8 tiles, and the tile updates of
// the fp64 path run on the FP64 tensor cores (DMMA, mma.sync m8n8k4.f64). State lives in the
// caller's buffers (D~ in Dhat, raw fills in their final C slots, y/x in x) and stays L2-resident
// (c4: 100 MB). Three grid-wide phases per level, separated by grid.sync():
//
//   P1 (one CTA per column c):   l.8  D^_c = chol(D~_c), blocked right-looking: 32 x 32 diagonal
//                                block by one warp (shuffles), panel TRSM, trailing update on DMMA;
//                                Alg. 6 l.4 y_c <- D^_c^{-1} y_c rides along as m extra rows of the
//                                panel TRSM / trailing update.
//   P2 (column x side x VT vectors): l.10 rows of C_r <- C_r D^_c^{-T}, l.12 columns of C_l <-
//                                D^_c^{-1} C_l: blocked forward substitution, 32 x 32 diagonal
//                                solves (lane per vector) + DMMA panel updates.
//   P3 (tiles):                  separators (owner-computes "pull"):
//                                D~_m -= C_r C_r^T (left child, l.11) then C_l^T C_l (right child, the
//                                update Alg. 4 defers to l.7/l.9) -- the paper's order, no races;
//                                fill (l.13) C_{l+1} = -C_r C_l; y_m -= C_r y_{m-s} + C_l^T y_{m+s}.
//   backward (one CTA per column): x_c = D^_c^{-T}(y_c - C_r^T x_{c+s} - C_l x_{c-s}) (Alg. 6 l.10-16).
//
// Tile sizes adapt to the level: wide tiles (fewer L2 reloads) while a level has many columns,
// narrow ones (more CTAs on the chain) at the top of the tree.
#pragma once
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include "btd_persist.cuh"

namespace btd {

constexpr int kP2Threads = 256;
constexpr int kP2Warps = kP2Threads / 32;
constexpr int kQ = 32;   // panel width (POTRF, TRSM)
constexpr int kKC = 32;  // k chunk of the P3 tile GEMMs

// smem leading dimension for an n-column block: n + 4 elements keeps the 8 x 4 DMMA fragment
// loads at the 2-wavefront minimum (row stride = 8 banks mod 32) and rows 16-byte aligned
__host__ __device__ constexpr int p2_ld(int n) { return n + 4; }

template <typename T>
struct Persist2Smem {
    static __host__ __device__ int vt_max() { return sizeof(T) == 8 ? 64 : 128; }
    static __host__ __device__ size_t elems(int n, int m) {
        const int np = (n + 31) / 32 * 32;
        const size_t ld = p2_ld(np);
        const size_t p1 = (size_t)(np + m) * ld + np;                   // A (+ y rows), dinv
        const size_t p2 = (size_t)np * ld + (size_t)vt_max() * ld + np;  // L, X, dinv
        const size_t p3 = 2 * (size_t)kKC * (64 + 4);                   // sA, sB
        const size_t bw = (size_t)np * ld + (size_t)n * m + np;         // L, v, dinv
        size_t e = p1 > p2 ? p1 : p2;
        e = e > p3 ? e : p3;
        return e > bw ? e : bw;
    }
    static __host__ __device__ size_t bytes(int n, int m) { return elems(n, m) * sizeof(T) + 64; }
};

// rows x cols block of global G (ld gld) -> smem S (ld sld) with every copy in flight at once
// (LDGSTS, 16 bytes when rows stay aligned); complete for the calling thread on return -- the caller's
// __syncthreads() makes it CTA-visible.
template <typename T>
__device__ __forceinline__ void cta_load_block(T *S, int sld, const T *G, int gld, int rows, int cols) {
    constexpr int W = 16 / (int)sizeof(T);
    if (cols % W == 0 && gld % W == 0 && sld % W == 0 && (((uintptr_t)G) & 15) == 0) {
        const int cw = cols / W;
        for (int q = threadIdx.x; q < rows * cw; q += blockDim.x) {
            const int i = q / cw, j = (q % cw) * W;
            __pipeline_memcpy_async(S + (size_t)i * sld + j, G + (size_t)i * gld + j, 16);
        }
    } else {
        for (int q = threadIdx.x; q < rows * cols; q += blockDim.x) {
            const int i = q / cols, j = q % cols;
            __pipeline_memcpy_async(S + (size_t)i * sld + j, G + (size_t)i * gld + j, sizeof(T));
        }
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
}

// cta_load_block without the commit/wait: several blocks share one commit group.
template <typename T>
__device__ __forceinline__ void cta_issue_block(T *S, int sld, const T *G, int gld, int rows, int cols) {
    constexpr int W = 16 / (int)sizeof(T);
    if (cols % W == 0 && gld % W == 0 && sld % W == 0 && (((uintptr_t)G) & 15) == 0) {
        const int cw = cols / W;
        for (int q = threadIdx.x; q < rows * cw; q += blockDim.x) {
            const int i = q / cw, j = (q % cw) * W;
            __pipeline_memcpy_async(S + (size_t)i * sld + j, G + (size_t)i * gld + j, 16);
        }
    } else {
        for (int q = threadIdx.x; q < rows * cols; q += blockDim.x) {
            const int i = q / cols, j = q % cols;
            __pipeline_memcpy_async(S + (size_t)i * sld + j, G + (size_t)i * gld + j, sizeof(T));
        }
    }
}

// d += a * b over one m8n8k4 step (fp64 tensor core). Fragments (lane = 4 g + t): a = A[g][t],
// b = B[t][g], d = {D[g][2t], D[g][2t+1]}.
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// One warp: C(8x8 at rows r0, cols c0 of S, ld lds) -= sum_{k<kb} P[r0+i][pk+k] Q[c0+j][pk+k], where P
// and Q are row-major smem blocks (ld lds) -- the rank-kb update of a tile by a panel. Rows/cols
// outside [0, rmax) / [0, cmax) are neither read nor written. T = double: DMMA; float: FFMA.
// PT / QT: P / Q stored transposed (element (i, k) at P[k * ldp + i]).
template <typename T, bool PT = false, bool QT = false>
__device__ __forceinline__ void tile8_sub(T *S, int lds, int r0, int c0, int rmax, int cmax, const T *P, int ldp,
                                          const T *Q, int ldq, int pk, int kb) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    auto pel = [&](int i, int k) { return PT ? P[k * ldp + i] : P[i * ldp + k]; };
    auto qel = [&](int j, int k) { return QT ? Q[k * ldq + j] : Q[j * ldq + k]; };
    if constexpr (sizeof(T) == 8) {
        double d[2];
        const int r = r0 + g, c = c0 + 2 * t;
        d[0] = (r < rmax && c < cmax) ? S[r * lds + c] : 0.0;
        d[1] = (r < rmax && c + 1 < cmax) ? S[r * lds + c + 1] : 0.0;
        const int pr = r0 + g, qr = c0 + g;
        for (int k = 0; k < kb; k += 4) {
            const int kk = pk + k + t;
            const double a = (pr < rmax && k + t < kb) ? -pel(pr, kk) : 0.0;
            const double b = (qr < cmax && k + t < kb) ? qel(qr, kk) : 0.0;
            dmma884(d, a, b);
        }
        if (r < rmax && c < cmax) S[r * lds + c] = d[0];
        if (r < rmax && c + 1 < cmax) S[r * lds + c + 1] = d[1];
    } else {
        // two outputs per lane, same footprint as the DMMA fragment
        const int r = r0 + g, c = c0 + 2 * t;
        if (r >= rmax) return;
        T d0 = c < cmax ? S[r * lds + c] : T(0), d1 = c + 1 < cmax ? S[r * lds + c + 1] : T(0);
        for (int k = 0; k < kb; ++k) {
            const T a = pel(r, pk + k);
            if (c < cmax) d0 = fma(-a, qel(c, pk + k), d0);
            if (c + 1 < cmax) d1 = fma(-a, qel(c + 1, pk + k), d1);
        }
        if (c < cmax) S[r * lds + c] = d0;
        if (c + 1 < cmax) S[r * lds + c + 1] = d1;
    }
}

// Padded order of the blocked kernels: n rounded up to the panel width. Rows/columns n..np-1 of
// a padded block are an identity diagonal (R2 in DESIGN.md: changes no output value), so every
// panel is a full 32 x 32 block and every loop below has a compile-time trip count.
__host__ __device__ constexpr int p2_np(int n) { return (n + kQ - 1) / kQ * kQ; }

// A (np x np in smem, ld lda) <- identity outside the leading n x n block.
template <typename T>
__device__ __forceinline__ void pad_identity(T *A, int lda, int n, int np) {
    if (n == np) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < np; i += nw)
        for (int j = (i < n ? n : 0) + lane; j < np; j += 32) A[i * lda + j] = (i == j) ? T(1) : T(0);
}

// Blocked right-looking Cholesky of the np x np (np = p2_np(n), identity-padded) block in smem A
// (row-major, ld lda; lower triangle read), CTA-wide, with `ext` extra rows np..np+ext-1 (right-hand
// sides stored transposed, zero-padded) carried through the panel TRSMs and trailing updates, so
// that on return they hold (L^{-1} y)^T. dinv[k] = 1/L[k][k]; strict upper triangle of L set to zero.
// Returns false if one of the first n pivots is <= 0 or NaN.
template <typename T, int Q = kQ>
__device__ bool cta_potrf_blocked(T *A, int lda, int n, int np, int ext, T *dinv) {
    __shared__ int s_ok;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ok = 1;
    const int rows = np + ext;
#ifdef BTD_TIMING
    // sub-phase cycles of CTA 0: 8 = diagonal blocks, 9 = panel TRSMs, 10 = trailing updates
    unsigned long long tq = clock64();
#define BTD_PSUB(id)                                                              \
    do {                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            const unsigned long long now_ = clock64();                            \
            atomicAdd(&btd_timing[(id)], now_ - tq);                              \
            tq = clock64();                                                       \
        }                                                                         \
    } while (0)
#else
#define BTD_PSUB(id) \
    do {             \
    } while (0)
#endif
    for (int k0 = 0; k0 < np; k0 += Q) {
        const int k1 = k0 + Q;
        // (1) diagonal block, one warp: lane i owns row k0 + i; right-looking, shuffles
        if (warp == 0) {
            T a[Q];
            const int i = lane;
#pragma unroll
            for (int j = 0; j < Q; ++j) a[j] = (i < Q && j <= i) ? A[(k0 + i) * lda + k0 + j] : ((i == j) ? T(1) : T(0));
            bool bad = false;
            T myinv = T(1);
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                const T akk = __shfl_sync(kFull, a[k], k);
                bad |= (k0 + k < n) && !(akk > T(0));
                T d, inv;
                pivot(akk, d, inv);
                // rows i < k update their (never stored) upper part too: no per-element selects
                a[k] = (i == k) ? d : a[k] * inv;
                myinv = (i == k) ? inv : myinv;
                // constant trip count (j > k becomes a compile-time predicate once unrolled): both
                // loops must flatten or a[] is demoted to local memory
#pragma unroll
                for (int j = 1; j < Q; ++j) {
                    if (j <= k) continue;
                    const T ljk = __shfl_sync(kFull, a[k], j);
                    a[j] = fma(-a[k], ljk, a[j]);
                }
            }
            if (i < Q) {  // lanes >= Q (Q < 32) carry don't-care rows
#pragma unroll
                for (int j = 0; j < Q; ++j)
                    if (j <= i) A[(k0 + i) * lda + k0 + j] = a[j];
                dinv[k0 + i] = myinv;
            }
            if (bad && lane == 0) s_ok = 0;
        }
        __syncthreads();
        BTD_PSUB(8);
        // (2) panel TRSM: rows r >= k1 (and the ext rows): x <- x L11^{-T}, one thread per row
        for (int r = k1 + tid; r < rows; r += blockDim.x) {
            T x[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j) x[j] = A[r * lda + k0 + j];
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                x[k] *= dinv[k0 + k];
#pragma unroll
                for (int j = 1; j < Q; ++j)
                    if (j > k) x[j] = fma(-x[k], A[(k0 + j) * lda + k0 + k], x[j]);
            }
#pragma unroll
            for (int j = 0; j < Q; ++j) A[r * lda + k0 + j] = x[j];
        }
        __syncthreads();
        BTD_PSUB(9);
        // (3) trailing update A22 -= L21 L21^T (lower 8 x 8 tiles), and the ext rows
        if (k1 < np) {
            const int nt = (np - k1) / 8;
            const int ntiles = nt * (nt + 1) / 2;
            for (int tt = warp; tt < ntiles; tt += blockDim.x / 32) {
                int ti = 0, q = tt;
                while (q > ti) {
                    q -= ti + 1;
                    ++ti;
                }
                tile8_sub<T>(A + (size_t)k1 * lda + k1, lda, 8 * ti, 8 * q, np - k1, np - k1, A + (size_t)k1 * lda, lda,
                             A + (size_t)k1 * lda, lda, k0, Q);
            }
            for (int q = tid; q < ext * (np - k1); q += blockDim.x) {
                const int r = np + q / (np - k1), j = k1 + q % (np - k1);
                T acc = A[r * lda + j];
#pragma unroll 8
                for (int k = 0; k < Q; ++k) acc = fma(-A[r * lda + k0 + k], A[j * lda + k0 + k], acc);
                A[r * lda + j] = acc;
            }
        }
        __syncthreads();
        BTD_PSUB(10);
    }
#undef BTD_PSUB
    for (int i = warp; i < np; i += blockDim.x >> 5)
        for (int j = i + 1 + lane; j < np; j += 32) A[i * lda + j] = T(0);
    __syncthreads();
    return s_ok != 0;
}

// X (nv vectors of padded length np, row v at X[v*ldx], zero beyond n) <- X L^{-T}, i.e. every
// vector x <- L^{-1} x, CTA-wide. L: np x np lower (identity-padded) in smem, ld lda; dinv[k] =
// 1/L[k][k]. Blocked: 32-column diagonal solves (one thread per vector), then the panel update of
// the remaining columns on 8 x 8 tiles (DMMA for fp64).
template <typename T, int Q = kQ>
__device__ void cta_trsm_blocked(T *X, int ldx, int nv, const T *L, int lda, int np, const T *dinv) {
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int k0 = 0; k0 < np; k0 += Q) {
        const int k1 = k0 + Q;
        for (int v = tid; v < nv; v += blockDim.x) {
            T x[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j) x[j] = X[v * ldx + k0 + j];
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                x[k] *= dinv[k0 + k];
#pragma unroll
                for (int j = 1; j < Q; ++j)
                    if (j > k) x[j] = fma(-x[k], L[(k0 + j) * lda + k0 + k], x[j]);
            }
#pragma unroll
            for (int j = 0; j < Q; ++j) X[v * ldx + k0 + j] = x[j];
        }
        __syncthreads();
        if (k1 < np) {
            // X[:, k1:] -= X[:, k0:k1] L[k1:, k0:k1]^T ; P = X (panel at column k0), Q = rows k1.. of L
            const int tr = (nv + 7) / 8, tc = (np - k1) / 8;
            for (int tt = warp; tt < tr * tc; tt += blockDim.x / 32) {
                const int ti = tt / tc, tj = tt % tc;
                tile8_sub<T>(X + k1, ldx, 8 * ti, 8 * tj, nv, np - k1, X, ldx, L + (size_t)k1 * lda, lda, k0, Q);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- P3 tile GEMM (CTA-wide)

// Stage one k-chunk of an operand into smem as sX[k][i] (k-major, ld TT + 4): element (i, k) of the
// operand is M[(i0 + i) * n + k0 + k] (ROW: the rows of M) or M[(k0 + k) * n + i0 + i] (COL: the
// columns of M); zero outside [0, n).
template <typename T, int TT, bool ROW>
__device__ __forceinline__ void stage_chunk(T *sX, const T *M, int n, int i0, int k0) {
    constexpr int LDS = TT + 4, PER = kKC * TT / kP2Threads;
    T v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {  // all loads in flight before the first store
        const int q = threadIdx.x + u * kP2Threads;
        // ROW: consecutive threads walk k (contiguous in M); COL: they walk i
        const int i = ROW ? q / kKC : q % TT, k = ROW ? q % kKC : q / TT;
        const int gi = i0 + i, gk = k0 + k;
        v[u] = (gi < n && gk < n) ? (ROW ? M[(size_t)gi * n + gk] : M[(size_t)gk * n + gi]) : T(0);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int q = threadIdx.x + u * kP2Threads;
        const int i = ROW ? q / kKC : q % TT, k = ROW ? q % kKC : q / TT;
        sX[k * LDS + i] = v[u];
    }
}

// acc (the warp's SUBR x SUBC 8 x 8 sub-tiles of a TT x TT tile) -= P Q^T over K = n, with P and Q
// given as (matrix, ROW/COL) operand forms at tile offsets i0 / j0.
template <typename T, int TT, bool PROW, bool QROW>
__device__ __forceinline__ void tile_gemm_sub(T (&acc)[TT / 32][TT / 16][2], const T *Pm, const T *Qm, int n, int i0,
                                              int j0, T *sA, T *sB) {
    constexpr int LDS = TT + 4, SUBR = TT / 32, SUBC = TT / 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int rb = (warp & 3) * 8 * SUBR, cb = (warp >> 2) * 8 * SUBC;
    for (int k0 = 0; k0 < n; k0 += kKC) {
        __syncthreads();
        stage_chunk<T, TT, PROW>(sA, Pm, n, i0, k0);
        stage_chunk<T, TT, QROW>(sB, Qm, n, j0, k0);
        __syncthreads();
        if constexpr (sizeof(T) == 8) {
#pragma unroll 2
            for (int kk = 0; kk < kKC; kk += 4) {
                double a[SUBR], b[SUBC];
#pragma unroll
                for (int r = 0; r < SUBR; ++r) a[r] = -sA[(kk + t) * LDS + rb + 8 * r + g];
#pragma unroll
                for (int c = 0; c < SUBC; ++c) b[c] = sB[(kk + t) * LDS + cb + 8 * c + g];
#pragma unroll
                for (int r = 0; r < SUBR; ++r)
#pragma unroll
                    for (int c = 0; c < SUBC; ++c) dmma884(acc[r][c], a[r], b[c]);
            }
        } else {
#pragma unroll 4
            for (int kk = 0; kk < kKC; ++kk) {
                T a[SUBR], b[SUBC][2];
#pragma unroll
                for (int r = 0; r < SUBR; ++r) a[r] = sA[kk * LDS + rb + 8 * r + g];
#pragma unroll
                for (int c = 0; c < SUBC; ++c) {
                    b[c][0] = sB[kk * LDS + cb + 8 * c + 2 * t];
                    b[c][1] = sB[kk * LDS + cb + 8 * c + 2 * t + 1];
                }
#pragma unroll
                for (int r = 0; r < SUBR; ++r)
#pragma unroll
                    for (int c = 0; c < SUBC; ++c) {
                        acc[r][c][0] = fma(-a[r], b[c][0], acc[r][c][0]);
                        acc[r][c][1] = fma(-a[r], b[c][1], acc[r][c][1]);
                    }
            }
        }
    }
}

// Load (init) or store the warp's accumulator fragments of the tile at (i0, j0) of block M (n x n).
template <typename T, int TT, bool STORE>
__device__ __forceinline__ void tile_io(T (&acc)[TT / 32][TT / 16][2], T *M, int n, int i0, int j0) {
    constexpr int SUBR = TT / 32, SUBC = TT / 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int rb = (warp & 3) * 8 * SUBR, cb = (warp >> 2) * 8 * SUBC;
#pragma unroll
    for (int r = 0; r < SUBR; ++r)
#pragma unroll
        for (int c = 0; c < SUBC; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = i0 + rb + 8 * r + g, j = j0 + cb + 8 * c + 2 * t + h;
                if (STORE) {
                    if (i < n && j < n) M[(size_t)i * n + j] = acc[r][c][h];
                } else {
                    acc[r][c][h] = (M && i < n && j < n) ? M[(size_t)i * n + j] : T(0);
                }
            }
}

// ---------------------------------------------------------------- the kernel

template <typename T>
__global__ void __launch_bounds__(kP2Threads, 1)
    btd_persist2_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat, T *C,
                        T *x, int32_t *info, Geo g, int batch, int fact, int solve) {
    cg::grid_group grid = cg::this_grid();
    BTD_STAMP_INIT();
    const int N = g.N, n = g.n, m = g.m;
    const size_t nn = (size_t)n * n;
    {   // phase 0: x <- b, info <- 0 (D~ is read from D at level 1 and written to Dhat: no copy)
        const size_t stride = (size_t)gridDim.x * blockDim.x;
        const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        const size_t nb = (size_t)batch * N * n * m;
        if (fact)
            for (size_t q = t0; q < (size_t)batch; q += stride) info[q] = 0;
        if (solve && bvec != x)
            for (size_t q = t0; q < nb; q += stride) x[q] = bvec[q];
        grid.sync();
    }
    extern __shared__ __align__(16) unsigned char psm2_raw[];
    T *sm = reinterpret_cast<T *>(psm2_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int np = p2_np(n);
    const int lda = p2_ld(np);

    auto Dh = [&](long long sy) { return Dhat + sy * N * nn; };
    auto Cs = [&](long long sy) { return C + sy * (size_t)g.nC * nn; };
    auto xs = [&](long long sy) { return x + sy * (size_t)N * n * m; };
    // D~ of block i: the input D until level-1 P3 has written every separator to Dhat
    auto Dsrc = [&](long long sy, int l, int i) -> const T * {
        return (l == 1 && fact ? D + sy * N * nn : Dh(sy)) + (size_t)(i - 1) * nn;
    };

    for (int l = 1; l <= g.L; ++l) {
        const int s = 1 << (l - 1);
        const int ncols = ((N / s) + 1) / 2;
        // ------------------------------------------------ P1: POTRF (+ forward y)
        for (long long task = blockIdx.x; task < (long long)batch * ncols; task += gridDim.x) {
            const long long sy = task / ncols;
            const int j = (int)(task % ncols);
            const int c = s * (2 * j + 1);
            const int ext = solve ? m : 0;
            T *A = sm;                            // (np + ext) x lda
            T *dinv = A + (size_t)(np + ext) * lda;
            const T *src = fact ? Dsrc(sy, l, c) : Dh(sy) + (size_t)(c - 1) * nn;
            cta_load_block<T>(A, lda, src, n, n, n);
            pad_identity<T>(A, lda, n, np);
            T *yc = solve ? xs(sy) + (size_t)(c - 1) * n * m : nullptr;
            for (int q = tid; q < ext * np; q += blockDim.x) {
                const int qq = q / np, i = q % np;
                A[(np + qq) * lda + i] = i < n ? yc[(size_t)i * m + qq] : T(0);
            }
            __syncthreads();
            if (fact) {
                const bool ok = cta_potrf_blocked<T>(A, lda, n, np, ext, dinv);
                if (!ok && tid == 0) report_fail(info + sy, c);
                T *dst = Dh(sy) + (size_t)(c - 1) * nn;
                for (int i = warp; i < n; i += kP2Warps)
                    for (int jj = lane; jj < n; jj += 32) dst[(size_t)i * n + jj] = A[i * lda + jj];
            } else {
                for (int i = tid; i < np; i += blockDim.x) dinv[i] = T(1) / A[i * lda + i];
                __syncthreads();
                cta_trsm_blocked<T>(A + (size_t)np * lda, lda, ext, A, lda, np, dinv);
            }
            for (int q = tid; q < ext * n; q += blockDim.x) {
                const int qq = q / n, i = q % n;
                yc[(size_t)i * m + qq] = A[(np + qq) * lda + i];
            }
            __syncthreads();
        }
        BTD_STAMP(0);
        grid.sync();
        BTD_STAMP(1);
        // ------------------------------------------------ P2: TRSMs (l.10, l.12)
        if (fact) {
            const long long per_sys = (long long)ncols * 2;
            int VT = Persist2Smem<T>::vt_max();
            while (VT > 16 && (long long)batch * per_sys * ((n + VT - 1) / VT) < (long long)gridDim.x) VT /= 2;
            const int nchunk = (n + VT - 1) / VT;
            const long long ntask = (long long)batch * per_sys * nchunk;
            for (long long task = blockIdx.x; task < ntask; task += gridDim.x) {
                const long long sy = task / (per_sys * nchunk);
                long long rem = task % (per_sys * nchunk);
                const int j = (int)(rem / (2 * nchunk));
                rem %= 2 * nchunk;
                const int side = (int)(rem / nchunk);  // 0: rows of C_r; 1: columns of C_l
                const int v0 = (int)(rem % nchunk) * VT;
                const int nv = (n - v0) < VT ? (n - v0) : VT;
                const int c = s * (2 * j + 1);
                if (!(side == 0 ? (c + s <= N) : (c > s))) continue;
                T *Ls = sm;
                T *X = Ls + (size_t)np * lda;
                T *dinv = X + (size_t)VT * lda;
                cta_load_block<T>(Ls, lda, Dh(sy) + (size_t)(c - 1) * nn, n, n, n);
                pad_identity<T>(Ls, lda, n, np);
                for (int q = tid; q < nv * (np - n); q += blockDim.x) X[(q / (np - n)) * lda + n + q % (np - n)] = T(0);
                const long long slot = cslot(g, l, side == 0 ? c / s : c / s - 1);
                const T *srcC = (l == 1) ? (E + sy * (size_t)(N - 1) * nn + (size_t)(side == 0 ? c - 1 : c - 2) * nn)
                                         : (Cs(sy) + slot * nn);
                T *dstC = Cs(sy) + slot * nn;
                if (side == 0) {
                    cta_load_block<T>(X, lda, srcC + (size_t)v0 * n, n, nv, n);
                } else {
                    // columns v0.. of C_l, transposed into rows of X (warps over i, lanes over v)
                    for (int i = warp; i < n; i += kP2Warps)
                        for (int v = lane; v < nv; v += 32) X[v * lda + i] = srcC[(size_t)i * n + v0 + v];
                }
                __syncthreads();
                for (int i = tid; i < np; i += blockDim.x) dinv[i] = T(1) / Ls[i * lda + i];
                __syncthreads();
                cta_trsm_blocked<T>(X, lda, nv, Ls, lda, np, dinv);
                if (side == 0) {
                    for (int v = warp; v < nv; v += kP2Warps)
                        for (int i = lane; i < n; i += 32) dstC[(size_t)(v0 + v) * n + i] = X[v * lda + i];
                } else {
                    for (int i = warp; i < n; i += kP2Warps)
                        for (int v = lane; v < nv; v += 32) dstC[(size_t)i * n + v0 + v] = X[v * lda + i];
                }
                __syncthreads();
            }
            BTD_STAMP(2);
            grid.sync();
            BTD_STAMP(3);
        }
        // ------------------------------------------------ P3: separators (pull), fills, y
        {
            const int nsep = N / (2 * s);  // separators m = 2s, 4s, ... <= N
            auto run_tiles = [&](auto tt_tag) {
                constexpr int TT = decltype(tt_tag)::value;
                const int nt = (n + TT - 1) / TT;
                const int sep_t = fact ? nt * (nt + 1) / 2 : 0, fill_t = fact ? nt * nt : 0;
                const int ytask = solve ? 1 : 0;
                const long long per_sys = (long long)nsep * (sep_t + ytask) + (long long)ncols * fill_t;
                T *sA = sm, *sB = sm + kKC * (TT + 4);
                for (long long task = blockIdx.x; task < (long long)batch * per_sys; task += gridDim.x) {
                    const long long sy = task / per_sys;
                    long long rem = task % per_sys;
                    if (rem < (long long)nsep * (sep_t + ytask)) {
                        const int js = (int)(rem / (sep_t + ytask));
                        const int kind = (int)(rem % (sep_t + ytask));
                        const int msep = 2 * s * (js + 1);
                        const bool hasRc = msep + s <= N;  // right child exists
                        const T *Cr = Cs(sy) + cslot(g, l, msep / s - 1) * nn;   // left child's C_r
                        const T *Cl = Cs(sy) + cslot(g, l, msep / s) * nn;       // right child's C_l
                        if (kind < sep_t) {
                            int ti = 0, q = kind;
                            while (q > ti) {
                                q -= ti + 1;
                                ++ti;
                            }
                            const int i0 = ti * TT, j0 = q * TT;
                            T acc[TT / 32][TT / 16][2];
                            tile_io<T, TT, false>(acc, const_cast<T *>(Dsrc(sy, l, msep)), n, i0, j0);
                            tile_gemm_sub<T, TT, true, true>(acc, Cr, Cr, n, i0, j0, sA, sB);       // l.11
                            if (hasRc) tile_gemm_sub<T, TT, false, false>(acc, Cl, Cl, n, i0, j0, sA, sB);  // l.7/l.9
                            tile_io<T, TT, true>(acc, Dh(sy) + (size_t)(msep - 1) * nn, n, i0, j0);
                        } else {
                            // y_m -= C_r y_{m-s}, then y_m -= C_l^T y_{m+s}
                            T *ym = xs(sy) + (size_t)(msep - 1) * n * m;
                            const T *yl = xs(sy) + (size_t)(msep - s - 1) * n * m;
                            const T *yr = xs(sy) + (size_t)(msep + s - 1) * n * m;
                            for (int q = tid; q < n * m; q += blockDim.x) {
                                const int i = q / m, qq = q % m;
                                T a = T(0), b2 = T(0);
#pragma unroll 16
                                for (int k = 0; k < n; ++k) a = fma(Cr[(size_t)i * n + k], yl[(size_t)k * m + qq], a);
                                if (hasRc) {
#pragma unroll 16
                                    for (int k = 0; k < n; ++k) b2 = fma(Cl[(size_t)k * n + i], yr[(size_t)k * m + qq], b2);
                                }
                                T v = ym[q] - a;
                                ym[q] = hasRc ? v - b2 : v;
                            }
                        }
                    } else {
                        rem -= (long long)nsep * (sep_t + ytask);
                        const int jc = (int)(rem / fill_t), t = (int)(rem % fill_t);
                        const int c = s * (2 * jc + 1);
                        if (!(c > s && c + s <= N)) continue;
                        const int i0 = (t / nt) * TT, j0 = (t % nt) * TT;
                        const T *Cr = Cs(sy) + cslot(g, l, c / s) * nn;
                        const T *Cl = Cs(sy) + cslot(g, l, c / s - 1) * nn;
                        T acc[TT / 32][TT / 16][2];
                        tile_io<T, TT, false>(acc, nullptr, n, i0, j0);
                        tile_gemm_sub<T, TT, true, false>(acc, Cr, Cl, n, i0, j0, sA, sB);  // -C_r C_l (l.13)
                        tile_io<T, TT, true>(acc, Cs(sy) + cslot(g, l + 1, (c - s) / (2 * s)) * nn, n, i0, j0);
                    }
                }
            };
            // wide tiles while the level has enough of them to fill the grid
            const int nt64 = (n + 63) / 64;
            const long long t64 = (long long)batch * ((long long)nsep * nt64 * (nt64 + 1) / 2 + (long long)ncols * nt64 * nt64);
            if (t64 >= (long long)gridDim.x)
                run_tiles(std::integral_constant<int, 64>{});
            else
                run_tiles(std::integral_constant<int, 32>{});
        }
        BTD_STAMP(4);
        grid.sync();
        BTD_STAMP(5);
    }

    // ------------------------------------------------ backward sweep (Alg. 6 l.10-16)
    if (solve) {
        for (int l = g.L; l >= 1; --l) {
            const int s = 1 << (l - 1);
            const int ncols = ((N / s) + 1) / 2;
            for (long long task = blockIdx.x; task < (long long)batch * ncols; task += gridDim.x) {
                const long long sy = task / ncols;
                const int j = (int)(task % ncols);
                const int c = s * (2 * j + 1);
                const bool hasL = c > s, hasR = c + s <= N;
                T *Ls = sm;                           // D^_c, ld lda
                T *v = Ls + (size_t)np * lda;         // n x m
                T *dinv = v + (size_t)n * m;
                cta_load_block<T>(Ls, lda, Dh(sy) + (size_t)(c - 1) * nn, n, n, n);
                const T *Cr = Cs(sy) + cslot(g, l, c / s) * nn;
                const T *Cl = Cs(sy) + cslot(g, l, (c / s >= 2 ? c / s : 2) - 1) * nn;
                const T *yc = xs(sy) + (size_t)(c - 1) * n * m;
                const T *xr = xs(sy) + (size_t)((hasR ? c + s : c) - 1) * n * m;
                const T *xl = xs(sy) + (size_t)((hasL ? c - s : c) - 1) * n * m;
                // v = y_c - C_r^T x_{c+s} (threads over i: columns of C_r, coalesced)
                for (int q = tid; q < n * m; q += blockDim.x) {
                    const int i = q / m, qq = q % m;
                    T a = T(0);
                    if (hasR) {
#pragma unroll 16
                        for (int k = 0; k < n; ++k) a = fma(Cr[(size_t)k * n + i], xr[(size_t)k * m + qq], a);
                    }
                    v[q] = yc[q] - a;
                }
                __syncthreads();
                // v -= C_l x_{c-s} (one warp per row i, lanes over k, coalesced)
                if (hasL) {
                    for (int r = warp; r < n * m; r += kP2Warps) {
                        const int i = r / m, qq = r % m;
                        T a = T(0);
                        for (int k = lane; k < n; k += 32) a = fma(Cl[(size_t)i * n + k], xl[(size_t)k * m + qq], a);
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
                        if (lane == 0) v[r] -= a;
                    }
                }
                for (int i = tid; i < n; i += blockDim.x) dinv[i] = T(1) / Ls[i * lda + i];
                __syncthreads();
                // v <- L^{-T} v: one warp per right-hand side, lane owns rows i = lane + 32 u (n <= 128)
                for (int qq = warp; qq < m; qq += kP2Warps) {
                    T r[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = lane + 32 * u;
                        r[u] = i < n ? v[(size_t)i * m + qq] : T(0);
                    }
                    for (int k = n - 1; k >= 0; --k) {
                        const int ow = k & 31, uk = k >> 5;
                        T mine = r[0];
#pragma unroll
                        for (int u = 1; u < 4; ++u) mine = (u == uk) ? r[u] : mine;
                        const T xk = __shfl_sync(kFull, mine, ow) * dinv[k];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int i = lane + 32 * u;
                            r[u] = (i == k) ? xk : (i < k ? fma(-Ls[k * lda + i], xk, r[u]) : r[u]);
                        }
                    }
                    T *dst = xs(sy) + (size_t)(c - 1) * n * m;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = lane + 32 * u;
                        if (i < n) dst[(size_t)i * m + qq] = r[u];
                    }
                }
                __syncthreads();
            }
            BTD_STAMP(6);
            grid.sync();
            BTD_STAMP(7);
        }
    }
}

}  // namespace btd
