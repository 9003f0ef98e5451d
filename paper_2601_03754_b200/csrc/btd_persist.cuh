// btd_persist.cuh -- PERSIST variant: one cooperative (grid-resident) launch for a whole
// factor+solve of long horizons and/or large blocks (n <= 128), e.g. BASELINE configs c2-c4.
//
// Algorithm 4 in its deferred form with state in the caller's buffers (as the
// LEVEL variant: D~ in Dhat, raw fill in its final C slot, y/x in x). Each level is split into
// three grid-wide phases separated by grid.sync(); inside a phase the work is a list of
// independent CTA tasks spread over every SM:
//
//   P1 (one task per column c):      l.7  D~_c -= E^_{l-1,2c/s}^T E^_{l-1,2c/s}   (deferred)
//                                    l.8  D^_c = chol(D~_c)
//                                    Alg. 6 forward: y_c -= (same)^T y_{c+s/2}; y_c <- D^_c^{-1} y_c
//   P2 (column x side x row tile):   l.10 rows of C_r <- C_r D^_c^{-T};  l.12 columns of C_l <- D^_c^{-1} C_l
//   P3 (column x output tile):       l.9 + l.11  D~_{c+s} -= E^_{l-1,2c/s+2}^T E^ + C_r C_r^T
//                                    l.13 fill  C_{l+1,(c-s)/2s} = -C_r C_l
//                                    Alg. 6: y_{c+s} -= E^^T y_{c+3s/2} + C_r y_c
//   backward (one task per column):  x_c = D^_c^{-T}(y_c - C_r^T x_{c+s} - C_l x_{c-s})   (Alg. 6 l.10-16)
//
// A task works on whole n x n blocks staged in shared memory with element-parallel loops over the
// CTA (no register arrays, n is a runtime value); the TRSMs run one warp per vector with the
// right-looking substitution broadcast by shuffles; the Schur/fill GEMMs are tiled 64 x 64 with a
// 4 x 4 register micro-tile per thread. Tasks read their operands from L2 (the whole state of
// c3/c4 is 9-85 MB, resident in the 126 MB L2).
#pragma once
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include "btd_kernels.cuh"

namespace btd {

namespace cg = cooperative_groups;

constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr int kPTile = 64;   // GEMM output tile
constexpr int kPKC = 32;     // GEMM k chunk
constexpr int kPRT = 32;     // TRSM vectors per task

template <typename T>
struct PersistSmem {
    // max over phases of the dynamic shared memory (elements)
    static __host__ __device__ size_t elems(int n, int m) {
        const size_t nn = (size_t)n * n;
        const size_t p1 = nn + (size_t)kPKC * 128 + 2 * (size_t)n * m + n + 256;
        const size_t p2 = (size_t)n * (n + 1) + (size_t)kPRT * n + n;
        const size_t p3 = 2 * (size_t)kPKC * (kPTile + 1);
        const size_t bw = nn + 3 * (size_t)n * m + n;
        size_t e = p1 > p2 ? p1 : p2;
        e = e > p3 ? e : p3;
        e = e > bw ? e : bw;
        return e;
    }
    static __host__ __device__ size_t bytes(int n, int m) { return elems(n, m) * sizeof(T) + 64; }
};

// ---------------------------------------------------------------- CTA helpers

// Global -> shared copy with every element in flight at once (LDGSTS), complete on return for the
// calling thread (a __syncthreads() makes it CTA-visible).
template <typename T>
__device__ __forceinline__ void cta_copy_in(T *dst, const T *src, size_t cnt) {
    for (size_t q = threadIdx.x; q < cnt; q += blockDim.x) __pipeline_memcpy_async(dst + q, src + q, sizeof(T));
    __pipeline_commit();
    __pipeline_wait_prior(0);
}

// Right-looking Cholesky of the n x n block A (row-major, ld n) in shared memory; only the lower
// triangle is read. colk (n elements) is scratch holding the current column. Returns true if every
// pivot was > 0. Upper triangle set to zero; dinv[k] = 1/L[k][k].
template <typename T>
__device__ bool cta_potrf(T *A, int n, T *dinv, T *colk) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        const T akk = A[k * n + k];
        const T d = sqrt_rn(akk);
        const T inv = rcp_rn(d);
        for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
            const T v = (i == k) ? d : A[i * n + k] * inv;
            colk[i] = v;
            if (i != k) A[i * n + k] = v;  // A[k][k] is rewritten after the barrier (others still read it)
        }
        if (threadIdx.x == 0) {
            dinv[k] = inv;
            if (!(akk > T(0))) s_ok = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) A[k * n + k] = d;
        // trailing update of the lower triangle: A[i][j] -= L[i][k] L[j][k], k < j <= i
        // rows over warps, columns over lanes (no integer division in the hot loop)
        {
            const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (int i = k + 1 + (threadIdx.x >> 5); i < n; i += nw) {
                const T li = colk[i];
                for (int j = k + 1 + lane; j <= i; j += 32) A[i * n + j] = fma(-li, colk[j], A[i * n + j]);
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = i + 1 + (threadIdx.x & 31); j < n; j += 32) A[i * n + j] = T(0);
    __syncthreads();
    return s_ok != 0;
}

// CTA-wide Cholesky with the block held in registers, 2-D block-cyclic (n <= 128, 256 threads):
// thread (warp w, lane) owns A[i][j] for i = w + 8r (r < 16), j = lane + 32c (c < 4). Optionally
// applies the deferred left downdate A -= Cd^T Cd first (Alg. 4 l.7; Cd global, staged through
// `chunk` kPKC rows at a time). Step k: the owners of column k publish it (double-buffered
// `colbuf`, 2n), one barrier, every thread forms L[i][k] = a_ik/d for its rows/columns and applies
// the rank-1 update to its elements right of column k; column k of L goes straight to A (shared
// memory). Returns true if every pivot was > 0; dinv[k] = 1/L[k][k]; strict upper triangle = 0.
template <typename T>
__device__ bool cta_chol_reg(T *A, int n, const T *Cd, T *chunk, T *colbuf, T *dinv) {
    constexpr int RR = 16, CC = 4, NP = 128;  // padded order: rows/cols >= n are identity
    __shared__ int s_ok2;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T a[RR][CC];
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int c = 0; c < CC; ++c) {
            const int i = w + 8 * r, j = lane + 32 * c;
            a[r][c] = (i < n && j < n) ? A[i * n + j] : (i == j ? T(1) : T(0));
        }
    if (threadIdx.x == 0) s_ok2 = 1;
    if (Cd) {
        for (int k0 = 0; k0 < n; k0 += kPKC) {
            const int kc = (n - k0) < kPKC ? (n - k0) : kPKC;
            __syncthreads();
            for (int kk = threadIdx.x >> 5; kk < kc; kk += blockDim.x >> 5)
                for (int i = lane; i < NP; i += 32) chunk[kk * NP + i] = i < n ? Cd[(size_t)(k0 + kk) * n + i] : T(0);
            __syncthreads();
            for (int kk = 0; kk < kc; ++kk) {
                T ci[RR], cj[CC];
#pragma unroll
                for (int r = 0; r < RR; ++r) ci[r] = chunk[kk * NP + w + 8 * r];
#pragma unroll
                for (int c = 0; c < CC; ++c) cj[c] = chunk[kk * NP + lane + 32 * c];
#pragma unroll
                for (int r = 0; r < RR; ++r)
#pragma unroll
                    for (int c = 0; c < CC; ++c) a[r][c] = fma(-ci[r], cj[c], a[r][c]);
            }
        }
    }
    for (int k = 0; k < n; ++k) {
        T *cb = colbuf + (k & 1) * NP;
        const int c0 = k >> 5;
        if (lane == (k & 31)) {
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                T v = a[r][0];
#pragma unroll
                for (int c = 1; c < CC; ++c) v = (c == c0) ? a[r][c] : v;
                cb[w + 8 * r] = v;
            }
        }
        __syncthreads();
        const T akk = cb[k];
        T d, inv;
        pivot(akk, d, inv);
        T li[RR], lj[CC];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            const T v = cb[w + 8 * r] * inv;
            li[r] = (w + 8 * r > k) ? v : T(0);
        }
#pragma unroll
        for (int c = 0; c < CC; ++c) {
            const T v = cb[lane + 32 * c] * inv;
            lj[c] = (lane + 32 * c > k) ? v : T(0);
        }
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
            for (int c = 0; c < CC; ++c) a[r][c] = fma(-li[r], lj[c], a[r][c]);
        if (lane == (k & 31)) {  // column k of L to shared memory (rows k..n-1)
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const int i = w + 8 * r;
                if (i >= k && i < n) A[i * n + k] = (i == k) ? d : li[r];
            }
        }
        if (threadIdx.x == 0) {
            dinv[k] = inv;
            if (!(akk > T(0))) s_ok2 = 0;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = i + 1 + lane; j < n; j += 32) A[i * n + j] = T(0);
    __syncthreads();
    return s_ok2 != 0;
}

// One warp: x <- L^{-1} x (forward) for nv <= 4 vectors X[v*n + i] (n <= 128) at once. Lane l
// holds elements i = l + 32 t of every vector in registers; step k broadcasts x_k of each vector
// from its owner lane and updates the lane's elements i > k with column k of L (Lt[k*ldt + i]).
template <typename T>
__device__ void warp_fwd_subst(T *X, int nv, const T *Lt, int ldt, const T *dinv, int n) {
    const int lane = threadIdx.x & 31;
    T x[4][4];
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = lane + 32 * t;
            x[v][t] = (v < nv && i < n) ? X[(size_t)v * n + i] : T(0);
        }
    for (int k = 0; k < n; ++k) {
        const int owner = k & 31, tk = k >> 5;
        const T dk = dinv[k];
        T l[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = lane + 32 * t;
            l[t] = (i > k && i < n) ? Lt[(size_t)k * ldt + i] : T(0);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            T mine = x[v][0];
#pragma unroll
            for (int t = 1; t < 4; ++t) mine = (tk == t) ? x[v][t] : mine;
            const T xk = __shfl_sync(kFull, mine * dk, owner);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const bool own = (lane == owner) && (t == tk);
                x[v][t] = own ? xk : fma(-xk, l[t], x[v][t]);
            }
        }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = lane + 32 * t;
            if (v < nv && i < n) X[(size_t)v * n + i] = x[v][t];
        }
}

// out(i,j) += sum_k opA(i,k) opB(j,k) over a 64 x 64 tile; opA(i,k) = A[i*lda+k] (ta=0) or A[k*lda+i]
// (ta=1); i in [i0, i0+rows), j in [j0, j0+cols), k in [0, K). Result returned through acc in
// registers (thread's 4 x 4 micro tile at (ty*4 + a, tx*4 + b), 16 x 16 threads).
template <typename T>
__device__ void cta_gemm_tile(T (&acc)[4][4], const T *A, int lda, int ta, const T *B, int ldb, int tb, int i0, int rows,
                              int j0, int cols, int K, T *sA, T *sB) {
    constexpr int LDS = kPTile + 1;  // padded: transposing stores stay conflict-free
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    for (int k0 = 0; k0 < K; k0 += kPKC) {
        const int kc = (K - k0) < kPKC ? (K - k0) : kPKC;
        __syncthreads();
        for (int q = threadIdx.x; q < kPKC * kPTile; q += blockDim.x) {
            // coalesced global reads: consecutive threads walk the contiguous dimension
            int kk = ta ? q / kPTile : q % kPKC;
            int ii = ta ? q % kPTile : q / kPKC;
            T va = T(0);
            if (kk < kc && ii < rows) va = ta ? A[(size_t)(k0 + kk) * lda + i0 + ii] : A[(size_t)(i0 + ii) * lda + k0 + kk];
            sA[kk * LDS + ii] = va;
            kk = tb ? q / kPTile : q % kPKC;
            ii = tb ? q % kPTile : q / kPKC;
            T vb = T(0);
            if (kk < kc && ii < cols) vb = tb ? B[(size_t)(k0 + kk) * ldb + j0 + ii] : B[(size_t)(j0 + ii) * ldb + k0 + kk];
            sB[kk * LDS + ii] = vb;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = sA[kk * LDS + ty * 4 + u];
                b[u] = sB[kk * LDS + tx * 4 + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
    }
}

// ---------------------------------------------------------------- the kernel

template <typename T>
__global__ void __launch_bounds__(kPThreads, 1)
    btd_persist_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat, T *C,
                       T *x, int32_t *info, Geo g, int batch, int fact, int solve) {
    cg::grid_group grid = cg::this_grid();
    BTD_STAMP_INIT();
    {   // phase 0 (a1): Dhat <- D, x <- b, info <- 0
        const size_t stride = (size_t)gridDim.x * blockDim.x;
        const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        const size_t nD = (size_t)batch * g.N * g.n * g.n, nb = (size_t)batch * g.N * g.n * g.m;
        if (fact) {
            if (D != Dhat)
                for (size_t q = t0; q < nD; q += stride) Dhat[q] = D[q];
            for (size_t q = t0; q < (size_t)batch; q += stride) info[q] = 0;
        }
        if (solve && bvec != x)
            for (size_t q = t0; q < nb; q += stride) x[q] = bvec[q];
        grid.sync();
    }
    extern __shared__ __align__(16) unsigned char psm_raw[];
    T *sm = reinterpret_cast<T *>(psm_raw);
    const int N = g.N, n = g.n, m = g.m;
    const size_t nn = (size_t)n * n;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ntile = (n + kPTile - 1) / kPTile;
    const int nrt = (n + kPRT - 1) / kPRT;

    auto Dh = [&](long long s) { return Dhat + s * N * nn; };
    auto Cs = [&](long long s) { return C + s * (size_t)g.nC * nn; };
    auto xs = [&](long long s) { return x + s * (size_t)N * n * m; };

    for (int l = 1; l <= g.L; ++l) {
        const int s = 1 << (l - 1);
        const int ncols = ((N / s) + 1) / 2;
        // ------------------------------------------------ P1: deferred l.7, potrf, forward y
        for (long long task = blockIdx.x; task < (long long)batch * ncols; task += gridDim.x) {
            const long long sy = task / ncols;
            const int j = (int)(task % ncols);
            const int c = s * (2 * j + 1);
            const bool defC = l > 1 && (c + s / 2 <= N);
            T *A = sm;                        // n x n
            T *chunk = A + nn;                // kPKC x 128
            T *yv = chunk + (size_t)kPKC * 128;  // n x m (y_c)
            T *ys = yv + (size_t)n * m;       // n x m (y_{c+s/2})
            T *dinv = ys + (size_t)n * m;     // n
            T *colk = dinv + n;               // 2 x 128 (double-buffered column)
            if (fact) cta_copy_in(A, Dh(sy) + (size_t)(c - 1) * nn, nn);
            else cta_copy_in(A, Dh(sy) + (size_t)(c - 1) * nn, nn);
            if (solve) {
                cta_copy_in(yv, xs(sy) + (size_t)(c - 1) * n * m, (size_t)n * m);
                if (defC) cta_copy_in(ys, xs(sy) + (size_t)(c + s / 2 - 1) * n * m, (size_t)n * m);
            }
            __syncthreads();
            const T *Cd = defC ? Cs(sy) + cslot(g, l - 1, 2 * c / s) * nn : nullptr;
            if (defC && solve) {  // y_c -= Cd^T y_{c+s/2}, Cd staged through `chunk`
                for (int k0 = 0; k0 < n; k0 += kPKC) {
                    const int kc = (n - k0) < kPKC ? (n - k0) : kPKC;
                    __syncthreads();
                    cta_copy_in(chunk, Cd + (size_t)k0 * n, (size_t)kc * n);
                    __syncthreads();
                    for (int q = tid; q < n * m; q += blockDim.x) {
                        const int i = q / m, qq = q % m;
                        T acc = T(0);
                        for (int kk = 0; kk < kc; ++kk) acc = fma(chunk[kk * n + i], ys[(k0 + kk) * m + qq], acc);
                        yv[q] -= acc;
                    }
                }
                __syncthreads();
            }
            if (fact) {
                // l.7 deferred downdate + l.8 POTRF, block in registers
                const bool ok = cta_chol_reg(A, n, Cd, chunk, colk, dinv);
                if (!ok && tid == 0) report_fail(info + sy, c);
                T *dst = Dh(sy) + (size_t)(c - 1) * nn;
                for (size_t q = tid; q < nn; q += blockDim.x) dst[q] = A[q];
            } else {
                for (int i = tid; i < n; i += blockDim.x) dinv[i] = rcp_rn(A[i * n + i]);
            }
            __syncthreads();
            if (solve) {
                // y_c <- L^{-1} y_c, one warp per right-hand side, left-looking (row i of L contiguous)
                for (int qq = warp; qq < m; qq += kPWarps) {
                    const int lane = tid & 31;
                    for (int i = 0; i < n; ++i) {
                        T acc = T(0);
                        for (int k = lane; k < i; k += 32) acc = fma(A[i * n + k], yv[k * m + qq], acc);
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
                        if (lane == 0) yv[i * m + qq] = (yv[i * m + qq] - acc) * dinv[i];
                        __syncwarp();
                    }
                }
                __syncthreads();
                T *dst = xs(sy) + (size_t)(c - 1) * n * m;
                for (int q = tid; q < n * m; q += blockDim.x) dst[q] = yv[q];
            }
            __syncthreads();
        }
        BTD_STAMP(0);
        grid.sync();
        BTD_STAMP(1);
        // ------------------------------------------------ P2: TRSMs (l.10, l.12)
        if (fact) {
            const long long ntask = (long long)batch * ncols * 2 * nrt;
            for (long long task = blockIdx.x; task < ntask; task += gridDim.x) {
                const long long sy = task / ((long long)ncols * 2 * nrt);
                long long rem = task % ((long long)ncols * 2 * nrt);
                const int j = (int)(rem / (2 * nrt));
                rem %= (2 * nrt);
                const int side = (int)(rem / nrt);  // 0 = right (rows of C_r), 1 = left (columns of C_l)
                const int rt = (int)(rem % nrt);
                const int c = s * (2 * j + 1);
                const bool has = side == 0 ? (c + s <= N) : (c > s);
                if (!has) continue;
                const int v0 = rt * kPRT, nv = (n - v0) < kPRT ? (n - v0) : kPRT;
                const int ldt = n + 1;
                T *Lt = sm;                         // L^T, padded rows
                T *X = Lt + (size_t)n * ldt;        // nv x n
                T *dinv = X + (size_t)kPRT * n;
                const T *Dc = Dh(sy) + (size_t)(c - 1) * nn;
                const long long slot = cslot(g, l, side == 0 ? c / s : c / s - 1);
                const T *src = (l == 1) ? (E + sy * (size_t)(N - 1) * nn + (size_t)(side == 0 ? c - 1 : c - 2) * nn)
                                        : (Cs(sy) + slot * nn);
                T *dst = Cs(sy) + slot * nn;
                for (int i = warp; i < n; i += kPWarps)  // Lt[k][i] = L[i][k] (lower part only)
                    for (int k = (tid & 31); k <= i; k += 32) Lt[(size_t)k * ldt + i] = Dc[(size_t)i * n + k];
                if (side == 0) {
                    for (int v = warp; v < nv; v += kPWarps)
                        for (int i = (tid & 31); i < n; i += 32) X[(size_t)v * n + i] = src[(size_t)(v0 + v) * n + i];
                } else {
                    for (int i = warp; i < n; i += kPWarps)
                        for (int v = (tid & 31); v < nv; v += 32) X[(size_t)v * n + i] = src[(size_t)i * n + v0 + v];
                }
                __syncthreads();
                for (int i = tid; i < n; i += blockDim.x) dinv[i] = rcp_rn(Lt[(size_t)i * ldt + i]);
                __syncthreads();
                // vectors split over warps
                const int per = (nv + kPWarps - 1) / kPWarps;
                const int a0 = warp * per, a1 = (a0 + per) < nv ? (a0 + per) : nv;
                if (a0 < a1) warp_fwd_subst(X + (size_t)a0 * n, a1 - a0, Lt, ldt, dinv, n);
                __syncthreads();
                if (side == 0) {
                    for (int v = warp; v < nv; v += kPWarps)
                        for (int i = (tid & 31); i < n; i += 32) dst[(size_t)(v0 + v) * n + i] = X[(size_t)v * n + i];
                } else {
                    for (int i = warp; i < n; i += kPWarps)
                        for (int v = (tid & 31); v < nv; v += 32) dst[(size_t)i * n + v0 + v] = X[(size_t)v * n + i];
                }
                __syncthreads();
            }
            BTD_STAMP(2);
            grid.sync();
            BTD_STAMP(3);
        }
        // ------------------------------------------------ P3: l.9 + l.11 syrk, l.13 fill, y pushes
        {
            const int nsy = ntile * (ntile + 1) / 2;  // lower tiles of D~_{c+s}
            const int nfi = ntile * ntile;            // fill tiles
            const int per_col = fact ? (nsy + nfi + (solve ? 1 : 0)) : 1;
            const long long ntask = (long long)batch * ncols * per_col;
            for (long long task = blockIdx.x; task < ntask; task += gridDim.x) {
                const long long sy = task / ((long long)ncols * per_col);
                long long rem = task % ((long long)ncols * per_col);
                const int j = (int)(rem / per_col);
                int kind = (int)(rem % per_col);
                const int c = s * (2 * j + 1);
                const bool hasL = c > s, hasR = c + s <= N;
                const bool defS = l > 1 && (c + s + s / 2 <= N);
                const T *Cr = Cs(sy) + cslot(g, l, c / s) * nn;
                if (!fact) kind = nsy + nfi;  // solve-only: the y task
                if (kind < nsy) {
                    if (!hasR) continue;
                    int ti = 0, q = kind;
                    while (q > ti) { q -= ti + 1; ++ti; }
                    const int tj = q;
                    const int i0 = ti * kPTile, j0 = tj * kPTile;
                    const int rows = (n - i0) < kPTile ? (n - i0) : kPTile, cols = (n - j0) < kPTile ? (n - j0) : kPTile;
                    T acc[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
                    T *sA = sm, *sB = sm + kPKC * (kPTile + 1);
                    if (defS) {
                        const T *Ce = Cs(sy) + cslot(g, l - 1, 2 * c / s + 2) * nn;
                        cta_gemm_tile(acc, Ce, n, 1, Ce, n, 1, i0, rows, j0, cols, n, sA, sB);  // Ce^T Ce
                    }
                    cta_gemm_tile(acc, Cr, n, 0, Cr, n, 0, i0, rows, j0, cols, n, sA, sB);       // C_r C_r^T
                    T *Dsep = Dh(sy) + (size_t)(c + s - 1) * nn;
                    const int tx = tid % 16, ty = tid / 16;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int i = ty * 4 + u, jj = tx * 4 + v;
                            if (i < rows && jj < cols) Dsep[(size_t)(i0 + i) * n + j0 + jj] -= acc[u][v];
                        }
                    __syncthreads();
                } else if (kind < nsy + nfi) {
                    if (!(hasL && hasR)) continue;
                    const int t = kind - nsy, ti = t / ntile, tj = t % ntile;
                    const int i0 = ti * kPTile, j0 = tj * kPTile;
                    const int rows = (n - i0) < kPTile ? (n - i0) : kPTile, cols = (n - j0) < kPTile ? (n - j0) : kPTile;
                    const T *Cl = Cs(sy) + cslot(g, l, c / s - 1) * nn;
                    T acc[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
                    T *sA = sm, *sB = sm + kPKC * (kPTile + 1);
                    cta_gemm_tile(acc, Cr, n, 0, Cl, n, 1, i0, rows, j0, cols, n, sA, sB);  // C_r C_l
                    T *F = Cs(sy) + cslot(g, l + 1, (c - s) / (2 * s)) * nn;
                    const int tx = tid % 16, ty = tid / 16;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int i = ty * 4 + u, jj = tx * 4 + v;
                            if (i < rows && jj < cols) F[(size_t)(i0 + i) * n + j0 + jj] = -acc[u][v];
                        }
                    __syncthreads();
                } else {
                    // y pushes into y_{c+s}: deferred left push of column c+3s/2 (level l-1) and right push of c
                    if (!solve || !hasR) continue;
                    T *ytgt = xs(sy) + (size_t)(c + s - 1) * n * m;
                    const T *yc = xs(sy) + (size_t)(c - 1) * n * m;
                    for (int q = tid; q < n * m; q += blockDim.x) {
                        const int i = q / m, qq = q % m;
                        T acc = T(0);
                        if (defS) {
                            const T *Ce = Cs(sy) + cslot(g, l - 1, 2 * c / s + 2) * nn;
                            const T *ysrc = xs(sy) + (size_t)(c + s + s / 2 - 1) * n * m;
                            for (int k = 0; k < n; ++k) acc = fma(Ce[(size_t)k * n + i], ysrc[k * m + qq], acc);
                        }
                        for (int k = 0; k < n; ++k) acc = fma(Cr[(size_t)i * n + k], yc[k * m + qq], acc);
                        ytgt[q] -= acc;
                    }
                    __syncthreads();
                }
            }
        }
        BTD_STAMP(4);
        grid.sync();
        BTD_STAMP(5);
    }

    // ------------------------------------------------ backward sweep
    if (solve) {
        for (int l = g.L; l >= 1; --l) {
            const int s = 1 << (l - 1);
            const int ncols = ((N / s) + 1) / 2;
            for (long long task = blockIdx.x; task < (long long)batch * ncols; task += gridDim.x) {
                const long long sy = task / ncols;
                const int j = (int)(task % ncols);
                const int c = s * (2 * j + 1);
                const bool hasL = c > s, hasR = c + s <= N;
                T *A = sm;                      // D^_c row-major
                T *v = A + nn;                  // n x m
                T *xr = v + (size_t)n * m;      // x_{c+s}
                T *xl = xr + (size_t)n * m;     // x_{c-s}
                T *dinv = xl + (size_t)n * m;
                cta_copy_in(A, Dh(sy) + (size_t)(c - 1) * nn, nn);
                cta_copy_in(v, xs(sy) + (size_t)(c - 1) * n * m, (size_t)n * m);
                if (hasR) cta_copy_in(xr, xs(sy) + (size_t)(c + s - 1) * n * m, (size_t)n * m);
                if (hasL) cta_copy_in(xl, xs(sy) + (size_t)(c - s - 1) * n * m, (size_t)n * m);
                __syncthreads();
                for (int i = tid; i < n; i += blockDim.x) dinv[i] = rcp_rn(A[i * n + i]);
                const T *Cr = Cs(sy) + cslot(g, l, c / s) * nn;
                const T *Cl = Cs(sy) + cslot(g, l, (c / s >= 2 ? c / s : 2) - 1) * nn;
                for (int q = tid; q < n * m; q += blockDim.x) {
                    const int i = q / m, qq = q % m;
                    T acc = T(0);
                    if (hasR)
                        for (int k = 0; k < n; ++k) acc = fma(Cr[(size_t)k * n + i], xr[k * m + qq], acc);
                    if (hasL)
                        for (int k = 0; k < n; ++k) acc = fma(Cl[(size_t)i * n + k], xl[k * m + qq], acc);
                    v[q] -= acc;
                }
                __syncthreads();
                // v <- L^{-T} v, one warp per right-hand side (row k of L contiguous)
                for (int qq = warp; qq < m; qq += kPWarps) {
                    const int lane = tid & 31;
                    for (int k = n - 1; k >= 0; --k) {
                        T xk = T(0);
                        if (lane == 0) {
                            xk = v[k * m + qq] * dinv[k];
                            v[k * m + qq] = xk;
                        }
                        xk = __shfl_sync(kFull, xk, 0);
                        for (int i = lane; i < k; i += 32) v[i * m + qq] = fma(-A[(size_t)k * n + i], xk, v[i * m + qq]);
                        __syncwarp();
                    }
                }
                __syncthreads();
                T *dst = xs(sy) + (size_t)(c - 1) * n * m;
                for (int q = tid; q < n * m; q += blockDim.x) dst[q] = v[q];
                __syncthreads();
            }
            BTD_STAMP(6);
            grid.sync();
            BTD_STAMP(7);
        }
    }
}

}  // namespace btd

namespace btd {
// ---------------------------------------------------------------- PERSIST-TEAM (n <= 32)
//
// Same dataflow as the LEVEL variant (Alg. 4 deferred form, one column op per team of lanes,
// state in the output buffers) but in ONE cooperative launch: tasks (system, column) of level l
// are spread over every team of every resident CTA and levels are separated by grid.sync(),
// so there is one launch per call instead of 2L+1 and the instruction stream stays warm.
template <typename T, int NB>
struct PTeamCfg {
    static constexpr int TS = LevelShape_TS<NB>::TS;
    static constexpr int THREADS = 256;
    static constexpr int NT = THREADS / TS;
    static constexpr int TSTR = LevelSmem<T, NB>::TSTR;
    static constexpr size_t BYTES = (size_t)NT * TSTR * sizeof(T);
};

template <typename T, int NB, bool FACT, bool SOLVE>
__global__ void __launch_bounds__(PTeamCfg<T, NB>::THREADS, 1)
    btd_persist_team_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat,
                            T *C, T *x, int32_t *info, Geo g, int batch) {
    using Cfg = PTeamCfg<T, NB>;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char ptsm_raw[];
    const int team = threadIdx.x / Cfg::TS;
    T *scr = reinterpret_cast<T *>(ptsm_raw) + (size_t)team * Cfg::TSTR;
    const long long gteam = (long long)blockIdx.x * Cfg::NT + team;
    const long long nteams = (long long)gridDim.x * Cfg::NT;
    {   // a1: Dhat <- D, x <- b, info <- 0
        const size_t stride = (size_t)gridDim.x * blockDim.x;
        const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        const size_t nD = (size_t)batch * g.N * g.n * g.n, nb = (size_t)batch * g.N * g.n * g.m;
        if (FACT) {
            if (D != Dhat)
                for (size_t q = t0; q < nD; q += stride) Dhat[q] = D[q];
            for (size_t q = t0; q < (size_t)batch; q += stride) info[q] = 0;
        }
        if (SOLVE && bvec != x)
            for (size_t q = t0; q < nb; q += stride) x[q] = bvec[q];
        grid.sync();
    }
    for (int l = 1; l <= g.L; ++l) {
        const int ncols = ((g.N >> (l - 1)) + 1) / 2;
        const long long ntask = (long long)batch * ncols;
        // all lanes of a warp iterate together (teams of one warp share the loop trip count)
        const long long first = gteam - (gteam % (32 / Cfg::TS));
        for (long long t0 = first; t0 < ntask; t0 += nteams) {
            const long long task = t0 + (gteam - first);
            const long long sys = task < ntask ? task / ncols : 0;
            const int j = task < ntask ? (int)(task % ncols) : ncols;  // j >= ncols: inactive team
            level_fwd_task<T, NB, Cfg::TS, FACT, SOLVE>(E, Dhat, C, x, info, g, l, sys, j, scr);
        }
        grid.sync();
    }
    if (SOLVE) {
        for (int l = g.L; l >= 1; --l) {
            const int ncols = ((g.N >> (l - 1)) + 1) / 2;
            const long long ntask = (long long)batch * ncols;
            const long long first = gteam - (gteam % (32 / Cfg::TS));
            for (long long t0 = first; t0 < ntask; t0 += nteams) {
                const long long task = t0 + (gteam - first);
                const long long sys = task < ntask ? task / ncols : 0;
                const int j = task < ntask ? (int)(task % ncols) : ncols;
                level_bwd_task<T, NB, Cfg::TS>(Dhat, C, x, g, l, sys, j, scr);
            }
            grid.sync();
        }
    }
}

}  // namespace btd
