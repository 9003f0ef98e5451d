// btd_wide.cuh -- WIDE variant: single long systems (BASELINE configs c2, c3), n <= 32.
//
// One cooperative launch; level l of Algorithm 4 (deferred form) is one
// grid-wide phase in which every column op is executed by a whole CTA (256 threads), and levels
// are separated by grid.sync(). Compared with one warp per column op (LEVEL / PERSIST-TEAM) this
// shortens the per-level critical path -- the quantity that sets single-system latency once the
// first levels no longer fill the GPU.
//
// Per column c of level l (stride s), every block staged in shared memory (ld NB+4, padded to
// NB in {8, 16, 32} with an identity diagonal / zeros), wide_fwd_task2:
//   l.7   A   = D~_c   - Cd^T Cd        Cd = E^_{l-1,2c/s}   (stored left coupling of column c+s/2)
//   l.9   Sep = D~_c+s - Ce^T Ce        Ce = E^_{l-1,2c/s+2} (stored left coupling of column c+3s/2)
//   l.8   A   = chol(A)                 -> Dhat[c]     (one warp; y_c rides along, Alg. 6 l.4)
//   l.10  Cr  = Cr A^-T                 -> C[slot(l, c/s)]
//   l.12  Cl  = A^-1 Cl                 -> C[slot(l, c/s-1)]
//   l.11  Sep -= Cr Cr^T                -> Dhat[c+s]
//   l.13  C[slot(l+1,(c-s)/2s)] = -Cr Cl
//   Alg. 6 forward: y_c -= Cd^T y_{c+s/2}; y_c = A^-1 y_c; y_{c+s} -= Ce^T y_{c+3s/2} + Cr y_c
// with the Schur/fill products on 8 x 8 tiles (DMMA for fp64), and the backward sweep
// x_c = A^-T (y_c - Cr^T x_{c+s} - Cl x_{c-s}) one CTA per column. The ATOMIC instantiation is
// Algorithm 5 (right-looking, atomic Schur updates; variant BTD_VARIANT_ATOMIC).
#pragma once
#include <cooperative_groups.h>

#include "btd_kernels.cuh"
#include "btd_persist2.cuh"

namespace btd {

constexpr int kWThreads = 256;

// Backward-task blocks are staged with a compile-time leading dimension NB+1 (NB in {8,16,32}
// >= n): the +1 keeps column walks conflict-free.
template <int n_>
constexpr int wide_nb() { return n_ <= 8 ? 8 : n_ <= 16 ? 16 : 32; }
template <typename T>
struct WideSmem {
    static __host__ __device__ int nb(int n) { return n <= 8 ? 8 : n <= 16 ? 16 : 32; }
    static __host__ __device__ size_t elems(int n, int m) {
        // forward task: A (+ m y rows), Cr, ClT, Cd, Ce, Sep, F with ld NB+4; ys, yt, yu; dinv
        const size_t fwd = (size_t)(7 * nb(n) + m) * (nb(n) + 4) + 3 * (size_t)n * m + nb(n);
        // backward task (ld NB+1)
        const size_t blk = (size_t)nb(n) * (nb(n) + 1);
        const size_t bwd = 4 * blk + 3 * (size_t)n * m + nb(n);
        return (fwd > bwd ? fwd : bwd) + 32;
    }
    static __host__ __device__ size_t bytes(int n, int m) { return elems(n, m) * sizeof(T); }
};

// One thread: x <- L^{-T} x (back substitution) for a vector of length n <= NB in registers, L lower
// in shared memory (ld NB+1), dinv the reciprocal diagonal; result to out[i*ostride]. Fully
// unrolled: the compiler hoists the shared-memory loads ahead of their uses.
template <typename T, int NB>
__device__ __forceinline__ void thread_trsv_upper_t(T (&x)[NB], const T *L, const T *dinv, int n, T *out,
                                                    int ostride) {
    constexpr int LD = NB + 1;
#pragma unroll
    for (int k = NB - 1; k >= 0; --k) {
        if (k < n) {  // padding rows/columns of L and dinv are never read
            x[k] *= dinv[k];
            out[(size_t)k * ostride] = x[k];
#pragma unroll
            for (int i = 0; i < k; ++i) x[i] = fma(-L[k * LD + i], x[k], x[i]);
        }
    }
}

// Asynchronous (LDGSTS) copy of an n x n global block into shared memory with leading dim ldd;
// completion: __pipeline_commit() + __pipeline_wait_prior(0) + __syncthreads() by the caller.
template <typename T>
__device__ __forceinline__ void wide_copy_block(T *dst, int ldd, const T *src, int n) {
    for (int q = threadIdx.x; q < n * n; q += blockDim.x)
        __pipeline_memcpy_async(dst + (q / n) * ldd + (q % n), src + q, sizeof(T));
}

// One column op of level l (Alg. 4 l.7-l.13 + Alg. 6 forward) by one CTA, built from the blocked
// PERSIST2 pieces at panel width NB: blocks staged with 16-byte copies (ld NB+4, identity/zero
// padded to NB), the deferred downdates (l.7, l.9), l.11 and the fill (l.13) as 8 x 8 tiles (DMMA
// for fp64), the POTRF by one warp with the y rows riding along (Alg. 6 l.4), both TRSMs as one
// batch of 2 NB vectors (rows of C_r, columns of C_l).
// ATOMIC: Algorithm 5, the fully right-looking schedule -- no deferred
// downdates; after its TRSMs the column pushes BOTH Schur updates, D~_{c-s} -= C_l^T C_l and
// D~_{c+s} -= C_r C_r^T (lower triangles), and both forward-sweep updates into the separators'
// y with atomic adds (contention <= 2). The per-level chain is potrf -> trsm -> syrk
// (3 ops instead of 4); the summation order at a separator is nondeterministic (A7).
template <typename T, int NB, bool ATOMIC = false>
__device__ void wide_fwd_task2(const T *__restrict__ E, T *Dhat, T *C, T *x, int32_t *info, const Geo &g, int l,
                               long long sys, int j, bool fact, bool solve, T *sm
#ifdef BTD_TIMING
                               , unsigned long long &btd_t_last
#endif
) {
    const int N = g.N, n = g.n, m = g.m;
    constexpr int LDW = NB + 4;
    constexpr size_t BLK = (size_t)NB * LDW;
    const size_t nn = (size_t)n * n;
    const int s = 1 << (l - 1);
    const int c = s * (2 * j + 1);
    const bool hasL = c > s, hasR = c + s <= N;
    const bool defC = !ATOMIC && l > 1 && (c + s / 2 <= N);
    const bool defS = !ATOMIC && l > 1 && (c + s + s / 2 <= N);
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;
    T *xs = x ? x + sys * (size_t)N * n * m : nullptr;
    const int ext = solve ? m : 0;
    T *A = sm;                                  // (NB + ext) x LDW: D~_c, then L; rows NB..: y_c^T
    T *Cr = A + (size_t)(NB + ext) * LDW;       // rows of C_r
    T *ClT = Cr + BLK;                          // columns of C_l as rows (must follow Cr)
    T *Cd = ClT + BLK, *Ce = Cd + BLK, *Sep = Ce + BLK, *F = Sep + BLK;
    T *ys = F + BLK, *yt = ys + (size_t)n * m, *yu = yt + (size_t)n * m;
    T *dinv = yu + (size_t)n * m;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    const long long sR = cslot(g, l, c / s), sL = cslot(g, l, hasL ? c / s - 1 : 1);
    const T *CrSrc = l == 1 ? Es + (size_t)(c - 1) * nn : Cs + sR * nn;
    const T *ClSrc = l == 1 ? Es + (size_t)(c - 2) * nn : Cs + sL * nn;

    // ---- one round of loads (LDGSTS) + padding
    cta_issue_block<T>(A, LDW, Dh + (size_t)(c - 1) * nn, n, n, n);
    if (fact && hasR) {
        cta_issue_block<T>(Cr, LDW, CrSrc, n, n, n);
        if (!ATOMIC) cta_issue_block<T>(Sep, LDW, Dh + (size_t)(c + s - 1) * nn, n, n, n);
    }
    if (!fact && hasR) cta_issue_block<T>(Cr, LDW, Cs + sR * nn, n, n, n);
    if (defC) cta_issue_block<T>(Cd, LDW, Cs + cslot(g, l - 1, 2 * c / s) * nn, n, n, n);
    if (defS) cta_issue_block<T>(Ce, LDW, Cs + cslot(g, l - 1, 2 * c / s + 2) * nn, n, n, n);
    __pipeline_commit();
    if ((fact || ATOMIC) && hasL) {  // columns of C_l, transposed (lanes over the contiguous index)
        const T *src = fact ? ClSrc : Cs + sL * nn;
        for (int i = warp; i < n; i += nw)
            for (int v = lane; v < n; v += 32) ClT[v * LDW + i] = src[(size_t)i * n + v];
    }
    if (solve) {
        for (int q = tid; q < n * m; q += blockDim.x) {
            const int i = q / m, r = q % m;
            A[(NB + r) * LDW + i] = xs[(size_t)(c - 1) * n * m + q];
            if (defC) ys[q] = xs[(size_t)(c + s / 2 - 1) * n * m + q];
            if (hasR && !ATOMIC) yt[q] = xs[(size_t)(c + s - 1) * n * m + q];
            if (defS) yu[q] = xs[(size_t)(c + s + s / 2 - 1) * n * m + q];
        }
        for (int q = tid; q < m * (NB - n); q += blockDim.x) A[(NB + q / (NB - n)) * LDW + n + q % (NB - n)] = T(0);
    }
    // padding: A identity, the other blocks zero, outside the leading n x n
    if (n < NB) {
        for (int q = tid; q < NB * NB; q += blockDim.x) {
            const int i = q / NB, jj = q % NB;
            if (i >= n || jj >= n) {
                A[i * LDW + jj] = (i == jj) ? T(1) : T(0);
                Cr[i * LDW + jj] = T(0);
                ClT[i * LDW + jj] = T(0);
            }
        }
    }
    if (fact && !hasR)
        for (int q = tid; q < NB * NB; q += blockDim.x) Cr[(q / NB) * LDW + q % NB] = T(0);
    if ((fact || ATOMIC) && !hasL)
        for (int q = tid; q < NB * NB; q += blockDim.x) ClT[(q / NB) * LDW + q % NB] = T(0);
    __pipeline_wait_prior(0);
    __syncthreads();
    BTD_STAMP(0);
    const int nt = (n + 7) / 8, ntri = nt * (nt + 1) / 2;
    // ---- l.7 / l.9 deferred left downdates  A -= Cd^T Cd,  Sep -= Ce^T Ce  (lower 8 x 8 tiles)
    if (fact && (defC || defS)) {
        for (int tt = warp; tt < 2 * ntri; tt += nw) {
            const bool second = tt >= ntri;
            if (second ? !defS : !defC) continue;
            int ti = 0, q = second ? tt - ntri : tt;
            while (q > ti) {
                q -= ti + 1;
                ++ti;
            }
            const T *M = second ? Ce : Cd;
            tile8_sub<T, true, true>(second ? Sep : A, LDW, 8 * ti, 8 * q, n, n, M, LDW, M, LDW, 0, n);
        }
    }
    if (solve && (defC || defS)) {  // y_c -= Cd^T y_{c+s/2} ;  y_{c+s} -= Ce^T y_{c+3s/2}
        for (int q = tid; q < 2 * n * m; q += blockDim.x) {
            const bool second = q >= n * m;
            if (second ? !defS : !defC) continue;
            const int qq = second ? q - n * m : q, i = qq / m, r = qq % m;
            const T *M = second ? Ce : Cd;
            const T *src = second ? yu : ys;
            T acc = T(0);
            for (int k = 0; k < n; ++k) acc = fma(M[k * LDW + i], src[k * m + r], acc);
            if (second)
                yt[qq] -= acc;
            else
                A[(NB + r) * LDW + i] -= acc;
        }
    }
    __syncthreads();
    BTD_STAMP(1);
    // ---- l.8 POTRF + Alg. 6 l.4 (the y rows)
    if (fact) {
        const bool ok = cta_potrf_blocked<T, NB>(A, LDW, n, NB, ext, dinv);
        if (!ok && tid == 0) report_fail(info + sys, c);
    } else {
        for (int i = tid; i < NB; i += blockDim.x) dinv[i] = T(1) / A[i * LDW + i];
        __syncthreads();
        if (ext) cta_trsm_blocked<T, NB>(A + (size_t)NB * LDW, LDW, ext, A, LDW, NB, dinv);
    }
    BTD_STAMP(2);
    // ---- l.10 / l.12 TRSMs: rows of C_r and columns of C_l, one batch of 2 NB vectors
    if (fact) cta_trsm_blocked<T, NB>(Cr, LDW, 2 * NB, A, LDW, NB, dinv);
    BTD_STAMP(3);
    // ---- stores of this column's L^ blocks and y_c
    if (fact) {
        T *dst = Dh + (size_t)(c - 1) * nn;
        for (int i = warp; i < n; i += nw)
            for (int jj = lane; jj < n; jj += 32) dst[(size_t)i * n + jj] = A[i * LDW + jj];
        if (hasR) {
            T *d2 = Cs + sR * nn;
            for (int i = warp; i < n; i += nw)
                for (int jj = lane; jj < n; jj += 32) d2[(size_t)i * n + jj] = Cr[i * LDW + jj];
        }
        if (hasL) {
            T *d2 = Cs + sL * nn;
            for (int i = warp; i < n; i += nw)
                for (int v = lane; v < n; v += 32) d2[(size_t)i * n + v] = ClT[v * LDW + i];
        }
    }
    if (solve)
        for (int q = tid; q < n * m; q += blockDim.x) xs[(size_t)(c - 1) * n * m + q] = A[(NB + q % m) * LDW + q / m];
    if constexpr (ATOMIC) {
        // ---- Alg. 5 l.9-l.11: S_R = C_r C_r^T (-> D~_{c+s}), S_L = C_l^T C_l (-> D~_{c-s}), fill
        T *SR = Sep, *SL = Ce;
        const bool fill = hasL && hasR;
        if (fact) {
            for (int q = tid; q < NB * NB; q += blockDim.x) {
                const int o = (q / NB) * LDW + q % NB;
                SR[o] = T(0);
                SL[o] = T(0);
                F[o] = T(0);
            }
            __syncthreads();
            for (int tt = warp; tt < 2 * ntri + (fill ? nt * nt : 0); tt += nw) {
                if (tt < 2 * ntri) {
                    const bool left = tt >= ntri;
                    if (left ? !hasL : !hasR) continue;
                    int ti = 0, q = left ? tt - ntri : tt;
                    while (q > ti) {
                        q -= ti + 1;
                        ++ti;
                    }
                    const T *M = left ? ClT : Cr;  // C_l^T C_l = sum_k ClT[i][k] ClT[j][k]
                    tile8_sub<T>(left ? SL : SR, LDW, 8 * ti, 8 * q, n, n, M, LDW, M, LDW, 0, n);
                } else {
                    const int t2 = tt - 2 * ntri;
                    tile8_sub<T>(F, LDW, 8 * (t2 / nt), 8 * (t2 % nt), n, n, Cr, LDW, ClT, LDW, 0, n);
                }
            }
            __syncthreads();
            // atomic pushes of the lower triangles (tiles hold -S); contention <= 2 per element
            for (int i = warp; i < n; i += nw)
                for (int jj = lane; jj <= i; jj += 32) {
                    if (hasR) atomicAdd(Dh + (size_t)(c + s - 1) * nn + (size_t)i * n + jj, SR[i * LDW + jj]);
                    if (hasL) atomicAdd(Dh + (size_t)(c - s - 1) * nn + (size_t)i * n + jj, SL[i * LDW + jj]);
                }
            if (fill) {
                T *dF = Cs + cslot(g, l + 1, (c - s) / (2 * s)) * nn;
                for (int i = warp; i < n; i += nw)
                    for (int jj = lane; jj < n; jj += 32) dF[(size_t)i * n + jj] = F[i * LDW + jj];
            }
        }
        if (solve) {  // y_{c+s} -= C_r y_c ; y_{c-s} -= C_l^T y_c   (atomic)
            for (int q = tid; q < 2 * n * m; q += blockDim.x) {
                const bool left = q >= n * m;
                if (left ? !hasL : !hasR) continue;
                const int qq = left ? q - n * m : q, i = qq / m, r = qq % m;
                const T *M = left ? ClT : Cr;
                T acc = T(0);
                for (int k = 0; k < n; ++k) acc = fma(M[i * LDW + k], A[(NB + r) * LDW + k], acc);
                atomicAdd(xs + (size_t)((left ? c - s : c + s) - 1) * n * m + qq, -acc);
            }
        }
    } else {
        // ---- l.11 right downdate  Sep -= Cr Cr^T  and l.13 fill  F = -Cr Cl  (8 x 8 tiles)
        if (fact && hasR) {
            const bool fill = hasL && hasR;
            if (fill)
                for (int q = tid; q < NB * NB; q += blockDim.x) F[(q / NB) * LDW + q % NB] = T(0);
            __syncthreads();
            for (int tt = warp; tt < ntri + (fill ? nt * nt : 0); tt += nw) {
                if (tt < ntri) {
                    int ti = 0, q = tt;
                    while (q > ti) {
                        q -= ti + 1;
                        ++ti;
                    }
                    tile8_sub<T>(Sep, LDW, 8 * ti, 8 * q, n, n, Cr, LDW, Cr, LDW, 0, n);
                } else {
                    const int t2 = tt - ntri;
                    tile8_sub<T>(F, LDW, 8 * (t2 / nt), 8 * (t2 % nt), n, n, Cr, LDW, ClT, LDW, 0, n);
                }
            }
            __syncthreads();
            T *dsep = Dh + (size_t)(c + s - 1) * nn;
            for (int i = warp; i < n; i += nw)
                for (int jj = lane; jj < n; jj += 32) dsep[(size_t)i * n + jj] = Sep[i * LDW + jj];
            if (fill) {
                T *dF = Cs + cslot(g, l + 1, (c - s) / (2 * s)) * nn;
                for (int i = warp; i < n; i += nw)
                    for (int jj = lane; jj < n; jj += 32) dF[(size_t)i * n + jj] = F[i * LDW + jj];
            }
        }
        if (solve && hasR) {  // y_{c+s} = yt - C_r y_c
            for (int q = tid; q < n * m; q += blockDim.x) {
                const int i = q / m, r = q % m;
                T acc = T(0);
                for (int k = 0; k < n; ++k) acc = fma(Cr[i * LDW + k], A[(NB + r) * LDW + k], acc);
                xs[(size_t)(c + s - 1) * n * m + q] = yt[q] - acc;
            }
        }
    }
    __syncthreads();
    BTD_STAMP(4);
}

template <typename T, int NB>
__device__ void wide_bwd_task(const T *Dhat, const T *C, T *x, const Geo &g, int l, long long sys, int j, T *sm) {
    const int N = g.N, n = g.n, m = g.m;
    constexpr int lda = NB + 1;
    const size_t nn = (size_t)n * n, blk = (size_t)NB * lda;
    const int s = 1 << (l - 1);
    const int c = s * (2 * j + 1);
    const bool hasL = c > s, hasR = c + s <= N;
    const T *Dh = Dhat + sys * N * nn;
    const T *Cs = C + sys * (size_t)g.nC * nn;
    T *xs = x + sys * (size_t)N * n * m;
    T *A = sm, *Cr = A + blk, *Cl = Cr + blk;
    T *v = Cl + 2 * blk, *xr = v + (size_t)n * m, *xl = xr + (size_t)n * m;  // Cl + guard
    T *dinv = xl + (size_t)n * m;
    const int tid = threadIdx.x;
    wide_copy_block(A, lda, Dh + (size_t)(c - 1) * nn, n);
    if (hasR) wide_copy_block(Cr, lda, Cs + cslot(g, l, c / s) * nn, n);
    if (hasL) wide_copy_block(Cl, lda, Cs + cslot(g, l, c / s - 1) * nn, n);
    for (int q = tid; q < n * m; q += blockDim.x) {
        v[q] = xs[(size_t)(c - 1) * n * m + q];
        if (hasR) xr[q] = xs[(size_t)(c + s - 1) * n * m + q];
        if (hasL) xl[q] = xs[(size_t)(c - s - 1) * n * m + q];
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) dinv[i] = rcp_fast(A[i * lda + i]);
    for (int q = tid; q < n * m; q += blockDim.x) {
        const int i = q / m, r = q % m;
        T acc = T(0);
        if (hasR)
            for (int k = 0; k < n; ++k) acc = fma(Cr[k * lda + i], xr[k * m + r], acc);
        if (hasL)
            for (int k = 0; k < n; ++k) acc = fma(Cl[i * lda + k], xl[k * m + r], acc);
        v[q] -= acc;
    }
    __syncthreads();
    // v <- L^{-T} v: thread r per right-hand side (unrolled back substitution)
    for (int r = tid; r < m; r += blockDim.x) {
        T w[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) w[k] = k < n ? v[k * m + r] : T(0);
        thread_trsv_upper_t<T, NB>(w, A, dinv, n, xs + (size_t)(c - 1) * n * m + r, m);
    }
    __syncthreads();
}

template <typename T, int NB, bool ATOMIC = false>
__global__ void __launch_bounds__(kWThreads, 1)
    btd_wide_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat, T *C, T *x,
                    int32_t *info, Geo g, int batch, int fact, int solve) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    BTD_STAMP_INIT();
    extern __shared__ __align__(16) unsigned char wsm_raw[];
    T *sm = reinterpret_cast<T *>(wsm_raw);
    {   // a1: Dhat <- D, x <- b, info <- 0
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
    for (int l = 1; l <= g.L; ++l) {
        const int ncols = ((g.N >> (l - 1)) + 1) / 2;
        for (long long task = blockIdx.x; task < (long long)batch * ncols; task += gridDim.x)
            wide_fwd_task2<T, NB, ATOMIC>(E, Dhat, C, x, info, g, l, task / ncols, (int)(task % ncols), fact, solve, sm
#ifdef BTD_TIMING
                                 , btd_t_last
#endif
            );
        grid.sync();
        BTD_STAMP(5);
    }
    if (solve) {
        for (int l = g.L; l >= 1; --l) {
            const int ncols = ((g.N >> (l - 1)) + 1) / 2;
            for (long long task = blockIdx.x; task < (long long)batch * ncols; task += gridDim.x)
                wide_bwd_task<T, NB>(Dhat, C, x, g, l, task / ncols, (int)(task % ncols), sm);
            BTD_STAMP(6);
            grid.sync();
            BTD_STAMP(7);
        }
    }
}

}  // namespace btd
