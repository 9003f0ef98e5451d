// btd_fused_r2.cuh -- FUSED-R2: the batched factor+solve kernel (config c5 and every batched
// small-block system with n == NB, one right-hand side).
//
// Same arithmetic as FUSED-R (btd_kernels.cuh; Algorithm 4 + Algorithm 6, PAPER.md:539-560 and
// 596-619): one CTA per system, teams of TS lanes x RPL rows, the column op's two TRSMs and y_c's
// forward substitution riding along the POTRF sweep (team_potrf_trsm), all levels and both
// sweeps in one launch. What changes is the shared-memory working set, cut so that three
// systems (CTAs) fit per SM instead of two:
//
//   * Separators D~ (even original blocks) live in "padded-lower" slots: row i keeps only its
//     first ceil((i+1)/W)*W elements (W = 16 B / sizeof(T)), which hold the lower triangle --
//     the only part ever read (A13). n = 12 fp32: 96 instead of 144 elements.
//   * Fills (Alg. 4 l.13) live in full slots indexed by ODD original blocks: the fill of column c
//     at level l (stride s) goes to odd slot c - s + 1. At level l >= 2 column c reads its left
//     coupling from odd slot c - s + 1 and its right one from odd slot c + 1 (the fills of its
//     two children), then overwrites the left slot with its own fill. Every fill is consumed by
//     exactly one column of the next level, so the slots never collide.
//   * Level-1 columns read D_c, E_{c-1}, E_c straight from HBM into registers (no staging).
//   * The left downdate C_l^T C_l is computed in phase Y from C_l (kept in registers across the
//     barrier) instead of being carried as a second block of registers.
//   * Backward-sweep cache (levels >= 3): D^_c goes back into column c's own (now dead) separator
//     slot -- it is lower triangular, so it fits; the coupling blocks of level l >= 3 go to odd
//     slots that died at level l-1 or earlier (slots of blocks 4k+3 after level 2, 8k+5 after
//     level 3, ...), assigned in order of death (R2Cache).
//
// Shared memory (elements of T): odd slots  NO * BLK,  even slots  NE * PLB,  Y  N * LD.
#pragma once
#include <cuda_pipeline.h>

#include "btd_kernels.cuh"

namespace btd {

// Padded-lower block layout: row i holds elements [0, len(i)) with len(i) = (i / W + 1) * W.
template <typename T, int NB>
struct PLow {
    static constexpr int W = VecT<T>::W;
    static constexpr int LD = Dims<T, NB>::LD;
    __host__ __device__ static constexpr int off(int i) {
        // sum_{r < i} (r / W + 1) W = W (W g (g + 1) / 2 + rem (g + 1)),  g = i / W, rem = i % W
        return W * (W * (i / W) * (i / W + 1) / 2 + (i % W) * (i / W + 1));
    }
    static constexpr int SZ0 = off(NB);
    // slot stride: odd multiple of 16 elements (= 64 B fp32) apart from a multiple of 32 banks, so
    // the two teams of a quarter-warp that touch neighbouring slots hit different banks
    static constexpr int SZ = (SZ0 % 32 == 0) ? SZ0 + 16 / (int)(sizeof(T) / 4) : SZ0;
};

template <typename T, int NB>
struct FusedR2Cfg {
    using R = FusedRCfg<T, NB>;
    static constexpr int TS = R::TS, RPL = R::RPL, THREADS = R::THREADS, NT = R::NT;
    static constexpr bool OK = R::OK;
    static constexpr int BLK = Dims<T, NB>::BLK, LD = Dims<T, NB>::LD, PLB = PLow<T, NB>::SZ;
    static __host__ __device__ int n_odd(int N) { return (N + 1) / 2; }
    static __host__ __device__ int n_even(int N) { return N / 2; }
    static __host__ __device__ size_t bytes(int N) {
        return ((size_t)n_odd(N) * BLK + (size_t)n_even(N) * PLB + (size_t)N * LD) * sizeof(T);
    }
};

// Lane's rows of a padded-lower block (entries above the diagonal read as zero).
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void pl_load_rows(T (&v)[RPL][NB], const T *blk, const Lane<NB, TS> &ln) {
    constexpr int W = VecT<T>::W;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i = ln.row(t);
        const T *p = blk + PLow<T, NB>::off(i);
        // only the row's own chunks (w <= i): the next row belongs to another lane (no shared reads
        // of words another lane may be storing)
#pragma unroll
        for (int w = 0; w < NB; w += W) {
            T tt[W];
            if (w <= i) {
                unpack(*reinterpret_cast<const typename VecT<T>::type *>(p + w), tt);
            } else {
#pragma unroll
                for (int q = 0; q < W; ++q) tt[q] = T(0);
            }
#pragma unroll
            for (int q = 0; q < W; ++q) v[t][w + q] = (w + q > i) ? T(0) : tt[q];
        }
    }
}

// Store the lane's rows (vector chunks up to and including the one holding the diagonal).
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void pl_store_rows(T *blk, const T (&v)[RPL][NB], const Lane<NB, TS> &ln) {
    constexpr int W = VecT<T>::W;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i = ln.row(t);
        T *p = blk + PLow<T, NB>::off(i);
#pragma unroll
        for (int w = 0; w < NB; w += W) {
            if (w <= i) {
                if (w + W <= NB) {
                    T tt[W];
#pragma unroll
                    for (int q = 0; q < W; ++q) tt[q] = v[t][w + q];
                    *reinterpret_cast<typename VecT<T>::type *>(p + w) = pack4(tt);
                } else {
#pragma unroll
                    for (int q = 0; q < W; ++q)
                        if (w + q < NB) p[w + q] = v[t][w + q];
                }
            }
        }
    }
}

// acc (lane's rows of a padded-lower separator) -= S (lower triangle, lane's rows).
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void pl_sub_rows(T *blk, const T (&S)[RPL][NB], const Lane<NB, TS> &ln) {
    T acc[RPL][NB];
    pl_load_rows<T, NB, TS, RPL>(acc, blk, ln);
#pragma unroll
    for (int t = 0; t < RPL; ++t)
#pragma unroll
        for (int q = 0; q < NB; ++q) acc[t][q] -= S[t][q];
    pl_store_rows<T, NB, TS, RPL>(blk, acc, ln);
}

// Backward-sweep cache of FUSED-R2: coupling block number q (levels >= LC in order, each level's
// blocks k = 1..N/s-1) -> odd slot index. Odd slot o = (c-1)/2 holds fills until its block's
// last use; slots with v2(o) = g die when level g + 2 ends. Entries are handed out in order of
// death (all v2 = 0 slots, then v2 = 1, ...), which keeps every entry of level l inside slots
// that died by the end of level l - 1 (checked on the host: tests/test_abi.py mirrors this).
struct R2Cache {
    int LC;
    __device__ static int ccount(int N, int l) { return (N >> (l - 1)) - 1; }
    __device__ static int group_count(int NO, int g) {  // #{o < NO : v2(o) = g}, o >= 1
        const int m = (NO - 1) >> g;
        return (m + 1) / 2;
    }
    __device__ void init(int N, int L) {
        // first level whose couplings fit, given the slots dead before it starts
        LC = L + 1;
        const int NO = (N + 1) / 2;
        for (int lc = 3; lc <= L; ++lc) {
            bool ok = true;
            int need = 0;
            for (int l = lc; l <= L && ok; ++l) {
                need += ccount(N, l);
                int have = 0;
                for (int g = 0; g <= l - 3; ++g) have += group_count(NO, g);
                ok = need <= have;
            }
            if (ok) {
                LC = lc;
                break;
            }
        }
    }
    __device__ int base(int N, int l) const {
        int q = 0;
        for (int l2 = LC; l2 < l; ++l2) q += ccount(N, l2);
        return q;
    }
    __device__ static int slot(int NO, int q) {
        int g = 0;
        for (;;) {
            const int cg = group_count(NO, g);
            if (q < cg) return (2 * q + 1) << g;
            q -= cg;
            ++g;
        }
    }
};

// ---------------------------------------------------------------- L2 eviction-priority hints
// Inputs (D, E, b) are read once and the outputs of the levels the backward sweep reads from the
// shared-memory cache are never read again: both stream through L2 with evict_first. The L^ blocks
// of the levels below the cache are re-read by the backward sweep: they are written evict_last
// and read back evict_first, so that they survive the other CTAs' streams in between.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void ldg_v(float (&t)[4], const float *p, uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(t[0]), "=f"(t[1]), "=f"(t[2]), "=f"(t[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ldg_v(double (&t)[2], const double *p, uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(t[0]), "=d"(t[1]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ float ldg_s(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ldg_s(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// coherent loads (no .nc): for blocks this kernel wrote earlier (the backward sweep's L^ reads)
__device__ __forceinline__ void ldc_v(float (&t)[4], const float *p, uint64_t pol) {
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(t[0]), "=f"(t[1]), "=f"(t[2]), "=f"(t[3]) : "l"(p), "l"(pol) : "memory");
}
__device__ __forceinline__ void ldc_v(double (&t)[2], const double *p, uint64_t pol) {
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(t[0]), "=d"(t[1]) : "l"(p), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ float ldc_s(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ double ldc_s(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ void stg_v(float *p, const float (&t)[4], uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(t[0]), "f"(t[1]), "f"(t[2]),
                 "f"(t[3]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void stg_v(double *p, const double (&t)[2], uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(t[0]), "d"(t[1]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void stg_s(float *p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_s(double *p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// Exact-size (n == NB, rows whole 16-byte vectors) block I/O of the lane's rows / columns with a
// policy; `on` false gives identity (id) or zero rows and stores nothing.
template <typename T, int NB, int TS, int RPL, bool COH = false>
__device__ __forceinline__ void h_load_rows(T (&v)[RPL][NB], const T *blk, const Lane<NB, TS> &ln, bool on, bool id,
                                            uint64_t pol) {
    constexpr int W = VecT<T>::W;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i = ln.row(t);
        if (on) {
#pragma unroll
            for (int w = 0; w < NB; w += W) {
                T tt[W];
                if (COH)
                    ldc_v(tt, blk + (size_t)i * NB + w, pol);
                else
                    ldg_v(tt, blk + (size_t)i * NB + w, pol);
#pragma unroll
                for (int q = 0; q < W; ++q) v[t][w + q] = tt[q];
            }
        } else {
#pragma unroll
            for (int j = 0; j < NB; ++j) v[t][j] = (id && j == i) ? T(1) : T(0);
        }
    }
}
template <typename T, int NB, int TS, int RPL, bool COH = false>
__device__ __forceinline__ void h_load_cols(T (&v)[RPL][NB], const T *blk, const Lane<NB, TS> &ln, bool on,
                                            uint64_t pol) {
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i = ln.row(t);
#pragma unroll
        for (int k = 0; k < NB; ++k) v[t][k] = on ? (COH ? ldc_s(blk + k * NB + i, pol) : ldg_s(blk + k * NB + i, pol)) : T(0);
    }
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void h_store_rows(T *blk, const T (&v)[RPL][NB], const Lane<NB, TS> &ln, bool on,
                                             uint64_t pol) {
    constexpr int W = VecT<T>::W;
    if (!on) return;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i = ln.row(t);
#pragma unroll
        for (int w = 0; w < NB; w += W) {
            T tt[W];
#pragma unroll
            for (int q = 0; q < W; ++q) tt[q] = v[t][w + q];
            stg_v(blk + (size_t)i * NB + w, tt, pol);
        }
    }
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void h_store_cols(T *blk, const T (&v)[RPL][NB], const Lane<NB, TS> &ln, bool on,
                                             uint64_t pol) {
    if (!on) return;
#pragma unroll
    for (int t = 0; t < RPL; ++t)
#pragma unroll
        for (int k = 0; k < NB; ++k) stg_s(blk + k * NB + ln.row(t), v[t][k], pol);
}

template <typename T, int NB, int TS, int NT, int MINB>
__global__ void __launch_bounds__(NT *TS, MINB)
    btd_fused_r2_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat, T *C,
                        T *x, int32_t *info, Geo g, int sys0) {
    using Cfg = FusedR2Cfg<T, NB>;
    constexpr int LD = Cfg::LD, BLK = Cfg::BLK, PLB = Cfg::PLB;
    constexpr int RPL = NB / TS;
    constexpr int TPW = 32 / TS;
    constexpr int W = VecT<T>::W;
    using V = typename VecT<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned s_fail;

    const int N = g.N;
    constexpr int n = NB;
    const int NO = Cfg::n_odd(N), NE = Cfg::n_even(N);
    T *odd = reinterpret_cast<T *>(smem_raw);
    T *even = odd + (size_t)NO * BLK;
    T *Y = even + (size_t)NE * PLB;
    auto OS = [&](int c) { return odd + (size_t)((c - 1) >> 1) * BLK; };  // odd block c's slot
    auto ES = [&](int c) { return even + (size_t)((c >> 1) - 1) * PLB; };  // even block c's slot

    const long long sys = (long long)blockIdx.x + sys0;
    constexpr size_t nn = (size_t)n * n;
    const T *Ds = D + sys * N * nn;
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;

    const int tid = threadIdx.x, warp = tid >> 5, team = tid / TS;
    const int lane = tid & 31;
    Lane<NB, TS> ln{lane % TS, lane - lane % TS};

    R2Cache bc;
    bc.init(N, g.L);
    if (tid == 0) s_fail = 0xffffffffu;

    // ---- a1: even D blocks -> padded-lower slots, b -> Y (asynchronous 16-byte copies). The odd
    // blocks are read by their level-1 columns straight from HBM (measured faster than staging
    // them: 3.65 M vs 3.51 M systems/s on c5).
    {
        constexpr int CH = LD / W;  // 16-byte chunks per full row
        const int tot = NE * NB * CH;
        for (int q = tid; q < tot; q += blockDim.x) {
            const int e = q / (NB * CH), rem = q % (NB * CH), i = rem / CH, w = rem % CH;
            if (w * W <= i) {
                const T *src = Ds + (size_t)(2 * e + 1) * nn + (size_t)i * n + w * W;
                __pipeline_memcpy_async(reinterpret_cast<V *>(even + (size_t)e * PLB + PLow<T, NB>::off(i) + w * W),
                                        reinterpret_cast<const V *>(src), 16);
            }
        }
        const T *bs = bvec + sys * (size_t)N * n;
        for (int q = tid; q < N * n / W; q += blockDim.x)
            __pipeline_memcpy_async(reinterpret_cast<V *>(Y) + q, reinterpret_cast<const V *>(bs) + q, 16);
        __pipeline_commit();
        __pipeline_wait_prior(0);
    }
    __syncthreads();

    for (int l = 1; l <= g.L; ++l) {
        const int s = 1 << (l - 1);
        const int ncols = ((N / s) + 1) / 2;
        const long long offL = g.off[l - 1];
        for (int j0 = 0; j0 < ncols; j0 += NT) {
            const int j = j0 + team;
            const bool wact = j0 + warp * TPW < ncols;
            const bool act = j < ncols;
            const int c = act ? s * (2 * j + 1) : s;  // inactive teams shadow a valid column, store nothing
            const bool hasL = act && c > s;
            const bool hasR = act && (c + s <= N);
            T cl[RPL][NB];  // lane's columns of the left coupling (kept for phase Y)
            if (wact) {
                T yv[NB];
                T cr[RPL][NB];
                T a[RPL][NB];
                // -- a4 operands and a3's block: level 1 from HBM, later levels from the slots.
                // A missing coupling (hasR / hasL false) reads some finite block: every use of it
                // below is guarded by the same flag.
                if (l == 1) {
                    const uint64_t pf = l2_evict_first();
                    h_load_rows<T, NB, TS, RPL>(a, Ds + (size_t)(c - 1) * nn, ln, act, true, pf);
                    h_load_rows<T, NB, TS, RPL>(cr, Es + (size_t)(c - 1) * nn, ln, hasR, false, pf);
                    h_load_cols<T, NB, TS, RPL>(cl, Es + (size_t)((c >= 2 ? c : 2) - 2) * nn, ln, hasL, pf);
                } else {
                    // inactive teams shadow column s, whose team may be writing D^_s into ES(s)
                    if (act) pl_load_rows<T, NB, TS, RPL>(a, ES(c), ln);
                    s_load_rows<T, NB, TS, RPL>(cr, OS(hasR ? c + 1 : c - s + 1), ln);
                    s_load_cols<T, NB, TS, RPL>(cl, OS(c - s + 1), ln);
                }
                if (act) {  // inactive teams shadow column s: they must not read the y it is writing
                    vload<T, NB>(yv, Y + (size_t)(c - 1) * LD);
                } else {
#pragma unroll
                    for (int k = 0; k < NB; ++k) yv[k] = T(0);
                    set_identity<T, NB, TS, RPL>(a, ln);
                }
                // -- a3 + a4 + a6 (Alg. 4 l.8, l.10, l.12; Alg. 6 l.4) in one sweep
                const int bad = team_potrf_trsm<T, NB, TS, RPL, true>(a, cr, cl, yv, ln);
                if (act && bad >= 0 && ln.q == 0) atomicMin(&s_fail, fail_key(c));
                if (l >= bc.LC && act) {  // backward-sweep cache (R2Cache)
                    pl_store_rows<T, NB, TS, RPL>(ES(c), a, ln);
                    const int qb = bc.base(N, l);
                    if (hasR) s_store_rows<T, NB, TS, RPL>(odd + (size_t)R2Cache::slot(NO, qb + c / s - 1) * BLK, cr, ln);
                    if (hasL) s_store_cols<T, NB, TS, RPL>(odd + (size_t)R2Cache::slot(NO, qb + c / s - 2) * BLK, cl, ln);
                }
                {
                    // levels below the backward cache are re-read by the backward sweep: keep them in L2
                    const uint64_t po = l >= bc.LC ? l2_evict_first() : l2_evict_last();
                    h_store_rows<T, NB, TS, RPL>(Dh + (size_t)(c - 1) * nn, a, ln, act, po);
                    h_store_rows<T, NB, TS, RPL>(Cs + (offL + c / s - 1) * nn, cr, ln, hasR, po);
                    h_store_cols<T, NB, TS, RPL>(Cs + (offL + c / s - 2) * nn, cl, ln, hasL, po);
                }
                // -- a6: y_c final for this level, y_{c+s} -= C_r y_c
                {
                    T *yc = Y + (size_t)(c - 1) * LD;
                    __syncwarp();
#pragma unroll
                    for (int t = 0; t < RPL; ++t) {
                        if (act) yc[ln.row(t)] = select_idx<T, NB>(yv, ln.row(t));
                        if (hasR) {
                            T d = T(0);
#pragma unroll
                            for (int k = 0; k < NB; ++k) d = fma(cr[t][k], yv[k], d);
                            Y[(size_t)(c + s - 1) * LD + ln.row(t)] -= d;
                        }
                    }
                }
                // -- a2 (right, Alg. 4 l.11): D~_{c+s} -= C_r C_r^T  (rows of C_r by shuffles, lower only)
                {
                    T SR[RPL][NB];
                    set_zero<T, NB, RPL>(SR);
#pragma unroll
                    for (int jj = 0; jj < NB; ++jj)
#pragma unroll
                        for (int k = 0; k < NB; ++k) {
                            const T v = __shfl_sync(kFull, cr[jj / TS][k], ln.base + jj % TS);  // C_r[jj][k]
#pragma unroll
                            for (int t = jj / TS; t < RPL; ++t) SR[t][jj] = fma(cr[t][k], v, SR[t][jj]);
                        }
                    if (hasR) pl_sub_rows<T, NB, TS, RPL>(ES(c + s), SR, ln);
                }
                // -- a5 (Alg. 4 l.13): fill -C_r C_l -> odd slot c - s + 1 (columns of C_l by shuffles)
                {
                    T F[RPL][NB];
                    set_zero<T, NB, RPL>(F);
#pragma unroll
                    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
                        for (int k = 0; k < NB; ++k) {
                            const T v = __shfl_sync(kFull, cl[bb / TS][k], ln.base + bb % TS);  // C_l[k][bb]
#pragma unroll
                            for (int t = 0; t < RPL; ++t) F[t][bb] = fma(-cr[t][k], v, F[t][bb]);
                        }
                    if (hasL && hasR) s_store_rows<T, NB, TS, RPL>(OS(c - s + 1), F, ln);
                }
            }
            __syncthreads();
            // ---- phase Y: left pushes (deferred left-looking part of Alg. 4, l.7/l.9; Alg. 6 l.5)
            if (wact) {
                T SL[RPL][NB];  // lane's rows of C_l^T C_l (lower)
                set_zero<T, NB, RPL>(SL);
#pragma unroll
                for (int bb = 0; bb < NB; ++bb)
#pragma unroll
                    for (int k = 0; k < NB; ++k) {
                        const T v = __shfl_sync(kFull, cl[bb / TS][k], ln.base + bb % TS);  // C_l[k][bb]
#pragma unroll
                        for (int t = bb / TS; t < RPL; ++t) SL[t][bb] = fma(cl[t][k], v, SL[t][bb]);
                    }
                if (hasL) {
                    pl_sub_rows<T, NB, TS, RPL>(ES(c - s), SL, ln);  // D~_{c-s} -= C_l^T C_l
                    const T *yc = Y + (size_t)(c - 1) * LD;
#pragma unroll
                    for (int t = 0; t < RPL; ++t)  // y_{c-s} -= C_l^T y_c
                        Y[(size_t)(c - s - 1) * LD + ln.row(t)] -= dot<T, NB>(cl[t], yc);
                }
            }
            __syncthreads();
        }
    }

    // ---- a7: backward sweep, l = L..1 (Alg. 6 lines 10-16)
    for (int l = g.L; l >= 1; --l) {
        const int s = 1 << (l - 1);
        const int ncols = ((N / s) + 1) / 2;
        const long long offL = g.off[l - 1];
        for (int j0 = 0; j0 < ncols; j0 += NT) {
            if (j0 + warp * TPW >= ncols) continue;  // warp-uniform
            const int j = j0 + team;
            const bool act = j < ncols;
            const int c = act ? s * (2 * j + 1) : s;
            const bool hasL = act && c > s;
            const bool hasR = act && (c + s <= N);
            T *yc = Y + (size_t)(c - 1) * LD;
            const int qb = l >= bc.LC ? bc.base(N, l) : 0;
            {
                // y_c - C_r^T x_{c+s} - C_l x_{c-s}: the couplings first, so that they are dead
                // before the whole of L^_c is brought into registers
                T crc[RPL][NB], clr[RPL][NB];
                if (l >= bc.LC) {  // upper levels: from the shared-memory cache
                    const T *sr = hasR ? odd + (size_t)R2Cache::slot(NO, qb + c / s - 1) * BLK : odd;
                    const T *sl = hasL ? odd + (size_t)R2Cache::slot(NO, qb + c / s - 2) * BLK : odd;
                    s_load_cols<T, NB, TS, RPL>(crc, sr, ln);
                    s_load_rows<T, NB, TS, RPL>(clr, sl, ln);
                } else {
                    const uint64_t pf = l2_evict_first();
                    h_load_cols<T, NB, TS, RPL, true>(crc, Cs + (offL + c / s - 1) * nn, ln, hasR, pf);
                    h_load_rows<T, NB, TS, RPL, true>(clr, Cs + (offL + (c / s >= 2 ? c / s : 2) - 2) * nn, ln, hasL, false,
                                                pf);
                }
                const T *xr = Y + (size_t)((hasR ? c + s : c) - 1) * LD;
                const T *xl = Y + (size_t)((hasL ? c - s : c) - 1) * LD;
                T mine[RPL];
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    // inactive teams (shadowing column s) read no y: column s's team is writing it
                    const T a = hasR ? dot<T, NB>(crc[t], xr) : T(0);   // (C_r^T x_{c+s})[i]
                    const T b2 = hasL ? dot<T, NB>(clr[t], xl) : T(0);  // (C_l x_{c-s})[i]
                    mine[t] = act ? yc[ln.row(t)] : T(0);
                    mine[t] -= hasR ? a : T(0);
                    mine[t] -= hasL ? b2 : T(0);
                }
                __syncwarp();
#pragma unroll
                for (int t = 0; t < RPL; ++t)
                    if (act) yc[ln.row(t)] = mine[t];
                __syncwarp();
            }
            T Lf[NB][NB], Linv[NB];
            if (l >= bc.LC) {
                const T *pd = ES(c);
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const T *pr = pd + PLow<T, NB>::off(i);  // row i: its own chunks only
#pragma unroll
                    for (int w = 0; w <= i; w += W) {
                        T tt[W];
                        unpack(*reinterpret_cast<const typename VecT<T>::type *>(pr + w), tt);
#pragma unroll
                        for (int q = 0; q < W; ++q)
                            if (w + q <= i) Lf[i][w + q] = tt[q];
                    }
                    Linv[i] = rcp_fast(Lf[i][i]);
                }
            } else {
                const uint64_t pf = l2_evict_first();
                const T *blk = Dh + (size_t)(c - 1) * nn;
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    T row[NB];
#pragma unroll
                    for (int w = 0; w < NB; w += W) {
                        T tt[W];
                        ldc_v(tt, blk + (size_t)i * NB + w, pf);
#pragma unroll
                        for (int q = 0; q < W; ++q) row[w + q] = tt[q];
                    }
#pragma unroll
                    for (int k = 0; k <= i; ++k) Lf[i][k] = row[k];
                    Linv[i] = rcp_fast(row[i]);
                }
            }
            T v[NB];
            if (act) {
                vload<T, NB>(v, yc);
            } else {
#pragma unroll
                for (int k = 0; k < NB; ++k) v[k] = T(0);
            }
            bwd_full<T, NB>(v, Lf, Linv);
            __syncwarp();
            // x_c is final: write it to Y (read by the lower levels) and straight to HBM
            T *xs = x + (sys * (size_t)N + (c - 1)) * n;
            const uint64_t px = l2_evict_first();
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                const T xv = select_idx<T, NB>(v, ln.row(t));
                if (act) yc[ln.row(t)] = xv;
                if (act) stg_s(xs + ln.row(t), xv, px);
            }
        }
        __syncthreads();
    }
    if (tid == 0) info[sys] = (s_fail == 0xffffffffu) ? 0 : (int)(s_fail & ((1u << 25) - 1));
}

}  // namespace btd
