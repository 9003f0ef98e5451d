// btd_kernels.cuh -- the level kernels of the multi-stage block-tridiagonal Cholesky.
//
// Two realisations of Algorithm 4 (factor) + Algorithm 6 (solve,
// PAPER.md:596-619), both built from the team primitives of btd_team.cuh:
//
//  FUSED  one CTA per system runs every level and both sweeps in one launch. The working
//         blocks live in shared memory in one slot per original block index:
//           slot[i] = D~_i (the Schur-updated diagonal block) until column i is eliminated,
//                     afterwards the raw fill coupling produced by column i (Alg. 4 l.13),
//         so a column c at level l reads its couplings from slot[c -+ s/2] (l > 1) or E (l = 1).
//         Schur downdates are owner-free pushes split in two phases per round of columns:
//         phase X pushes to the right separator (Alg. 4 l.11), phase Y -- after a CTA barrier --
//         to the left separator (the update Alg. 4 defers to the next level, l.7/l.9), so a
//         separator always receives left child then right child, race-free and deterministic.
//         L^ streams to HBM once; the backward sweep re-reads it (L2-resident).
//
//  LEVEL  one launch per level for factor(+forward) and one per level for the backward sweep,
//         state in the caller's output buffers (D~ in Dhat, raw fill in its final C slot, y/x
//         in x). This is Algorithm 4's literal deferred form: column i at level l first applies
//         the left downdates of level l-1 to D^_i (l.7) and D^_{i+s} (l.9), then potrf (l.8),
//         trsm (l.10/l.12), the right downdate (l.11) and the fill gemm (l.13). Used when a
//         system does not fit in one SM's shared memory (long horizons, large n).
//
// Indices: original blocks are 1-based; slot (l, k) of C is at off[l-1] + k - 1 (include/btd.h).
#pragma once
#include "btd_team.cuh"

namespace btd {

struct Geo {
    int N, n, m, L;
    long long nC;       // coupling blocks per system
    long long off[34];  // off[l-1] = first slot of level l (l = 1..L+1)
};

__device__ __forceinline__ long long cslot(const Geo &g, int l, int k) { return g.off[l - 1] + k - 1; }

// ============================================================================ FUSED
//
// Shared memory (elements of T):
//   slots   N * BLK            (FACT only)
//   Y       N * m * LD         (SOLVE only; y then x, one padded row per block and rhs)
//   scratch NT * TSTR          (3 blocks per team: sLt (later reused as sCl), sCr, sClT;
//                               TSTR padded by 64 B so the two teams of a warp hit different banks)
template <typename T, int NB, int NT>
struct FusedSmem {
    static constexpr int LD = Dims<T, NB>::LD;
    static constexpr int BLK = Dims<T, NB>::BLK;
    static constexpr int TSTR = 3 * BLK + 64 / (int)sizeof(T);
    static __host__ __device__ size_t bytes(int N, int m, bool fact, bool solve) {
        size_t e = (fact ? (size_t)N * BLK : 0) + (solve ? (size_t)N * m * LD : 0) + (size_t)NT * TSTR;
        return e * sizeof(T);
    }
};

// Launch shape of the fused kernel for block size NB: team width TS, CTA threads, min CTAs/SM.
template <typename T, int NB>
struct FusedCfg {
    static constexpr int TS = NB <= 1 ? 1 : NB <= 2 ? 2 : NB <= 4 ? 4 : NB <= 8 ? 8 : NB <= 16 ? 16 : 32;
    static constexpr int LIM = sizeof(T) == 4 ? 16 : 8;  // register rows per lane that fit 128 regs
    static constexpr int THREADS = NB <= LIM ? 256 : 128;
    static constexpr int NT = THREADS / TS;
    static constexpr int MINB = NB <= LIM ? 2 : 1;
};

// MR = number of right-hand sides if fixed at compile time (1), 0 = runtime g.m.
template <typename T, int NB, int TS, int NT, bool FACT, bool SOLVE, int MR>
__global__ void __launch_bounds__(NT *TS, FusedCfg<T, NB>::MINB)
    btd_fused_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat, T *C,
                     T *x, int32_t *info, Geo g, int sys0) {
    using S = FusedSmem<T, NB, NT>;
    constexpr int LD = S::LD, BLK = S::BLK;
    constexpr int TPW = 32 / TS;  // teams per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *smem = reinterpret_cast<T *>(smem_raw);
    T *slots = smem;
    T *Y = smem + (FACT ? (size_t)g.N * BLK : 0);
    __shared__ unsigned s_fail;

    const int N = g.N, n = g.n;
    const int m = MR > 0 ? MR : g.m;
    T *scr = Y + (SOLVE ? (size_t)N * m * LD : 0);
    const long long sys = (long long)blockIdx.x + sys0;
    const size_t nn = (size_t)n * n;
    const T *Ds = D ? D + sys * N * nn : nullptr;
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int team = tid / TS;
    const int r = lane % TS;
    const int base = lane - r;
    const bool rv = r < NB;  // lane owns a (possibly padded) row
    const int rr = rv ? r : 0;
    T *sLt = scr + (size_t)team * S::TSTR;
    T *sCl = sLt;  // reuses sLt once both TRSMs are done
    T *sCr = sLt + BLK;
    T *sClT = sCr + BLK;

    if (tid == 0) s_fail = 0xffffffffu;
    // ---- a1: load.  slots <- D (padded with identity); Y <- b.
    if (FACT) {
        if (n == NB && LD == NB) {
            constexpr int W = VecT<T>::W;
            const size_t tot = (size_t)N * nn;
            if (tot % W == 0) {
                using V = typename VecT<T>::type;
                const V *src = reinterpret_cast<const V *>(Ds);
                V *dst = reinterpret_cast<V *>(slots);
                for (size_t q = tid; q < tot / W; q += blockDim.x) dst[q] = src[q];
            } else {
                for (size_t q = tid; q < tot; q += blockDim.x) slots[q] = Ds[q];
            }
        } else {
            for (size_t q = tid; q < (size_t)N * BLK; q += blockDim.x) {
                const int i = (int)(q / BLK), r2 = (int)((q % BLK) / LD), c2 = (int)(q % LD);
                T v = T(0);
                if (r2 < n && c2 < n)
                    v = Ds[(size_t)i * nn + (size_t)r2 * n + c2];
                else if (r2 == c2)
                    v = T(1);
                slots[q] = v;
            }
        }
    }
    if (SOLVE) {
        const T *bs = bvec + sys * (size_t)N * n * m;
        for (size_t q = tid; q < (size_t)N * m * LD; q += blockDim.x) {
            const int i = (int)(q / ((size_t)m * LD)), rem = (int)(q % ((size_t)m * LD));
            const int qq = rem / LD, r2 = rem % LD;
            Y[q] = (r2 < n) ? bs[((size_t)i * n + r2) * m + qq] : T(0);
        }
    }
    __syncthreads();

    // ---- levels l = 1..L (stride s): a2-a6
    for (int l = 1; l <= g.L; ++l) {
        const int s = 1 << (l - 1);
        const int ncols = ((N / s) + 1) / 2;
        const long long offL = g.off[l - 1];
        const long long offN = g.off[l];
        for (int j0 = 0; j0 < ncols; j0 += NT) {
            const int j = j0 + team;
            const bool wact = j0 + warp * TPW < ncols;  // warp has at least one active team
            const bool act = j < ncols;
            const int c = s * (2 * j + 1);
            const bool hasL = act && c > s;
            const bool hasR = act && (c + s <= N);
            T cl[NB];
            if (wact) {
                // -- a3: D~_c -> D^_c
                T dl[NB];
                if (FACT) {
                    vload<T, NB>(dl, slots + (size_t)((act ? c : 1) - 1) * BLK + rr * LD);
                    if (!(act && rv)) {
#pragma unroll
                        for (int q = 0; q < NB; ++q) dl[q] = (q == r) ? T(1) : T(0);
                    }
                    const int bad = team_potrf<T, NB>(dl, r, base);
                    if (act && bad >= 0 && r == 0) atomicMin(&s_fail, fail_key(c));
                    g_store_row<T, NB>(Dh + (size_t)(c - 1) * nn, dl, n, r, act);
                } else {
                    g_load_row<T, NB>(dl, Dh + (size_t)(c - 1) * nn, n, r, act, true);
                }
                team_put_Lt<T, NB>(sLt, dl, r);

                // -- a4: couplings. cr = row r of the right coupling, cl = column r of the left one.
                T cr[NB];
                if (FACT) {
                    if (l == 1) {
                        g_load_row<T, NB>(cr, Es + (size_t)(c - 1) * nn, n, r, hasR, false);  // E_c   = (c+1, c)
                        g_load_col<T, NB>(cl, Es + (size_t)(c - 2) * nn, n, r, hasL, false);  // E_c-1 = (c, c-1)
                    } else {
                        vload<T, NB>(cr, slots + (size_t)((hasR ? c + s / 2 : 1) - 1) * BLK + rr * LD);
                        const T *pl = slots + (size_t)((hasL ? c - s / 2 : 1) - 1) * BLK + rr;
#pragma unroll
                        for (int q = 0; q < NB; ++q) cl[q] = pl[q * LD];
#pragma unroll
                        for (int q = 0; q < NB; ++q) {
                            cr[q] = (hasR && rv) ? cr[q] : T(0);
                            cl[q] = (hasL && rv) ? cl[q] : T(0);
                        }
                    }
                    __syncwarp();
                    tri_solve<T, NB>(cr, sLt);  // Alg. 4 l.10: C_r <- C_r D^^{-T}
                    tri_solve<T, NB>(cl, sLt);  // Alg. 4 l.12: C_l <- D^^{-1} C_l
                    g_store_row<T, NB>(Cs + (offL + c / s - 1) * nn, cr, n, r, hasR);
                    g_store_col<T, NB>(Cs + (offL + c / s - 2) * nn, cl, n, r, hasL);
                } else {
                    g_load_row<T, NB>(cr, Cs + (offL + c / s - 1) * nn, n, r, hasR, false);
                    g_load_col<T, NB>(cl, Cs + (offL + c / s - 2) * nn, n, r, hasL, false);
                }
                T inv_r = T(1);
                if (SOLVE) {
                    __syncwarp();
                    inv_r = sLt[rr * LD + rr];  // 1/L[r][r] (team_put_Lt)
                }
                __syncwarp();  // sLt is dead from here on; sCl reuses it
                if (rv) {
                    vstore<T, NB>(sCr + r * LD, cr);
                    vstore<T, NB>(sClT + r * LD, cl);
#pragma unroll
                    for (int q = 0; q < NB; ++q) sCl[q * LD + r] = cl[q];
                }
                __syncwarp();

                if (FACT) {
                    // -- a5: fill  C_{l+1,(c-s)/2s} = -C_r C_l  -> slot[c] (column c's D~ is consumed)
                    if (hasL && hasR && rv) {
                        T f[NB];
#pragma unroll
                        for (int q = 0; q < NB; ++q) f[q] = T(0);
                        rowmat_sub<T, NB>(f, cr, sCl);
                        vstore<T, NB>(slots + (size_t)(c - 1) * BLK + r * LD, f);
                    }
                    // -- a2 (right): D~_{c+s} -= C_r C_r^T
                    if (hasR && rv) {
                        T acc[NB];
                        T *p = slots + (size_t)(c + s - 1) * BLK + r * LD;
                        vload<T, NB>(acc, p);
                        rowdot_sub<T, NB>(acc, cr, sCr);
                        vstore<T, NB>(p, acc);
                    }
                }
                (void)offN;
                // -- a6: y_c <- D^^{-1} y_c ; y_{c+s} -= C_r y_c
                if (SOLVE) {
                    for (int q = 0; q < m; ++q) {
                        T *yc = Y + ((size_t)((act ? c : 1) - 1) * m + q) * LD;
                        T yv = yc[rr];
                        yv = (act && rv) ? yv : T(0);
                        yv = team_fwd<T, NB>(yv, dl, inv_r, r, base);
                        if (act && rv) yc[r] = yv;
                    }
                    __syncwarp();
                    if (hasR && rv) {
                        for (int q = 0; q < m; ++q) {
                            const T d = dot<T, NB>(cr, Y + ((size_t)(c - 1) * m + q) * LD);
                            Y[((size_t)(c + s - 1) * m + q) * LD + r] -= d;
                        }
                    }
                }
            }
            __syncthreads();
            // ---- phase Y: left pushes (deferred left-looking part of Alg. 4, l.7/l.9)
            if (wact && hasL && rv) {
                if (FACT) {
                    T acc[NB];
                    T *p = slots + (size_t)(c - s - 1) * BLK + r * LD;
                    vload<T, NB>(acc, p);
                    rowdot_sub<T, NB>(acc, cl, sClT);  // D~_{c-s} -= C_l^T C_l
                    vstore<T, NB>(p, acc);
                }
                if (SOLVE) {
                    for (int q = 0; q < m; ++q) {
                        const T d = dot<T, NB>(cl, Y + ((size_t)(c - 1) * m + q) * LD);
                        Y[((size_t)(c - s - 1) * m + q) * LD + r] -= d;  // y_{c-s} -= C_l^T y_c
                    }
                }
            }
            __syncthreads();
        }
    }

    // ---- a7: backward sweep, l = L..1 (Alg. 6 lines 10-16)
    if (SOLVE) {
        for (int l = g.L; l >= 1; --l) {
            const int s = 1 << (l - 1);
            const int ncols = ((N / s) + 1) / 2;
            const long long offL = g.off[l - 1];
            for (int j0 = 0; j0 < ncols; j0 += NT) {
                if (j0 + warp * TPW >= ncols) continue;  // warp-uniform
                const int j = j0 + team;
                const bool act = j < ncols;
                const int c = s * (2 * j + 1);
                const bool hasL = act && c > s;
                const bool hasR = act && (c + s <= N);
                T lc[NB], crc[NB], clr[NB];
                g_load_col<T, NB>(lc, Dh + (size_t)(c - 1) * nn, n, r, act, true);
                g_load_col<T, NB>(crc, Cs + (offL + c / s - 1) * nn, n, r, hasR, false);
                g_load_row<T, NB>(clr, Cs + (offL + c / s - 2) * nn, n, r, hasL, false);
                const T dg = Dh[(size_t)((act ? c : 1) - 1) * nn + (size_t)(r < n ? r : 0) * (n + 1)];
                const T inv_r = (act && r < n) ? T(1) / dg : T(1);
                for (int q = 0; q < m; ++q) {
                    T *yc = Y + ((size_t)((act ? c : 1) - 1) * m + q) * LD;
                    T v = yc[rr];
                    v = (act && rv) ? v : T(0);
                    const T a = dot<T, NB>(crc, Y + ((size_t)((hasR ? c + s : 1) - 1) * m + q) * LD);
                    const T b2 = dot<T, NB>(clr, Y + ((size_t)((hasL ? c - s : 1) - 1) * m + q) * LD);
                    v -= hasR ? a : T(0);
                    v -= hasL ? b2 : T(0);
                    v = team_bwd<T, NB>(v, lc, inv_r, r, base);
                    if (act && rv) yc[r] = v;
                }
            }
            __syncthreads();
        }
        T *xs = x + sys * (size_t)N * n * m;
        for (size_t q = tid; q < (size_t)N * n * m; q += blockDim.x) {
            const int i = (int)(q / ((size_t)n * m)), rem = (int)(q % ((size_t)n * m));
            const int r2 = rem / m, qq = rem % m;
            xs[q] = Y[((size_t)i * m + qq) * LD + r2];
        }
    }
    if (FACT && tid == 0) info[sys] = (s_fail == 0xffffffffu) ? 0 : (int)(s_fail & ((1u << 25) - 1));
}


// ============================================================================ LEVEL
//
// init: Dhat <- D (raw, full blocks), x <- b, info <- 0.
template <typename T>
__global__ void btd_level_init_kernel(const T *__restrict__ D, const T *__restrict__ bvec, T *Dhat, T *x,
                                      int32_t *info, long long nD, long long nb, int batch, int fact, int solve) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (fact) {
        for (long long q = t0; q < nD; q += stride) Dhat[q] = D[q];
        for (long long q = t0; q < batch; q += stride) info[q] = 0;
    }
    if (solve && bvec != x)
        for (long long q = t0; q < nb; q += stride) x[q] = bvec[q];
}

// One level l of Alg. 4 (FACT) and/or the forward sweep of Alg. 6 (SOLVE), deferred form.
// grid = (ceil(ncols / NT), batch); one team per column; dynamic smem NT * LevelSmem::TSTR.
template <typename T, int NB>
struct LevelSmem {
    static constexpr int BLK = Dims<T, NB>::BLK;
    static constexpr int TSTR = 3 * BLK + 64 / (int)sizeof(T);
};

template <typename T, int NB, int TS, int NT, bool FACT, bool SOLVE>
__global__ void __launch_bounds__(NT *TS) btd_level_fwd_kernel(const T *__restrict__ E, T *Dhat, T *C, T *x,
                                                              int32_t *info, Geo g, int l, int sys0) {
    constexpr int LD = Dims<T, NB>::LD, BLK = Dims<T, NB>::BLK;
    extern __shared__ __align__(16) unsigned char lsm_raw[];
    T *scr_all = reinterpret_cast<T *>(lsm_raw);

    const int N = g.N, n = g.n, m = g.m;
    const long long sys = (long long)blockIdx.y + sys0;
    const size_t nn = (size_t)n * n;
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;
    T *xs = x ? x + sys * (size_t)N * n * m : nullptr;

    const int tid = threadIdx.x, lane = tid & 31, team = tid / TS, r = lane % TS, base = lane - r;
    const bool rv = r < NB;
    T *sLt = scr_all + team * LevelSmem<T, NB>::TSTR;
    T *sB = sLt + BLK;  // right coupling rows / deferred coupling rows / y broadcast
    T *sCl = sB + BLK;  // left coupling, row-major

    const int s = 1 << (l - 1);
    const int ncols = ((N / s) + 1) / 2;
    const int j = blockIdx.x * NT + team;
    const bool act = j < ncols;
    const int c = s * (2 * j + 1);
    const bool hasL = act && c > s;
    const bool hasR = act && (c + s <= N);
    const bool defC = act && l > 1 && (c + s / 2 <= N);      // Alg. 4 l.7
    const bool defS = act && l > 1 && (c + s + s / 2 <= N);  // Alg. 4 l.9

    // Deferred left downdate (Alg. 4 l.7 / l.9):  acc -= Cd^T Cd  where Cd is the stored left
    // coupling of column ysrc at level l-1 (lane r: acc[j] -= sum_k Cd[k][r] Cd[k][j]), and its
    // forward-sweep analogue  y_tgt -= Cd^T y_ysrc.
    auto deferred = [&](T(&acc)[NB], bool on, long long slot, int ysrc, int ytgt) {
        T cdc[NB];
        g_load_col<T, NB>(cdc, Cs + slot * nn, n, r, on, false);
        if (FACT) {
            __syncwarp();
            if (rv) {
                T row[NB];
                g_load_row<T, NB>(row, Cs + slot * nn, n, r, on, false);
                vstore<T, NB>(sB + r * LD, row);
            }
            __syncwarp();
            if (on) rowmat_sub<T, NB>(acc, cdc, sB);
        }
        if (SOLVE && on && r < n) {
            for (int q = 0; q < m; ++q) {
                T sum = T(0);
#pragma unroll
                for (int k = 0; k < NB; ++k)
                    if (k < n) sum = fma(cdc[k], xs[((size_t)(ysrc - 1) * n + k) * m + q], sum);
                xs[((size_t)(ytgt - 1) * n + r) * m + q] -= sum;
            }
        }
    };

    // ---- D^_c: l.7 then l.8
    {
        T dl[NB];
        g_load_row<T, NB>(dl, Dh + (size_t)(c - 1) * nn, n, r, act, true);
        if (l > 1) deferred(dl, defC, cslot(g, l - 1, 2 * c / s), c + s / 2, c);
        if (FACT) {
            const int bad = team_potrf<T, NB>(dl, r, base);
            if (act && bad >= 0 && r == 0) report_fail(info + sys, c);
            g_store_row<T, NB>(Dh + (size_t)(c - 1) * nn, dl, n, r, act);
        } else {
#pragma unroll
            for (int q = 0; q < NB; ++q)
                if (q > r) dl[q] = T(0);
        }
        __syncwarp();
        team_put_Lt<T, NB>(sLt, dl, r);
    }
    // ---- separator D^_{c+s}: l.9 (deferred, level l-1) then l.11 (this level)
    T cr[NB];
    if (FACT) {
        if (l == 1)
            g_load_row<T, NB>(cr, Es + (size_t)(c - 1) * nn, n, r, hasR, false);  // E_c = block (c+1, c)
        else
            g_load_row<T, NB>(cr, Cs + cslot(g, l, c / s) * nn, n, r, hasR, false);
        __syncwarp();
        tri_solve<T, NB>(cr, sLt);  // l.10
        g_store_row<T, NB>(Cs + cslot(g, l, c / s) * nn, cr, n, r, hasR);
        T sep[NB];
        g_load_row<T, NB>(sep, Dh + (size_t)(c + s - 1) * nn, n, r, hasR, false);
        if (l > 1) deferred(sep, defS, cslot(g, l - 1, 2 * c / s + 2), c + s + s / 2, c + s);
        __syncwarp();
        if (rv) vstore<T, NB>(sB + r * LD, cr);
        __syncwarp();
        if (hasR) {
            rowdot_sub<T, NB>(sep, cr, sB);  // l.11: D^_{c+s} -= C_r C_r^T
            g_store_row<T, NB>(Dh + (size_t)(c + s - 1) * nn, sep, n, r, hasR);
        }
        {
            T cl[NB];
            if (l == 1)
                g_load_col<T, NB>(cl, Es + (size_t)(c - 2) * nn, n, r, hasL, false);  // E_{c-1} = (c, c-1)
            else
                g_load_col<T, NB>(cl, Cs + cslot(g, l, c / s - 1) * nn, n, r, hasL, false);
            tri_solve<T, NB>(cl, sLt);  // l.12
            g_store_col<T, NB>(Cs + cslot(g, l, c / s - 1) * nn, cl, n, r, hasL);
            if (rv) {
#pragma unroll
                for (int q = 0; q < NB; ++q) sCl[q * LD + r] = cl[q];
            }
        }
        __syncwarp();
        if (hasL && hasR) {  // l.13: fill -> its final slot (trsm'd in place at level l+1)
            T f[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) f[q] = T(0);
            rowmat_sub<T, NB>(f, cr, sCl);
            g_store_row<T, NB>(Cs + cslot(g, l + 1, (c - s) / (2 * s)) * nn, f, n, r, true);
        }
    } else {
        g_load_row<T, NB>(cr, Cs + cslot(g, l, c / s) * nn, n, r, hasR, false);
        if (l > 1) {
            T dummy[NB];
            deferred(dummy, defS, cslot(g, l - 1, 2 * c / s + 2), c + s + s / 2, c + s);
        }
    }
    if (SOLVE) {
        // Alg. 6 l.4-5: y_c <- D^_c^{-1} y_c ; y_{c+s} -= C_r y_c   (l.6 is deferred like l.7/l.9)
        T dl[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) dl[k] = (rv && k < r) ? sLt[k * LD + r] : T(0);
        T inv_r = T(1);
#pragma unroll
        for (int k = 0; k < NB; ++k)
            if (k == r) inv_r = sLt[k * LD + k];
        for (int q = 0; q < m; ++q) {
            T yv = (act && r < n) ? xs[((size_t)(c - 1) * n + r) * m + q] : T(0);
            yv = team_fwd<T, NB>(yv, dl, inv_r, r, base);
            if (act && r < n) xs[((size_t)(c - 1) * n + r) * m + q] = yv;
            __syncwarp();
            if (rv) sB[r] = yv;
            __syncwarp();
            if (hasR && r < n) {
                T sum = T(0);
#pragma unroll
                for (int k = 0; k < NB; ++k) sum = fma(cr[k], sB[k], sum);
                xs[((size_t)(c + s - 1) * n + r) * m + q] -= sum;
            }
        }
    }
}


// Backward sweep level l (Alg. 6 lines 10-16): x_c = D^_c^{-T}(y_c - C_r^T x_{c+s} - C_l x_{c-s}).
template <typename T, int NB, int TS, int NT>
__global__ void __launch_bounds__(NT *TS) btd_level_bwd_kernel(const T *Dhat, const T *C, T *x, Geo g, int l,
                                                              int sys0) {
    __shared__ __align__(16) T sx[NT][2][NB];
    const int N = g.N, n = g.n, m = g.m;
    const long long sys = (long long)blockIdx.y + sys0;
    const size_t nn = (size_t)n * n;
    const T *Dh = Dhat + sys * N * nn;
    const T *Cs = C + sys * (size_t)g.nC * nn;
    T *xs = x + sys * (size_t)N * n * m;
    const int tid = threadIdx.x, lane = tid & 31, team = tid / TS, r = lane % TS, base = lane - r;
    const bool rv = r < NB;
    const int s = 1 << (l - 1);
    const int ncols = ((N / s) + 1) / 2;
    const int j = blockIdx.x * NT + team;
    const bool act = j < ncols;
    const int c = s * (2 * j + 1);
    const bool hasL = act && c > s;
    const bool hasR = act && (c + s <= N);
    T lc[NB], crc[NB], clr[NB];
    g_load_col<T, NB>(lc, Dh + (size_t)(c - 1) * nn, n, r, act, true);
    g_load_col<T, NB>(crc, Cs + cslot(g, l, c / s) * nn, n, r, hasR, false);
    g_load_row<T, NB>(clr, Cs + cslot(g, l, c / s - 1) * nn, n, r, hasL, false);
    const T inv_r = (act && r < n) ? T(1) / Dh[(size_t)(c - 1) * nn + (size_t)r * n + r] : T(1);
    for (int q = 0; q < m; ++q) {
        if (rv) {
            sx[team][0][r] = (hasR && r < n) ? xs[((size_t)(c + s - 1) * n + r) * m + q] : T(0);
            sx[team][1][r] = (hasL && r < n) ? xs[((size_t)(c - s - 1) * n + r) * m + q] : T(0);
        }
        __syncwarp();
        T v = (act && r < n) ? xs[((size_t)(c - 1) * n + r) * m + q] : T(0);
        T a = T(0), b2 = T(0);
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            a = fma(crc[k], sx[team][0][k], a);
            b2 = fma(clr[k], sx[team][1][k], b2);
        }
        v -= a;
        v -= b2;
        v = team_bwd<T, NB>(v, lc, inv_r, r, base);
        if (act && r < n) xs[((size_t)(c - 1) * n + r) * m + q] = v;
        __syncwarp();
    }
}

}  // namespace btd
