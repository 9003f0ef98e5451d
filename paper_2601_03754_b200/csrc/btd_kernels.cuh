// btd_kernels.cuh -- the level kernels of the multi-stage block-tridiagonal Cholesky.
//
// Realisations of Algorithm 4 (factor) + Algorithm 6 (solve),
// all built from the team primitives of btd_team.cuh:
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
//         Two team layouts:
//           FUSED-R (small blocks: fp32 n <= 12, fp64 n <= 8): TS lanes x RPL rows per lane with
//                   RPL = NB/TS, the whole factor L^ of the column held in every lane's registers
//                   (TRSMs and the forward/backward solves need no communication), GEMM operands
//                   exchanged by warp shuffles -- no shared-memory scratch, so two systems fit
//                   per SM.
//           FUSED-S (larger blocks): one row per lane, L^ and the coupling rows staged in a
//                   per-team shared-memory scratch and read as broadcasts.
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
#include <cuda_pipeline.h>

#include "btd_team.cuh"

#ifndef BTD_FR_MINB
#define BTD_FR_MINB 2
#endif
namespace btd {

struct Geo {
    int N, n, m, L;
    long long nC;       // coupling blocks per system
    long long off[34];  // off[l-1] = first slot of level l (l = 1..L+1)
};

__device__ __forceinline__ long long cslot(const Geo &g, int l, int k) { return g.off[l - 1] + k - 1; }

// Optional phase timing (build with -DBTD_TIMING): CTA 0 accumulates clock64() deltas per phase id
// into btd_timing[] (read back with cudaMemcpyFromSymbol by tools/phase_times.py).
#ifdef BTD_TIMING
static __device__ unsigned long long btd_timing[32];
// fire-and-forget reduction (RED): the stamp adds no load latency to the phase it closes
#define BTD_STAMP(id)                                                         \
    do {                                                                      \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                            \
            const unsigned long long now_ = clock64();                        \
            atomicAdd(&btd_timing[(id)], now_ - btd_t_last);                  \
            btd_t_last = clock64();                                           \
        }                                                                     \
    } while (0)
#define BTD_STAMP_INIT() unsigned long long btd_t_last = clock64(), btd_t_sub = btd_t_last
// sub-phase stamps on their own clock (do not disturb the phase totals)
#define BTD_SUB_INIT()                                                        \
    do {                                                                      \
        if (blockIdx.x == 0 && threadIdx.x == 0) btd_t_sub = clock64();       \
    } while (0)
#define BTD_SUB(cond, id)                                                     \
    do {                                                                      \
        if ((cond) && blockIdx.x == 0 && threadIdx.x == 0) {                  \
            const unsigned long long now_ = clock64();                        \
            atomicAdd(&btd_timing[(id)], now_ - btd_t_sub);                   \
            btd_t_sub = clock64();                                            \
        }                                                                     \
    } while (0)
#else
#define BTD_SUB_INIT() \
    do {               \
    } while (0)
#define BTD_SUB(cond, id) \
    do {                  \
    } while (0)
#define BTD_STAMP(id) \
    do {              \
    } while (0)
#define BTD_STAMP_INIT() \
    do {                 \
    } while (0)
#endif

// ---------------------------------------------------------------------------- shared pieces

// slots <- D (padded with identity), Y <- b (padded rows), cooperative over the CTA.
// sp >= 0: only blocks [0, sp) and b are waited for on return (asynchronous copies); the copies of
// blocks [sp, N) stay in flight in the most recent commit group (caller: __pipeline_wait_prior(0)).
template <typename T, int NB, bool FACT, bool SOLVE>
__device__ __forceinline__ void fused_load_inputs(T *slots, T *Y, const T *Ds, const T *bs, int N, int n, int m,
                                                  int sp = -1) {
    constexpr int LD = Dims<T, NB>::LD, BLK = Dims<T, NB>::BLK;
    const int tid = threadIdx.x;
    const size_t nn = (size_t)n * n;
    size_t rest0 = 0, rest1 = 0;  // 16-byte chunks of D still to copy after b
    if (FACT) {
        if (n == NB && LD == NB) {
            constexpr int W = VecT<T>::W;
            const size_t tot = (size_t)N * nn;
            if (tot % W == 0) {
                // asynchronous 16-byte copies (LDGSTS): every thread keeps all of its loads in flight
                using V = typename VecT<T>::type;
                const V *src = reinterpret_cast<const V *>(Ds);
                V *dst = reinterpret_cast<V *>(slots);
                const size_t cut = (sp >= 0 && sp < N && ((size_t)sp * nn) % W == 0) ? (size_t)sp * nn / W : tot / W;
                for (size_t q = tid; q < cut; q += blockDim.x) __pipeline_memcpy_async(dst + q, src + q, 16);
                __pipeline_commit();
                rest0 = cut;
                rest1 = tot / W;
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
        if (m == 1 && n == LD && ((size_t)N * n) % VecT<T>::W == 0) {
            using V = typename VecT<T>::type;
            for (size_t q = tid; q < (size_t)N * n / VecT<T>::W; q += blockDim.x)
                __pipeline_memcpy_async(reinterpret_cast<V *>(Y) + q, reinterpret_cast<const V *>(bs) + q, 16);
            __pipeline_commit();
        } else {
            for (size_t q = tid; q < (size_t)N * m * LD; q += blockDim.x) {
                const int i = (int)(q / ((size_t)m * LD)), rem = (int)(q % ((size_t)m * LD));
                const int qq = rem / LD, r2 = rem % LD;
                Y[q] = (r2 < n) ? bs[((size_t)i * n + r2) * m + qq] : T(0);
            }
        }
    }
    if (rest0 < rest1) {
        using V = typename VecT<T>::type;
        const V *src = reinterpret_cast<const V *>(Ds);
        V *dst = reinterpret_cast<V *>(slots);
        for (size_t q = rest0 + tid; q < rest1; q += blockDim.x) __pipeline_memcpy_async(dst + q, src + q, 16);
        __pipeline_commit();
        __pipeline_wait_prior(1);
    } else {
        __pipeline_wait_prior(0);
    }
}

template <typename T, int NB>
__device__ __forceinline__ void fused_store_x(T *xs, const T *Y, int N, int n, int m) {
    constexpr int LD = Dims<T, NB>::LD;
    for (size_t q = threadIdx.x; q < (size_t)N * n * m; q += blockDim.x) {
        const int i = (int)(q / ((size_t)n * m)), rem = (int)(q % ((size_t)n * m));
        const int r2 = rem / m, qq = rem % m;
        xs[q] = Y[((size_t)i * m + qq) * LD + r2];
    }
}

// v[k] of the lane's row k... select v[i] for a runtime index i without dynamic register indexing.
template <typename T, int NB>
__device__ __forceinline__ T select_idx(const T (&v)[NB], int i) {
    T out = v[0];
#pragma unroll
    for (int k = 1; k < NB; ++k) out = (i == k) ? v[k] : out;
    return out;
}

// ============================================================================ FUSED-R
//
// Shared memory (elements of T): slots N * BLK (FACT), Y N * m * LD (SOLVE). No scratch.
template <typename T, int NB>
struct FusedRCfg {
    // team width: NB / TS rows per lane, every lane busy (TS divides NB and 32)
    static constexpr int TS = sizeof(T) == 4 ? (NB == 12 ? 4 : NB == 8 ? 4 : NB == 6 ? 2 : NB == 4 ? 2 : 1)
                                             : (NB == 8 ? 4 : NB == 6 ? 2 : NB == 4 ? 2 : 1);
    static constexpr int RPL = NB / TS;
    static constexpr int THREADS = 128;
    static constexpr int NT = THREADS / TS;
    static constexpr bool OK = (sizeof(T) == 4 ? NB <= 12 : NB <= 8) && NB % TS == 0;
    static __host__ __device__ size_t bytes(int N, int m, bool fact, bool solve) {
        return ((fact ? (size_t)N * Dims<T, NB>::BLK : 0) + (solve ? (size_t)N * m * Dims<T, NB>::LD : 0)) *
               sizeof(T);
    }
};

// Cholesky of the team's block with every lane collecting the whole factor: on return Lf[j][k]
// (j >= k) = L[j][k] and Linv[k] = 1/L[k][k] in every lane; a[][] holds the lane's rows of L.
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ int team_potrf_full(T (&a)[RPL][NB], T (&Lf)[NB][NB], T (&Linv)[NB],
                                               const Lane<NB, TS> &ln) {
    int bad = -1;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T akk = __shfl_sync(kFull, a[k / TS][k], ln.base + k % TS);
        bad = (!(akk > T(0)) && bad < 0) ? k : bad;
        T d, inv;
        pivot(akk, d, inv);
        Lf[k][k] = d;
        Linv[k] = inv;
#pragma unroll
        for (int t = 0; t < RPL; ++t) a[t][k] = (ln.row(t) == k) ? d : a[t][k] * inv;
#pragma unroll
        for (int j = k + 1; j < NB; ++j) {
            const T ljk = __shfl_sync(kFull, a[j / TS][k], ln.base + j % TS);
            Lf[j][k] = ljk;
#pragma unroll
            for (int t = 0; t < RPL; ++t) a[t][j] = fma(-a[t][k], ljk, a[t][j]);
        }
    }
#pragma unroll
    for (int t = 0; t < RPL; ++t)
#pragma unroll
        for (int j = 0; j < NB; ++j) a[t][j] = (j > ln.row(t)) ? T(0) : a[t][j];
    return bad;
}

// team_potrf_full fused with the column op's two TRSMs (Alg. 4 l.10, l.12) and, with WY, the
// forward substitution of y_c (Alg. 6 l.4): the lane's rows of C_r, columns of C_l and y are
// eliminated as extra rows of the factorization, reusing its pivots and column shuffles, so no
// copy of L is kept. Operation for operation the same arithmetic as team_potrf_full followed by
// tri_solve_reg(cr), tri_solve_reg(cl) and fwd_full(y) -- bitwise identical results.
template <typename T, int NB, int TS, int RPL, bool WY>
__device__ __forceinline__ int team_potrf_trsm(T (&a)[RPL][NB], T (&cr)[RPL][NB], T (&cl)[RPL][NB], T (&y)[NB],
                                               const Lane<NB, TS> &ln) {
    int bad = -1;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T akk = __shfl_sync(kFull, a[k / TS][k], ln.base + k % TS);
        bad = (!(akk > T(0)) && bad < 0) ? k : bad;
        T d, inv;
        pivot(akk, d, inv);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            a[t][k] = (ln.row(t) == k) ? d : a[t][k] * inv;
            cr[t][k] *= inv;
            cl[t][k] *= inv;
        }
        if (WY) y[k] *= inv;
        // constant trip count (j > k as a compile-time predicate after unrolling): the unroller
        // must flatten both loops or the register arrays are demoted to local memory
#pragma unroll
        for (int j = 1; j < NB; ++j) {
            if (j <= k) continue;
            const T ljk = __shfl_sync(kFull, a[j / TS][k], ln.base + j % TS);
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                a[t][j] = fma(-a[t][k], ljk, a[t][j]);
                cr[t][j] = fma(-cr[t][k], ljk, cr[t][j]);
                cl[t][j] = fma(-cl[t][k], ljk, cl[t][j]);
            }
            if (WY) y[j] = fma(-y[k], ljk, y[j]);
        }
    }
#pragma unroll
    for (int t = 0; t < RPL; ++t)
#pragma unroll
        for (int j = 0; j < NB; ++j) a[t][j] = (j > ln.row(t)) ? T(0) : a[t][j];
    return bad;
}

// x <- L^{-1} x with L in registers (per-lane vectors).
template <typename T, int NB, int RPL>
__device__ __forceinline__ void tri_solve_reg(T (&x)[RPL][NB], const T (&Lf)[NB][NB], const T (&Linv)[NB]) {
#pragma unroll
    for (int k = 0; k < NB; ++k)
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            x[t][k] *= Linv[k];
#pragma unroll
            for (int j = k + 1; j < NB; ++j) x[t][j] = fma(-x[t][k], Lf[j][k], x[t][j]);
        }
}

template <typename T, int NB>
__device__ __forceinline__ void fwd_full(T (&y)[NB], const T (&Lf)[NB][NB], const T (&Linv)[NB]) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        y[k] *= Linv[k];
#pragma unroll
        for (int j = k + 1; j < NB; ++j) y[j] = fma(-y[k], Lf[j][k], y[j]);
    }
}

template <typename T, int NB>
__device__ __forceinline__ void bwd_full(T (&v)[NB], const T (&Lf)[NB][NB], const T (&Linv)[NB]) {
#pragma unroll
    for (int k = NB - 1; k >= 0; --k) {
        v[k] *= Linv[k];
#pragma unroll
        for (int i = 0; i < k; ++i) v[i] = fma(-Lf[k][i], v[k], v[i]);
    }
}

// Whole L^ diagonal block of original block c into registers (every lane), from global Dhat.
template <typename T, int NB>
__device__ __forceinline__ void load_L_full(T (&Lf)[NB][NB], T (&Linv)[NB], const T *blk, int n) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        T row[NB];
        g_load_row1<T, NB>(row, blk, n, i, true, true);
#pragma unroll
        for (int k = 0; k <= i; ++k) Lf[i][k] = row[k];
        Linv[i] = rcp_fast(row[i]);
    }
}

// Backward-sweep cache of FUSED-R (factor+solve). The L^ blocks of levels l >= LC are also written
// to shared-memory slots that are dead by then, so the backward sweep reads the upper levels from
// shared memory instead of L2/HBM. The slot of an odd block (its level-1 fill) is dead after level 2,
// the slot of a block = 2 mod 4 (its level-2 fill) after level 3. Cache entry q lives in the slot of
// block 2q+1 (q < H1) or 4(q-H1)+2; level l's entries are the D^ blocks of its columns
// j = 0..ncols-1, then its coupling blocks k = 1..N/s-1 (the C layout).
struct BwdCache {
    int LC, H1;
    __device__ static int count(int N, int l) {
        const int s = 1 << (l - 1);
        return ((N / s) + 1) / 2 + (N / s) - 1;
    }
    __device__ void init(int N, int L) {
        H1 = (N + 1) / 2;
        const int H2 = (N + 2) / 4;
        LC = L + 1;
        for (int lc = 3; lc <= 4 && lc <= L; ++lc) {
            int tot = 0;
            for (int l = lc; l <= L; ++l) tot += count(N, l);
            if (tot <= H1 + H2 && count(N, lc) <= (lc == 3 ? H1 : H1 + H2)) {
                LC = lc;
                break;
            }
        }
    }
    __device__ int base(int N, int l) const {  // first cache index of level l >= LC
        int q = 0;
        for (int l2 = LC; l2 < l; ++l2) q += count(N, l2);
        return q;
    }
    __device__ int slot(int q) const { return q < H1 ? 2 * q : 4 * (q - H1) + 1; }  // 0-based slot
};

// EX: n == NB at compile time (no padding): the generic padded load/store paths are not
// compiled, which keeps the kernel's code (and its instruction-cache footprint) small.
template <typename T, int NB, int TS, int NT, bool FACT, bool SOLVE, int MR, bool EX>
__global__ void __launch_bounds__(NT *TS, BTD_FR_MINB)
    btd_fused_r_kernel(const T *__restrict__ D, const T *__restrict__ E, const T *__restrict__ bvec, T *Dhat, T *C,
                       T *x, int32_t *info, Geo g, int sys0) {
    constexpr int LD = Dims<T, NB>::LD, BLK = Dims<T, NB>::BLK;
    constexpr int RPL = NB / TS;
    constexpr int TPW = 32 / TS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *slots = reinterpret_cast<T *>(smem_raw);
    __shared__ unsigned s_fail;

    const int N = g.N, n = EX ? NB : g.n;
    const int m = MR > 0 ? MR : g.m;
    T *Y = slots + (FACT ? (size_t)N * BLK : 0);
    const long long sys = (long long)blockIdx.x + sys0;
    const size_t nn = (size_t)n * n;
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, team = tid / TS;
    Lane<NB, TS> ln{lane % TS, lane - lane % TS};

    BTD_STAMP_INIT();
    BwdCache bc;
    bc.init(N, g.L);
    if (!(FACT && SOLVE)) bc.LC = g.L + 1;  // LC > L: no cache (factor-only or solve-only)
    if (tid == 0) s_fail = 0xffffffffu;
    // level 1's first round touches blocks < 2 NT only: the rest of D lands while it runs
    fused_load_inputs<T, NB, FACT, SOLVE>(slots, Y, D ? D + sys * N * nn : nullptr,
                                          SOLVE ? bvec + sys * (size_t)N * n * m : nullptr, N, n, m, 2 * NT);
    __syncthreads();
    BTD_STAMP(0);

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
            T SL[RPL][NB];  // lane's rows of C_l^T C_l (left downdate, applied in phase Y)
            if (wact) {
                // FY: factor + single right-hand side -- the TRSMs and y_c's forward substitution
                // ride along the POTRF (team_potrf_trsm) and no copy of L is kept
                constexpr bool FY = FACT && SOLVE && MR == 1;
                T Lf[FY ? 1 : NB][NB], Linv[FY ? 1 : NB];
                T yv[NB];
                T cr[RPL][NB];
                BTD_SUB_INIT();
                if (FACT) {
                    // -- a4 operands: couplings (row q+TS t of the right one, column q+TS t of the
                    // left one); level 1 reads them from HBM, later levels from the fill slots
                    if (l == 1) {
                        g_load_rows<T, NB, TS, RPL>(cr, Es + (size_t)(c - 1) * nn, n, ln, hasR, false);
                        g_load_cols<T, NB, TS, RPL>(cl, Es + (size_t)((c >= 2 ? c : 2) - 2) * nn, n, ln, hasL, false);
                    } else {
                        // a missing coupling (hasR / hasL false) reads some finite block: every use
                        // of it below is guarded by the same flag
                        s_load_rows<T, NB, TS, RPL>(cr, slots + (size_t)((hasR ? c + s / 2 : c) - 1) * BLK, ln);
                        s_load_cols<T, NB, TS, RPL>(cl, slots + (size_t)((hasL ? c - s / 2 : c) - 1) * BLK, ln);
                    }
                    if (FY) {  // inactive teams shadow column s: no reads of the y it is writing
                        if (act) {
                            vload<T, NB>(yv, Y + (size_t)(c - 1) * LD);
                        } else {
#pragma unroll
                            for (int k = 0; k < NB; ++k) yv[k] = T(0);
                        }
                    }
                    // -- a3: D~_c -> D^_c
                    T a[RPL][NB];
                    s_load_rows<T, NB, TS, RPL>(a, slots + (size_t)(c - 1) * BLK, ln);
                    if (!act) set_identity<T, NB, TS, RPL>(a, ln);
                    int bad;
                    if constexpr (FY) {
                        // Alg. 4 l.8, l.10 (C_r <- C_r D^^{-T}), l.12 (C_l <- D^^{-1} C_l); Alg. 6 l.4
                        bad = team_potrf_trsm<T, NB, TS, RPL, true>(a, cr, cl, yv, ln);
                    } else {
                        bad = team_potrf_full<T, NB, TS, RPL>(a, Lf, Linv, ln);
                        tri_solve_reg<T, NB, RPL>(cr, Lf, Linv);  // Alg. 4 l.10: C_r <- C_r D^^{-T}
                        tri_solve_reg<T, NB, RPL>(cl, Lf, Linv);  // Alg. 4 l.12: C_l <- D^^{-1} C_l
                    }
                    if (act && bad >= 0 && ln.q == 0) atomicMin(&s_fail, fail_key(c));
                    BTD_SUB(l >= 3, 20);
                    if (SOLVE && l >= bc.LC && act) {  // backward-sweep cache (see BwdCache)
                        const int qb = bc.base(N, l);
                        s_store_rows<T, NB, TS, RPL>(slots + (size_t)bc.slot(qb + j) * BLK, a, ln);
                        if (hasR) s_store_rows<T, NB, TS, RPL>(slots + (size_t)bc.slot(qb + ncols + c / s - 1) * BLK, cr, ln);
                        if (hasL) s_store_cols<T, NB, TS, RPL>(slots + (size_t)bc.slot(qb + ncols + c / s - 2) * BLK, cl, ln);
                    }
                    g_store_rows<T, NB, TS, RPL>(Dh + (size_t)(c - 1) * nn, a, n, ln, act);
                    g_store_rows<T, NB, TS, RPL>(Cs + (offL + c / s - 1) * nn, cr, n, ln, hasR);
                    g_store_cols<T, NB, TS, RPL>(Cs + (offL + c / s - 2) * nn, cl, n, ln, hasL);
                }
                if constexpr (!FACT && !FY) {
                    load_L_full<T, NB>(Lf, Linv, Dh + (size_t)(c - 1) * nn, n);
                    g_load_rows<T, NB, TS, RPL>(cr, Cs + (offL + c / s - 1) * nn, n, ln, hasR, false);
                    g_load_cols<T, NB, TS, RPL>(cl, Cs + (offL + (c / s >= 2 ? c / s : 2) - 2) * nn, n, ln, hasL,
                                                false);
                }
                BTD_SUB(l >= 3, 21);
                // -- a6: y_c <- D^^{-1} y_c (redundantly in every lane of the team), y_{c+s} -= C_r y_c
                if (SOLVE) {
                    for (int q = 0; q < m; ++q) {
                        T *yc = Y + ((size_t)(c - 1) * m + q) * LD;
                        if constexpr (!FY) {
                            if (act) {
                                vload<T, NB>(yv, yc);
                            } else {
#pragma unroll
                                for (int k = 0; k < NB; ++k) yv[k] = T(0);
                            }
                            fwd_full<T, NB>(yv, Lf, Linv);
                        }
                        __syncwarp();
#pragma unroll
                        for (int t = 0; t < RPL; ++t) {
                            if (act) yc[ln.row(t)] = select_idx<T, NB>(yv, ln.row(t));
                            if (hasR) {
                                T d = T(0);
#pragma unroll
                                for (int k = 0; k < NB; ++k) d = fma(cr[t][k], yv[k], d);
                                Y[((size_t)(c + s - 1) * m + q) * LD + ln.row(t)] -= d;
                            }
                        }
                    }
                }
                BTD_SUB(l >= 3, 22);
                if (FACT) {
                    // -- a2 (right): D~_{c+s} -= C_r C_r^T   (rows of C_r exchanged by shuffles)
                    {
                        T SR[RPL][NB];
                        set_zero<T, NB, RPL>(SR);
#pragma unroll
                        for (int jj = 0; jj < NB; ++jj)
#pragma unroll
                            for (int k = 0; k < NB; ++k) {
                                const T v = __shfl_sync(kFull, cr[jj / TS][k], ln.base + jj % TS);  // C_r[jj][k]
                                // lower triangle only (row q + TS t >= jj needs t >= jj / TS): the
                                // separator's upper triangle is never read (potrf reads the lower one)
#pragma unroll
                                for (int t = jj / TS; t < RPL; ++t) SR[t][jj] = fma(cr[t][k], v, SR[t][jj]);
                            }
                        if (hasR) {
                            T *p = slots + (size_t)(c + s - 1) * BLK;
#pragma unroll
                            for (int t = 0; t < RPL; ++t) {
                                T acc[NB];
                                vload<T, NB>(acc, p + ln.row(t) * LD);
#pragma unroll
                                for (int q = 0; q < NB; ++q) acc[q] -= SR[t][q];
                                vstore<T, NB>(p + ln.row(t) * LD, acc);
                            }
                        }
                    }
                    BTD_SUB(l >= 3, 23);
                    // -- a5 fill -C_r C_l -> slot[c], and C_l^T C_l for phase Y (columns of C_l shuffled)
                    {
                        T F[RPL][NB];
                        set_zero<T, NB, RPL>(F);
                        set_zero<T, NB, RPL>(SL);
#pragma unroll
                        for (int bb = 0; bb < NB; ++bb)
#pragma unroll
                            for (int k = 0; k < NB; ++k) {
                                const T v = __shfl_sync(kFull, cl[bb / TS][k], ln.base + bb % TS);  // C_l[k][bb]
#pragma unroll
                                for (int t = 0; t < RPL; ++t) {
                                    F[t][bb] = fma(-cr[t][k], v, F[t][bb]);
                                    if (t >= bb / TS) SL[t][bb] = fma(cl[t][k], v, SL[t][bb]);  // lower only
                                }
                            }
                        if (hasL && hasR) s_store_rows<T, NB, TS, RPL>(slots + (size_t)(c - 1) * BLK, F, ln);
                    }
                    BTD_SUB(l >= 3, 24);
                }
            }
            __syncthreads();
            BTD_STAMP(l < 11 ? 5 + l : 1);
            // ---- phase Y: left pushes (deferred left-looking part of Alg. 4, l.7/l.9)
            if (wact && hasL) {
                if (FACT) {
                    T *p = slots + (size_t)(c - s - 1) * BLK;
#pragma unroll
                    for (int t = 0; t < RPL; ++t) {
                        T acc[NB];
                        vload<T, NB>(acc, p + ln.row(t) * LD);
#pragma unroll
                        for (int q = 0; q < NB; ++q) acc[q] -= SL[t][q];  // D~_{c-s} -= C_l^T C_l
                        vstore<T, NB>(p + ln.row(t) * LD, acc);
                    }
                }
                if (SOLVE) {
                    for (int q = 0; q < m; ++q) {
                        const T *yc = Y + ((size_t)(c - 1) * m + q) * LD;
#pragma unroll
                        for (int t = 0; t < RPL; ++t)  // y_{c-s} -= C_l^T y_c
                            Y[((size_t)(c - s - 1) * m + q) * LD + ln.row(t)] -= dot<T, NB>(cl[t], yc);
                    }
                }
            }
            if (l == 1 && j0 == 0) __pipeline_wait_prior(0);  // rest of D (fused_load_inputs)
            __syncthreads();
            BTD_STAMP(2);
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
                const int c = act ? s * (2 * j + 1) : s;
                const bool hasL = act && c > s;
                const bool hasR = act && (c + s <= N);
                T Lf[NB][NB], Linv[NB];
                T crc[RPL][NB], clr[RPL][NB];
                if (l >= bc.LC) {  // upper levels: L^ from the shared-memory cache
                    const int qb = bc.base(N, l);
                    const T *pd = slots + (size_t)bc.slot(qb + (act ? j : 0)) * BLK;
#pragma unroll
                    for (int i = 0; i < NB; ++i) {
                        T row[NB];
                        vload<T, NB>(row, pd + i * LD);
#pragma unroll
                        for (int k = 0; k < i; ++k) Lf[i][k] = row[k];
                        Lf[i][i] = row[i];
                        Linv[i] = rcp_fast(row[i]);
                    }
                    s_load_cols<T, NB, TS, RPL>(crc, hasR ? slots + (size_t)bc.slot(qb + ncols + c / s - 1) * BLK : pd, ln);
                    s_load_rows<T, NB, TS, RPL>(clr, hasL ? slots + (size_t)bc.slot(qb + ncols + c / s - 2) * BLK : pd, ln);
                } else {
                    load_L_full<T, NB>(Lf, Linv, Dh + (size_t)(c - 1) * nn, n);
                    g_load_cols<T, NB, TS, RPL>(crc, Cs + (offL + c / s - 1) * nn, n, ln, hasR, false);
                    g_load_rows<T, NB, TS, RPL>(clr, Cs + (offL + (c / s >= 2 ? c / s : 2) - 2) * nn, n, ln, hasL,
                                                false);
                }
                for (int q = 0; q < m; ++q) {
                    T *yc = Y + ((size_t)(c - 1) * m + q) * LD;
                    const T *xr = Y + ((size_t)((hasR ? c + s : c) - 1) * m + q) * LD;
                    const T *xl = Y + ((size_t)((hasL ? c - s : c) - 1) * m + q) * LD;
                    T v[NB];
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
                    if (act) {
                        vload<T, NB>(v, yc);
                    } else {
#pragma unroll
                        for (int k = 0; k < NB; ++k) v[k] = T(0);
                    }
                    bwd_full<T, NB>(v, Lf, Linv);
                    __syncwarp();
                    // x_c is final: write it to Y (read by the lower levels) and straight to HBM
                    T *xs = x + (sys * (size_t)N + (c - 1)) * n * m + q;
#pragma unroll
                    for (int t = 0; t < RPL; ++t) {
                        const T xv = select_idx<T, NB>(v, ln.row(t));
                        if (act) yc[ln.row(t)] = xv;
                        if (act && ln.row(t) < n) xs[(size_t)ln.row(t) * m] = xv;
                    }
                }
            }
            __syncthreads();
            BTD_STAMP(l >= 3 ? 25 : 24 + l);  // backward: 25 = levels >= 3, 26 = level 2, 27 = level 1
        }

    }
    if (FACT && tid == 0) info[sys] = (s_fail == 0xffffffffu) ? 0 : (int)(s_fail & ((1u << 25) - 1));
}

// ============================================================================ FUSED-S
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

// Launch shape of the FUSED-S kernel for block size NB: team width TS, CTA threads, min CTAs/SM.
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
    constexpr int RPL = 1;
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
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, team = tid / TS;
    Lane<NB, TS> ln{lane % TS, lane - lane % TS};
    const bool rv = ln.valid(0);
    T *sLt = scr + (size_t)team * S::TSTR;
    T *sCl = sLt;  // reuses sLt once both TRSMs are done
    T *sCr = sLt + BLK;
    T *sClT = sCr + BLK;

    if (tid == 0) s_fail = 0xffffffffu;
    fused_load_inputs<T, NB, FACT, SOLVE>(slots, Y, D ? D + sys * N * nn : nullptr,
                                          SOLVE ? bvec + sys * (size_t)N * n * m : nullptr, N, n, m);
    __syncthreads();

    for (int l = 1; l <= g.L; ++l) {
        const int s = 1 << (l - 1);
        const int ncols = ((N / s) + 1) / 2;
        const long long offL = g.off[l - 1];
        for (int j0 = 0; j0 < ncols; j0 += NT) {
            const int j = j0 + team;
            const bool wact = j0 + warp * TPW < ncols;
            const bool act = j < ncols;
            const int c = act ? s * (2 * j + 1) : s;
            const bool hasL = act && c > s;
            const bool hasR = act && (c + s <= N);
            T cl[RPL][NB];
            if (wact) {
                T dl[RPL][NB], dinv[RPL];
                if (FACT) {
                    s_load_rows<T, NB, TS, RPL>(dl, slots + (size_t)(c - 1) * BLK, ln);
                    if (!act) set_identity<T, NB, TS, RPL>(dl, ln);
                    const int bad = team_potrf<T, NB, TS, RPL>(dl, dinv, ln);
                    if (act && bad >= 0 && ln.q == 0) atomicMin(&s_fail, fail_key(c));
                    g_store_rows<T, NB, TS, RPL>(Dh + (size_t)(c - 1) * nn, dl, n, ln, act);
                } else {
                    g_load_rows<T, NB, TS, RPL>(dl, Dh + (size_t)(c - 1) * nn, n, ln, act, true);
                    dinv[0] = T(1);
#pragma unroll
                    for (int k = 0; k < NB; ++k) dinv[0] = (k == ln.q) ? rcp_rn(dl[0][k]) : dinv[0];
                }
                team_put_Lt<T, NB, TS, RPL>(sLt, dl, dinv, ln);

                T cr[RPL][NB];
                if (FACT) {
                    if (l == 1) {
                        g_load_rows<T, NB, TS, RPL>(cr, Es + (size_t)(c - 1) * nn, n, ln, hasR, false);
                        g_load_cols<T, NB, TS, RPL>(cl, Es + (size_t)((c >= 2 ? c : 2) - 2) * nn, n, ln, hasL, false);
                    } else {
                        s_load_rows<T, NB, TS, RPL>(cr, slots + (size_t)((hasR ? c + s / 2 : c) - 1) * BLK, ln);
                        s_load_cols<T, NB, TS, RPL>(cl, slots + (size_t)((hasL ? c - s / 2 : c) - 1) * BLK, ln);
#pragma unroll
                        for (int q = 0; q < NB; ++q) {
                            cr[0][q] = (hasR && rv) ? cr[0][q] : T(0);
                            cl[0][q] = (hasL && rv) ? cl[0][q] : T(0);
                        }
                    }
                    __syncwarp();
                    tri_solve<T, NB, RPL>(cr, sLt);  // Alg. 4 l.10: C_r <- C_r D^^{-T}
                    tri_solve<T, NB, RPL>(cl, sLt);  // Alg. 4 l.12: C_l <- D^^{-1} C_l
                    g_store_rows<T, NB, TS, RPL>(Cs + (offL + c / s - 1) * nn, cr, n, ln, hasR);
                    g_store_cols<T, NB, TS, RPL>(Cs + (offL + c / s - 2) * nn, cl, n, ln, hasL);
                } else {
                    g_load_rows<T, NB, TS, RPL>(cr, Cs + (offL + c / s - 1) * nn, n, ln, hasR, false);
                    g_load_cols<T, NB, TS, RPL>(cl, Cs + (offL + (c / s >= 2 ? c / s : 2) - 2) * nn, n, ln, hasL,
                                                false);
                }
                __syncwarp();  // sLt is dead from here on; sCl reuses it
                s_store_rows<T, NB, TS, RPL>(sCr, cr, ln);
                s_store_rows<T, NB, TS, RPL>(sClT, cl, ln);
                s_store_cols<T, NB, TS, RPL>(sCl, cl, ln);
                __syncwarp();

                if (FACT) {
                    // -- a5: fill  C_{l+1,(c-s)/2s} = -C_r C_l  -> slot[c] (column c's D~ is consumed)
                    if (hasL && hasR) {
                        T f[RPL][NB];
                        set_zero<T, NB, RPL>(f);
                        rowmat_sub<T, NB, RPL>(f, cr, sCl);
                        s_store_rows<T, NB, TS, RPL>(slots + (size_t)(c - 1) * BLK, f, ln);
                    }
                    // -- a2 (right): D~_{c+s} -= C_r C_r^T
                    if (hasR) {
                        T acc[RPL][NB];
                        T *p = slots + (size_t)(c + s - 1) * BLK;
                        s_load_rows<T, NB, TS, RPL>(acc, p, ln);
                        rowdot_sub<T, NB, RPL>(acc, cr, sCr);
                        s_store_rows<T, NB, TS, RPL>(p, acc, ln);
                    }
                }
                // -- a6: y_c <- D^^{-1} y_c ; y_{c+s} -= C_r y_c
                if (SOLVE) {
                    for (int q = 0; q < m; ++q) {
                        T *yc = Y + ((size_t)(c - 1) * m + q) * LD;
                        T yv[RPL];
                        yv[0] = (act && rv) ? yc[ln.q] : T(0);  // inactive teams read no y
                        team_fwd<T, NB, TS, RPL>(yv, dl, dinv, ln);
                        if (act && rv) yc[ln.q] = yv[0];
                    }
                    __syncwarp();
                    if (hasR && rv) {
                        for (int q = 0; q < m; ++q) {
                            const T d = dot<T, NB>(cr[0], Y + ((size_t)(c - 1) * m + q) * LD);
                            Y[((size_t)(c + s - 1) * m + q) * LD + ln.q] -= d;
                        }
                    }
                }
            }
            __syncthreads();
            // ---- phase Y: left pushes (deferred left-looking part of Alg. 4, l.7/l.9)
            if (wact && hasL) {
                if (FACT) {
                    T acc[RPL][NB];
                    T *p = slots + (size_t)(c - s - 1) * BLK;
                    s_load_rows<T, NB, TS, RPL>(acc, p, ln);
                    rowdot_sub<T, NB, RPL>(acc, cl, sClT);  // D~_{c-s} -= C_l^T C_l
                    s_store_rows<T, NB, TS, RPL>(p, acc, ln);
                }
                if (SOLVE && rv) {
                    for (int q = 0; q < m; ++q) {
                        const T d = dot<T, NB>(cl[0], Y + ((size_t)(c - 1) * m + q) * LD);
                        Y[((size_t)(c - s - 1) * m + q) * LD + ln.q] -= d;  // y_{c-s} -= C_l^T y_c
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
                const int c = act ? s * (2 * j + 1) : s;
                const bool hasL = act && c > s;
                const bool hasR = act && (c + s <= N);
                T lc[RPL][NB], crc[RPL][NB], clr[RPL][NB], dinv[RPL];
                g_load_cols<T, NB, TS, RPL>(lc, Dh + (size_t)(c - 1) * nn, n, ln, act, true);
                g_load_cols<T, NB, TS, RPL>(crc, Cs + (offL + c / s - 1) * nn, n, ln, hasR, false);
                g_load_rows<T, NB, TS, RPL>(clr, Cs + (offL + (c / s >= 2 ? c / s : 2) - 2) * nn, n, ln, hasL,
                                            false);
                dinv[0] = T(1);
#pragma unroll
                for (int k = 0; k < NB; ++k) dinv[0] = (k == ln.q) ? rcp_rn(lc[0][k]) : dinv[0];
                for (int q = 0; q < m; ++q) {
                    T *yc = Y + ((size_t)(c - 1) * m + q) * LD;
                    T v[RPL];
                    v[0] = (act && rv) ? yc[ln.q] : T(0);  // inactive teams read no y
                    const T a = hasR ? dot<T, NB>(crc[0], Y + ((size_t)(c + s - 1) * m + q) * LD) : T(0);
                    const T b2 = hasL ? dot<T, NB>(clr[0], Y + ((size_t)(c - s - 1) * m + q) * LD) : T(0);
                    v[0] -= hasR ? a : T(0);
                    v[0] -= hasL ? b2 : T(0);
                    team_bwd<T, NB, TS, RPL>(v, lc, dinv, ln);
                    if (act && rv) yc[ln.q] = v[0];
                }
            }
            __syncthreads();
        }
        fused_store_x<T, NB>(x + sys * (size_t)N * n * m, Y, N, n, m);
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

template <int NB>
struct LevelShape_TS {
    static constexpr int TS = NB <= 1 ? 1 : NB <= 2 ? 2 : NB <= 4 ? 4 : NB <= 8 ? 8 : NB <= 16 ? 16 : 32;
};

// One level l of Alg. 4 (FACT) and/or the forward sweep of Alg. 6 (SOLVE), deferred form.
// grid = (ceil(ncols / NT), batch); one team (one row per lane) per column; dynamic smem NT * TSTR.
template <typename T, int NB>
struct LevelSmem {
    static constexpr int BLK = Dims<T, NB>::BLK;
    static constexpr int TSTR = 3 * BLK + 64 / (int)sizeof(T);
};

// One column op of level l for (system sys, column index j): the body shared by the LEVEL kernel
// (one launch per level) and the PERSIST-TEAM kernel (one cooperative launch, grid.sync per level).
// `scr` is this team's shared-memory scratch (LevelSmem::TSTR elements). Warp-collective.
template <typename T, int NB, int TS, bool FACT, bool SOLVE>
__device__ __forceinline__ void level_fwd_task(const T *__restrict__ E, T *Dhat, T *C, T *x, int32_t *info,
                                               const Geo &g, int l, long long sys, int j, T *scr) {
    constexpr int LD = Dims<T, NB>::LD, BLK = Dims<T, NB>::BLK;
    constexpr int RPL = 1;
    const int N = g.N, n = g.n, m = g.m;
    const size_t nn = (size_t)n * n;
    const T *Es = E ? E + sys * (size_t)(N - 1) * nn : nullptr;
    T *Dh = Dhat + sys * N * nn;
    T *Cs = C + sys * (size_t)g.nC * nn;
    T *xs = x ? x + sys * (size_t)N * n * m : nullptr;

    const int lane = threadIdx.x & 31;
    Lane<NB, TS> ln{lane % TS, lane - lane % TS};
    const int r = ln.q;
    const bool rv = ln.valid(0);
    T *sLt = scr;
    T *sB = sLt + BLK;  // right coupling rows / deferred coupling rows / y broadcast
    T *sCl = sB + BLK;  // left coupling, row-major

    const int s = 1 << (l - 1);
    const int ncols = ((N / s) + 1) / 2;
    const bool act = j < ncols;
    const int c = act ? s * (2 * j + 1) : s;
    const bool hasL = act && c > s;
    const bool hasR = act && (c + s <= N);
    const bool defC = act && l > 1 && (c + s / 2 <= N);      // Alg. 4 l.7
    const bool defS = act && l > 1 && (c + s + s / 2 <= N);  // Alg. 4 l.9

    // Deferred left downdate (Alg. 4 l.7 / l.9):  acc -= Cd^T Cd  where Cd is the stored left
    // coupling of column ysrc at level l-1 (lane r: acc[j] -= sum_k Cd[k][r] Cd[k][j]), and its
    // forward-sweep analogue  y_tgt -= Cd^T y_ysrc.
    auto deferred = [&](T(&acc)[RPL][NB], bool on, long long slot, int ysrc, int ytgt) {
        T cdc[RPL][NB];
        g_load_cols<T, NB, TS, RPL>(cdc, Cs + slot * nn, n, ln, on, false);
        if (FACT) {
            __syncwarp();
            T row[RPL][NB];
            g_load_rows<T, NB, TS, RPL>(row, Cs + slot * nn, n, ln, on, false);
            s_store_rows<T, NB, TS, RPL>(sB, row, ln);
            __syncwarp();
            if (on) rowmat_sub<T, NB, RPL>(acc, cdc, sB);
        }
        if (SOLVE && on && r < n) {
            for (int q = 0; q < m; ++q) {
                T sum = T(0);
#pragma unroll
                for (int k = 0; k < NB; ++k)
                    if (k < n) sum = fma(cdc[0][k], xs[((size_t)(ysrc - 1) * n + k) * m + q], sum);
                xs[((size_t)(ytgt - 1) * n + r) * m + q] -= sum;
            }
        }
    };

    // ---- D^_c: l.7 then l.8
    T dinv[RPL];
    {
        T dl[RPL][NB];
        g_load_rows<T, NB, TS, RPL>(dl, Dh + (size_t)(c - 1) * nn, n, ln, act, true);
        if (l > 1) deferred(dl, defC, cslot(g, l - 1, 2 * c / s), c + s / 2, c);
        if (FACT) {
            const int bad = team_potrf<T, NB, TS, RPL>(dl, dinv, ln);
            if (act && bad >= 0 && r == 0) report_fail(info + sys, c);
            g_store_rows<T, NB, TS, RPL>(Dh + (size_t)(c - 1) * nn, dl, n, ln, act);
        } else {
#pragma unroll
            for (int q = 0; q < NB; ++q) dl[0][q] = (q > r) ? T(0) : dl[0][q];
            dinv[0] = T(1);
#pragma unroll
            for (int k = 0; k < NB; ++k) dinv[0] = (k == r) ? rcp_rn(dl[0][k]) : dinv[0];
        }
        __syncwarp();
        team_put_Lt<T, NB, TS, RPL>(sLt, dl, dinv, ln);
    }
    // ---- separator D^_{c+s}: l.9 (deferred, level l-1) then l.11 (this level)
    T cr[RPL][NB];
    if (FACT) {
        if (l == 1)
            g_load_rows<T, NB, TS, RPL>(cr, Es + (size_t)(c - 1) * nn, n, ln, hasR, false);  // E_c = (c+1, c)
        else
            g_load_rows<T, NB, TS, RPL>(cr, Cs + cslot(g, l, c / s) * nn, n, ln, hasR, false);
        __syncwarp();
        tri_solve<T, NB, RPL>(cr, sLt);  // l.10
        g_store_rows<T, NB, TS, RPL>(Cs + cslot(g, l, c / s) * nn, cr, n, ln, hasR);
        T sep[RPL][NB];
        g_load_rows<T, NB, TS, RPL>(sep, Dh + (size_t)((hasR ? c + s : c) - 1) * nn, n, ln, hasR, false);
        if (l > 1) deferred(sep, defS, cslot(g, l - 1, 2 * c / s + 2), c + s + s / 2, c + s);
        __syncwarp();
        s_store_rows<T, NB, TS, RPL>(sB, cr, ln);
        __syncwarp();
        if (hasR) {
            rowdot_sub<T, NB, RPL>(sep, cr, sB);  // l.11: D^_{c+s} -= C_r C_r^T
            g_store_rows<T, NB, TS, RPL>(Dh + (size_t)(c + s - 1) * nn, sep, n, ln, hasR);
        }
        {
            T cl[RPL][NB];
            if (l == 1)
                g_load_cols<T, NB, TS, RPL>(cl, Es + (size_t)((c >= 2 ? c : 2) - 2) * nn, n, ln, hasL, false);
            else
                g_load_cols<T, NB, TS, RPL>(cl, Cs + cslot(g, l, (c / s >= 2 ? c / s : 2) - 1) * nn, n, ln, hasL,
                                            false);
            tri_solve<T, NB, RPL>(cl, sLt);  // l.12
            g_store_cols<T, NB, TS, RPL>(Cs + cslot(g, l, c / s - 1) * nn, cl, n, ln, hasL);
            s_store_cols<T, NB, TS, RPL>(sCl, cl, ln);
        }
        __syncwarp();
        if (hasL && hasR) {  // l.13: fill -> its final slot (trsm'd in place at level l+1)
            T f[RPL][NB];
            set_zero<T, NB, RPL>(f);
            rowmat_sub<T, NB, RPL>(f, cr, sCl);
            g_store_rows<T, NB, TS, RPL>(Cs + cslot(g, l + 1, (c - s) / (2 * s)) * nn, f, n, ln, true);
        }
    } else {
        g_load_rows<T, NB, TS, RPL>(cr, Cs + cslot(g, l, c / s) * nn, n, ln, hasR, false);
        if (l > 1) {
            T dummy[RPL][NB];
            set_zero<T, NB, RPL>(dummy);
            deferred(dummy, defS, cslot(g, l - 1, 2 * c / s + 2), c + s + s / 2, c + s);
        }
    }
    if (SOLVE) {
        // Alg. 6 l.4-5: y_c <- D^_c^{-1} y_c ; y_{c+s} -= C_r y_c   (l.6 is deferred like l.7/l.9)
        T dl[RPL][NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) dl[0][k] = (rv && k < r) ? sLt[k * LD + (rv ? r : 0)] : T(0);
        for (int q = 0; q < m; ++q) {
            T yv[RPL];
            yv[0] = (act && r < n) ? xs[((size_t)(c - 1) * n + r) * m + q] : T(0);
            team_fwd<T, NB, TS, RPL>(yv, dl, dinv, ln);
            if (act && r < n) xs[((size_t)(c - 1) * n + r) * m + q] = yv[0];
            __syncwarp();
            if (rv) sB[r] = yv[0];
            __syncwarp();
            if (hasR && r < n) {
                T sum = T(0);
#pragma unroll
                for (int k = 0; k < NB; ++k) sum = fma(cr[0][k], sB[k], sum);
                xs[((size_t)(c + s - 1) * n + r) * m + q] -= sum;
            }
        }
    }
}

template <typename T, int NB, int TS, int NT, bool FACT, bool SOLVE>
__global__ void __launch_bounds__(NT *TS) btd_level_fwd_kernel(const T *__restrict__ E, T *Dhat, T *C, T *x,
                                                              int32_t *info, Geo g, int l, int sys0) {
    extern __shared__ __align__(16) unsigned char lsm_raw[];
    T *scr = reinterpret_cast<T *>(lsm_raw) + (threadIdx.x / TS) * LevelSmem<T, NB>::TSTR;
    level_fwd_task<T, NB, TS, FACT, SOLVE>(E, Dhat, C, x, info, g, l, (long long)blockIdx.y + sys0,
                                           blockIdx.x * NT + (int)(threadIdx.x / TS), scr);
}

// Backward sweep of one column (Alg. 6 lines 10-16): x_c = D^_c^{-T}(y_c - C_r^T x_{c+s} - C_l x_{c-s}).
// sx: 2*NB elements of this team's shared scratch. Warp-collective.
template <typename T, int NB, int TS>
__device__ __forceinline__ void level_bwd_task(const T *Dhat, const T *C, T *x, const Geo &g, int l, long long sys,
                                               int j, T *sxs) {
    constexpr int RPL = 1;
    const int N = g.N, n = g.n, m = g.m;
    const size_t nn = (size_t)n * n;
    const T *Dh = Dhat + sys * N * nn;
    const T *Cs = C + sys * (size_t)g.nC * nn;
    T *xs = x + sys * (size_t)N * n * m;
    const int lane = threadIdx.x & 31;
    Lane<NB, TS> ln{lane % TS, lane - lane % TS};
    const int r = ln.q;
    const bool rv = ln.valid(0);
    const int s = 1 << (l - 1);
    const int ncols = ((N / s) + 1) / 2;
    const bool act = j < ncols;
    const int c = act ? s * (2 * j + 1) : s;
    const bool hasL = act && c > s;
    const bool hasR = act && (c + s <= N);
    T lc[RPL][NB], crc[RPL][NB], clr[RPL][NB], dinv[RPL];
    g_load_cols<T, NB, TS, RPL>(lc, Dh + (size_t)(c - 1) * nn, n, ln, act, true);
    g_load_cols<T, NB, TS, RPL>(crc, Cs + cslot(g, l, c / s) * nn, n, ln, hasR, false);
    g_load_rows<T, NB, TS, RPL>(clr, Cs + cslot(g, l, (c / s >= 2 ? c / s : 2) - 1) * nn, n, ln, hasL, false);
    dinv[0] = T(1);
#pragma unroll
    for (int k = 0; k < NB; ++k) dinv[0] = (k == r) ? rcp_rn(lc[0][k]) : dinv[0];
    for (int q = 0; q < m; ++q) {
        if (rv) {
            sxs[r] = (hasR && r < n) ? xs[((size_t)(c + s - 1) * n + r) * m + q] : T(0);
            sxs[NB + r] = (hasL && r < n) ? xs[((size_t)(c - s - 1) * n + r) * m + q] : T(0);
        }
        __syncwarp();
        T v[RPL];
        v[0] = (act && r < n) ? xs[((size_t)(c - 1) * n + r) * m + q] : T(0);
        T a = T(0), b2 = T(0);
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            a = fma(crc[0][k], sxs[k], a);
            b2 = fma(clr[0][k], sxs[NB + k], b2);
        }
        v[0] -= a;
        v[0] -= b2;
        team_bwd<T, NB, TS, RPL>(v, lc, dinv, ln);
        if (act && r < n) xs[((size_t)(c - 1) * n + r) * m + q] = v[0];
        __syncwarp();
    }
}

template <typename T, int NB, int TS, int NT>
__global__ void __launch_bounds__(NT *TS) btd_level_bwd_kernel(const T *Dhat, const T *C, T *x, Geo g, int l,
                                                              int sys0) {
    __shared__ __align__(16) T sx[NT][2 * NB];
    level_bwd_task<T, NB, TS>(Dhat, C, x, g, l, (long long)blockIdx.y + sys0, blockIdx.x * NT + (int)(threadIdx.x / TS),
                              sx[threadIdx.x / TS]);
}

}  // namespace btd
