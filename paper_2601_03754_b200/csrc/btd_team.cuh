// btd_team.cuh -- register-tiled "team" primitives for one n x n block column op group.
//
// A team is TS consecutive lanes of a warp (TS divides 32). Lane q of the team owns the
// RPL = NB / TS rows  i = q + TS*t  (t = 0..RPL-1) of every block it works on -- or the
// same-numbered columns of the left coupling -- held in registers as T v[RPL][NB]. NB is
// the compiled (padded) block size; rows/columns n <= i < NB are an identity/zero padding
// that changes no real value. With RPL > 1 (e.g. n = 12: 4 lanes x 3 rows) every lane of
// the warp does useful work and a warp runs 32/TS column op groups side by side.
//
// Shared-memory scratch per team (leading dimension LD = NB rounded up to 16 bytes):
//   sLt [NB][LD]  L^T, i.e. column k of L^ contiguous: sLt[k][j] = L[j][k] (j > k),
//                 with the reciprocal 1/L[k][k] on the diagonal
//   sCr [NB][LD]  right coupling, row-major
//   sClT[NB][LD]  left coupling transposed (row i = column i of C_l)
//   sCl [NB][LD]  left coupling, row-major
//
// The elementary operations are those of Table 1; their use inside the
// level loop follows Algorithm 4 and Algorithm 6.
//
// All numerics are branch-free in the lane's row index: data-dependent predicates on it
// would let the compiler re-roll the unrolled loops into runtime-bounded loops and demote
// the register arrays to local memory.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace btd {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
struct VecT;
template <>
struct VecT<float> {
    using type = float4;
    static constexpr int W = 4;
};
template <>
struct VecT<double> {
    using type = double2;
    static constexpr int W = 2;
};

template <typename T, int NB>
struct Dims {
    static constexpr int W = 16 / (int)sizeof(T);
    static constexpr int LD = ((NB + W - 1) / W) * W;  // padded leading dimension (elements)
    static constexpr int BLK = NB * LD;                  // one padded block (elements)
};

__device__ __forceinline__ void unpack(const float4 &t, float *d) {
    d[0] = t.x; d[1] = t.y; d[2] = t.z; d[3] = t.w;
}
__device__ __forceinline__ void unpack(const double2 &t, double *d) {
    d[0] = t.x; d[1] = t.y;
}
__device__ __forceinline__ float4 pack4(const float *d) { return make_float4(d[0], d[1], d[2], d[3]); }
__device__ __forceinline__ double2 pack4(const double *d) { return make_double2(d[0], d[1]); }

// IEEE-rounded reciprocal and square root (same results as 1/x and sqrt(x) without fast-math).
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return 1.0 / x; }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_rn(double x) { return sqrt(x); }

// Pivot of a Cholesky step: d = sqrt(a), inv = 1/d. fp32 uses the MUFU reciprocal square root
// refined by one Newton step (<= 2 ulp, exact for powers of two) instead of the IEEE sqrt and
// divide sequences, which sit on the POTRF critical path; fp64 keeps the IEEE operations.
__device__ __forceinline__ void pivot(float a, float &d, float &inv) {
    float r = rsqrtf(a);
    r = r * fmaf(-0.5f * a * r, r, 1.5f);
    inv = r;
    d = a * r;
}
__device__ __forceinline__ void pivot(double a, double &d, double &inv) {
    // MUFU double-precision rsqrt seed (~2^-23) + two Newton steps (quadratic: ~2^-46, then
    // ~full precision); keeps the IEEE sqrt/divide sequences off the POTRF critical path.
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    r = r * fma(-0.5 * a * r, r, 1.5);
    r = r * fma(-0.5 * a * r, r, 1.5);
    inv = r;
    d = a * r;
}
// Reciprocal: fp32 MUFU approximation + one Newton step; fp64 IEEE divide.
__device__ __forceinline__ float rcp_fast(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * fmaf(-x, r, 2.0f);
}
__device__ __forceinline__ double rcp_fast(double x) { return 1.0 / x; }

// v[0..NB) <- p[0..NB), p 16-byte aligned (shared or global).
template <typename T, int NB>
__device__ __forceinline__ void vload(T (&v)[NB], const T *p) {
    constexpr int W = VecT<T>::W;
#pragma unroll
    for (int i = 0; i < NB; i += W) {
        if (i + W <= NB) {
            T t[W];
            unpack(*reinterpret_cast<const typename VecT<T>::type *>(p + i), t);
#pragma unroll
            for (int q = 0; q < W; ++q) v[i + q] = t[q];
        } else {
#pragma unroll
            for (int q = 0; q < W; ++q)
                if (i + q < NB) v[i + q] = p[i + q];
        }
    }
}

// p[0..NB) <- v, p 16-byte aligned.
template <typename T, int NB>
__device__ __forceinline__ void vstore(T *p, const T (&v)[NB]) {
    constexpr int W = VecT<T>::W;
#pragma unroll
    for (int i = 0; i < NB; i += W) {
        if (i + W <= NB) {
            T t[W];
#pragma unroll
            for (int q = 0; q < W; ++q) t[q] = v[i + q];
            *reinterpret_cast<typename VecT<T>::type *>(p + i) = pack4(t);
        } else {
#pragma unroll
            for (int q = 0; q < W; ++q)
                if (i + q < NB) p[i + q] = v[i + q];
        }
    }
}

// Team geometry of one lane.
template <int NB, int TS>
struct Lane {
    static constexpr int RPL = (NB + TS - 1) / TS;  // rows per lane
    int q;     // lane index inside the team
    int base;  // first lane of the team inside the warp
    __device__ __forceinline__ int row(int t) const { return q + TS * t; }
    __device__ __forceinline__ bool valid(int t) const { return q + TS * t < NB; }
};

// ------------------------------------------------------------------ global-memory block I/O
// A global block is n x n row-major with leading dimension n (the C-ABI layout). Padded
// rows/columns read as identity (identity_pad) or zero.

template <typename T, int NB>
__device__ __forceinline__ void g_load_row1(T (&v)[NB], const T *blk, int n, int i, bool on, bool identity_pad) {
    if (on && i < n) {
        if ((NB * (int)sizeof(T)) % 16 == 0 && n == NB) {
            vload<T, NB>(v, blk + (size_t)i * NB);
        } else {
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const T t = blk[(size_t)i * n + (j < n ? j : n - 1)];
                v[j] = (j < n) ? t : T(0);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < NB; ++j) v[j] = (identity_pad && j == i) ? T(1) : T(0);
    }
}

// v[k] = blk[k][i] (column i).
template <typename T, int NB>
__device__ __forceinline__ void g_load_col1(T (&v)[NB], const T *blk, int n, int i, bool on, bool identity_pad) {
    if (n == NB) {  // unpadded: compile-time strides, no clamps
        if (on && i < NB) {
#pragma unroll
            for (int k = 0; k < NB; ++k) v[k] = blk[k * NB + i];
        } else {
#pragma unroll
            for (int k = 0; k < NB; ++k) v[k] = (identity_pad && k == i) ? T(1) : T(0);
        }
        return;
    }
    const bool ok = on && i < n;
    const int ic = ok ? i : 0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        T t = T(0);
        if (ok) t = blk[(size_t)(k < n ? k : n - 1) * n + ic];
        v[k] = ok ? ((k < n) ? t : T(0)) : ((identity_pad && k == i) ? T(1) : T(0));
    }
}

template <typename T, int NB>
__device__ __forceinline__ void g_store_row1(T *blk, const T (&v)[NB], int n, int i, bool on) {
    if (!(on && i < n)) return;
    if ((NB * (int)sizeof(T)) % 16 == 0 && n == NB) {
        vstore<T, NB>(blk + (size_t)i * NB, v);
    } else {
        const unsigned long long msk = (n >= 64) ? ~0ull : ((1ull << n) - 1);
#pragma unroll
        for (int j = 0; j < NB; ++j)
            if ((msk >> j) & 1ull) blk[(size_t)i * n + j] = v[j];
    }
}

template <typename T, int NB>
__device__ __forceinline__ void g_store_col1(T *blk, const T (&v)[NB], int n, int i, bool on) {
    if (!(on && i < n)) return;
    if (n == NB) {
#pragma unroll
        for (int k = 0; k < NB; ++k) blk[k * NB + i] = v[k];
        return;
    }
    const unsigned long long msk = (n >= 64) ? ~0ull : ((1ull << n) - 1);
#pragma unroll
    for (int k = 0; k < NB; ++k)
        if ((msk >> k) & 1ull) blk[(size_t)k * n + i] = v[k];
}

// RPL-row versions: lane-owned rows (or columns) i = q + TS t.
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void g_load_rows(T (&v)[RPL][NB], const T *blk, int n, const Lane<NB, TS> &ln, bool on,
                                            bool identity_pad) {
#pragma unroll
    for (int t = 0; t < RPL; ++t) g_load_row1<T, NB>(v[t], blk, n, ln.row(t), on, identity_pad);
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void g_load_cols(T (&v)[RPL][NB], const T *blk, int n, const Lane<NB, TS> &ln, bool on,
                                            bool identity_pad) {
#pragma unroll
    for (int t = 0; t < RPL; ++t) g_load_col1<T, NB>(v[t], blk, n, ln.row(t), on, identity_pad);
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void g_store_rows(T *blk, const T (&v)[RPL][NB], int n, const Lane<NB, TS> &ln, bool on) {
#pragma unroll
    for (int t = 0; t < RPL; ++t) g_store_row1<T, NB>(blk, v[t], n, ln.row(t), on);
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void g_store_cols(T *blk, const T (&v)[RPL][NB], int n, const Lane<NB, TS> &ln, bool on) {
#pragma unroll
    for (int t = 0; t < RPL; ++t) g_store_col1<T, NB>(blk, v[t], n, ln.row(t), on);
}

// Shared-memory padded block (NB rows x LD): rows / columns owned by the lane.
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void s_load_rows(T (&v)[RPL][NB], const T *blk, const Lane<NB, TS> &ln) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int t = 0; t < RPL; ++t) vload<T, NB>(v[t], blk + (ln.valid(t) ? ln.row(t) : 0) * LD);
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void s_store_rows(T *blk, const T (&v)[RPL][NB], const Lane<NB, TS> &ln) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int t = 0; t < RPL; ++t)
        if (ln.valid(t)) vstore<T, NB>(blk + ln.row(t) * LD, v[t]);
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void s_load_cols(T (&v)[RPL][NB], const T *blk, const Lane<NB, TS> &ln) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i = ln.valid(t) ? ln.row(t) : 0;
#pragma unroll
        for (int k = 0; k < NB; ++k) v[t][k] = blk[k * LD + i];
    }
}
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void s_store_cols(T *blk, const T (&v)[RPL][NB], const Lane<NB, TS> &ln) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int t = 0; t < RPL; ++t)
        if (ln.valid(t)) {
#pragma unroll
            for (int k = 0; k < NB; ++k) blk[k * LD + ln.row(t)] = v[t][k];
        }
}

template <typename T, int NB, int RPL>
__device__ __forceinline__ void set_zero(T (&v)[RPL][NB]) {
#pragma unroll
    for (int t = 0; t < RPL; ++t)
#pragma unroll
        for (int j = 0; j < NB; ++j) v[t][j] = T(0);
}

template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void set_identity(T (&v)[RPL][NB], const Lane<NB, TS> &ln) {
#pragma unroll
    for (int t = 0; t < RPL; ++t)
#pragma unroll
        for (int j = 0; j < NB; ++j) v[t][j] = (j == ln.row(t)) ? T(1) : T(0);
}

// ------------------------------------------------------------------ team numerics

// In-place Cholesky of the team's block (rows in a[][]): right-looking; pivot and column k
// broadcast by shuffles. Returns the first failing pivot row (<= 0 or NaN) or -1, uniform over
// the team; dinv[t] receives 1/L[i][i] of owned row i. Entries above the diagonal end as 0.
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ int team_potrf(T (&a)[RPL][NB], T (&dinv)[RPL], const Lane<NB, TS> &ln) {
    int bad = -1;
#pragma unroll
    for (int t = 0; t < RPL; ++t) dinv[t] = T(1);
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T akk = __shfl_sync(kFull, a[k / TS][k], ln.base + k % TS);
        bad = (!(akk > T(0)) && bad < 0) ? k : bad;
        T d, inv;
        pivot(akk, d, inv);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int i = ln.row(t);
            a[t][k] = (i == k) ? d : a[t][k] * inv;
            dinv[t] = (i == k) ? inv : dinv[t];
        }
#pragma unroll
        for (int j = k + 1; j < NB; ++j) {
            const T ljk = __shfl_sync(kFull, a[j / TS][k], ln.base + j % TS);
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

// Write the lane's rows of L into the column-major scratch sLt (diag = 1/L[i][i]).
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void team_put_Lt(T *sLt, const T (&a)[RPL][NB], const T (&dinv)[RPL],
                                            const Lane<NB, TS> &ln) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        if (!ln.valid(t)) continue;
        const int i = ln.row(t);
#pragma unroll
        for (int k = 0; k < NB; ++k) sLt[k * LD + i] = (k == i) ? dinv[t] : a[t][k];
    }
}

// x <- L^{-1} x for each of the lane's vectors (forward substitution, L from sLt).
// Used for both TRSMs of Alg. 4: rows of C_r (C_r D^^{-T}) and columns of C_l (D^^{-1} C_l).
template <typename T, int NB, int RPL>
__device__ __forceinline__ void tri_solve(T (&x)[RPL][NB], const T *sLt) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        T col[NB];
        vload<T, NB>(col, sLt + k * LD);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            x[t][k] *= col[k];
#pragma unroll
            for (int j = k + 1; j < NB; ++j) x[t][j] = fma(-x[t][k], col[j], x[t][j]);
        }
    }
}

// acc[t][j] -= sum_k u[t][k] * S[j][k] (S row-major in shared memory): the lane's rows of
// U S^T. Used for both SYRK downdates ("syrk").
template <typename T, int NB, int RPL>
__device__ __forceinline__ void rowdot_sub(T (&acc)[RPL][NB], const T (&u)[RPL][NB], const T *S) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        T row[NB];
        vload<T, NB>(row, S + j * LD);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            T s = T(0);
#pragma unroll
            for (int k = 0; k < NB; ++k) s = fma(u[t][k], row[k], s);
            acc[t][j] -= s;
        }
    }
}

// acc[t][j] -= sum_k u[t][k] * S[k][j]: the lane's rows of U S. Used for the fill GEMM.
template <typename T, int NB, int RPL>
__device__ __forceinline__ void rowmat_sub(T (&acc)[RPL][NB], const T (&u)[RPL][NB], const T *S) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        T row[NB];
        vload<T, NB>(row, S + k * LD);
#pragma unroll
        for (int t = 0; t < RPL; ++t)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[t][j] = fma(-u[t][k], row[j], acc[t][j]);
    }
}

// Forward substitution of one right-hand-side column distributed over the team: the lane holds
// y[t] for its rows, its rows of L (a) and dinv; on exit y = L^{-1} y.
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void team_fwd(T (&y)[RPL], const T (&a)[RPL][NB], const T (&dinv)[RPL],
                                         const Lane<NB, TS> &ln) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T xk = __shfl_sync(kFull, y[k / TS] * dinv[k / TS], ln.base + k % TS);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int i = ln.row(t);
            const T upd = fma(-a[t][k], xk, y[t]);
            y[t] = (i == k) ? xk : ((i > k) ? upd : y[t]);
        }
    }
}

// Back substitution with L^T: the lane holds v[t], its columns of L (lc[t][k] = L[k][i]) and
// dinv; on exit v = L^{-T} v.
template <typename T, int NB, int TS, int RPL>
__device__ __forceinline__ void team_bwd(T (&v)[RPL], const T (&lc)[RPL][NB], const T (&dinv)[RPL],
                                         const Lane<NB, TS> &ln) {
#pragma unroll
    for (int k = NB - 1; k >= 0; --k) {
        const T xk = __shfl_sync(kFull, v[k / TS] * dinv[k / TS], ln.base + k % TS);
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int i = ln.row(t);
            const T upd = fma(-lc[t][k], xk, v[t]);
            v[t] = (i == k) ? xk : ((i < k) ? upd : v[t]);
        }
    }
}

template <typename T, int NB>
__device__ __forceinline__ T dot(const T (&u)[NB], const T *p) {
    T row[NB];
    vload<T, NB>(row, p);
    T s = T(0);
#pragma unroll
    for (int k = 0; k < NB; ++k) s = fma(u[k], row[k], s);
    return s;
}

// Failure key ordering "(level, index)": level of original block i is 1 + v2(i) = ffs(i).
__device__ __forceinline__ unsigned fail_key(int idx) {
    return ((unsigned)__ffs(idx) << 25) | (unsigned)idx;
}

// Record failing pivot block idx into info (0 = ok) keeping the smallest (level, index).
__device__ __forceinline__ void report_fail(int32_t *info, int idx) {
    int old = *(volatile int32_t *)info;
    const unsigned key = fail_key(idx);
    while (true) {
        if (old != 0 && fail_key(old) <= key) break;
        const int prev = atomicCAS(info, old, idx);
        if (prev == old) break;
        old = prev;
    }
}

}  // namespace btd
