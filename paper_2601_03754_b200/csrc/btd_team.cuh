// btd_team.cuh -- register-tiled "team" primitives for one n x n block column op group.
//
// A team is TS consecutive lanes of a warp (TS = power of two >= NB, <= 32); lane r of the
// team owns row r of every block it works on (or column r for the left coupling, see below),
// held in registers as T v[NB]. NB is the compiled (padded) block size; rows/columns
// n <= i < NB are an identity/zero padding that changes no real value.
//
// Shared-memory scratch per team (leading dimension LD = NB rounded up to 16 bytes):
//   sLt [NB][LD]  L^T, i.e. column k of L^ contiguous: sLt[k][j] = L[j][k] (j > k),
//                 with the reciprocal 1/L[k][k] on the diagonal
//   sCr [NB][LD]  right coupling, row-major (row r = lane r's register row)
//   sClT[NB][LD]  left coupling transposed (row r = column r of C_l)
//   sCl [NB][LD]  left coupling, row-major
//
// The elementary operations are those of Table 1; their use inside the
// level loop follows Algorithm 4 and Algorithm 6.
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

// ------------------------------------------------------------------ global-memory block I/O
// A global block is n x n row-major with leading dimension n (the C-ABI layout). Row r of the
// padded NB x NB block: real rows/cols copy, padding is identity (diag = 1) or zero.

template <typename T, int NB>
__device__ __forceinline__ void g_load_row(T (&v)[NB], const T *blk, int n, int r, bool act,
                                           bool identity_pad) {
    if (act && r < n) {
        if ((NB * (int)sizeof(T)) % 16 == 0 && n == NB) {
            vload<T, NB>(v, blk + (size_t)r * NB);
        } else {
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const T t = blk[(size_t)r * n + (j < n ? j : n - 1)];
                v[j] = (j < n) ? t : T(0);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < NB; ++j) v[j] = (identity_pad && j == r) ? T(1) : T(0);
    }
}

// v[i] = blk[i][r] (column r), zero padding.
template <typename T, int NB>
__device__ __forceinline__ void g_load_col(T (&v)[NB], const T *blk, int n, int r, bool act,
                                           bool identity_pad) {
    const bool on = act && r < n;
    const int rc = on ? r : 0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        T t = T(0);
        if (on) t = blk[(size_t)(i < n ? i : n - 1) * n + rc];
        v[i] = on ? ((i < n) ? t : T(0)) : ((identity_pad && i == r) ? T(1) : T(0));
    }
}

template <typename T, int NB>
__device__ __forceinline__ void g_store_row(T *blk, const T (&v)[NB], int n, int r, bool act) {
    if (!(act && r < n)) return;
    if ((NB * (int)sizeof(T)) % 16 == 0 && n == NB) {
        vstore<T, NB>(blk + (size_t)r * NB, v);
    } else {
        const unsigned long long msk = (n >= 64) ? ~0ull : ((1ull << n) - 1);
#pragma unroll
        for (int j = 0; j < NB; ++j)
            if ((msk >> j) & 1ull) blk[(size_t)r * n + j] = v[j];
    }
}

template <typename T, int NB>
__device__ __forceinline__ void g_store_col(T *blk, const T (&v)[NB], int n, int r, bool act) {
    if (!(act && r < n)) return;
    const unsigned long long msk = (n >= 64) ? ~0ull : ((1ull << n) - 1);
#pragma unroll
    for (int i = 0; i < NB; ++i)
        if ((msk >> i) & 1ull) blk[(size_t)i * n + r] = v[i];
}

// ------------------------------------------------------------------ team numerics

// In-place Cholesky of the team's block (row r in a[]): right-looking, column k pivot
// broadcast by shuffle. Returns the first failing pivot row (<= 0 or NaN) or -1; the
// return value is uniform over the team. Entries above the diagonal are set to 0.
template <typename T, int NB>
__device__ __forceinline__ int team_potrf(T (&a)[NB], int r, int base) {
    // Branch-free on the lane row r: every lane updates its whole register row (entries above
    // the diagonal become don't-care values and are cleared at the end). Data-dependent
    // predicates on r would let the compiler re-roll the unrolled loops into a runtime-bounded
    // loop and demote a[] to local memory.
    int bad = -1;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T akk = __shfl_sync(kFull, a[k], base + k);
        bad = (!(akk > T(0)) && bad < 0) ? k : bad;
        const T d = sqrt(akk);
        const T inv = T(1) / d;
        a[k] = (r == k) ? d : a[k] * inv;
#pragma unroll
        for (int j = k + 1; j < NB; ++j) {
            const T ljk = __shfl_sync(kFull, a[k], base + j);
            a[j] = fma(-a[k], ljk, a[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) a[j] = (j > r) ? T(0) : a[j];
    return bad;
}

// Write lane r's row of L into the column-major scratch sLt (diag = 1/L[r][r]).
template <typename T, int NB>
__device__ __forceinline__ void team_put_Lt(T *sLt, const T (&a)[NB], int r) {
    constexpr int LD = Dims<T, NB>::LD;
    if (r >= NB) return;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T v = (k < r) ? a[k] : ((k == r) ? T(1) / a[k] : T(0));
        sLt[k * LD + r] = v;
    }
}

// x <- L^{-1} x for a per-lane vector x (forward substitution, L from sLt).
// Used for both TRSMs of Alg. 4: a row of C_r (C_r D^^{-T}) and a column of C_l (D^^{-1} C_l).
template <typename T, int NB>
__device__ __forceinline__ void tri_solve(T (&x)[NB], const T *sLt) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        T col[NB];
        vload<T, NB>(col, sLt + k * LD);
        x[k] *= col[k];
#pragma unroll
        for (int j = k + 1; j < NB; ++j) x[j] = fma(-x[k], col[j], x[j]);
    }
}

// acc[j] -= sum_k u[k] * S[j][k] for all j (S row-major NB x LD in shared memory):
// lane-row r of  U S^T  where lane r holds row r of U. Used for both SYRK downdates
// (S = the coupling's rows, resp. its columns) -- PAPER.md:163-178 "syrk".
template <typename T, int NB>
__device__ __forceinline__ void rowdot_sub(T (&acc)[NB], const T (&u)[NB], const T *S) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        T row[NB];
        vload<T, NB>(row, S + j * LD);
        T s = T(0);
#pragma unroll
        for (int k = 0; k < NB; ++k) s = fma(u[k], row[k], s);
        acc[j] -= s;
    }
}

// acc[j] -= sum_k u[k] * S[k][j]  (lane-row r of U S).  Used for the fill GEMM.
template <typename T, int NB>
__device__ __forceinline__ void rowmat_sub(T (&acc)[NB], const T (&u)[NB], const T *S) {
    constexpr int LD = Dims<T, NB>::LD;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        T row[NB];
        vload<T, NB>(row, S + k * LD);
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[j] = fma(-u[k], row[j], acc[j]);
    }
}

// Forward substitution of one right-hand-side column distributed over the team:
// lane r holds y_r and row r of L (a[]) and inv_r = 1/L[r][r]; on exit y_r = (L^{-1} y)_r.
template <typename T, int NB>
__device__ __forceinline__ T team_fwd(T y, const T (&a)[NB], T inv_r, int r, int base) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const T xk = __shfl_sync(kFull, y * inv_r, base + k);
        const T upd = fma(-a[k], xk, y);
        y = (r == k) ? xk : ((r > k) ? upd : y);
    }
    return y;
}

// Back substitution with L^T: lane r holds v_r and column r of L (lc[k] = L[k][r]) and
// inv_r; on exit v_r = (L^{-T} v)_r.
template <typename T, int NB>
__device__ __forceinline__ T team_bwd(T v, const T (&lc)[NB], T inv_r, int r, int base) {
#pragma unroll
    for (int k = NB - 1; k >= 0; --k) {
        const T xk = __shfl_sync(kFull, v * inv_r, base + k);
        const T upd = fma(-lc[k], xk, v);
        v = (r == k) ? xk : ((r < k) ? upd : v);
    }
    return v;
}

// v[r] for a runtime lane row r without dynamic register indexing (1 for padding lanes r >= NB).
template <typename T, int NB>
__device__ __forceinline__ T pick(const T (&v)[NB], int r) {
    T out = T(1);
#pragma unroll
    for (int k = 0; k < NB; ++k)
        if (k == r) out = v[k];
    return out;
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
