// Microbenchmark: one-warp Cholesky of a 32 x 32 fp64 block (the diagonal-block step on the
// single-system critical path: WIDE n = 32, PERSIST2 panels). Lane i owns row i; the column is
// broadcast by shuffles; the update is unconditional (the upper part is never stored).
//   V0  pivot = rsqrt.approx.f64 + 2 Newton steps, l_ik = a_ik * inv, update with l_ik l_jk
//   V1  as V0 with 1 Newton step
//   V2  reciprocal form: column shuffled BEFORE the pivot (off the chain), update
//       a_ij -= (a_ik / a_kk) a_jk with rcp.approx.f64 + 2 Newton; L column = a_ik * rsqrt (off chain)
//   V3  as V2, rcp Newton 1 step
// V4 rolled loop, rotating register window, column published in smem (small code).
// Cycles per factorization: warm (best of reps) and cold (first call: instruction cache cold), one warp alone on an SM; max |L - L_V0|.
#include <cstdio>
#include <cmath>
#include "../../paper_2601_03754_b200/csrc/btd_team.cuh"
using namespace btd;

__device__ __forceinline__ void piv_n(double a, double &d, double &inv, int newton) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    const double h = 0.5 * a;
    r = r * fma(-h * r, r, 1.5);
    if (newton > 1) r = r * fma(-h * r, r, 1.5);
    inv = r;
    d = a * r;
}
__device__ __forceinline__ double rcp_n(double a, int newton) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    double e = fma(-a, r, 1.0);
    r = fma(r, e, r);
    if (newton > 1) {
        e = fma(-a, r, 1.0);
        r = fma(r, e, r);
    }
    return r;
}

template <int V>
__global__ void k(const double *A, double *L, long long *out, int reps) {
    const int i = threadIdx.x;
    double a[32];
    __shared__ double col[32][33];
    long long best = 1ll << 60, first = 0;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
        for (int j = 0; j < 32; ++j) a[j] = (j <= i) ? A[i * 32 + j] : 0.0;
        __syncwarp();
        const long long t0 = clock64();
        if (V == 4) {
            // rolled loop, rotating register window: a[0] is always the current column
            for (int kk = 0; kk < 32; ++kk) {
                const double akk = __shfl_sync(kFull, a[0], kk);
                double d, inv;
                piv_n(akk, d, inv, 2);
                const double l = (i == kk) ? d : a[0] * inv;
                col[i][kk] = l;
                __syncwarp();
#pragma unroll
                for (int jj = 1; jj < 32; ++jj) a[jj - 1] = fma(-l, col[kk + jj < 32 ? kk + jj : 31][kk], a[jj]);
                a[31] = 0.0;
                __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = col[i][j];
        } else if (V <= 1) {
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
                const double akk = __shfl_sync(kFull, a[kk], kk);
                double d, inv;
                piv_n(akk, d, inv, V == 0 ? 2 : 1);
                a[kk] = (i == kk) ? d : a[kk] * inv;
#pragma unroll
                for (int j = 1; j < 32; ++j) {
                    if (j <= kk) continue;
                    const double ljk = __shfl_sync(kFull, a[kk], j);
                    a[j] = fma(-a[kk], ljk, a[j]);
                }
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
                double col[32];
#pragma unroll
                for (int j = 1; j < 32; ++j)
                    if (j > kk) col[j] = __shfl_sync(kFull, a[kk], j);  // raw column, independent of the pivot
                const double akk = __shfl_sync(kFull, a[kk], kk);
                const double rk = rcp_n(akk, V == 2 ? 2 : 1);
                const double t = a[kk] * rk;
#pragma unroll
                for (int j = 1; j < 32; ++j)
                    if (j > kk) a[j] = fma(-t, col[j], a[j]);
                double d, inv;
                piv_n(akk, d, inv, 2);  // L column: off the chain
                a[kk] = (i == kk) ? d : a[kk] * inv;
            }
        }
        __syncwarp();
        const long long t1 = clock64();
        best = (t1 - t0) < best ? (t1 - t0) : best;
        if (rep == 0) first = t1 - t0;
#pragma unroll
        for (int j = 0; j < 32; ++j) L[i * 32 + j] = (j <= i) ? a[j] : 0.0;
    }
    if (i == 0) {
        out[0] = best;
        out[1] = first;
    }
}

int main() {
    static double h[1024], l0[1024], l1[1024];
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j) ? 40.0 + i : 1.0 / (1 + i + j);
    double *A, *L; long long *o, c[2];
    cudaMalloc(&A, sizeof h); cudaMalloc(&L, sizeof h); cudaMalloc(&o, 16);
    cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
    const char *nm[] = {"V0 rsqrt+2 Newton", "V1 rsqrt+1 Newton", "V2 rcp form, 2 Newton", "V3 rcp form, 1 Newton",
                        "V4 rolled, rotating window"};
    for (int v = 0; v < 5; ++v) {
        if (v == 0) k<0><<<1, 32>>>(A, L, o, 20);
        if (v == 1) k<1><<<1, 32>>>(A, L, o, 20);
        if (v == 2) k<2><<<1, 32>>>(A, L, o, 20);
        if (v == 3) k<3><<<1, 32>>>(A, L, o, 20);
        if (v == 4) k<4><<<1, 32>>>(A, L, o, 20);
        cudaMemcpy(c, o, 16, cudaMemcpyDeviceToHost);
        cudaMemcpy(v == 0 ? l0 : l1, L, sizeof h, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int q = 0; q < 1024; ++q) err = fmax(err, fabs(l1[q] - l0[q]) / fabs(l0[q] == 0 ? 1 : l0[q]));
        printf("potrf 32x32 fp64, one warp, %-26s warm %6lld  cold (first call) %6lld cycles   max rel diff vs V0 %.2e\n",
               nm[v], c[0], c[1], v ? err : 0.0);
    }
    return 0;
}
