// Variants of the per-step TRSV inner loop to find what limits it (one CTA, 64 active threads).
#include <cstdio>
#include "../../paper_2601_03754_b200/csrc/btd_wide.cuh"
constexpr int NB = 32, LD = NB + 1;

template <typename T, int V>
__global__ void k(int n, int reps, long long *out) {
    __shared__ T L[2 * NB * LD], dinv[NB], X[64 * LD];
    for (int q = threadIdx.x; q < NB * LD; q += blockDim.x) L[q] = (q % (LD + 1) == 0) ? T(2) : T(0.01);
    for (int q = threadIdx.x; q < NB; q += blockDim.x) dinv[q] = T(0.5);
    long long acc = 0;
    for (int r = 0; r < reps; ++r) {
        for (int q = threadIdx.x; q < 64 * LD; q += blockDim.x) X[q] = T(1);
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < 64) {
            T x[NB];
            for (int j = 0; j < NB; ++j) x[j] = X[threadIdx.x * LD + j];
            T *out_ = X + threadIdx.x * LD;
            if (V == 0) {  // baseline: loads inside the step
                for (int kk = 0; kk < n; ++kk) {
                    const T xk = x[0] * dinv[kk];
                    out_[kk] = xk;
                    const T *col = L + kk * (LD + 1);
#pragma unroll
                    for (int jj = 1; jj < NB; ++jj) x[jj - 1] = fma(-xk, col[jj * LD], x[jj]);
                    x[NB - 1] = T(0);
                }
            } else if (V == 1) {  // column prefetched one step ahead into registers
                T c[NB];
#pragma unroll
                for (int jj = 0; jj < NB; ++jj) c[jj] = L[jj * LD];
                for (int kk = 0; kk < n; ++kk) {
                    T cn[NB];
                    const T *coln = L + (kk + 1) * (LD + 1);
#pragma unroll
                    for (int jj = 0; jj < NB; ++jj) cn[jj] = coln[jj * LD];
                    const T xk = x[0] * dinv[kk];
                    out_[kk] = xk;
#pragma unroll
                    for (int jj = 1; jj < NB; ++jj) x[jj - 1] = fma(-xk, c[jj], x[jj]);
                    x[NB - 1] = T(0);
#pragma unroll
                    for (int jj = 0; jj < NB; ++jj) c[jj] = cn[jj];
                }
            } else if (V == 2) {  // fully unrolled, register-indexed, no rotation
#pragma unroll
                for (int kk = 0; kk < NB; ++kk) {
                    x[kk] *= dinv[kk];
                    out_[kk] = x[kk];
#pragma unroll
                    for (int jj = kk + 1; jj < NB; ++jj) x[jj] = fma(-x[kk], L[jj * LD + kk], x[jj]);
                }
            } else if (V == 3) {  // empty: measurement overhead
                out_[0] = x[0] + x[NB - 1];
            }
        }
        __syncthreads();
        acc += clock64() - t0;
    }
    if (threadIdx.x == 0) out[0] = acc / reps;
}

int main() {
    long long *out, c;
    cudaMalloc(&out, 8);
    k<float, 3><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f32 V3 empty     %lld\n", c);
    k<float, 0><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f32 V0 baseline  %lld\n", c);
    k<float, 1><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f32 V1 prefetch  %lld\n", c);
    k<float, 2><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f32 V2 unrolled  %lld\n", c);
    k<double, 0><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f64 V0 baseline  %lld\n", c);
    k<double, 1><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f64 V1 prefetch  %lld\n", c);
    k<double, 2><<<1, 256>>>(32, 20, out); cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); printf("f64 V2 unrolled  %lld  (%s)\n", c, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
