// Microbenchmark: cycles per call of the WIDE kernel's building blocks (one CTA, one warp / quads).
#include <cstdio>
#include "../../paper_2601_03754_b200/csrc/btd_wide.cuh"

template <typename T>
__global__ void kpotrf(T *gA, int n, int reps, long long *out, int *bad) {
    __shared__ T A[2 * 32 * 33], dinv[32], y[32];
    long long acc = 0;
    for (int r = 0; r < reps; ++r) {
        for (int q = threadIdx.x; q < n * n; q += blockDim.x) A[(q / n) * (n + 1) + q % n] = gA[q];
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < 32) bad[0] = btd::warp_potrf_rot<T, 32>(A, n, dinv, y, 1);
        __syncthreads();
        acc += clock64() - t0;
    }
    if (threadIdx.x == 0) out[0] = acc / reps;
}

template <typename T>
__global__ void ktrsv(T *gA, int n, int reps, long long *out) {
    __shared__ T A[2 * 32 * 33], dinv[32], X[64 * 33];
    for (int q = threadIdx.x; q < n * n; q += blockDim.x) A[(q / n) * (n + 1) + q % n] = q / n == q % n ? T(2) : T(0.01);
    for (int q = threadIdx.x; q < n; q += blockDim.x) dinv[q] = T(0.5);
    long long acc = 0;
    for (int r = 0; r < reps; ++r) {
        for (int q = threadIdx.x; q < 64 * 33; q += blockDim.x) X[q] = T(1);
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < 64) {
            T x[32];
            for (int k = 0; k < 32; ++k) x[k] = X[threadIdx.x * 33 + k];
            btd::thread_trsv_lower<T, 32>(x, A, dinv, n, X + threadIdx.x * 33, 1);
        }
        __syncthreads();
        acc += clock64() - t0;
    }
    if (threadIdx.x == 0) out[0] = acc / reps;
}

__global__ void kdfma(double *o, int iters, long long *out) {
    double a = o[threadIdx.x], b = 1.0000001, c = 0.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    o[threadIdx.x] = a;
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
    const int n = 32;
    double hA[n * n];
    float fA[n * n];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) hA[i * n + j] = fA[i * n + j] = (i == j) ? 40.0 : 1.0 / (1 + i + j);
    double *dA; float *fdA; long long *out; int *bad; double *o;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&fdA, sizeof fA); cudaMalloc(&out, 64); cudaMalloc(&bad, 4);
    cudaMalloc(&o, 4096);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(fdA, fA, sizeof fA, cudaMemcpyHostToDevice);
    long long c;
    kpotrf<double><<<1, 256>>>(dA, n, 20, out, bad);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("warp_potrf_rot<double,32> n=32: %lld cycles  (%s)\n", c, cudaGetErrorString(cudaGetLastError()));
    kpotrf<float><<<1, 256>>>(fdA, n, 20, out, bad);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("warp_potrf_rot<float,32>  n=32: %lld cycles\n", c);
    ktrsv<double><<<1, 256>>>(dA, n, 20, out);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("thread_trsv_lower<double> n=32 (64 vectors): %lld cycles\n", c);
    ktrsv<float><<<1, 256>>>(fdA, n, 20, out);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("thread_trsv_lower<float>  n=32 (64 vectors): %lld cycles\n", c);
    kdfma<<<1, 32>>>(o, 10000, out);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("dependent DFMA latency: %lld cycles\n", c);
    return 0;
}
