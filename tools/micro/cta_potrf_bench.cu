// Microbenchmark: cycles of the PERSIST kernel's CTA-wide POTRF (n = 128, one CTA of 256 threads).
#include <cstdio>
#include "../../paper_2601_03754_b200/csrc/btd_persist.cuh"

template <typename T, int V>
__global__ void k(const T *gA, int n, int reps, long long *out, int *ok) {
    extern __shared__ unsigned char raw[];
    T *A = reinterpret_cast<T *>(raw);
    T *dinv = A + n * n, *colk = dinv + n;  // colk: 2n colbuf + chunk (unused)
    long long acc = 0;
    for (int r = 0; r < reps; ++r) {
        for (int q = threadIdx.x; q < n * n; q += blockDim.x) A[q] = gA[q];
        __syncthreads();
        long long t0 = clock64();
        const bool good = V ? btd::cta_chol_reg<T>(A, n, nullptr, colk + 2 * n, colk, dinv)
                            : btd::cta_potrf(A, n, dinv, colk);
        __syncthreads();
        acc += clock64() - t0;
        if (threadIdx.x == 0) ok[0] = good;
    }
    if (threadIdx.x == 0) out[0] = acc / reps;
}

int main() {
    const int n = 128;
    static double h[n * n];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) h[i * n + j] = (i == j) ? 200.0 : 1.0 / (1 + i + j);
    double *d; long long *out; int *ok;
    cudaMalloc(&d, sizeof h); cudaMalloc(&out, 8); cudaMalloc(&ok, 4);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    size_t smem = (n * n + 8 * n) * sizeof(double);
    long long c; int g;
    cudaFuncSetAttribute(k<double, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k<double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<double, 0><<<1, 256, smem>>>(d, n, 5, out, ok);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&g, ok, 4, cudaMemcpyDeviceToHost);
    printf("cta_potrf<double> n=128: %lld cycles ok=%d (%s)\n", c, g, cudaGetErrorString(cudaGetLastError()));
    k<double, 1><<<1, 256, smem>>>(d, n, 5, out, ok);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&g, ok, 4, cudaMemcpyDeviceToHost);
    printf("cta_chol_reg<double> n=128: %lld cycles ok=%d (%s)\n", c, g, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
