// Microbenchmark: FFMA / DFMA throughput per SM (one CTA of 256 threads, 8 independent chains/thread).
#include <cstdio>

template <typename T>
__global__ void k(T *o, int iters, long long *out) {
    T a0 = o[threadIdx.x], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const T b = (T)1.0000001, c = (T)0.5;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    o[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
    double *o; long long *out, c;
    cudaMalloc(&o, 1 << 16); cudaMalloc(&out, 8);
    const int iters = 4096, threads = 256;
    k<float><<<1, threads>>>((float *)o, iters, out);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("FFMA: %.1f per clk per SM\n", (double)iters * 8 * threads / c);
    k<double><<<1, threads>>>(o, iters, out);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("DFMA: %.1f per clk per SM\n", (double)iters * 8 * threads / c);
    return 0;
}
