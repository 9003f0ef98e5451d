// Microbenchmark: FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) vs DFMA throughput per SM and the
// latency of one dependent DMMA, on one SM (one CTA, `threads` threads, independent chains).
// Decides DMMA vs FFMA64 for the large-n (c4) Schur updates.
#include <cstdio>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double *o, int iters, long long *out) {
    double acc[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = o[threadIdx.x] + c;
    const double a = 1.0000001, b = 0.5;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
    o[threadIdx.x] = s;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_dfma(double *o, int iters, long long *out) {
    double a0 = o[threadIdx.x], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 0.5;
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
    const int iters = 4096;
    for (int threads : {128, 256, 512, 1024}) {
        k_dmma<8><<<1, threads>>>(o, iters, out);
        cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        // one m8n8k4 = 256 FMA per warp
        printf("DMMA m8n8k4 f64, %4d threads, 8 chains: %.1f FMA/clk/SM (%.2f clk per warp-MMA per SM)\n", threads,
               (double)iters * 8 * (threads / 32) * 256 / c, (double)c / (iters * 8.0 * (threads / 32)));
        k_dfma<<<1, threads>>>(o, iters, out);
        cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        printf("DFMA,              %4d threads, 8 chains: %.1f FMA/clk/SM\n", threads, (double)iters * 8 * threads / c);
    }
    k_dmma<1><<<1, 32>>>(o, iters, out);
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("DMMA dependent latency: %.1f clk\n", (double)c / iters);
    return 0;
}
