// Microbenchmark: cost of cooperative_groups grid.sync() vs a hand-rolled flag barrier on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long *out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// sense-reversing barrier: one atomicAdd per CTA, spin on a generation word
__global__ void k_flag(int iters, unsigned int *count, volatile unsigned int *gen, unsigned long long *out) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int g0 = *gen;
            __threadfence();
            if (atomicAdd(count, 1) == gridDim.x - 1) {
                *count = 0;
                __threadfence();
                *gen = g0 + 1;
            } else {
                while (*gen == g0) {
                }
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
    unsigned long long *d;
    unsigned int *cnt, *gen;
    cudaMalloc(&d, 8);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    int iters = 1000;
    for (int grid : {4, 32, 148, 296}) {
        for (int threads : {256}) {
            void *args[] = {&iters, &d};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaLaunchCooperativeKernel((void *)k_cg, grid, threads, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)k_cg, grid, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long cyc;
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            printf("cg grid.sync grid=%d: %.3f us per sync (%.0f cycles), err=%s\n", grid, ms * 1e3 / iters,
                   (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
            void *args2[] = {&iters, &cnt, &gen, &d};
            cudaLaunchCooperativeKernel((void *)k_flag, grid, threads, args2, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)k_flag, grid, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            printf("flag barrier grid=%d: %.3f us per sync (%.0f cycles), err=%s\n", grid, ms * 1e3 / iters,
                   (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // empty cooperative launch latency (graph-free)
    return 0;
}
