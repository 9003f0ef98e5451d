// Critical-path floor of one level (SURVEY.md §8(d) "Per-regime roofline statement"): the latency
// of the dependent chain potrf -> trsm -> syrk of ONE column op, executed by one CTA (256 threads)
// with its blocks already in shared memory (no HBM/L2 traffic, no grid barrier), with the library's
// own device functions (btd_persist2.cuh / btd_wide.cuh); plus the back-substitution of the
// backward sweep and one grid.sync(). t_chain(n) x L is the floor a level-synchronous schedule can
// reach for a single system; bench.py reports it next to the measured latencies.
// Writes JSON lines: {"n":..,"dtype":..,"potrf_cyc":..,"trsm_cyc":..,"syrk_cyc":..,"bwd_cyc":..}
#include <cooperative_groups.h>
#include <cstdio>

#include "../../paper_2601_03754_b200/csrc/btd_wide.cuh"
using namespace btd;

// One op per kernel (keeps each kernel's register allocation that of the library code): setup,
// one warm-up call (instruction cache), then the timed call; cycles of thread 0.
template <typename T, int NP, int VT>
struct Bufs {
    static constexpr int LD = NP + 4;
    static __device__ void setup(T *sm, const T *Ag, T *&A, T *&X, T *&S, T *&dinv) {
        A = sm;
        X = A + (size_t)(NP + 1) * LD;
        S = X + (size_t)VT * LD;
        dinv = S + (size_t)NP * LD;
        for (int q = threadIdx.x; q < NP * NP; q += blockDim.x) A[(q / NP) * LD + q % NP] = Ag[q];
        for (int q = threadIdx.x; q < LD; q += blockDim.x) A[NP * LD + q] = T(1);
        for (int q = threadIdx.x; q < VT * NP; q += blockDim.x) X[(q / NP) * LD + q % NP] = T(1) / (1 + q % 7);
        for (int q = threadIdx.x; q < NP * LD; q += blockDim.x) S[q] = T(0);
        for (int q = threadIdx.x; q < NP; q += blockDim.x) dinv[q] = T(1) / Ag[q * NP + q];
        __syncthreads();
    }
};

template <typename T, int NP, int VT, int OP>
__global__ void __launch_bounds__(256, 1) k_op(const T *Ag, unsigned long long *out, int n) {
    extern __shared__ __align__(16) unsigned char raw[];
    constexpr int LD = NP + 4, Q = NP < 32 ? NP : 32;
    T *A, *X, *S, *dinv;
    unsigned long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
        Bufs<T, NP, VT>::setup(reinterpret_cast<T *>(raw), Ag, A, X, S, dinv);
        // OP 1 / 3 (TRSM, back substitution) get an already factored A from k_factor: a factorization
        // in the same kernel raises register pressure and made the TRSM spill (3.5 KB stack), which
        // the library kernels (btd_wide_kernel: no stack) do not.
        t0 = clock64();
        if (OP == 0) {
            cta_potrf_blocked<T, Q>(A, LD, n, NP, 1, dinv);  // + one y row
        } else if (OP == 1) {
            // sizes as runtime values, as in the library's call sites (compile-time constants let
            // the compiler hoist every L element into registers and spill)
            const int rt = n < 0;
            cta_trsm_blocked<T, Q>(X, LD + rt, VT + rt, A, LD + rt, NP + rt, dinv);
        } else if (OP == 2) {  // S -= X X^T (lower 8 x 8 tiles), the l.11 downdate
            const int m = VT < n ? VT : n, nt = (m + 7) / 8, ntri = nt * (nt + 1) / 2;
            for (int tt = threadIdx.x >> 5; tt < ntri; tt += blockDim.x >> 5) {
                int ti = 0, q = tt;
                while (q > ti) { q -= ti + 1; ++ti; }
                tile8_sub<T>(S, LD, 8 * ti, 8 * q, m, m, X, LD, X, LD, 0, n);
            }
        } else if (threadIdx.x < 32) {  // backward: v <- L^{-T} v, one warp, lane owns i = lane + 32 u
            constexpr int U = NP / 32 > 0 ? NP / 32 : 1;
            const int lane = threadIdx.x;
            T r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = T(1);
            for (int k = n - 1; k >= 0; --k) {
                const int ow = k & 31, uk = k >> 5;
                T mine = r[0];
#pragma unroll
                for (int u = 1; u < U; ++u) mine = (u == uk) ? r[u] : mine;
                const T xk = __shfl_sync(0xffffffffu, mine, ow) * dinv[k];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = lane + 32 * u;
                    r[u] = (i == k) ? xk : (i < k ? fma(-A[k * LD + i], xk, r[u]) : r[u]);
                }
            }
            if (lane == 0) S[0] += r[0];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[OP] = clock64() - t0;
}

// The factor L of A (in place, lower triangle; A's diagonal is replaced by L's) for OP 1 / 3.
template <typename T, int NP, int VT>
__global__ void __launch_bounds__(256, 1) k_factor(const T *Ag, T *Lg, int n) {
    extern __shared__ __align__(16) unsigned char raw[];
    constexpr int LD = NP + 4, Q = NP < 32 ? NP : 32;
    T *A, *X, *S, *dinv;
    Bufs<T, NP, VT>::setup(reinterpret_cast<T *>(raw), Ag, A, X, S, dinv);
    cta_potrf_blocked<T, Q>(A, LD, n, NP, 0, dinv);
    __syncthreads();
    for (int q = threadIdx.x; q < NP * NP; q += blockDim.x) Lg[q] = A[(q / NP) * LD + q % NP];
}

template <typename T, int NP, int VT>
void run(int n, const char *dt) {
    T *hA = new T[NP * NP];
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) hA[i * NP + j] = (i == j) ? T(4 * NP) : T(1) / T(1 + i + j);
    T *dA;
    unsigned long long *dout, h[4] = {0, 0, 0, 0};
    cudaMalloc(&dA, sizeof(T) * NP * NP);
    cudaMalloc(&dout, 32);
    cudaMemset(dout, 0, 32);
    cudaMemcpy(dA, hA, sizeof(T) * NP * NP, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(T) * ((size_t)(NP + 1) * (NP + 4) + (size_t)VT * (NP + 4) + (size_t)NP * (NP + 4) + NP);
    cudaError_t e = cudaSuccess;
    void (*ks[4])(const T *, unsigned long long *, int) = {k_op<T, NP, VT, 0>, k_op<T, NP, VT, 1>, k_op<T, NP, VT, 2>,
                                                          k_op<T, NP, VT, 3>};
    T *dL;
    cudaMalloc(&dL, sizeof(T) * NP * NP);
    cudaFuncSetAttribute(k_factor<T, NP, VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_factor<T, NP, VT><<<1, 256, smem>>>(dA, dL, n);
    e = cudaDeviceSynchronize();
    for (int op = 0; op < 4 && e == cudaSuccess; ++op) {
        cudaFuncSetAttribute(ks[op], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        ks[op]<<<1, 256, smem>>>((op == 1 || op == 3) ? dL : dA, dout, n);
        e = cudaDeviceSynchronize();
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    cudaMemcpy(h, dout, 32, cudaMemcpyDeviceToHost);
    printf("{\"n\": %d, \"dtype\": \"%s\", \"trsm_vectors\": %d, \"potrf_cyc\": %llu, \"trsm_cyc\": %llu, "
           "\"syrk_cyc\": %llu, \"bwd_cyc\": %llu, \"err\": \"%s\"}\n",
           n, dt, VT, h[0], h[1], h[2], h[3], cudaGetErrorString(e));
    cudaFree(dA);
    cudaFree(dL);
    cudaFree(dout);
    delete[] hA;
}

__global__ void k_sync(int iters, unsigned long long *out) {
    cooperative_groups::grid_group g = cooperative_groups::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / iters;
}

int main() {
    run<double, 8, 16>(2, "f64");
    run<double, 16, 32>(16, "f64");
    run<double, 32, 64>(32, "f64");
    run<float, 32, 64>(32, "f32");
    // n = 128 (c4) is not measured here: its blocks (280 KB with the scratch) exceed shared memory
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int iters = 200;
    void *args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((const void *)k_sync, dim3(nsm), dim3(256), args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    printf("{\"gridsync_cyc\": %llu, \"grid\": %d, \"sm_khz\": %d}\n", h, nsm, mhz);
    return 0;
}
