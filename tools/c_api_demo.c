/* c_api_demo.c -- the C ABI of include/btd.h used from plain C (no Python, no torch):
 * plan -> device buffers -> btd_factor_solve -> check against the known solution.
 *
 * System: B independent systems with D_i = 4 I + (i mod 3) I / 8, E_i = -I (n x n blocks), a
 * diagonally dominant SPD block-tridiagonal matrix, and b = Psi x* for x*_i[r] = 1 + (i + r) mod 5.
 * Prints one line "c_api_demo ok max_err=<e>" (exit 0) or the failing status (exit 1).
 * Build: gcc -std=c11 tools/c_api_demo.c -Iinclude -I$CUDA/include -Lpaper_2601_03754_b200 -lbtd -lcudart
 *        (rpath set by paper_2601_03754_b200/build.py:build_c_demo)
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "btd.h"

#define CHECK_CUDA(x)                                                             \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

int main(int argc, char **argv) {
    const int64_t N = argc > 1 ? atoll(argv[1]) : 100, n = argc > 2 ? atoll(argv[2]) : 6, B = 3, m = 1;
    btd_plan *plan = NULL;
    btd_status st = btd_plan_create(&plan, N, n, B, m, BTD_F64);
    if (st != BTD_OK) {
        fprintf(stderr, "btd_plan_create: %s\n", btd_status_string(st));
        return 1;
    }
    const int64_t nC = btd_num_coupling_blocks(plan), nn = n * n;
    const size_t sD = (size_t)B * N * nn, sE = (size_t)B * (N - 1) * nn, sb = (size_t)B * N * n * m;
    const size_t sC = (size_t)B * nC * nn;
    double *hD = calloc(sD, 8), *hE = calloc(sE, 8), *hb = calloc(sb, 8), *hx = calloc(sb, 8), *xs = calloc(sb, 8);
    for (int64_t j = 0; j < B; ++j)
        for (int64_t i = 0; i < N; ++i) {
            for (int64_t r = 0; r < n; ++r) {
                hD[((j * N + i) * n + r) * n + r] = 4.0 + (double)(i % 3) / 8.0;
                if (i < N - 1) hE[((j * (N - 1) + i) * n + r) * n + r] = -1.0;
                xs[(j * N + i) * n + r] = 1.0 + (double)((i + r) % 5);
            }
        }
    for (int64_t j = 0; j < B; ++j)  /* b = Psi x* (D, E diagonal here) */
        for (int64_t i = 0; i < N; ++i)
            for (int64_t r = 0; r < n; ++r) {
                double v = hD[((j * N + i) * n + r) * n + r] * xs[(j * N + i) * n + r];
                if (i > 0) v -= xs[(j * N + i - 1) * n + r];
                if (i < N - 1) v -= xs[(j * N + i + 1) * n + r];
                hb[(j * N + i) * n + r] = v;
            }
    double *dD, *dE, *db, *dDh, *dC, *dx;
    int32_t *dinfo, hinfo[3];
    CHECK_CUDA(cudaMalloc((void **)&dD, sD * 8));
    CHECK_CUDA(cudaMalloc((void **)&dE, sE * 8));
    CHECK_CUDA(cudaMalloc((void **)&db, sb * 8));
    CHECK_CUDA(cudaMalloc((void **)&dDh, sD * 8));
    CHECK_CUDA(cudaMalloc((void **)&dC, sC * 8));
    CHECK_CUDA(cudaMalloc((void **)&dx, sb * 8));
    CHECK_CUDA(cudaMalloc((void **)&dinfo, B * sizeof(int32_t)));
    CHECK_CUDA(cudaMemcpy(dD, hD, sD * 8, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(dE, hE, sE * 8, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(db, hb, sb * 8, cudaMemcpyHostToDevice));
    st = btd_factor_solve(plan, dD, dE, db, dDh, dC, dx, dinfo, NULL);
    if (st != BTD_OK) {
        fprintf(stderr, "btd_factor_solve: %s %s\n", btd_status_string(st), btd_last_error());
        return 1;
    }
    CHECK_CUDA(cudaMemcpy(hx, dx, sb * 8, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(hinfo, dinfo, B * sizeof(int32_t), cudaMemcpyDeviceToHost));
    double err = 0.0;
    for (size_t q = 0; q < sb; ++q) err = fmax(err, fabs(hx[q] - xs[q]) / 5.0);
    const int ok = err <= 1e-12 && hinfo[0] == 0 && hinfo[1] == 0 && hinfo[2] == 0;
    printf("c_api_demo %s variant=%d levels=%d max_err=%.3e\n", ok ? "ok" : "FAILED", btd_plan_variant(plan),
           btd_num_levels(plan), err);
    btd_plan_destroy(plan);
    cudaFree(dD); cudaFree(dE); cudaFree(db); cudaFree(dDh); cudaFree(dC); cudaFree(dx); cudaFree(dinfo);
    free(hD); free(hE); free(hb); free(hx); free(xs);
    return ok ? 0 : 1;
}
