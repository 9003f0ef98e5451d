// btd_persist.cu -- launcher of the PERSIST variant (cooperative launch, one kernel per call).
#include "btd_internal.h"
#include "btd_persist.cuh"
#include "btd_persist2.cuh"
#include "btd_wide.cuh"

namespace btd {

// PERSIST2 (btd_persist2.cuh): blocked POTRF / TRSM, DMMA tile updates, pull-form separators.
template <typename T>
static btd_status run_persist2(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat,
                               void *C, void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    const int n = (int)p->n, m = (int)p->m, N = (int)p->N;
    const size_t smem = Persist2Smem<T>::bytes(n, m);
    auto kern = btd_persist2_kernel<T>;
    if (btd_status rs = ensure_smem_attr((const void *)kern, smem); rs != BTD_OK) return rs;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kP2Threads, smem);
    if (e != cudaSuccess) return record_cuda_error(e);
    if (per_sm < 1) return BTD_EUNSUPPORTED;
    const size_t nn = (size_t)n * n;
    const T *Dt = op != 1 ? (const T *)D + sys0 * N * nn : nullptr;
    const T *Et = E ? (const T *)E + sys0 * (size_t)(N - 1) * nn : nullptr;
    const T *bt = b ? (const T *)b + sys0 * (size_t)N * n * m : nullptr;
    T *Dh = (T *)Dhat + sys0 * N * nn;
    T *Ct = (T *)C + sys0 * (size_t)p->geo.nC * nn;
    T *xt = x ? (T *)x + sys0 * (size_t)N * n * m : nullptr;
    int32_t *inf = info ? info + sys0 : nullptr;
    Geo g = p->geo;
    int batch = (int)count, fact = op != 1, solve = op != 0;
    // every SM: level 1 has up to (N/2) x tiles of work; the top levels need the CTAs for their tiles
    const long long maxg = (long long)nsm * per_sm;
    int grid = (int)maxg;
    void *args[] = {(void *)&Dt, (void *)&Et, (void *)&bt, (void *)&Dh, (void *)&Ct, (void *)&xt, (void *)&inf,
                    (void *)&g, (void *)&batch, (void *)&fact, (void *)&solve};
    e = cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(kP2Threads), args, smem, st);
    if (e != cudaSuccess) return record_cuda_error(e);
    return BTD_OK;
}

template <typename T>
btd_status run_persist(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat, void *C,
                       void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    if (p->use_persist2) return run_persist2<T>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    const int n = (int)p->n, m = (int)p->m, N = (int)p->N;
    const size_t smem = PersistSmem<T>::bytes(n, m);
    auto kern = btd_persist_kernel<T>;
    if (btd_status rs = ensure_smem_attr((const void *)kern, smem); rs != BTD_OK) return rs;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPThreads, smem);
    if (e != cudaSuccess) return record_cuda_error(e);
    if (per_sm < 1) return BTD_EUNSUPPORTED;
    const size_t nn = (size_t)n * n;
    const T *Dt = (const T *)D + (op != 1 ? sys0 * N * nn : 0);
    const T *Et = E ? (const T *)E + sys0 * (size_t)(N - 1) * nn : nullptr;
    const T *bt = b ? (const T *)b + sys0 * (size_t)N * n * m : nullptr;
    T *Dh = (T *)Dhat + sys0 * N * nn;
    T *Ct = (T *)C + sys0 * (size_t)p->geo.nC * nn;
    T *xt = x ? (T *)x + sys0 * (size_t)N * n * m : nullptr;
    int32_t *inf = info ? info + sys0 : nullptr;
    if (op == 1) Dt = nullptr;
    Geo g = p->geo;
    int batch = (int)count, fact = op != 1, solve = op != 0;
    // enough CTAs for the widest phase, but never more than can be co-resident
    long long want = (long long)count * ((N + 1) / 2) * 2 * ((n + kPRT - 1) / kPRT);
    long long maxg = (long long)nsm * per_sm;
    int grid = (int)(want < maxg ? (want > 0 ? want : 1) : maxg);
    void *args[] = {(void *)&Dt, (void *)&Et, (void *)&bt, (void *)&Dh, (void *)&Ct, (void *)&xt, (void *)&inf,
                    (void *)&g, (void *)&batch, (void *)&fact, (void *)&solve};
    e = cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(kPThreads), args, smem, st);
    if (e != cudaSuccess) return record_cuda_error(e);
    return BTD_OK;
}

template <typename T, int NB, bool ATOMIC>
static btd_status launch_wide(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat,
                              void *C, void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    const int n = (int)p->n, m = (int)p->m, N = (int)p->N;
    const size_t smem = WideSmem<T>::bytes(n, m);
    auto kern = btd_wide_kernel<T, NB, ATOMIC>;
    if (btd_status rs = ensure_smem_attr((const void *)kern, smem); rs != BTD_OK) return rs;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWThreads, smem);
    if (e != cudaSuccess) return record_cuda_error(e);
    if (per_sm < 1) return BTD_EUNSUPPORTED;
    const size_t nn = (size_t)n * n;
    const T *Dt = op != 1 ? (const T *)D + sys0 * N * nn : nullptr;
    const T *Et = E ? (const T *)E + sys0 * (size_t)(N - 1) * nn : nullptr;
    const T *bt = b ? (const T *)b + sys0 * (size_t)N * n * m : nullptr;
    T *Dh = (T *)Dhat + sys0 * N * nn;
    T *Ct = (T *)C + sys0 * (size_t)p->geo.nC * nn;
    T *xt = x ? (T *)x + sys0 * (size_t)N * n * m : nullptr;
    int32_t *inf = info ? info + sys0 : nullptr;
    Geo g = p->geo;
    int batch = (int)count, fact = op != 1, solve = op != 0;
    const long long want = (long long)count * ((N + 1) / 2);
    const long long maxg = (long long)nsm * per_sm;
    int grid = (int)(want < maxg ? (want > 0 ? want : 1) : maxg);
    void *args[] = {(void *)&Dt, (void *)&Et, (void *)&bt, (void *)&Dh, (void *)&Ct, (void *)&xt, (void *)&inf,
                    (void *)&g, (void *)&batch, (void *)&fact, (void *)&solve};
    e = cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(kWThreads), args, smem, st);
    if (e != cudaSuccess) return record_cuda_error(e);
    return BTD_OK;
}

template <typename T>
btd_status run_wide(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat, void *C,
                    void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    if (p->variant == BTD_VARIANT_ATOMIC) {
        if (p->n <= 8) return launch_wide<T, 8, true>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
        if (p->n <= 16) return launch_wide<T, 16, true>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
        return launch_wide<T, 32, true>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    }
    if (p->n <= 8) return launch_wide<T, 8, false>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    if (p->n <= 16) return launch_wide<T, 16, false>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    return launch_wide<T, 32, false>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
}

template btd_status run_wide<float>(const btd_plan *, int, const void *, const void *, const void *, void *, void *,
                                    void *, int32_t *, int64_t, int64_t, cudaStream_t);
template btd_status run_wide<double>(const btd_plan *, int, const void *, const void *, const void *, void *, void *,
                                     void *, int32_t *, int64_t, int64_t, cudaStream_t);

template btd_status run_persist<float>(const btd_plan *, int, const void *, const void *, const void *, void *, void *,
                                       void *, int32_t *, int64_t, int64_t, cudaStream_t);
template btd_status run_persist<double>(const btd_plan *, int, const void *, const void *, const void *, void *,
                                        void *, void *, int32_t *, int64_t, int64_t, cudaStream_t);
}  // namespace btd

#ifdef BTD_TIMING
extern "C" int btd_debug_timing_wide(unsigned long long *host16, int reset) {
    if (reset) {
        unsigned long long z[32] = {0};
        return (int)cudaMemcpyToSymbol(btd::btd_timing, z, sizeof z);
    }
    return (int)cudaMemcpyFromSymbol(host16, btd::btd_timing, 32 * sizeof(unsigned long long));
}
#endif
