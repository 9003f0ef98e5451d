// btd_inst.cu -- typed launchers; compiled once per (dtype, NB) with -DBTD_T=<float|double> -DBTD_NB=<n>
// so the 20 instantiations build in parallel (see paper_2601_03754_b200/build.py).
#include "btd_fused_r2.cuh"
#include "btd_internal.h"
#include "btd_persist.cuh"

namespace btd {
static btd_status cuda_fail(cudaError_t e) { return record_cuda_error(e); }

template <typename T, int NB, bool FACT, bool SOLVE, int MR>
static btd_status launch_fused_mr(const btd_plan *p, const T *D, const T *E, const T *b, T *Dhat, T *C, T *x,
                                  int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    constexpr bool R = FusedRCfg<T, NB>::OK;
    constexpr int TS = R ? FusedRCfg<T, NB>::TS : FusedCfg<T, NB>::TS;
    constexpr int NT = R ? FusedRCfg<T, NB>::NT : FusedCfg<T, NB>::NT;
    void (*kern)(const T *, const T *, const T *, T *, T *, T *, int32_t *, Geo, int);
    if constexpr (R)
        kern = p->n == NB ? btd_fused_r_kernel<T, NB, TS, NT, FACT, SOLVE, MR, true>
                          : btd_fused_r_kernel<T, NB, TS, NT, FACT, SOLVE, MR, false>;
    else
        kern = btd_fused_kernel<T, NB, TS, NT, FACT, SOLVE, MR>;
    if constexpr (FACT && SOLVE && MR == 1 && r2_capable<T, NB>()) {
        if (p->n == NB && p->use_r2) {
            auto k2 = p->r2_minb == 2 ? btd_fused_r2_kernel<T, NB, TS, NT, 2> : btd_fused_r2_kernel<T, NB, TS, NT, 3>;
            const size_t sm2 = FusedR2Cfg<T, NB>::bytes((int)p->N);
            if (btd_status rs = ensure_smem_attr((const void *)k2, sm2); rs != BTD_OK) return rs;
            for (int64_t s0 = 0; s0 < count; s0 += (1ll << 30)) {
                const int64_t cnt = (count - s0) < (1ll << 30) ? (count - s0) : (1ll << 30);
                k2<<<(unsigned)cnt, NT * TS, sm2, st>>>(D, E, b, Dhat, C, x, info, p->geo, (int)(sys0 + s0));
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) return cuda_fail(e);
            }
            return BTD_OK;
        }
    }
    const size_t smem = fused_bytes<T, NB>(p, FACT, SOLVE);
    // opt in to > 48 KB dynamic smem per (device, KERNEL): the exact-n (EX) and padded FUSED-R
    // instantiations are two kernels behind one launcher
    if (btd_status rs = ensure_smem_attr((const void *)kern, smem); rs != BTD_OK) return rs;
    for (int64_t s0 = 0; s0 < count; s0 += (1ll << 30)) {
        const int64_t cnt = (count - s0) < (1ll << 30) ? (count - s0) : (1ll << 30);
        kern<<<(unsigned)cnt, NT * TS, smem, st>>>(D, E, b, Dhat, C, x, info, p->geo, (int)(sys0 + s0));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e);
    }
    return BTD_OK;
}

template <typename T, int NB, bool FACT, bool SOLVE>
static btd_status launch_fused(const btd_plan *p, const T *D, const T *E, const T *b, T *Dhat, T *C, T *x,
                               int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    if constexpr (SOLVE) {
        if (p->m == 1) return launch_fused_mr<T, NB, FACT, SOLVE, 1>(p, D, E, b, Dhat, C, x, info, sys0, count, st);
    }
    return launch_fused_mr<T, NB, FACT, SOLVE, 0>(p, D, E, b, Dhat, C, x, info, sys0, count, st);
}

template <typename T, int NB, bool FACT, bool SOLVE>
static btd_status launch_level(const btd_plan *p, const T *D, const T *E, const T *b, T *Dhat, T *C, T *x,
                               int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    constexpr int TS = LevelShape<T, NB>::TS, NT = LevelShape<T, NB>::NT;
    constexpr int SMEM = NT * LevelShape<T, NB>::BYTES;
    const int64_t N = p->N, n = p->n, m = p->m;
    const size_t nn = (size_t)n * n;
    {   // init: Dhat <- D, x <- b, info <- 0 (for the slice)
        const long long nD = FACT ? (long long)(count * N * nn) : 0;
        const long long nb = SOLVE ? (long long)(count * N * n * m) : 0;
        long long work = nD > nb ? nD : nb;
        if (work < count) work = count;
        int blocks = (int)((work + 255) / 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        if (blocks < 1) blocks = 1;
        btd_level_init_kernel<T><<<blocks, 256, 0, st>>>(
            FACT ? D + sys0 * N * nn : nullptr, SOLVE ? b + sys0 * N * n * m : nullptr,
            FACT ? Dhat + sys0 * N * nn : nullptr, SOLVE ? x + sys0 * N * n * m : nullptr,
            FACT ? info + sys0 : nullptr, nD, nb, (int)count, FACT ? 1 : 0, SOLVE ? 1 : 0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e);
    }
    for (int64_t s0 = 0; s0 < count; s0 += 65535) {
        const int64_t cnt = (count - s0) < 65535 ? (count - s0) : 65535;
        const int base = (int)(sys0 + s0);
        for (int l = 1; l <= p->L; ++l) {
            const int64_t s = 1ll << (l - 1);
            const int64_t ncols = ((N / s) + 1) / 2;
            dim3 grid((unsigned)((ncols + NT - 1) / NT), (unsigned)cnt);
            btd_level_fwd_kernel<T, NB, TS, NT, FACT, SOLVE>
                <<<grid, NT * TS, SMEM, st>>>(E, Dhat, C, x, info, p->geo, l, base);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e);
        }
        if (SOLVE) {
            for (int l = p->L; l >= 1; --l) {
                const int64_t s = 1ll << (l - 1);
                const int64_t ncols = ((N / s) + 1) / 2;
                dim3 grid((unsigned)((ncols + NT - 1) / NT), (unsigned)cnt);
                btd_level_bwd_kernel<T, NB, TS, NT><<<grid, NT * TS, 0, st>>>(Dhat, C, x, p->geo, l, base);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) return cuda_fail(e);
            }
        }
    }
    return BTD_OK;
}

template <typename T, int NB, bool FACT, bool SOLVE>
static btd_status launch_persist_team(const btd_plan *p, const T *D, const T *E, const T *b, T *Dhat, T *C, T *x,
                                      int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    using Cfg = PTeamCfg<T, NB>;
    auto kern = btd_persist_team_kernel<T, NB, FACT, SOLVE>;
    const size_t smem = Cfg::BYTES;
    if (btd_status rs = ensure_smem_attr((const void *)kern, smem); rs != BTD_OK) return rs;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS, smem);
    if (e != cudaSuccess) return cuda_fail(e);
    if (per_sm < 1) return BTD_EUNSUPPORTED;
    const int64_t N = p->N, n = p->n, m = p->m;
    const size_t nn = (size_t)n * n;
    const T *Dt = FACT ? D + sys0 * N * nn : nullptr;
    const T *Et = (FACT && E) ? E + sys0 * (size_t)(N - 1) * nn : nullptr;
    const T *bt = SOLVE ? b + sys0 * (size_t)N * n * m : nullptr;
    T *Dh = Dhat + sys0 * N * nn;
    T *Ct = C + sys0 * (size_t)p->geo.nC * nn;
    T *xt = SOLVE ? x + sys0 * (size_t)N * n * m : nullptr;
    int32_t *inf = FACT ? info + sys0 : nullptr;
    Geo g = p->geo;
    int batch = (int)count;
    const long long want = ((long long)count * ((N + 1) / 2) + Cfg::NT - 1) / Cfg::NT;
    const long long maxg = (long long)nsm * per_sm;
    int grid = (int)(want < maxg ? (want > 0 ? want : 1) : maxg);
    void *args[] = {(void *)&Dt, (void *)&Et, (void *)&bt, (void *)&Dh, (void *)&Ct,
                    (void *)&xt, (void *)&inf, (void *)&g, (void *)&batch};
    e = cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(Cfg::THREADS), args, smem, st);
    if (e != cudaSuccess) return cuda_fail(e);
    return BTD_OK;
}

template <typename T, int NB>
btd_status run_typed(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat,
                            void *C, void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    const T *Dt = (const T *)D, *Et = (const T *)E, *bt = (const T *)b;
    T *Dh = (T *)Dhat, *Ct = (T *)C, *xt = (T *)x;
    if (p->variant == BTD_VARIANT_PERSIST) {
        if (op == 0) return launch_persist_team<T, NB, true, false>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
        if (op == 1) return launch_persist_team<T, NB, false, true>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
        return launch_persist_team<T, NB, true, true>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
    }
    if (p->variant == BTD_VARIANT_FUSED) {
        if (op == 0) return launch_fused<T, NB, true, false>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
        if (op == 1) return launch_fused<T, NB, false, true>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
        return launch_fused<T, NB, true, true>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
    }
    if (op == 0) return launch_level<T, NB, true, false>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
    if (op == 1) return launch_level<T, NB, false, true>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
    return launch_level<T, NB, true, true>(p, Dt, Et, bt, Dh, Ct, xt, info, sys0, count, st);
}


#if defined(BTD_TIMING) && defined(BTD_NB) && BTD_NB == 12
}  // namespace btd
#define BTD_CAT2(a, b) a##b
#define BTD_CAT(a, b) BTD_CAT2(a, b)
extern "C" int BTD_CAT(btd_debug_timing_, BTD_T)(unsigned long long *host16, int reset) {
    if (reset) {
        unsigned long long z[32] = {0};
        return (int)cudaMemcpyToSymbol(btd::btd_timing, z, sizeof z);
    }
    return (int)cudaMemcpyFromSymbol(host16, btd::btd_timing, 32 * sizeof(unsigned long long));
}
namespace btd {
#endif

#if defined(BTD_T) && defined(BTD_NB)
template btd_status run_typed<BTD_T, BTD_NB>(const btd_plan *, int, const void *, const void *, const void *,
                                             void *, void *, void *, int32_t *, int64_t, int64_t, cudaStream_t);
#endif
}  // namespace btd
