// btd_internal.h -- plan structure and typed-launcher declarations shared by btd.cu and btd_inst.cu.
#pragma once
#include <cuda_runtime.h>

#include "../../include/btd.h"
#include "btd_fused_r2.cuh"

struct btd_plan {
    int64_t N, n, batch, m;
    btd_dtype dtype;
    int L;
    int NB;        // compiled block size
    int variant;   // BTD_VARIANT_FUSED / BTD_VARIANT_LEVEL
    size_t smem_fs, smem_f, smem_s;  // fused smem bytes: factor+solve, factor, solve
    size_t smem_persist;             // PERSIST kernel dynamic smem bytes
    int r2_minb;                     // FUSED-R2 min CTAs/SM (register cap): 3 (default) or 2 (env BTD_R2_MINB)
    bool use_persist2;               // n > 32: PERSIST2 (env BTD_PERSIST2=0 selects the round-1 PERSIST kernel)
    bool use_r2;                     // factor+solve, m = 1, n == NB: FUSED-R2 (env BTD_FUSED_R2=0 disables)
    btd::Geo geo;
};


namespace btd {
btd_status record_cuda_error(cudaError_t e);

// Opt kernel `kern` in to `bytes` of dynamic shared memory on the CURRENT device (the attribute is
// per device context). Remembered per (device, kernel) under a mutex, so concurrent callers and
// processes driving several GPUs each set it once per device.
btd_status ensure_smem_attr(const void *kern, size_t bytes);

template <int NB>
struct TeamShape {
    static constexpr int TS = NB <= 1 ? 1 : NB <= 2 ? 2 : NB <= 4 ? 4 : NB <= 8 ? 8 : NB <= 16 ? 16 : 32;
    static constexpr int NT = 128 / TS;  // teams per CTA, fused kernel
};

template <typename T, int NB>
struct LevelShape {
    static constexpr int TS = TeamShape<NB>::TS;
    static constexpr int BYTES = LevelSmem<T, NB>::TSTR * (int)sizeof(T);
    static constexpr int CAP = 24 * 1024 / BYTES;
    static constexpr int NT = CAP < 1 ? 1 : (CAP < 128 / TS ? CAP : 128 / TS);
};

constexpr size_t kMaxSmem = 227 * 1024 - 64;  // minus the kernel's static shared bytes

// FUSED-R2 (btd_fused_r2.cuh) handles factor+solve with m = 1 for the FUSED-R sizes whose rows
// are whole 16-byte vectors (fp32 n in {4, 8, 12}, fp64 n in {2, 4, 6, 8}).
template <typename T, int NB>
constexpr bool r2_capable() {
    return FusedRCfg<T, NB>::OK && Dims<T, NB>::LD == NB;
}

template <typename T, int NB>
size_t fused_bytes(const btd_plan *p, bool fact, bool solve) {
    if constexpr (r2_capable<T, NB>()) {
        if (fact && solve && p->m == 1 && p->n == NB && p->use_r2) {
            // (N * LD) elements of Y + odd full slots + even padded-lower slots
            const int N = (int)p->N;
            const size_t e = (size_t)((N + 1) / 2) * Dims<T, NB>::BLK + (size_t)(N / 2) * PLow<T, NB>::SZ +
                             (size_t)N * Dims<T, NB>::LD;
            return e * sizeof(T);
        }
    }
    if (FusedRCfg<T, NB>::OK) return FusedRCfg<T, NB>::bytes((int)p->N, (int)p->m, fact, solve);
    return FusedSmem<T, NB, FusedCfg<T, NB>::NT>::bytes((int)p->N, (int)p->m, fact, solve);
}

// Defined in btd_persist.cu (any n <= 128, cooperative launch).
template <typename T>
btd_status run_persist(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat, void *C,
                       void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st);

// Defined in btd_persist.cu (n <= 32, one CTA per column op, cooperative launch).
template <typename T>
btd_status run_wide(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat, void *C,
                    void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st);

// Defined in btd_inst.cu, explicitly instantiated once per (T, NB) translation unit.
template <typename T, int NB>
btd_status run_typed(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat, void *C,
                     void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st);
}  // namespace btd
