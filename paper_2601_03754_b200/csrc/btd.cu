// btd.cu -- C ABI (include/btd.h): plan (symbolic analysis a0), argument checks, dispatch.
//
// The plan derives everything from (N, n, batch, m, dtype): L = floor(log2 N)+1 levels
// (PAPER.md:569), slot offsets off(l) = sum_{l'<l} (floor(N/2^(l'-1)) - 1), the compiled block
// size NB >= n (identity padding), the team width and the kernel variant. No device tables:
// every index is closed form in (level, column) and passed as kernel arguments.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <utility>
#include <vector>

#include "btd_internal.h"
#include "btd_persist.cuh"
#include "btd_persist2.cuh"
#include "btd_wide.cuh"

using namespace btd;

static thread_local char g_last_error[256] = "";

btd_status btd::record_cuda_error(cudaError_t e) {
    snprintf(g_last_error, sizeof g_last_error, "%s", cudaGetErrorString(e));
    return BTD_ECUDA;
}
static btd_status cuda_fail(cudaError_t e) { return record_cuda_error(e); }

btd_status btd::ensure_smem_attr(const void *kern, size_t bytes) {
    if (bytes <= 48 * 1024) return BTD_OK;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    size_t &have = done[{dev, kern}];
    if (bytes <= have) return BTD_OK;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_fail(e);
    have = bytes;
    return BTD_OK;
}

// Device buffers are read and written with 16-byte vector accesses (LDGSTS / LDG.128 / STG.128)
// from their base address; the per-system strides are handled inside the kernels.
static bool al16(const void *p) { return ((uintptr_t)p & 15u) == 0; }
static bool al4(const void *p) { return ((uintptr_t)p & 3u) == 0; }

static const int kSizes[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};

// Largest N for which ONE system runs faster in the one-CTA FUSED kernel (no grid barriers) than in
// the cooperative WIDE kernel, per dtype and compiled block size (measured on B200,
// profiles/r02/fused_vs_wide_single.txt; e.g. fp64 n = 4, N = 64: 23 vs 73 us; n = 12: FUSED up to
// N = 64, WIDE from 128; n = 16: FUSED only at N = 16).
static int64_t fused_max_n_single(bool f32, int NB) {
    if (f32) return NB <= 8 ? 1024 : NB <= 12 ? 128 : NB <= 16 ? 64 : NB <= 24 ? 16 : 11;
    return NB <= 4 ? 1024 : NB <= 8 ? 192 : NB <= 12 ? 96 : NB <= 24 ? 16 : 3;
}

static int pick_nb(int64_t n) {
    for (int s : kSizes)
        if (n <= s) return s;
    return -1;
}

template <typename T>
static btd_status run_dtype(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat,
                            void *C, void *x, int32_t *info, int64_t sys0, int64_t count, cudaStream_t st) {
    switch (p->NB) {
#define BTD_CASE(S) \
    case S: return run_typed<T, S>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
        BTD_CASE(1) BTD_CASE(2) BTD_CASE(3) BTD_CASE(4) BTD_CASE(6) BTD_CASE(8) BTD_CASE(12) BTD_CASE(16)
        BTD_CASE(24) BTD_CASE(32)
#undef BTD_CASE
        default: return BTD_EUNSUPPORTED;
    }
}

template <typename T>
static size_t fused_bytes_dt(const btd_plan *p, bool fact, bool solve) {
    switch (p->NB) {
#define BTD_CASE(S) \
    case S: return fused_bytes<T, S>(p, fact, solve);
        BTD_CASE(1) BTD_CASE(2) BTD_CASE(3) BTD_CASE(4) BTD_CASE(6) BTD_CASE(8) BTD_CASE(12) BTD_CASE(16)
        BTD_CASE(24) BTD_CASE(32)
#undef BTD_CASE
        default: return ~(size_t)0;
    }
}

static btd_status run(const btd_plan *p, int op, const void *D, const void *E, const void *b, void *Dhat, void *C,
                      void *x, int32_t *info, int64_t sys0, int64_t count, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (p->variant == BTD_VARIANT_WIDE || p->variant == BTD_VARIANT_ATOMIC) {
        if (p->dtype == BTD_F32) return run_wide<float>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
        return run_wide<double>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    }
    if (p->variant == BTD_VARIANT_PERSIST && p->NB < 0) {  // n > 32: CTA-wide block ops
        if (p->dtype == BTD_F32) return run_persist<float>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
        return run_persist<double>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    }
    if (p->dtype == BTD_F32) return run_dtype<float>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
    return run_dtype<double>(p, op, D, E, b, Dhat, C, x, info, sys0, count, st);
}

// Streams and events of btd_factor_solve_host, created once per (host thread, device) and kept for
// the thread's lifetime (one thread's calls are issued in order, so reusing an event is safe: each
// cudaStreamWaitEvent captures the record made just before it).
struct HostPipe {
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t fork = nullptr, done = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_out;
};

static btd_status host_pipe(int nch, HostPipe **out) {
    static thread_local std::map<int, HostPipe> pipes;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    HostPipe &hp = pipes[dev];
    if (!hp.up && (e = cudaStreamCreateWithFlags(&hp.up, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e);
    if (!hp.down && (e = cudaStreamCreateWithFlags(&hp.down, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e);
    if (!hp.fork && (e = cudaEventCreateWithFlags(&hp.fork, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e);
    if (!hp.done && (e = cudaEventCreateWithFlags(&hp.done, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e);
    while ((int)hp.ev_in.size() < nch) {
        cudaEvent_t a = nullptr, b = nullptr;
        if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e);
        if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) {
            cudaEventDestroy(a);
            return cuda_fail(e);
        }
        hp.ev_in.push_back(a);
        hp.ev_out.push_back(b);
    }
    *out = &hp;
    return BTD_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

btd_status btd_plan_create_ex(btd_plan **out, int64_t N, int64_t n, int64_t batch, int64_t m, btd_dtype dtype,
                              btd_variant variant) {
    if (!out) return BTD_EINVAL;
    *out = nullptr;
    if (N < 1 || n < 1 || batch < 1 || m < 1 || (dtype != BTD_F32 && dtype != BTD_F64)) return BTD_EINVAL;
    if (N > (1ll << 24) || m > 4096) return BTD_EINVAL;
    if (n > 128) return BTD_EUNSUPPORTED;
    if (variant < BTD_VARIANT_AUTO || variant > BTD_VARIANT_ATOMIC) return BTD_EINVAL;
    const int NB = pick_nb(n);  // -1 for n > 32: only PERSIST handles those
    if (NB < 0 && (variant == BTD_VARIANT_FUSED || variant == BTD_VARIANT_LEVEL || variant == BTD_VARIANT_WIDE ||
                   variant == BTD_VARIANT_ATOMIC))
        return BTD_EUNSUPPORTED;
    btd_plan *p = new (std::nothrow) btd_plan();
    if (!p) return BTD_ENOMEM;
    p->N = N; p->n = n; p->batch = batch; p->m = m; p->dtype = dtype; p->NB = NB;
    {
        const char *ev = getenv("BTD_FUSED_R2");  // dev knob for A/B measurements (default on)
        p->use_r2 = !(ev && ev[0] == '0');
        const char *mb = getenv("BTD_R2_MINB");
        p->r2_minb = (mb && mb[0] == '2') ? 2 : 3;
        const char *p2 = getenv("BTD_PERSIST2");
        p->use_persist2 = !(p2 && p2[0] == '0');
    }
    int L = 0;
    while ((1ll << L) <= N) ++L;  // floor(log2 N) + 1
    p->L = L;
    memset(&p->geo, 0, sizeof p->geo);
    p->geo.N = (int)N; p->geo.n = (int)n; p->geo.m = (int)m; p->geo.L = L;
    long long off = 0;
    for (int l = 1; l <= L + 1; ++l) {
        p->geo.off[l - 1] = off;
        if (l <= L) off += (N >> (l - 1)) - 1;
    }
    p->geo.nC = off;
    const bool f32 = dtype == BTD_F32;
    if (NB > 0) {
        p->smem_fs = f32 ? fused_bytes_dt<float>(p, true, true) : fused_bytes_dt<double>(p, true, true);
        p->smem_f = f32 ? fused_bytes_dt<float>(p, true, false) : fused_bytes_dt<double>(p, true, false);
        p->smem_s = f32 ? fused_bytes_dt<float>(p, false, true) : fused_bytes_dt<double>(p, false, true);
    } else {
        p->smem_fs = p->smem_f = p->smem_s = ~(size_t)0;
    }
    size_t psm = 0;
    if (NB < 0)
        psm = p->use_persist2 ? (f32 ? Persist2Smem<float>::bytes((int)n, (int)m) : Persist2Smem<double>::bytes((int)n, (int)m))
                              : (f32 ? PersistSmem<float>::bytes((int)n, (int)m) : PersistSmem<double>::bytes((int)n, (int)m));
    const bool fits = p->smem_fs <= kMaxSmem;
    if ((variant == BTD_VARIANT_FUSED && !fits) || (variant == BTD_VARIANT_PERSIST && psm > kMaxSmem)) {
        delete p;
        return BTD_EUNSUPPORTED;
    }
    const size_t wsm = f32 ? WideSmem<float>::bytes((int)n, (int)m) : WideSmem<double>::bytes((int)n, (int)m);
    if ((variant == BTD_VARIANT_WIDE || variant == BTD_VARIANT_ATOMIC) && wsm > kMaxSmem) {
        delete p;
        return BTD_EUNSUPPORTED;
    }
    if (variant == BTD_VARIANT_AUTO) {
        // few independent systems with enough level-1 columns to spread over the SMs: latency path.
        // One system: WIDE up to 2048 (fp64) / 1024 (fp32) level-1 columns, where the cooperative
        // PERSIST kernel takes over; with many right-hand sides (m >= 16, e.g. the partition
        // chunks' border columns) WIDE whenever the system does not fit FUSED (measured,
        // profiles/r02/wide_vs_persist.txt: fp64 N = 2048: 615 vs 890 us; m = 65: 1.3 vs 8.9 ms).
        const long long cols = batch * ((N + 1) / 2);
        // several long systems: the single-system crossover holds for fp64 n = 32 (WIDE's DMMA tiles),
        // PERSIST wins the others (profiles/r02/wide_vs_persist_batched.txt: 4 x fp64 N = 512 n = 32:
        // 535 vs 775 us; 4 x fp64 N = 1024 n = 16: 407 vs 312 us)
        const long long wide_cols = batch > 1 ? ((!f32 && NB == 32) ? 2048 : 4 * 148) : (f32 ? 1024 : 2048);
        // short systems: FUSED (one CTA) wins below 16 blocks except for 32-wide blocks, where one CTA per
        // column op already pays from N = 4 (fp64) / 12 (fp32) (profiles/r02/small_n.txt: fp64 n = 32,
        // N = 8: 104 vs 141 us; N = 15: 105 vs 208 us)
        const bool long_enough = N >= 16 || (NB == 32 && N >= (f32 ? 12 : 4));
        const bool wide_ok = NB > 0 && wsm <= kMaxSmem && long_enough && (cols <= wide_cols || (m >= 16 && !fits));
        // up to one system per SM the FUSED CTAs all run at once: the single-system crossover applies
        const bool fused_first = batch <= 148 && fits && N <= fused_max_n_single(f32, NB);
        p->variant = fused_first ? BTD_VARIANT_FUSED : wide_ok ? BTD_VARIANT_WIDE : fits ? BTD_VARIANT_FUSED
                                                                                      : BTD_VARIANT_PERSIST;
        if (p->variant == BTD_VARIANT_PERSIST && NB < 0 && psm > kMaxSmem) {  // e.g. n = 128 fp64 with m >= 32
            delete p;
            return BTD_EUNSUPPORTED;
        }
    } else {
        p->variant = variant;
    }
    p->smem_persist = psm;
    *out = p;
    return BTD_OK;
}

btd_status btd_plan_create(btd_plan **out, int64_t N, int64_t n, int64_t batch, int64_t m, btd_dtype dtype) {
    return btd_plan_create_ex(out, N, n, batch, m, dtype, BTD_VARIANT_AUTO);
}

void btd_plan_destroy(btd_plan *plan) { delete plan; }

int32_t btd_num_levels(const btd_plan *p) { return p ? p->L : -1; }

int64_t btd_num_coupling_blocks(const btd_plan *p) { return p ? p->geo.nC : -1; }

int64_t btd_level_offset(const btd_plan *p, int32_t level) {
    if (!p || level < 1 || level > p->L + 1) return -1;
    return p->geo.off[level - 1];
}

btd_status btd_permutation(const btd_plan *p, int64_t *host_perm) {
    if (!p || !host_perm) return BTD_EINVAL;
    int64_t q = 0;
    for (int l = 1; l <= p->L; ++l) {
        const int64_t s = 1ll << (l - 1);
        for (int64_t c = s; c <= p->N; c += 2 * s) host_perm[q++] = c - 1;
    }
    return BTD_OK;
}

int32_t btd_plan_variant(const btd_plan *p) { return p ? p->variant : -1; }

int32_t btd_plan_launches(const btd_plan *p, int32_t op) {
    if (!p || op < 0 || op > 2) return -1;
    if (p->variant != BTD_VARIANT_LEVEL) return 1;
    const int64_t chunks = (p->batch + 65534) / 65535;
    const int per = op == 0 ? p->L : op == 1 ? 2 * p->L : 2 * p->L;
    return (int32_t)(1 + chunks * per);
}

int64_t btd_plan_smem_bytes(const btd_plan *p) {
    if (!p) return -1;
    if (p->variant == BTD_VARIANT_PERSIST) return (int64_t)p->smem_persist;
    return p->variant == BTD_VARIANT_FUSED ? (int64_t)p->smem_fs : 0;
}

btd_status btd_factor(const btd_plan *p, const void *D, const void *E, void *Dhat, void *C, int32_t *info,
                      void *stream) {
    if (!p || !D || !Dhat || (!C && p->geo.nC > 0) || !info || (p->N > 1 && !E)) return BTD_EINVAL;
    if (!al16(D) || !al16(E) || !al16(Dhat) || !al16(C) || !al4(info)) return BTD_EINVAL;
    return run(p, 0, D, E, nullptr, Dhat, C, nullptr, info, 0, p->batch, stream);
}

btd_status btd_solve(const btd_plan *p, const void *Dhat, const void *C, const void *b, void *x, void *stream) {
    if (!p || !Dhat || (!C && p->geo.nC > 0) || !b || !x) return BTD_EINVAL;
    if (!al16(Dhat) || !al16(C) || !al16(b) || !al16(x)) return BTD_EINVAL;
    return run(p, 1, nullptr, nullptr, b, (void *)Dhat, (void *)C, x, nullptr, 0, p->batch, stream);
}

btd_status btd_factor_solve(const btd_plan *p, const void *D, const void *E, const void *b, void *Dhat, void *C,
                            void *x, int32_t *info, void *stream) {
    if (!p || !D || !b || !Dhat || (!C && p->geo.nC > 0) || !x || !info || (p->N > 1 && !E)) return BTD_EINVAL;
    if (!al16(D) || !al16(E) || !al16(b) || !al16(Dhat) || !al16(C) || !al16(x) || !al4(info)) return BTD_EINVAL;
    return run(p, 2, D, E, b, Dhat, C, x, info, 0, p->batch, stream);
}

btd_status btd_factor_solve_host(const btd_plan *p, const void *hD, const void *hE, const void *hb, void *hDhat,
                                 void *hC, void *hx, int32_t *hinfo, void *dD, void *dE, void *db, void *dDhat,
                                 void *dC, void *dx, int32_t *dinfo, int32_t chunks, void *stream) {
    if (!p || !hD || !hb || !hDhat || ((!hC || !dC) && p->geo.nC > 0) || !hx || !hinfo || !dD || !db || !dDhat || !dx || !dinfo ||
        chunks < 1)
        return BTD_EINVAL;
    if (p->N > 1 && (!hE || !dE)) return BTD_EINVAL;
    if (!al16(dD) || !al16(dE) || !al16(db) || !al16(dDhat) || !al16(dC) || !al16(dx) || !al4(dinfo))
        return BTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t w = p->dtype == BTD_F32 ? 4 : 8;
    const size_t nn = (size_t)p->n * p->n;
    const size_t sD = p->N * nn * w, sE = (p->N - 1) * nn * w, sb = p->N * p->n * p->m * w,
                 sC = (size_t)p->geo.nC * nn * w;
    const int64_t per = (p->batch + chunks - 1) / chunks;
    const int nch = (int)((p->batch + per - 1) / per);
    // Three-stage pipeline: host->device copies on stream `up`, compute on the caller's stream,
    // device->host copies on stream `down` (the two copy directions run on separate copy engines),
    // chained per slice by events; the caller's stream finally waits for `down`, so the call stays
    // asynchronous and ordered on `stream`. The two streams and the events are created once per
    // (host thread, device) and reused by every later call (HostPipe).
    HostPipe *hp = nullptr;
    btd_status rs = host_pipe(nch, &hp);
    if (rs != BTD_OK) return rs;
    cudaStream_t up = hp->up, down = hp->down;
    cudaError_t e = cudaSuccess;
#define CK(call)                         \
    do {                                 \
        e = (call);                      \
        if (e != cudaSuccess) {          \
            return cuda_fail(e);         \
        }                                \
    } while (0)
    CK(cudaEventRecord(hp->fork, st));  // everything queued on `stream` before this call comes first
    CK(cudaStreamWaitEvent(up, hp->fork, 0));
    CK(cudaStreamWaitEvent(down, hp->fork, 0));
    for (int c = 0; c < nch; ++c) {
        const int64_t s0 = c * per;
        const int64_t cnt = (p->batch - s0) < per ? (p->batch - s0) : per;
        CK(cudaMemcpyAsync((char *)dD + s0 * sD, (const char *)hD + s0 * sD, cnt * sD, cudaMemcpyHostToDevice, up));
        if (sE)
            CK(cudaMemcpyAsync((char *)dE + s0 * sE, (const char *)hE + s0 * sE, cnt * sE, cudaMemcpyHostToDevice, up));
        CK(cudaMemcpyAsync((char *)db + s0 * sb, (const char *)hb + s0 * sb, cnt * sb, cudaMemcpyHostToDevice, up));
        CK(cudaEventRecord(hp->ev_in[c], up));
        CK(cudaStreamWaitEvent(st, hp->ev_in[c], 0));
        rs = run(p, 2, dD, dE, db, dDhat, dC, dx, dinfo, s0, cnt, stream);
        if (rs != BTD_OK) return rs;
        CK(cudaEventRecord(hp->ev_out[c], st));
        CK(cudaStreamWaitEvent(down, hp->ev_out[c], 0));
        CK(cudaMemcpyAsync((char *)hDhat + s0 * sD, (const char *)dDhat + s0 * sD, cnt * sD, cudaMemcpyDeviceToHost, down));
        if (sC)
            CK(cudaMemcpyAsync((char *)hC + s0 * sC, (const char *)dC + s0 * sC, cnt * sC, cudaMemcpyDeviceToHost, down));
        CK(cudaMemcpyAsync((char *)hx + s0 * sb, (const char *)dx + s0 * sb, cnt * sb, cudaMemcpyDeviceToHost, down));
        CK(cudaMemcpyAsync(hinfo + s0, dinfo + s0, cnt * sizeof(int32_t), cudaMemcpyDeviceToHost, down));
    }
    CK(cudaEventRecord(hp->done, down));
    CK(cudaStreamWaitEvent(st, hp->done, 0));
#undef CK
    return BTD_OK;
}

const char *btd_status_string(btd_status s) {
    switch (s) {
        case BTD_OK: return "BTD_OK";
        case BTD_EINVAL: return "BTD_EINVAL: invalid argument";
        case BTD_ECUDA: return "BTD_ECUDA: CUDA error";
        case BTD_ENOMEM: return "BTD_ENOMEM: host allocation failed";
        case BTD_EUNSUPPORTED: return "BTD_EUNSUPPORTED: size not supported by this build";
    }
    return "BTD_UNKNOWN";
}

const char *btd_last_error(void) { return g_last_error; }

}  // extern "C"
