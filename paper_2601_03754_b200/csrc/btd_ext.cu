// btd_ext.cu -- the SURVEY.md §8(f) rows built on top of the core factor/solve (include/btd.h):
//
//   f4a  mixed precision: binary32 factorization + binary64 iterative refinement
//   f4b  block-tridiagonal-arrow systems, border eliminated last
//   f4c  block-banded systems of block bandwidth w, solved as super-block tridiagonal
//   f3   partition permutation (Algorithm 2): per-chunk local elimination,
//        pivot-system assembly and the chunk back-substitution, one chunk per rank
//
// Every kernel here is HBM- or latency-bound glue around the core path: packing of right-hand
// sides, block-tridiagonal residuals in binary64, small dense border Cholesky factorizations,
// Schur-complement contributions. The O(N n^3) work always runs in the core kernels through the
// public C ABI (btd_factor_solve / btd_solve).
#include <cuda_runtime.h>

#include <cstdint>

#include "btd_internal.h"

using btd::record_cuda_error;

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work) {
    int64_t g = (work + kThreads - 1) / kThreads;
    const int64_t cap = 148ll * 16;  // grid-stride beyond 16 CTAs per SM
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

inline btd_status launched() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BTD_OK : record_cuda_error(e);
}

inline bool al16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// ------------------------------------------------------------------------- f4a: mixed precision

// binary64 -> binary32 rounding of a contiguous array (16-byte loads of double pairs).
__global__ void k_demote(const double *__restrict__ a, float *__restrict__ o, int64_t cnt) {
    const int64_t pairs = cnt >> 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < pairs; q += stride) {
        const double2 v = reinterpret_cast<const double2 *>(a)[q];
        reinterpret_cast<float2 *>(o)[q] = make_float2((float)v.x, (float)v.y);
    }
    if ((cnt & 1) && blockIdx.x == 0 && threadIdx.x == 0) o[cnt - 1] = (float)a[cnt - 1];
}

// One refinement step, one thread per element (j, i, r, c) of x:
//   x_next = x_prev + d                                     (binary64; x_prev absent for x_0)
//   r      = b - Psi x_next                                 (binary64, D lower-authoritative)
// and either r rounded to binary32 (input of the next binary32 solve) or the per-system squared
// norms of r and b (final step). The neighbours' x_next values are recomputed from (x_prev, d)
// by every thread that needs them, so no thread reads a value another thread writes.
template <bool PREV, bool WR, bool NRM>
__global__ void k_ir_step(int B, int N, int n, int m, const double *__restrict__ D, const double *__restrict__ E,
                          const double *__restrict__ b, const double *__restrict__ xp, const float *__restrict__ d,
                          double *__restrict__ xn, float *__restrict__ r32, double *__restrict__ nrm) {
    const int64_t total = (int64_t)B * N * n * m;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nn = (int64_t)n * n, nm = (int64_t)n * m;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int c = (int)(e % m);
        int64_t t = e / m;
        const int r = (int)(t % n);
        t /= n;
        const int i = (int)(t % N);
        const int64_t j = t / N;
        auto X = [&](int64_t idx) -> double {
            double v = (double)d[idx];
            if (PREV) v += xp[idx];
            return v;
        };
        xn[e] = X(e);
        if (!WR && !NRM) continue;
        const int64_t xi = (j * N + i) * nm + c;  // x(i, 0, c)
        const double *Di = D + (j * N + i) * nn;
        double acc = b[e];
        for (int k = 0; k < n; ++k) {
            const double dv = k <= r ? Di[(int64_t)r * n + k] : Di[(int64_t)k * n + r];
            acc = fma(-dv, X(xi + (int64_t)k * m), acc);
        }
        if (i > 0) {
            const double *Em = E + (j * (N - 1) + i - 1) * nn;  // block (i, i-1): row r
            for (int k = 0; k < n; ++k) acc = fma(-Em[(int64_t)r * n + k], X(xi - nm + (int64_t)k * m), acc);
        }
        if (i < N - 1) {
            const double *Ep = E + (j * (N - 1) + i) * nn;  // block (i+1, i)^T: column r
            for (int k = 0; k < n; ++k) acc = fma(-Ep[(int64_t)k * n + r], X(xi + nm + (int64_t)k * m), acc);
        }
        if (WR) r32[e] = (float)acc;
        if (NRM) {
            atomicAdd(&nrm[2 * j], acc * acc);
            atomicAdd(&nrm[2 * j + 1], b[e] * b[e]);
        }
    }
}

__global__ void k_ir_finish(int B, const double *__restrict__ nrm, double *__restrict__ resid) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < B) resid[j] = nrm[2 * j + 1] > 0 ? sqrt(nrm[2 * j] / nrm[2 * j + 1]) : sqrt(nrm[2 * j]);
}

struct MixedWs {
    float *D32, *E32, *r32, *d32;
    double *xtmp, *nrm;
};

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

size_t mixed_layout(const btd_plan *p, char *base, MixedWs *w) {
    const size_t nn = (size_t)p->n * p->n, B = (size_t)p->batch, N = (size_t)p->N;
    const size_t nx = B * N * p->n * p->m;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *q = base ? base + off : nullptr;
        off += align_up(bytes);
        return q;
    };
    MixedWs t;
    t.D32 = (float *)take(B * N * nn * 4);
    t.E32 = (float *)take(B * (N - 1) * nn * 4);
    t.r32 = (float *)take(nx * 4);
    t.d32 = (float *)take(nx * 4);
    t.xtmp = (double *)take(nx * 8);
    t.nrm = (double *)take(2 * B * 8);
    if (w) *w = t;
    return off;
}

// ------------------------------------------------------------------------- f4b: arrowhead

// R[j][i][r][c] = G_i^T[r][c] (c < na) | b_i[r][c - na]   (right-hand sides [G^T | b])
template <typename T>
__global__ void k_arrow_pack(int B, int N, int n, int na, int mb, const T *__restrict__ G, const T *__restrict__ b,
                             T *__restrict__ R) {
    const int mR = na + mb;
    const int64_t total = (int64_t)B * N * n * mR;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int c = (int)(e % mR);
        const int64_t t = e / mR;  // (j, i, r)
        const int r = (int)(t % n);
        const int64_t ji = t / n;
        R[e] = c < na ? G[(ji * na + c) * n + r] : b[t * mb + (c - na)];
    }
}

// Same output, tiled: a CTA owns TB consecutive (system, block) pairs; their G blocks (contiguous in
// memory) are staged in shared memory with coalesced loads, then R is written in its own order
// (coalesced), reading G^T from shared memory. The direct kernel above reads G with stride n.
template <typename T>
__global__ void k_arrow_pack_tiled(int64_t nblk, int n, int na, int mb, int TB, const T *__restrict__ G,
                                   const T *__restrict__ b, T *__restrict__ R) {
    extern __shared__ unsigned char smraw[];
    T *sG = reinterpret_cast<T *>(smraw);  // [TB][na][n]
    const int mR = na + mb, gsz = na * n, rsz = n * mR;
    for (int64_t t0 = (int64_t)blockIdx.x * TB; t0 < nblk; t0 += (int64_t)gridDim.x * TB) {
        const int tb = (int)(nblk - t0 < TB ? nblk - t0 : TB);
        __syncthreads();
        for (int q = threadIdx.x; q < tb * gsz; q += blockDim.x) sG[q] = G[t0 * gsz + q];
        __syncthreads();
        for (int q = threadIdx.x; q < tb * rsz; q += blockDim.x) {
            const int bi = q / rsz, w = q % rsz, r = w / mR, c = w % mR;
            R[t0 * rsz + q] = c < na ? sG[bi * gsz + c * n + r] : b[((t0 + bi) * n + r) * mb + (c - na)];
        }
    }
}

// One CTA per system: S = Z - sum_i G_i V_i, t = b_a - sum_i G_i u_i with Y_i = [V_i | u_i];
// L_Z = chol(S) (right-looking, in shared memory); x_a = L_Z^{-T} L_Z^{-1} t.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_arrow_schur(int N, int n, int na, int mb, int IB, const T *__restrict__ G,
                                                          const T *__restrict__ Z, const T *__restrict__ ba,
                                                          const T *__restrict__ Y, T *__restrict__ LZ,
                                                          T *__restrict__ xa, int32_t *__restrict__ info) {
    extern __shared__ unsigned char smraw[];
    T *S = reinterpret_cast<T *>(smraw);  // [na][mR]
    __shared__ int fail;
    const int mR = na + mb;
    const int64_t j = blockIdx.x;
    const T *Gj = G + j * (int64_t)N * na * n;
    const T *Yj = Y + j * (int64_t)N * n * mR;
    // sum over the N n border rows, split over `groups` thread groups when the outputs do not fill
    // the CTA; the partial sums are combined in group order (deterministic)
    const int O = na * mR;
    const int groups = O >= (int)blockDim.x ? 1 : (int)blockDim.x / O;
    T *part = S + O;  // [groups][O] when groups > 1
    if (IB > 0) {
        // staged: chunks of IB blocks of G and Y copied to shared memory with coalesced loads
        T *sG = part + blockDim.x, *sY = sG + (size_t)IB * na * n;
        const int t = threadIdx.x;
        const int g = groups > 1 ? t / O : 0;
        T acc[4] = {0, 0, 0, 0};  // groups == 1: up to 4 outputs per thread (O <= 4 * blockDim)
        for (int i0 = 0; i0 < N; i0 += IB) {
            const int ib = N - i0 < IB ? N - i0 : IB;
            __syncthreads();
            for (int q = t; q < ib * na * n; q += blockDim.x) sG[q] = Gj[(int64_t)i0 * na * n + q];
            for (int q = t; q < ib * n * mR; q += blockDim.x) sY[q] = Yj[(int64_t)i0 * n * mR + q];
            __syncthreads();
            for (int u = 0; u < 4; ++u) {
                const int o = groups > 1 ? t % O : u * blockDim.x + t;
                if (g >= groups || o >= O || (groups > 1 && u > 0)) break;
                const int a = o / mR, c = o % mR;
                T v = acc[u];
                for (int bi = (groups > 1 ? (g - i0 % groups + groups) % groups : 0); bi < ib;
                     bi += (groups > 1 ? groups : 1)) {
                    const T *Gi = sG + (size_t)bi * na * n + (size_t)a * n;
                    const T *Yi = sY + (size_t)bi * n * mR + c;
                    for (int r = 0; r < n; ++r) v = fma(Gi[r], Yi[r * mR], v);
                }
                acc[u] = v;
            }
        }
        for (int u = 0; u < 4; ++u) {
            const int o = groups > 1 ? t % O : u * blockDim.x + t;
            if (g >= groups || o >= O || (groups > 1 && u > 0)) break;
            if (groups > 1) part[g * O + o] = acc[u];
            else S[o] = acc[u];
        }
    } else {
    for (int o0 = 0; o0 < O; o0 += blockDim.x) {
        const int t = threadIdx.x;
        const int g = groups > 1 ? t / O : 0, o = groups > 1 ? t % O : o0 + t;
        if (g < groups && o < O) {
            const int a = o / mR, c = o % mR;
            T acc = 0;
            for (int i = g; i < N; i += groups) {
                const T *Gi = Gj + (int64_t)i * na * n + (int64_t)a * n;
                const T *Yi = Yj + (int64_t)i * n * mR + c;
                for (int r = 0; r < n; ++r) acc = fma(Gi[r], Yi[(int64_t)r * mR], acc);
            }
            if (groups > 1) part[g * O + o] = acc;
            else S[o] = acc;
        }
        if (groups > 1) break;
    }
    }
    if (groups > 1) {
        __syncthreads();
        for (int o = threadIdx.x; o < O; o += blockDim.x) {
            T acc = 0;
            for (int g = 0; g < groups; ++g) acc += part[g * O + o];
            S[o] = acc;
        }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < O; o += blockDim.x) {
        const int a = o / mR, c = o % mR;
        T base;
        if (c < na) {
            const int hi = a >= c ? a : c, lo = a >= c ? c : a;  // Z lower-authoritative
            base = Z[j * na * na + (int64_t)hi * na + lo];
        } else {
            base = ba[(j * na + a) * mb + (c - na)];
        }
        S[o] = base - S[o];
    }
    if (threadIdx.x == 0) fail = 0;
    __syncthreads();
    for (int k = 0; k < na; ++k) {
        const T piv = S[k * mR + k];
        if (!(piv > T(0))) {  // NaN or <= 0
            if (threadIdx.x == 0) fail = 1;
            break;
        }
        const T dk = sqrt(piv);
        __syncthreads();
        for (int i = k + 1 + threadIdx.x; i < na; i += blockDim.x) S[i * mR + k] /= dk;
        if (threadIdx.x == 0) S[k * mR + k] = dk;
        __syncthreads();
        const int rem = na - k - 1;
        for (int o = threadIdx.x; o < rem * rem; o += blockDim.x) {
            const int i = k + 1 + o / rem, l = k + 1 + o % rem;
            if (l <= i) S[i * mR + l] -= S[i * mR + k] * S[l * mR + k];
        }
        __syncthreads();
    }
    __syncthreads();
    if (fail) {
        if (threadIdx.x == 0 && info[j] == 0) info[j] = N + 1;  // the border is pivot block N+1
        return;
    }
    for (int o = threadIdx.x; o < na * na; o += blockDim.x) {
        const int a = o / na, c = o % na;
        LZ[j * na * na + o] = c <= a ? S[a * mR + c] : T(0);
    }
    // forward then backward substitution, one thread per right-hand side column
    for (int c = threadIdx.x; c < mb; c += blockDim.x) {
        T *t = S + na + c;  // column c of the rhs part, stride mR
        for (int a = 0; a < na; ++a) {
            T v = t[a * mR];
            for (int k = 0; k < a; ++k) v -= S[a * mR + k] * t[k * mR];
            t[a * mR] = v / S[a * mR + a];
        }
        for (int a = na - 1; a >= 0; --a) {
            T v = t[a * mR];
            for (int k = a + 1; k < na; ++k) v -= S[k * mR + a] * t[k * mR];
            t[a * mR] = v / S[a * mR + a];
        }
        for (int a = 0; a < na; ++a) xa[(j * na + a) * mb + c] = t[a * mR];
    }
}

// x_i = u_i - V_i x_a
template <typename T>
__global__ void k_arrow_update(int B, int N, int n, int na, int mb, const T *__restrict__ Y, const T *__restrict__ xa,
                               T *__restrict__ x) {
    const int mR = na + mb;
    const int64_t total = (int64_t)B * N * n * mb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int c = (int)(e % mb);
        const int64_t t = e / mb;  // (j, i, r)
        const int64_t j = t / ((int64_t)N * n);
        const T *Yr = Y + t * mR;
        T v = Yr[na + c];
        for (int a = 0; a < na; ++a) v = fma(-Yr[a], xa[(j * na + a) * mb + c], v);
        x[e] = v;
    }
}

// ------------------------------------------------------------------------- f4c: block banded

// Super-block tridiagonal (D', E', b') of a block-banded system: super-block I holds blocks
// I w .. I w + w - 1 (0-based); padding blocks (index >= N) are identity / zero.
template <typename T>
__global__ void k_band_pack(int B, int N, int n, int w, int m, int Np, const T *__restrict__ D,
                            const T *__restrict__ A, const T *__restrict__ b, T *__restrict__ Dp, T *__restrict__ Ep,
                            T *__restrict__ bp) {
    const int s = w * n;
    const int64_t nD = (int64_t)B * Np * s * s, nE = (int64_t)B * (Np - 1) * s * s, nb = (int64_t)B * Np * s * m;
    const int64_t nn = (int64_t)n * n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto Ablk = [&](int64_t j, int k, int col, int r, int cc) -> T {  // block (col + k, col), k = 1..w
        return A[(((j * w + (k - 1)) * N + col) * nn) + (int64_t)r * n + cc];
    };
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nD + nE + nb; e += stride) {
        if (e < nD) {
            const int Cc = (int)(e % s), R = (int)((e / s) % s);
            const int64_t JI = e / ((int64_t)s * s);
            const int I = (int)(JI % Np);
            const int64_t j = JI / Np;
            const int pr = R / n, r = R % n, pc = Cc / n, cc = Cc % n;
            const int br = I * w + pr, bc = I * w + pc;
            T v;
            if (br >= N || bc >= N) v = R == Cc ? T(1) : T(0);
            else if (pr == pc) v = r >= cc ? D[(j * N + br) * nn + (int64_t)r * n + cc] : T(0);
            else if (pr > pc) v = Ablk(j, pr - pc, bc, r, cc);
            else v = Ablk(j, pc - pr, br, cc, r);
            Dp[e] = v;
        } else if (e < nD + nE) {
            const int64_t f = e - nD;
            const int Cc = (int)(f % s), R = (int)((f / s) % s);
            const int64_t JI = f / ((int64_t)s * s);
            const int I = (int)(JI % (Np - 1));
            const int64_t j = JI / (Np - 1);
            const int pr = R / n, r = R % n, pc = Cc / n, cc = Cc % n;
            const int br = (I + 1) * w + pr, bc = I * w + pc;
            const int dist = br - bc;
            Ep[f] = (br < N && dist <= w) ? Ablk(j, dist, bc, r, cc) : T(0);
        } else {
            const int64_t f = e - nD - nE;
            const int c = (int)(f % m);
            const int R = (int)((f / m) % s);
            const int64_t JI = f / ((int64_t)m * s);
            const int I = (int)(JI % Np);
            const int64_t j = JI / Np;
            const int bi = I * w + R / n;
            bp[f] = bi < N ? b[((j * N + bi) * n + R % n) * m + c] : T(0);
        }
    }
}

// x[j] = the first N n m entries of x'[j] (same element order inside a system).
template <typename T>
__global__ void k_band_unpack(int B, int64_t per, int64_t perp, const T *__restrict__ xp, T *__restrict__ x) {
    const int64_t total = (int64_t)B * per;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride)
        x[e] = xp[(e / per) * perp + e % per];
}

// ------------------------------------------------------------------------- f3: partition

// R[i][r][c]: [B_k at block 0 | F_k^T at block N_k - 1 | b_k], column widths nb, nf, m.
template <typename T>
__global__ void k_part_pack(int Nk, int n, int m, int nb, int nf, const T *__restrict__ Bk, const T *__restrict__ Fk,
                            const T *__restrict__ b, T *__restrict__ R) {
    const int mR = nb + nf + m;
    const int64_t total = (int64_t)Nk * n * mR;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int c = (int)(e % mR);
        const int64_t t = e / mR;
        const int r = (int)(t % n);
        const int i = (int)(t / n);
        T v;
        if (c < nb) v = i == 0 ? Bk[r * n + c] : T(0);
        else if (c < nb + nf) v = i == Nk - 1 ? Fk[(c - nb) * n + r] : T(0);
        else v = b[t * m + (c - nb - nf)];
        R[e] = v;
    }
}

// Packet of chunk k (3 n^2 + 2 n m entries; absent terms are zero):
//   [0] SB = A_k - B_k^T Y_0[:, B]        [1] SF = F_k Y_last[:, F]     [2] H = -F_k Y_last[:, B]
//   [3] tB = a_k - B_k^T Y_0[:, b]        [4] tF = F_k Y_last[:, b]
template <typename T>
__global__ void k_part_contrib(int Nk, int n, int m, int nb, int nf, const T *__restrict__ Bk,
                               const T *__restrict__ Fk, const T *__restrict__ Ak, const T *__restrict__ ak,
                               const T *__restrict__ Y, T *__restrict__ P) {
    const int mR = nb + nf + m;
    const int nn = n * n;
    const int total = 3 * nn + 2 * n * m;
    const T *Y0 = Y;                                  // block 0 rows
    const T *YL = Y + (int64_t)(Nk - 1) * n * mR;     // last block rows
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        T v = 0;
        if (o < nn) {  // SB
            if (nb) {
                const int a = o / n, c = o % n;
                const int hi = a >= c ? a : c, lo = a >= c ? c : a;
                T acc = 0;
                for (int r = 0; r < n; ++r) acc = fma(Bk[r * n + a], Y0[(int64_t)r * mR + c], acc);
                v = Ak[hi * n + lo] - acc;
            }
        } else if (o < 2 * nn) {  // SF
            if (nf) {
                const int a = (o - nn) / n, c = (o - nn) % n;
                T acc = 0;
                for (int r = 0; r < n; ++r) acc = fma(Fk[a * n + r], YL[(int64_t)r * mR + nb + c], acc);
                v = acc;
            }
        } else if (o < 3 * nn) {  // H
            if (nb && nf) {
                const int a = (o - 2 * nn) / n, c = (o - 2 * nn) % n;
                T acc = 0;
                for (int r = 0; r < n; ++r) acc = fma(Fk[a * n + r], YL[(int64_t)r * mR + c], acc);
                v = -acc;
            }
        } else if (o < 3 * nn + n * m) {  // tB
            if (nb) {
                const int q = o - 3 * nn, a = q / m, c = q % m;
                T acc = 0;
                for (int r = 0; r < n; ++r) acc = fma(Bk[r * n + a], Y0[(int64_t)r * mR + nb + nf + c], acc);
                v = ak[a * m + c] - acc;
            }
        } else {  // tF
            if (nf) {
                const int q = o - 3 * nn - n * m, a = q / m, c = q % m;
                T acc = 0;
                for (int r = 0; r < n; ++r) acc = fma(Fk[a * n + r], YL[(int64_t)r * mR + nb + nf + c], acc);
                v = acc;
            }
        }
        P[o] = v;
    }
}

// Pivot system (p - 1 blocks, block tridiagonal) from the p packets:
//   DS[q] = SB(q+2) - SF(q+1),  ES[q] = H(q+2),  bS[q] = tB(q+2) - tF(q+1)    (chunks 1-based)
template <typename T>
__global__ void k_part_assemble(int p, int n, int m, const T *__restrict__ P, T *__restrict__ DS, T *__restrict__ ES,
                                T *__restrict__ bS) {
    const int nn = n * n, ps = 3 * nn + 2 * n * m;
    const int q1 = p - 1;
    const int64_t nD = (int64_t)q1 * nn, nE = (int64_t)(q1 - 1) * nn, nb = (int64_t)q1 * n * m;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nD + nE + nb; e += stride) {
        if (e < nD) {
            const int q = (int)(e / nn), o = (int)(e % nn);
            DS[e] = P[(int64_t)(q + 1) * ps + o] - P[(int64_t)q * ps + nn + o];
        } else if (e < nD + nE) {
            const int64_t f = e - nD;
            const int q = (int)(f / nn), o = (int)(f % nn);
            ES[f] = P[(int64_t)(q + 1) * ps + 2 * nn + o];
        } else {
            const int64_t f = e - nD - nE;
            const int q = (int)(f / (n * m)), o = (int)(f % (n * m));
            bS[f] = P[(int64_t)(q + 1) * ps + 3 * nn + o] - P[(int64_t)q * ps + 3 * nn + n * m + o];
        }
    }
}

// x_i = Y_i[:, b] - Y_i[:, B] xL - Y_i[:, F] xR
template <typename T>
__global__ void k_part_finish(int Nk, int n, int m, int nb, int nf, const T *__restrict__ Y, const T *__restrict__ xL,
                              const T *__restrict__ xR, T *__restrict__ x) {
    const int mR = nb + nf + m;
    const int64_t total = (int64_t)Nk * n * m;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int c = (int)(e % m);
        const int64_t t = e / m;
        const T *Yr = Y + t * mR;
        T v = Yr[nb + nf + c];
        for (int a = 0; a < nb; ++a) v = fma(-Yr[a], xL[a * m + c], v);
        for (int a = 0; a < nf; ++a) v = fma(-Yr[nb + a], xR[a * m + c], v);
        x[e] = v;
    }
}

}  // namespace

// ------------------------------------------------------------------------- C ABI
// (C linkage comes from the declarations in include/btd.h.)

btd_status btd_mixed_workspace_bytes(const btd_plan *p, size_t *bytes) {
    if (!p || !bytes || p->dtype != BTD_F32) return BTD_EINVAL;
    *bytes = mixed_layout(p, nullptr, nullptr);
    return BTD_OK;
}

// The refinement loop shared by btd_mixed_factor_solve and btd_mixed_solve: on entry w.d32 holds
// x_0 = solve32(fl32(b)); x_j for j = 0..iters alternates buffers so that x_iters lands in x.
static btd_status mixed_refine(const btd_plan *p, const double *D, const double *E, const double *b,
                               const float *Dhat, const float *C, double *x, int32_t iters, double *resid,
                               const MixedWs &w, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int B = (int)p->batch, N = (int)p->N, n = (int)p->n, m = (int)p->m;
    const int64_t nx = (int64_t)B * N * n * m;
    auto xbuf = [&](int j) { return ((iters - j) % 2 == 0) ? x : w.xtmp; };
    const int g = grid_for(nx);
    for (int k = 0; k <= iters; ++k) {
        const double *xp = k == 0 ? nullptr : xbuf(k - 1);
        double *xn = xbuf(k);
        const bool last = k == iters;
        if (!last) {
            if (k == 0)
                k_ir_step<false, true, false><<<g, kThreads, 0, st>>>(B, N, n, m, D, E, b, xp, w.d32, xn, w.r32, nullptr);
            else
                k_ir_step<true, true, false><<<g, kThreads, 0, st>>>(B, N, n, m, D, E, b, xp, w.d32, xn, w.r32, nullptr);
            if (btd_status rs = launched(); rs != BTD_OK) return rs;
            if (btd_status rs = btd_solve(p, Dhat, C, w.r32, w.d32, stream); rs != BTD_OK) return rs;
        } else if (resid) {
            cudaError_t e = cudaMemsetAsync(w.nrm, 0, 2 * (size_t)B * sizeof(double), st);
            if (e != cudaSuccess) return record_cuda_error(e);
            if (k == 0)
                k_ir_step<false, false, true><<<g, kThreads, 0, st>>>(B, N, n, m, D, E, b, xp, w.d32, xn, nullptr, w.nrm);
            else
                k_ir_step<true, false, true><<<g, kThreads, 0, st>>>(B, N, n, m, D, E, b, xp, w.d32, xn, nullptr, w.nrm);
            k_ir_finish<<<(B + 127) / 128, 128, 0, st>>>(B, w.nrm, resid);
        } else {
            if (k == 0)
                k_ir_step<false, false, false><<<g, kThreads, 0, st>>>(B, N, n, m, D, E, b, xp, w.d32, xn, nullptr, nullptr);
            else
                k_ir_step<true, false, false><<<g, kThreads, 0, st>>>(B, N, n, m, D, E, b, xp, w.d32, xn, nullptr, nullptr);
        }
    }
    return launched();
}

btd_status btd_mixed_factor_solve(const btd_plan *p, const double *D, const double *E, const double *b,
                                  float *Dhat, float *C, double *x, int32_t *info, int32_t iters, double *resid,
                                  void *work, void *stream) {
    if (!p || p->dtype != BTD_F32 || !D || !b || !Dhat || (!C && p->geo.nC > 0) || !x || !info || !work ||
        iters < 0 || (p->N > 1 && !E))
        return BTD_EINVAL;
    if (!al16(D) || !al16(E) || !al16(b) || !al16(x) || !al16(work)) return BTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    MixedWs w;
    mixed_layout(p, (char *)work, &w);
    const int B = (int)p->batch, N = (int)p->N, n = (int)p->n, m = (int)p->m;
    const int64_t nn = (int64_t)n * n, nx = (int64_t)B * N * n * m;
    k_demote<<<grid_for((int64_t)B * N * nn / 2), kThreads, 0, st>>>(D, w.D32, (int64_t)B * N * nn);
    if (N > 1) k_demote<<<grid_for((int64_t)B * (N - 1) * nn / 2), kThreads, 0, st>>>(E, w.E32, (int64_t)B * (N - 1) * nn);
    k_demote<<<grid_for(nx / 2), kThreads, 0, st>>>(b, w.r32, nx);
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    // x_0 = solve32(fl32(b)), then iters x (x_k = x_{k-1} + d_k, r = b - Psi x_k, d = solve32(r)).
    if (btd_status rs = btd_factor_solve(p, w.D32, N > 1 ? w.E32 : nullptr, w.r32, Dhat, C, w.d32, info, stream);
        rs != BTD_OK)
        return rs;
    return mixed_refine(p, D, E, b, Dhat, C, x, iters, resid, w, stream);
}

btd_status btd_mixed_solve(const btd_plan *p, const double *D, const double *E, const double *b, const float *Dhat,
                           const float *C, double *x, int32_t iters, double *resid, void *work, void *stream) {
    if (!p || p->dtype != BTD_F32 || !D || !b || !Dhat || (!C && p->geo.nC > 0) || !x || !work || iters < 0 ||
        (p->N > 1 && !E))
        return BTD_EINVAL;
    if (!al16(D) || !al16(E) || !al16(b) || !al16(x) || !al16(work) || !al16(Dhat) || !al16(C)) return BTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    MixedWs w;
    mixed_layout(p, (char *)work, &w);
    const int64_t nx = (int64_t)p->batch * p->N * p->n * p->m;
    k_demote<<<grid_for(nx / 2), kThreads, 0, st>>>(b, w.r32, nx);
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    if (btd_status rs = btd_solve(p, Dhat, C, w.r32, w.d32, stream); rs != BTD_OK) return rs;
    return mixed_refine(p, D, E, b, Dhat, C, x, iters, resid, w, stream);
}

template <typename T>
static btd_status arrow_impl(const btd_plan *p, int64_t na, const void *D, const void *E, const void *G,
                             const void *Z, const void *b, const void *ba, void *Dhat, void *C, void *R, void *Y,
                             void *LZ, void *x, void *xa, int32_t *info, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int B = (int)p->batch, N = (int)p->N, n = (int)p->n, mb = (int)(p->m - na);
    const int64_t nR = (int64_t)B * N * n * p->m;
    const size_t gblk = (size_t)na * n * sizeof(T);
    if (gblk <= 16384) {
        const int TB = (int)(49152 / gblk) < 64 ? (int)(49152 / gblk) : 64;
        const int64_t nblk = (int64_t)B * N;
        int64_t grid = (nblk + TB - 1) / TB;
        if (grid > 148 * 8) grid = 148 * 8;
        k_arrow_pack_tiled<T><<<(int)grid, kThreads, TB * gblk, st>>>(nblk, n, (int)na, mb, TB, (const T *)G,
                                                                      (const T *)b, (T *)R);
    } else {
        k_arrow_pack<T><<<grid_for(nR), kThreads, 0, st>>>(B, N, n, (int)na, mb, (const T *)G, (const T *)b, (T *)R);
    }
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    // factor, then one solve with the na + mb right-hand sides: with many right-hand sides the
    // batched fused factor+solve holds all of them in shared memory for the whole factorization
    // (1 CTA/SM at c5 size, m = 9: 10.3 ms) while the separate calls keep the factor at full
    // occupancy (c5, m = 9: 1.6 + 4.4 ms; measured in profiles/r02/arrow_exp.txt)
    if (btd_status rs = btd_factor(p, D, E, Dhat, C, info, stream); rs != BTD_OK) return rs;
    if (btd_status rs = btd_solve(p, Dhat, C, R, Y, stream); rs != BTD_OK) return rs;
    // S + group partial sums, then IB staged blocks of G and Y when 4 * 256 threads cover the outputs
    const size_t base = ((size_t)na * p->m + kThreads) * sizeof(T);
    const size_t perb = ((size_t)na * n + (size_t)n * p->m) * sizeof(T);
    int IB = (na * p->m <= 4 * kThreads && base + perb <= 96 * 1024) ? (int)((96 * 1024 - base) / perb) : 0;
    if (IB > 32) IB = 32;
    const size_t smem = base + (size_t)IB * perb;
    if (btd_status rs = btd::ensure_smem_attr((const void *)k_arrow_schur<T>, smem); rs != BTD_OK) return rs;
    k_arrow_schur<T><<<B, kThreads, smem, st>>>(N, n, (int)na, mb, IB, (const T *)G, (const T *)Z, (const T *)ba,
                                                 (const T *)Y, (T *)LZ, (T *)xa, info);
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    k_arrow_update<T><<<grid_for((int64_t)B * N * n * mb), kThreads, 0, st>>>(B, N, n, (int)na, mb, (const T *)Y,
                                                                               (const T *)xa, (T *)x);
    return launched();
}

btd_status btd_arrow_factor_solve(const btd_plan *p, int64_t na, const void *D, const void *E, const void *G,
                                  const void *Z, const void *b, const void *ba, void *Dhat, void *C, void *R, void *Y,
                                  void *LZ, void *x, void *xa, int32_t *info, void *stream) {
    if (!p || na < 1 || na >= p->m || !D || !G || !Z || !b || !ba || !Dhat || (!C && p->geo.nC > 0) || !R || !Y ||
        !LZ || !x || !xa || !info || (p->N > 1 && !E))
        return BTD_EINVAL;
    const size_t w = p->dtype == BTD_F32 ? 4 : 8;
    if (((size_t)na * p->m + kThreads) * w > btd::kMaxSmem) return BTD_EUNSUPPORTED;
    if (!al16(D) || !al16(E) || !al16(R) || !al16(Y) || !al16(Dhat) || !al16(C)) return BTD_EINVAL;
    if (p->dtype == BTD_F32) return arrow_impl<float>(p, na, D, E, G, Z, b, ba, Dhat, C, R, Y, LZ, x, xa, info, stream);
    return arrow_impl<double>(p, na, D, E, G, Z, b, ba, Dhat, C, R, Y, LZ, x, xa, info, stream);
}

template <typename T>
static btd_status banded_impl(const btd_plan *p, int64_t N, int64_t n, int64_t w, const void *D, const void *A,
                              const void *b, void *Dp, void *Ep, void *bp, void *Dhat, void *C, void *xp, void *x,
                              int32_t *info, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int B = (int)p->batch, Np = (int)p->N, m = (int)p->m;
    const int64_t s = w * n;
    const int64_t work = (int64_t)B * Np * s * s + (int64_t)B * (Np - 1) * s * s + (int64_t)B * Np * s * m;
    k_band_pack<T><<<grid_for(work), kThreads, 0, st>>>(B, (int)N, (int)n, (int)w, m, Np, (const T *)D, (const T *)A,
                                                        (const T *)b, (T *)Dp, (T *)Ep, (T *)bp);
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    if (btd_status rs = btd_factor_solve(p, Dp, Np > 1 ? Ep : nullptr, bp, Dhat, C, xp, info, stream); rs != BTD_OK)
        return rs;
    const int64_t per = N * n * m, perp = (int64_t)Np * s * m;
    k_band_unpack<T><<<grid_for(B * per), kThreads, 0, st>>>(B, per, perp, (const T *)xp, (T *)x);
    return launched();
}

btd_status btd_banded_factor_solve(const btd_plan *p, int64_t N, int64_t n, int64_t w, const void *D, const void *A,
                                   const void *b, void *Dp, void *Ep, void *bp, void *Dhat, void *C, void *xp,
                                   void *x, int32_t *info, void *stream) {
    if (!p || N < 1 || n < 1 || w < 1 || !D || (!A && N > 1) || !b || !Dp || !bp || !Dhat || !xp || !x || !info)
        return BTD_EINVAL;
    if (p->n != w * n || p->N != (N + w - 1) / w) return BTD_EINVAL;
    if (p->N > 1 && (!Ep || (!C && p->geo.nC > 0))) return BTD_EINVAL;
    if (!al16(Dp) || !al16(Ep) || !al16(bp) || !al16(xp) || !al16(Dhat) || !al16(C)) return BTD_EINVAL;
    if (p->dtype == BTD_F32) return banded_impl<float>(p, N, n, w, D, A, b, Dp, Ep, bp, Dhat, C, xp, x, info, stream);
    return banded_impl<double>(p, N, n, w, D, A, b, Dp, Ep, bp, Dhat, C, xp, x, info, stream);
}

template <typename T>
static btd_status part_local_impl(const btd_plan *p, const void *D, const void *E, const void *Bk, const void *Fk,
                                  const void *Ak, const void *ak, const void *b, void *R, void *Dhat, void *C,
                                  void *Y, void *packet, int32_t *info, int nb, int nf, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int Nk = (int)p->N, n = (int)p->n, m = (int)p->m - nb - nf;
    k_part_pack<T><<<grid_for((int64_t)Nk * n * p->m), kThreads, 0, st>>>(Nk, n, m, nb, nf, (const T *)Bk,
                                                                          (const T *)Fk, (const T *)b, (T *)R);
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    if (btd_status rs = btd_factor_solve(p, D, Nk > 1 ? E : nullptr, R, Dhat, C, Y, info, stream); rs != BTD_OK)
        return rs;
    const int total = 3 * n * n + 2 * n * m;
    k_part_contrib<T><<<(total + kThreads - 1) / kThreads, kThreads, 0, st>>>(
        Nk, n, m, nb, nf, (const T *)Bk, (const T *)Fk, (const T *)Ak, (const T *)ak, (const T *)Y, (T *)packet);
    return launched();
}

btd_status btd_partition_local(const btd_plan *p, const void *D, const void *E, const void *Bk, const void *Fk,
                               const void *Ak, const void *ak, const void *b, void *R, void *Dhat, void *C, void *Y,
                               void *packet, int32_t *info, void *stream) {
    if (!p || p->batch != 1 || !D || !b || !R || !Dhat || (!C && p->geo.nC > 0) || !Y || !packet || !info ||
        (p->N > 1 && !E))
        return BTD_EINVAL;
    if ((Bk == nullptr) != (Ak == nullptr) || (Bk == nullptr) != (ak == nullptr)) return BTD_EINVAL;
    const int nb = Bk ? (int)p->n : 0, nf = Fk ? (int)p->n : 0;
    if (p->m - nb - nf < 1) return BTD_EINVAL;
    if (!al16(D) || !al16(E) || !al16(R) || !al16(Y) || !al16(Dhat) || !al16(C)) return BTD_EINVAL;
    if (p->dtype == BTD_F32)
        return part_local_impl<float>(p, D, E, Bk, Fk, Ak, ak, b, R, Dhat, C, Y, packet, info, nb, nf, stream);
    return part_local_impl<double>(p, D, E, Bk, Fk, Ak, ak, b, R, Dhat, C, Y, packet, info, nb, nf, stream);
}

btd_status btd_partition_reduce(const btd_plan *ps, int32_t p, const void *packets, void *DS, void *ES, void *bS,
                                void *DhatS, void *CS, void *xS, int32_t *infoS, void *stream) {
    if (!ps || p < 2 || ps->N != p - 1 || ps->batch != 1 || !packets || !DS || !bS || !DhatS || !xS || !infoS)
        return BTD_EINVAL;
    if (p > 2 && (!ES || !CS)) return BTD_EINVAL;
    if (!al16(DS) || !al16(ES) || !al16(bS) || !al16(DhatS) || !al16(CS) || !al16(xS)) return BTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int n = (int)ps->n, m = (int)ps->m;
    const int64_t work = (int64_t)(2 * (p - 1) - 1) * n * n + (int64_t)(p - 1) * n * m;
    if (ps->dtype == BTD_F32)
        k_part_assemble<float><<<grid_for(work), kThreads, 0, st>>>(p, n, m, (const float *)packets, (float *)DS,
                                                                    (float *)ES, (float *)bS);
    else
        k_part_assemble<double><<<grid_for(work), kThreads, 0, st>>>(p, n, m, (const double *)packets, (double *)DS,
                                                                     (double *)ES, (double *)bS);
    if (btd_status rs = launched(); rs != BTD_OK) return rs;
    return btd_factor_solve(ps, DS, p > 2 ? ES : nullptr, bS, DhatS, CS, xS, infoS, stream);
}

btd_status btd_partition_finish(const btd_plan *p, const void *Y, const void *xL, const void *xR, void *x,
                                void *stream) {
    if (!p || p->batch != 1 || !Y || !x) return BTD_EINVAL;
    const int nb = xL ? (int)p->n : 0, nf = xR ? (int)p->n : 0;
    const int m = (int)p->m - nb - nf;
    if (m < 1) return BTD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int Nk = (int)p->N, n = (int)p->n;
    if (p->dtype == BTD_F32)
        k_part_finish<float><<<grid_for((int64_t)Nk * n * m), kThreads, 0, st>>>(
            Nk, n, m, nb, nf, (const float *)Y, (const float *)xL, (const float *)xR, (float *)x);
    else
        k_part_finish<double><<<grid_for((int64_t)Nk * n * m), kThreads, 0, st>>>(
            Nk, n, m, nb, nf, (const double *)Y, (const double *)xL, (const double *)xR, (double *)x);
    return launched();
}
