// k_tpu.cu -- "threads per H-unit" detector for small per-subcarrier channels
// (C1 2x2 QPSK, C2 4x4 16-QAM; any even NR <= 4, NL <= NR).
//
// Mapping (DESIGN.md §"Kernels"): a CTA owns TU consecutive subcarriers of one
// slot (TU H-units, 14 x TU REs) and G warps-worth of threads. Thread (g, u)
// serves unit u; the G threads of a unit split its work either by layer
// (LAYER_SPLIT: thread g owns W~ rows [g NL/G, (g+1) NL/G) for all 14 symbols)
// or by symbol (thread g owns all layers of symbols g, g+G, ...).
//   1. thread 0 issues 14 cp.async.bulk copies (one per OFDM symbol row, TU*NR*8
//      contiguous bytes) of the CTA's y tile into shared memory, each completing
//      on its own mbarrier -- the whole tile is in flight at once with no
//      register cost;
//   2. meanwhile every thread loads its unit's H (256-bit loads) and runs rows
//      a2-a5 fully unrolled in registers, in fp64 by default (reading R18: an
//      fp32 setup misses the 1e-4 x~ bound on square 4x4 channels, SURVEY.md
//      §8(c)); W~ rows (in PAM level units) and LLR slopes are rounded once to
//      fp32; with LAYER_SPLIT each thread forms only its own rows of
//      G^-1 and W~;
//   3. per symbol it waits on that row's mbarrier, reads y from shared memory,
//      forms its x~ = W~ y (row a6), demaps exactly (row a7) and writes its
//      LLRs with 256-bit stores (whole 32-byte sectors).
// The 14 REs of a unit reuse W~ held in registers.
#include <type_traits>

#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;

template <typename T>
struct Cx {
    T x, y;
};
template <typename T>
__device__ __forceinline__ Cx<T> cx(T x, T y) {
    return Cx<T>{x, y};
}
template <typename T>  // acc + a*b
__device__ __forceinline__ Cx<T> mac(Cx<T> acc, Cx<T> a, Cx<T> b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}
template <typename T>  // acc + conj(a)*b
__device__ __forceinline__ Cx<T> macc(Cx<T> acc, Cx<T> a, Cx<T> b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
    return acc;
}
template <typename T>  // acc + a*conj(b)
__device__ __forceinline__ Cx<T> macb(Cx<T> acc, Cx<T> a, Cx<T> b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.y, b.x, acc.y);
    acc.y = fma(-a.x, b.y, acc.y);
    return acc;
}
template <typename T>  // acc - a*conj(b)
__device__ __forceinline__ Cx<T> msubc(Cx<T> acc, Cx<T> a, Cx<T> b) {
    acc.x = fma(-a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(-a.y, b.x, acc.y);
    acc.y = fma(a.x, b.y, acc.y);
    return acc;
}
__device__ __forceinline__ double rsq(double v) { return rsqrt(v); }
__device__ __forceinline__ float rsq(float v) { return rsqrtf(v); }

template <int NR, int NL>
struct SetupOut {
    float2 w[NL][NR];  // W~ * sqrt(norm), fp32
    float slope[NL];   // SINR * llr_scale / norm
    float sinr[NL];
    bool fail;
};

// Rows a2-a5 in registers, scalar type T (double by default), fully unrolled:
//   a2 G = H^H H + s2 I;  a3 G = L L^H (left-looking, guard R17);
//   a4 X = L^-1;  B = X H^H;  W = X^H B = G^-1 H^H;  A_kk = sum_i |X_ik|^2;
//   a5 mu_k = 1 - s2 A_kk, SINR_k = mu_k / (s2 A_kk), W~_k = W_k sqrt(norm) / mu_k.
template <typename T, int NR, int NL>
__device__ __forceinline__ void setup_unit(const float2 (&hf)[NR][NL], float sigma2, float norm, float llr_scale,
                                           SetupOut<NR, NL>& o) {
    const float sqn = sqrtf(norm);
    {
        const T s2 = (T)sigma2;
        Cx<T> h[NR][NL];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int l = 0; l < NL; ++l) h[r][l] = cx<T>((T)hf[r][l].x, (T)hf[r][l].y);

        // a2: Gram (lower triangle) into L
        Cx<T> L[NL][NL];
        T gmax = 0;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
#pragma unroll
            for (int j = 0; j < i; ++j) {
                Cx<T> acc = cx<T>(0, 0);
#pragma unroll
                for (int r = 0; r < NR; ++r) acc = macc(acc, h[r][i], h[r][j]);
                L[i][j] = acc;
            }
            T d = s2;
#pragma unroll
            for (int r = 0; r < NR; ++r) d = fma(h[r][i].x, h[r][i].x, fma(h[r][i].y, h[r][i].y, d));
            L[i][i] = cx<T>(d, 0);
            gmax = gmax > d ? gmax : d;
        }
        // a3: left-looking Cholesky in place, keep 1/L_jj; guard p_j > tau max G_ii (R17, NaN-safe)
        T dinv[NL];
        bool fail = !(gmax == gmax);
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            T p = L[j][j].x;
#pragma unroll
            for (int k = 0; k < j; ++k) p = fma(-L[j][k].x, L[j][k].x, fma(-L[j][k].y, L[j][k].y, p));
            if (!(p > (T)kPivotTau * gmax)) {
                fail = true;
                p = 1;
            }
            dinv[j] = rsq(p);
#pragma unroll
            for (int i = j + 1; i < NL; ++i) {
                Cx<T> s = L[i][j];
#pragma unroll
                for (int k = 0; k < j; ++k) s = msubc(s, L[i][k], L[j][k]);
                L[i][j] = cx<T>(s.x * dinv[j], s.y * dinv[j]);
            }
        }
        // a4: X = L^-1 (lower): X_jj = 1/L_jj, X_ij = -(1/L_ii) sum_{m=j}^{i-1} L_im X_mj
        Cx<T> X[NL][NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            X[j][j] = cx<T>(dinv[j], 0);
#pragma unroll
            for (int i = j + 1; i < NL; ++i) {
                Cx<T> s = cx<T>(0, 0);
#pragma unroll
                for (int m = j; m < i; ++m) s = mac(s, L[i][m], X[m][j]);
                X[i][j] = cx<T>(-s.x * dinv[i], -s.y * dinv[i]);
            }
        }
        // B = X H^H (NL x NR): B_ir = sum_{m<=i} X_im conj(H_rm)
        Cx<T> B[NL][NR];
#pragma unroll
        for (int i = 0; i < NL; ++i)
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                Cx<T> s = cx<T>(0, 0);
#pragma unroll
                for (int m = 0; m <= i; ++m) s = macb(s, X[i][m], h[r][m]);
                B[i][r] = s;
            }
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            T A = 0;
#pragma unroll
            for (int i = k; i < NL; ++i) A = fma(X[i][k].x, X[i][k].x, fma(X[i][k].y, X[i][k].y, A));
            const T mu = fma(-s2, A, (T)1);  // in T: no cancellation loss
            // a5 in fp32 (readings R3, R4, R11)
            float sinr, f;
            if (sigma2 == 0.f) {
                sinr = __int_as_float(0x7f800000);
                f = sqn;
            } else {
                sinr = (float)mu / (float)(s2 * A);
                f = sqn / (float)mu;
            }
            const bool dead = !(mu > 0) || fail;
            if (dead) {
                sinr = 0.f;
                f = 0.f;
            }
            o.sinr[k] = sinr;
            o.slope[k] = sinr / norm * llr_scale;
            // W_kr = sum_{i>=k} conj(X_ik) B_ir, scaled once to fp32 level units
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                Cx<T> s = cx<T>(0, 0);
#pragma unroll
                for (int i = k; i < NL; ++i) s = macc(s, X[i][k], B[i][r]);
                o.w[k][r] = dead ? make_float2(0.f, 0.f) : make_float2((float)s.x * f, (float)s.y * f);
            }
        }
        o.fail = fail;
    }
}

// y staging modes
constexpr int kYBulk = 0;    // cp.async.bulk per symbol row into smem, one mbarrier per row
constexpr int kYLdg = 1;     // direct 256-bit loads, software-pipelined PF symbols ahead
constexpr int kYAsync = 2;   // per-thread cp.async 16 B into smem, one commit group per symbol

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// wait until at most n groups are pending (n folds to a constant after unrolling)
template <int MAXN>
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
    if constexpr (MAXN > 0) {
        if (n >= MAXN) {
            cp_async_wait<MAXN>();
            return;
        }
        cp_async_wait_dyn<MAXN - 1>(n);
    } else {
        cp_async_wait<0>();
    }
}

template <int NR, int NL, int QM, int LT, bool ZF>
__device__ __forceinline__ void apply_re(const DetectArgs& a, const SetupOut<NR, NL>& o, const float2 (&yv)[NR],
                                         size_t re) {
    constexpr int kLlrBytes = NL * QM * LlrTraits<LT>::bytes;
    constexpr int kWords = (kLlrBytes + 3) / 4;
    float2 x[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc = cmac(acc, o.w[k][r], yv[r]);
        x[k] = acc;
    }
    if (a.llr) {
        float v[NL * QM];
#pragma unroll
        for (int k = 0; k < NL; ++k) demap_layer<QM, ZF, LT>(x[k], o.slope[k], v + k * QM);
        uint32_t w[kWords];
        pack_llr<LT, NL * QM, ZF>(v, w);
        store_bytes<kLlrBytes>((char*)a.llr + re * kLlrBytes, w);
    }
    if (a.xhat) {
        const float ia = rsqrtf((float)qam_norm(QM));
        uint32_t w[2 * NL];
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            w[2 * k] = __float_as_uint(x[k].x * ia);
            w[2 * k + 1] = __float_as_uint(x[k].y * ia);
        }
        store_bytes<NL * 8>(a.xhat + re * NL, w);
    }
}

template <int NR, int NL, int QM, int LT, int TU, int G, int YL, bool ZF, int SPH>
__device__ __forceinline__ void apply_symbols(const DetectArgs& a, const SetupOut<NR, NL>& o, const float2* sy,
                                              uint64_t* bars, int slot, int sc, int ul, int g, bool active,
                                              float2 (*pf)[NR]) {
    constexpr int NS = (SPH + G - 1) / G;  // symbols per thread (upper bound)
    if constexpr (YL == kYBulk) {
#pragma unroll 1
        for (int s = g; s < SPH; s += G) {
            mbar_wait(&bars[s], 0);
            if (!active) continue;
            float2 yv[NR];
            const float2* ys = sy + (s * TU + ul) * NR;
#pragma unroll
            for (int r = 0; r < NR; ++r) yv[r] = ys[r];
            apply_re<NR, NL, QM, LT, ZF>(a, o, yv, (size_t)(slot * SPH + s) * a.n_sc + sc);
        }
    } else if constexpr (YL == kYAsync) {
        if (!active) return;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            const int s = g + i * G;
            if (s < SPH) {
                cp_async_wait_dyn<NS>(NS - 1 - i);
                float2 yv[NR];
                const float2* ys = sy + (s * TU + ul) * NR;
#pragma unroll
                for (int r = 0; r < NR; ++r) yv[r] = ys[r];
                apply_re<NR, NL, QM, LT, ZF>(a, o, yv, (size_t)(slot * SPH + s) * a.n_sc + sc);
            }
        }
    } else {
        if (!active) return;
        constexpr int PF = 2;  // prefetch distance (pf holds PF in-flight symbols)
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            const int s = g + i * G;
            if (s < SPH) {
                float2 yv[NR];
#pragma unroll
                for (int r = 0; r < NR; ++r) yv[r] = pf[i % PF][r];
                const int sn = s + PF * G;
                if (sn < SPH)
                    load_bytes<NR * 8>(a.y + ((size_t)(slot * SPH + sn) * a.n_sc + sc) * NR,
                                       reinterpret_cast<uint32_t*>(&pf[i % PF][0]));
                apply_re<NR, NL, QM, LT, ZF>(a, o, yv, (size_t)(slot * SPH + s) * a.n_sc + sc);
            }
        }
    }
}

// Shared-memory layout: [SPH <= 14 mbarriers | pad to 128 B][y tile SPH x TU x NR float2]
//                       [W~ broadcast: NL*NR float2 x TU][slopes: NL x TU] (SHARE only)
template <int NR, int NL, int TU, int YL, bool SHARE, int SPH>
constexpr int smem_bytes() {
    return 128 + (YL == kYLdg ? 0 : SPH * TU * NR * 8) + (SHARE ? TU * (NL * NR * 8 + NL * 4) : 0);
}

// SHARE: only warp 0 runs the setup and broadcasts W~ / slopes through shared
// memory to the other G-1 warps (no duplicated fp64 work).
template <int NR, int NL, int QM, int LT, int TU, int G, int YL, typename ST, bool SHARE, int SPH>
__global__ void __launch_bounds__(TU* G) k_tpu(DetectArgs a) {
    static_assert(NR % 2 == 0, "16-byte y rows");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    float2* sy = reinterpret_cast<float2*>(smem + 128);
    float2* sW = reinterpret_cast<float2*>(smem + 128 + (YL == kYLdg ? 0 : SPH * TU * NR * 8));
    float* sSlope = reinterpret_cast<float*>(sW + NL * NR * TU);
    constexpr int NS = (SPH + G - 1) / G;

    // PDL: let the next detect call on this stream start its (read-only) prologue now.
    pdl_launch_dependents();

    const int slot = blockIdx.y;
    const int sc0 = blockIdx.x * TU;
    const int nvalid = min(TU, a.n_sc - sc0);
    const int t = threadIdx.x;
    const int ul = t % TU, g = t / TU;
    const bool active = ul < nvalid;
    const int sc = sc0 + ul;
    const size_t unit = (size_t)slot * a.n_sc + sc;
    const bool does_setup = active && (!SHARE || g == 0);

    // a1: H first (it is on the setup's critical path), then the y tile
    float2 hf[NR][NL];
    if (does_setup) load_bytes<NR * NL * 8>(a.H + unit * NR * NL, reinterpret_cast<uint32_t*>(&hf[0][0]));

    float2 pf[2][NR];
    if constexpr (YL == kYBulk) {
        if (t == 0) {
#pragma unroll
            for (int s = 0; s < SPH; ++s) mbar_init(&bars[s], 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (t == 0) {
            const uint32_t row_bytes = (uint32_t)nvalid * NR * 8u;
#pragma unroll 1
            for (int s = 0; s < SPH; ++s) {
                mbar_arrive_expect_tx(&bars[s], row_bytes);
                bulk_g2s(sy + s * TU * NR, a.y + ((size_t)(slot * SPH + s) * a.n_sc + sc0) * NR, row_bytes,
                         &bars[s]);
            }
        }
    } else if constexpr (YL == kYAsync) {
        if (active) {
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                const int s = g + i * G;
                if (s < SPH) {
                    const float2* src = a.y + ((size_t)(slot * SPH + s) * a.n_sc + sc) * NR;
                    float2* dst = sy + (s * TU + ul) * NR;
#pragma unroll
                    for (int c = 0; c < NR / 2; ++c) cp_async16(dst + 2 * c, src + 2 * c);
                }
                cp_async_commit();
            }
        }
    } else {
        if (active) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int s = g + i * G;
                if (s < SPH)
                    load_bytes<NR * 8>(a.y + ((size_t)(slot * SPH + s) * a.n_sc + sc) * NR,
                                       reinterpret_cast<uint32_t*>(&pf[i][0]));
            }
        }
    }

    SetupOut<NR, NL> o;
    if (does_setup) setup_unit<ST, NR, NL>(hf, block_sigma2(a, slot), (float)qam_norm(QM), a.llr_scale, o);
    if constexpr (SHARE) {
        if (does_setup) {
#pragma unroll
            for (int k = 0; k < NL; ++k) {
#pragma unroll
                for (int r = 0; r < NR; ++r) sW[(k * NR + r) * TU + ul] = o.w[k][r];
                sSlope[k * TU + ul] = o.slope[k];
            }
        }
        __syncthreads();
        if (active && g != 0) {
#pragma unroll
            for (int k = 0; k < NL; ++k) {
#pragma unroll
                for (int r = 0; r < NR; ++r) o.w[k][r] = sW[(k * NR + r) * TU + ul];
                o.slope[k] = sSlope[k * TU + ul];
            }
        }
    }
    // PDL: all global writes come after the previous grid has completed.
    pdl_wait();
    if (does_setup && g == 0) {
        if (o.fail) atomicAdd(a.fail_count, 1ull);
        if (a.sinr) {
#pragma unroll
            for (int k = 0; k < NL; ++k) a.sinr[unit * NL + k] = o.sinr[k];
        }
    }
    if (a.sigma2 > 0.f)
        apply_symbols<NR, NL, QM, LT, TU, G, YL, false, SPH>(a, o, sy, bars, slot, sc, ul, g, active, pf);
    else
        apply_symbols<NR, NL, QM, LT, TU, G, YL, true, SPH>(a, o, sy, bars, slot, sc, ul, g, active, pf);
}

template <int NR, int NL, int QM, int LT, int TU, int G, int YL, typename ST, bool SH, int SPH>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_sc <= 0 || a.n_slots <= 0) return cudaSuccess;
    dim3 grid((a.n_sc + TU - 1) / TU, a.n_slots);
    return launch_kernel(k_tpu<NR, NL, QM, LT, TU, G, YL, ST, SH, SPH>, grid, dim3(TU * G),
                         smem_bytes<NR, NL, TU, YL, SH, SPH>(), s, a.overlap, a);
}

template <int NR, int NL, int QM, int LT, int TU, int G, int YL, typename ST, bool SH, int SPH>
cudaError_t prepare() {
    constexpr int smem = smem_bytes<NR, NL, TU, YL, SH, SPH>();
    if (smem > 48 * 1024)
        return cudaFuncSetAttribute(k_tpu<NR, NL, QM, LT, TU, G, YL, ST, SH, SPH>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaSuccess;
}

#define TPU_ENTRY3(NAME, NR, NL, QM, LT, TU, G, YL, ST, SH, SPH)                              \
    KernelEntry {                                                                              \
        NAME, NR, NL, QM, 1, SPH, LT, 32, 1, launch<NR, NL, QM, LT, TU, G, YL, ST, SH, SPH>,  \
            prepare<NR, NL, QM, LT, TU, G, YL, ST, SH, SPH>                                    \
    }
#define TPU_ENTRY2(NAME, NR, NL, QM, LT, TU, G, YL, ST, SH) TPU_ENTRY3(NAME, NR, NL, QM, LT, TU, G, YL, ST, SH, 14)
#define TPU_ENTRY(NAME, NR, NL, QM, LT, TU, G, YL, ST) TPU_ENTRY2(NAME, NR, NL, QM, LT, TU, G, YL, ST, false)

// First entry matching a plan wins (the default); another entry of the same
// shape is selectable by name through mimo_plan_desc_t.kernel.
const KernelEntry kEntries[] = {
    TPU_ENTRY("tpu_2x2_q2_f32", 2, 2, 2, kLlrF32, 32, 1, kYBulk, double),                 // C1
    TPU_ENTRY2("tpu_4x4_q4_f32", 4, 4, 4, kLlrF32, 64, 2, kYBulk, double, true),          // C2, paper 4x4
    TPU_ENTRY("tpu_2x2_q4_f32", 2, 2, 4, kLlrF32, 32, 1, kYBulk, double),
    TPU_ENTRY("tpu_2x1_q2_f32", 2, 1, 2, kLlrF32, 32, 1, kYBulk, double),
    TPU_ENTRY2("tpu_4x2_q4_f32", 4, 2, 4, kLlrF32, 64, 2, kYBulk, double, true),
    TPU_ENTRY2("tpu_4x4_q4_f16", 4, 4, 4, kLlrF16, 64, 2, kYBulk, double, true),
    TPU_ENTRY2("tpu_4x4_q4_i8", 4, 4, 4, kLlrI8, 64, 2, kYBulk, double, true),
    TPU_ENTRY2("tpu_4x4_q2_f32", 4, 4, 2, kLlrF32, 64, 2, kYBulk, double, true),
    TPU_ENTRY2("tpu_4x4_q6_f32", 4, 4, 6, kLlrF32, 64, 2, kYBulk, double, true),
    TPU_ENTRY2("tpu_4x4_q8_f32", 4, 4, 8, kLlrF32, 64, 2, kYBulk, double, true),
    // time-varying channels (NEXT-3): H every SPH < 14 symbols; one CTA per (H block, 64 subcarriers)
    TPU_ENTRY3("tpu_4x4_q4_f32_s7", 4, 4, 4, kLlrF32, 64, 2, kYBulk, double, true, 7),
    TPU_ENTRY3("tpu_4x4_q4_f32_s2", 4, 4, 4, kLlrF32, 64, 1, kYBulk, double, false, 2),
    TPU_ENTRY3("tpu_4x4_q4_f32_s1", 4, 4, 4, kLlrF32, 64, 1, kYBulk, double, false, 1),
    TPU_ENTRY3("tpu_2x2_q2_f32_s7", 2, 2, 2, kLlrF32, 32, 1, kYBulk, double, false, 7),
    TPU_ENTRY3("tpu_2x2_q2_f32_s1", 2, 2, 2, kLlrF32, 32, 1, kYBulk, double, false, 1),
};

}  // namespace

const KernelEntry* tpu_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
