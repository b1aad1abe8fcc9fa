// k_big.cu -- massive-MIMO per-PRB detector (C5: 64 rx x 16 layers, 64-QAM,
// int8, H per PRB). The per-RE filter x~ = W~ y is a dense complex contraction
// (16 x 64 per RE, 1024 cMAC): C5 is FP32-bound, not HBM-bound (SURVEY.md
// §8(d)), so the kernels are organised around the FFMA pipe.
//
//   k_big_setup (rows a2-a5), one CTA (256 threads) per PRB-unit, fp32
//     (reading R18; cond(G) <= ~10 on C5): G = H^H H + s2 I (one entry per
//     thread), Cholesky by 16 lanes of warp 0 (lane k holds row k, pivots and
//     columns by __shfl_sync; guard R17), X = L^-1 column per lane, G^-1 = X^H X,
//     W~ = diag(sqrt(norm)/mu) G^-1 H^H (4 entries per thread), written to the
//     plan workspace as [unit][r][k] plus slopes.
//   k_big_apply (rows a6-a7), one CTA per PRB-unit: the unit's 168 y vectors
//     are bulk-copied into shared memory at a padded 528-byte stride
//     (conflict-free 128-bit reads) and W~ [r][k] next to them; thread
//     (RE pair, layer half) accumulates its 2 x 8 complex outputs over r with
//     128-bit shared loads (register-tiled SIMT GEMM, 12.8 FFMA per load),
//     then demaps its 16 layer-REs and stores 48 contiguous LLR bytes per RE.
#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;
constexpr int kSc = 12;
constexpr int kRe = kSym * kSc;  // 168 REs per PRB-unit

template <int NR, int NL>
struct BigWs {
    static constexpr int w_floats = NR * NL * 2;                 // W~ [r][k] float2
    static constexpr int stride = (w_floats + NL + 31) / 32 * 32; // floats per unit (128-byte multiple)
};

__device__ __forceinline__ float2 shfl2(float2 v, int src) {
    return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <int NR, int NL, int QM>
__global__ void __launch_bounds__(256) k_big_setup(DetectArgs a) {
    static_assert(NL == 16 && NR % 4 == 0, "k_big_setup: 16 layers");
    constexpr int WS = BigWs<NR, NL>::stride;
    __shared__ __align__(16) float2 sH[NR * NL];      // [r][l]
    __shared__ float2 sG[NL * NL];                    // G, then X = L^-1 ([i][j]), then G^-1
    __shared__ float2 sL[NL * NL];
    __shared__ float sDinv[NL], sFac[NL], sSinr[NL];
    __shared__ int sFail;

    pdl_launch_dependents();
    const int t = threadIdx.x;
    const long long u = blockIdx.x;
    const float s2 = a.sigma2;
    const float norm = (float)qam_norm(QM);
    {
        const float4* src = reinterpret_cast<const float4*>(a.H + u * NR * NL);
        float4* dst = reinterpret_cast<float4*>(sH);
        for (int i = t; i < NR * NL / 2; i += 256) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    // a2: G_ij = sum_r conj(H_ri) H_rj (+ s2 on the diagonal), one entry per thread
    {
        const int i = t / NL, j = t % NL;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll 8
        for (int r = 0; r < NR; ++r) {
            const float2 hi = sH[r * NL + i], hj = sH[r * NL + j];
            acc.x = fmaf(hi.x, hj.x, fmaf(hi.y, hj.y, acc.x));
            acc.y = fmaf(hi.x, hj.y, fmaf(-hi.y, hj.x, acc.y));
        }
        if (i == j) acc = make_float2(acc.x + s2, 0.f);
        sG[i * NL + j] = acc;
    }
    __syncthreads();
    // a3: Cholesky by lanes 0..15 of warp 0 (lane k holds row k, right-looking)
    if (t < 32) {
        const int k = t & 15;
        float2 g[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) g[j] = sG[k * NL + j];
        float gmax = g[0].x;
#pragma unroll
        for (int j = 0; j < NL; ++j)
            if (j == k) gmax = g[j].x;
#pragma unroll
        for (int off = 1; off < NL; off <<= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
        bool fail = !(gmax == gmax);
        float my_dinv = 0.f;
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            float p = __shfl_sync(0xffffffffu, g[j].x, j);
            if (!(p > (float)kPivotTau * gmax)) {
                fail = true;
                p = 1.f;
            }
            const float dinv = rsqrtf(p);
            if (k == j) my_dinv = dinv;
            if (k > j) g[j] = make_float2(g[j].x * dinv, g[j].y * dinv);
#pragma unroll
            for (int m = j + 1; m < NL; ++m) {
                const float2 lmj = shfl2(g[j], m);
                if (k >= m) {
                    g[m].x = fmaf(-g[j].x, lmj.x, fmaf(-g[j].y, lmj.y, g[m].x));
                    g[m].y = fmaf(-g[j].y, lmj.x, fmaf(g[j].x, lmj.y, g[m].y));
                }
            }
        }
        if (t < NL) {
#pragma unroll
            for (int j = 0; j < NL; ++j) sL[k * NL + j] = (j < k) ? g[j] : make_float2(0.f, 0.f);
            sDinv[k] = my_dinv;
            if (k == 0) sFail = fail;
        }
    }
    __syncthreads();
    // a4: X = L^-1, column k per thread (k < 16): X_kk = 1/L_kk, X_ik = -(1/L_ii) sum_{m<i} L_im X_mk
    if (t < NL) {
        const int k = t;
        float2 x[NL];
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = 0; m < i; ++m) sv = cmac(sv, sL[i * NL + m], x[m]);
            const float di = sDinv[i];
            x[i] = (i == k) ? make_float2(di, 0.f) : (i < k ? make_float2(0.f, 0.f) : make_float2(-sv.x * di, -sv.y * di));
        }
#pragma unroll
        for (int i = 0; i < NL; ++i) sG[i * NL + k] = x[i];
    }
    __syncthreads();
    // G^-1 = X^H X (one entry per thread), mu / SINR / factor
    float2 gi;
    {
        const int i = t / NL, j = t % NL;
        float2 sv = make_float2(0.f, 0.f);
        for (int m = (i > j ? i : j); m < NL; ++m) {
            const float2 xi = sG[m * NL + i], xj = sG[m * NL + j];
            sv.x = fmaf(xi.x, xj.x, fmaf(xi.y, xj.y, sv.x));
            sv.y = fmaf(xi.x, xj.y, fmaf(-xi.y, xj.x, sv.y));
        }
        gi = sv;
    }
    __syncthreads();
    {
        const int i = t / NL, j = t % NL;
        sL[i * NL + j] = gi;  // G^-1 into sL
        if (i == j) {
            const float A = gi.x;
            const float mu = fmaf(-s2, A, 1.f);
            float sinr, fac;
            if (s2 == 0.f) {
                sinr = __int_as_float(0x7f800000);
                fac = sqrtf(norm);
            } else {
                sinr = __fdividef(mu, s2 * A);
                fac = __fdividef(sqrtf(norm), mu);
            }
            if (!(mu > 0.f) || sFail) {
                sinr = 0.f;
                fac = 0.f;
            }
            sFac[i] = fac;
            sSinr[i] = sinr;
        }
    }
    __syncthreads();
    // W~[r][k] = fac_k sum_j G^-1_kj conj(H_rj): 4 entries per thread, k fastest
    float2 wv[NR * NL / 256];
#pragma unroll
    for (int q = 0; q < NR * NL / 256; ++q) {
        const int idx = t + 256 * q;
        const int r = idx / NL, k = idx % NL;
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const float2 g2 = sL[k * NL + j], h = sH[r * NL + j];
            sv.x = fmaf(g2.x, h.x, fmaf(g2.y, h.y, sv.x));
            sv.y = fmaf(g2.y, h.x, fmaf(-g2.x, h.y, sv.y));
        }
        const float fac = sFac[k];
        wv[q] = fac > 0.f ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
    }
    pdl_wait();  // the previous call may still read the workspace
    float* ws = reinterpret_cast<float*>(a.ws) + u * WS;
#pragma unroll
    for (int q = 0; q < NR * NL / 256; ++q) reinterpret_cast<float2*>(ws)[t + 256 * q] = wv[q];
    if (t < NL) {
        ws[NR * NL * 2 + t] = sSinr[t] / norm * a.llr_scale;
        if (a.sinr) a.sinr[u * NL + t] = sSinr[t];
    }
    if (t == 0 && sFail) atomicAdd(a.fail_count, 1ull);
}

template <int NR, int NL>
struct BigSmem {
    static constexpr int YS = NR * 8 + 16;                 // bytes per RE (padded 16 B)
    static constexpr size_t bar = 0;
    static constexpr size_t y = 128;                       // [168][YS]
    static constexpr size_t W = y + (size_t)kRe * YS;      // [NR][NL] float2
    static constexpr size_t total = W + (size_t)NR * NL * 8;
};

// thread (pair p, half h): REs 2p, 2p+1 of the unit, layers 8h .. 8h+7
template <int NR, int NL, int QM, int LT>
__global__ void __launch_bounds__(kRe) k_big_apply(DetectArgs a) {
    static_assert(NL == 16 && NR % 2 == 0, "k_big_apply: 16 layers");
    using SM = BigSmem<NR, NL>;
    constexpr int WS = BigWs<NR, NL>::stride;
    constexpr int KH = NL / 2;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::bar);
    unsigned char* sy = smem + SM::y;
    const float2* sW = reinterpret_cast<const float2*>(smem + SM::W);

    pdl_launch_dependents();
    const int t = threadIdx.x;
    const long long u = blockIdx.x;
    const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
    if (t == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        mbar_arrive_expect_tx(&bar[0], (uint32_t)kRe * NR * 8u);
        mbar_arrive_expect_tx(&bar[1], (uint32_t)NR * NL * 8u);
    }
    __syncthreads();
    {  // thread t copies RE t (symbol t / 12, subcarrier t % 12) into its padded slot
        const int s = t / kSc, f = t % kSc;
        bulk_g2s(sy + (size_t)t * SM::YS, a.y + ((size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f) * NR, NR * 8u,
                 &bar[0]);
    }
    pdl_wait();  // W~ of this call's setup kernel is complete
    if (t == 0)
        bulk_g2s(smem + SM::W, reinterpret_cast<const float*>(a.ws) + u * WS, NR * NL * 8u, &bar[1]);
    const int p = t >> 1, h = t & 1;
    float slope[KH];
    {
        const float* wsu = reinterpret_cast<const float*>(a.ws) + u * WS + NR * NL * 2;
#pragma unroll
        for (int k = 0; k < KH; ++k) slope[k] = wsu[h * KH + k];
    }
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1], 0);

    float2 acc0[KH], acc1[KH];
#pragma unroll
    for (int k = 0; k < KH; ++k) acc0[k] = acc1[k] = make_float2(0.f, 0.f);
    const float4* y0 = reinterpret_cast<const float4*>(sy + (size_t)(2 * p) * SM::YS);
    const float4* y1 = reinterpret_cast<const float4*>(sy + (size_t)(2 * p + 1) * SM::YS);
    const float4* wq = reinterpret_cast<const float4*>(sW) + h * (KH / 2);
#pragma unroll 2
    for (int r2 = 0; r2 < NR / 2; ++r2) {
        const float4 ya = y0[r2], yb = y1[r2];  // (y_r, y_r+1) of each RE
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float2 va = c ? make_float2(ya.z, ya.w) : make_float2(ya.x, ya.y);
            const float2 vb = c ? make_float2(yb.z, yb.w) : make_float2(yb.x, yb.y);
            const float4* wr = wq + (2 * r2 + c) * (NL / 2);
#pragma unroll
            for (int k2 = 0; k2 < KH / 2; ++k2) {
                const float4 w2 = wr[k2];
                const float2 wa = make_float2(w2.x, w2.y), wb = make_float2(w2.z, w2.w);
                acc0[2 * k2] = cmac(acc0[2 * k2], wa, va);
                acc0[2 * k2 + 1] = cmac(acc0[2 * k2 + 1], wb, va);
                acc1[2 * k2] = cmac(acc1[2 * k2], wa, vb);
                acc1[2 * k2 + 1] = cmac(acc1[2 * k2 + 1], wb, vb);
            }
        }
    }
    constexpr int kBytes = KH * QM * LlrTraits<LT>::bytes;  // this thread's half of an RE record
    constexpr int kWords = (kBytes + 3) / 4;
    const bool zf = !(a.sigma2 > 0.f);
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int ri = 2 * p + e;
        const int s = ri / kSc, f = ri % kSc;
        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
        const float2* acc = e ? acc1 : acc0;
        if (a.llr) {
            float v[KH * QM];
            uint32_t wd[kWords];
            if (!zf) {
#pragma unroll
                for (int k = 0; k < KH; ++k) demap_layer<QM, false, LT>(acc[k], slope[k], v + k * QM);
                pack_llr<LT, KH * QM, false>(v, wd);
            } else {
#pragma unroll
                for (int k = 0; k < KH; ++k) demap_layer<QM, true, LT>(acc[k], slope[k], v + k * QM);
                pack_llr<LT, KH * QM, true>(v, wd);
            }
            store_bytes<kBytes>((char*)a.llr + re * (NL * QM * LlrTraits<LT>::bytes) + h * kBytes, wd);
        }
        if (a.xhat) {
#pragma unroll
            for (int k = 0; k < KH; ++k) a.xhat[re * NL + h * KH + k] = make_float2(acc[k].x * ia, acc[k].y * ia);
        }
    }
}

template <int NR, int NL>
size_t workspace(const DetectArgs& a) {
    return (size_t)a.n_units * BigWs<NR, NL>::stride * 4;
}

template <int NR, int NL, int QM, int LT>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    cudaError_t e = launch_kernel(k_big_setup<NR, NL, QM>, dim3((unsigned)a.n_units), dim3(256), 0, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    return launch_kernel(k_big_apply<NR, NL, QM, LT>, dim3((unsigned)a.n_units), dim3(kRe), BigSmem<NR, NL>::total, s,
                         a.overlap, a);
}

template <int NR, int NL, int QM, int LT>
cudaError_t prepare() {
    return cudaFuncSetAttribute(k_big_apply<NR, NL, QM, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)BigSmem<NR, NL>::total);
}

#define BIG_ENTRY(NAME, NR, NL, QM, LT) \
    KernelEntry { NAME, NR, NL, QM, kSc, 14, LT, 32, 2, launch<NR, NL, QM, LT>, prepare<NR, NL, QM, LT>, workspace<NR, NL> }

const KernelEntry kEntries[] = {
    BIG_ENTRY("big_64x16_q6_i8", 64, 16, 6, kLlrI8),  // C5
    BIG_ENTRY("big_64x16_q6_f16", 64, 16, 6, kLlrF16),
    BIG_ENTRY("big_64x16_q6_f32", 64, 16, 6, kLlrF32),
    BIG_ENTRY("big_64x16_q8_i8", 64, 16, 8, kLlrI8),
    BIG_ENTRY("big_64x16_q4_i8", 64, 16, 4, kLlrI8),
    BIG_ENTRY("big_32x16_q6_i8", 32, 16, 6, kLlrI8),
};

}  // namespace

const KernelEntry* big_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
