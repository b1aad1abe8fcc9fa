// k_big.cu -- massive-MIMO per-PRB detector (C5: 64 rx x 16 layers, 64-QAM,
// int8, H per PRB). The per-RE filter x~ = W~ y is a dense complex contraction
// (16 x 64 per RE, 1024 cMAC): C5 is FP32-bound, not HBM-bound (SURVEY.md
// §8(d)), so the kernels are organised around the FFMA pipe.
//
//   k_big_setup (rows a2-a5), one warp per PRB-unit, warp-synchronous, fp32
//     (reading R18; cond(G) <= ~10 on C5): G = H^H H + s2 I (half a row per
//     lane, broadcast 128-bit H reads), Cholesky with lane k holding row k
//     (pivots and columns by __shfl_sync; guard R17), X = L^-1 column per lane,
//     row k of G^-1 = X^H X per lane, W~ = diag(sqrt(norm)/mu) G^-1 H^H (lane
//     (k, half) covers half the antennas), written to the plan workspace as
//     [unit][r][k] plus slopes.
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

// One warp per PRB-unit (UPB units per CTA), warp-synchronous, no CTA barriers.
template <int NR, int NL>
struct SetupSmem {
    static constexpr size_t per_unit = (size_t)NR * NL * 8 + 3 * NL * NL * 8 + 3 * NL * 4 + 16;
};

template <int NR, int NL, int QM, int UPB>
__global__ void __launch_bounds__(32 * UPB) k_big_setup(DetectArgs a) {
    static_assert(NL == 16 && NR % 32 == 0, "k_big_setup: 16 layers, NR multiple of 32");
    constexpr int WS = BigWs<NR, NL>::stride;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem + (size_t)warp * SetupSmem<NR, NL>::per_unit;
    float2* sH = reinterpret_cast<float2*>(base);                 // [r][l]
    float2* sG = sH + NR * NL;                                    // G
    float2* sX = sG + NL * NL;                                    // L rows, then X = L^-1 [i][j]
    float2* sGi = sX + NL * NL;                                   // G^-1
    float* sDinv = reinterpret_cast<float*>(sGi + NL * NL);

    pdl_launch_dependents();
    const long long u = (long long)blockIdx.x * UPB + warp;
    const bool valid = u < a.n_units;
    const float s2 = a.sigma2;
    const float norm = (float)qam_norm(QM);
    if (valid) {
        const float4* src = reinterpret_cast<const float4*>(a.H + u * NR * NL);
        float4* dst = reinterpret_cast<float4*>(sH);
#pragma unroll 4
        for (int i = lane; i < NR * NL / 2; i += 32) dst[i] = __ldg(src + i);
    }
    __syncwarp();
    // a2: lane -> row i = lane/2, columns 8h .. 8h+7 of G (full rows, broadcast H reads)
    {
        const int i = lane >> 1, h = lane & 1;
        float2 g[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) g[q] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int r = 0; r < NR; ++r) {
            const float2 hi = sH[r * NL + i];
            const float4* hr = reinterpret_cast<const float4*>(sH + r * NL + 8 * h);
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
                const float4 v = hr[q2];
                g[2 * q2].x = fmaf(hi.x, v.x, fmaf(hi.y, v.y, g[2 * q2].x));
                g[2 * q2].y = fmaf(hi.x, v.y, fmaf(-hi.y, v.x, g[2 * q2].y));
                g[2 * q2 + 1].x = fmaf(hi.x, v.z, fmaf(hi.y, v.w, g[2 * q2 + 1].x));
                g[2 * q2 + 1].y = fmaf(hi.x, v.w, fmaf(-hi.y, v.z, g[2 * q2 + 1].y));
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int j = 8 * h + q;
            sG[i * NL + j] = (i == j) ? make_float2(g[q].x + s2, 0.f) : g[q];
        }
    }
    __syncwarp();
    // a3: Cholesky, lane k (and its duplicate k+16) holds row k
    const int k = lane & 15;
    float2 g[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) g[j] = sG[k * NL + j];
    float gmax = 0.f;
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
    if (lane < NL) {
#pragma unroll
        for (int j = 0; j < NL; ++j) sX[k * NL + j] = (j < k) ? g[j] : make_float2(0.f, 0.f);
        sDinv[k] = my_dinv;
    }
    __syncwarp();
    // a4: X = L^-1, column k per lane (lanes 16..31 duplicate)
    float2 x[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < i; ++m) sv = cmac(sv, sX[i * NL + m], x[m]);
        const float di = sDinv[i];
        x[i] = (i == k) ? make_float2(di, 0.f) : (i < k ? make_float2(0.f, 0.f) : make_float2(-sv.x * di, -sv.y * di));
    }
    __syncwarp();
    if (lane < NL) {
#pragma unroll
        for (int i = 0; i < NL; ++i) sX[i * NL + k] = x[i];
    }
    __syncwarp();
    // row k of G^-1 = X^H X (lane k; x = column k of X), A_kk
    float2 gi[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = j; m < NL; ++m) {
            const float2 xm = x[m], xmj = sX[m * NL + j];
            sv.x = fmaf(xm.x, xmj.x, fmaf(xm.y, xmj.y, sv.x));
            sv.y = fmaf(xm.x, xmj.y, fmaf(-xm.y, xmj.x, sv.y));
        }
        gi[j] = sv;
    }
    float A = 0.f;
#pragma unroll
    for (int j = 0; j < NL; ++j)
        if (j == k) A = gi[j].x;
    const float mu = fmaf(-s2, A, 1.f);
    float sinr, fac;
    if (s2 == 0.f) {
        sinr = __int_as_float(0x7f800000);
        fac = sqrtf(norm);
    } else {
        sinr = __fdividef(mu, s2 * A);
        fac = __fdividef(sqrtf(norm), mu);
    }
    if (!(mu > 0.f) || fail) {
        sinr = 0.f;
        fac = 0.f;
    }
    // W~[r][k] = fac_k sum_j G^-1_kj conj(H_rj): lane (k, half) covers r in [half*NR/2, (half+1)*NR/2)
    const int half = lane >> 4;
    pdl_wait();  // the previous call may still read the workspace
    if (valid) {
        float2* ws = reinterpret_cast<float2*>(reinterpret_cast<float*>(a.ws) + u * WS);
#pragma unroll 2
        for (int rr = 0; rr < NR / 2; ++rr) {
            const int r = half * (NR / 2) + rr;
            const float4* hr = reinterpret_cast<const float4*>(sH + r * NL);
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int j2 = 0; j2 < NL / 2; ++j2) {
                const float4 v = hr[j2];
                sv.x = fmaf(gi[2 * j2].x, v.x, fmaf(gi[2 * j2].y, v.y, sv.x));
                sv.y = fmaf(gi[2 * j2].y, v.x, fmaf(-gi[2 * j2].x, v.y, sv.y));
                sv.x = fmaf(gi[2 * j2 + 1].x, v.z, fmaf(gi[2 * j2 + 1].y, v.w, sv.x));
                sv.y = fmaf(gi[2 * j2 + 1].y, v.z, fmaf(-gi[2 * j2 + 1].x, v.w, sv.y));
            }
            ws[r * NL + k] = fac > 0.f ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
        }
        if (lane < NL) {
            reinterpret_cast<float*>(ws)[NR * NL * 2 + k] = sinr / norm * a.llr_scale;
            if (a.sinr) a.sinr[u * NL + k] = sinr;
        }
        if (lane == 0 && fail) atomicAdd(a.fail_count, 1ull);
    }
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
    constexpr int UPB = 4;
    cudaError_t e = launch_kernel(k_big_setup<NR, NL, QM, UPB>, dim3((unsigned)((a.n_units + UPB - 1) / UPB)),
                                  dim3(32 * UPB), UPB * SetupSmem<NR, NL>::per_unit, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    return launch_kernel(k_big_apply<NR, NL, QM, LT>, dim3((unsigned)a.n_units), dim3(kRe), BigSmem<NR, NL>::total, s,
                         a.overlap, a);
}

template <int NR, int NL, int QM, int LT>
cudaError_t prepare() {
    cudaError_t e = cudaFuncSetAttribute(k_big_setup<NR, NL, QM, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(4 * SetupSmem<NR, NL>::per_unit));
    if (e != cudaSuccess) return e;
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
