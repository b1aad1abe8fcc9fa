// k_big.cu -- 16-layer per-PRB detectors on the FP32 SIMT pipe (n_rx = 32 / 64;
// any Qm and LLR type): the SIMT setup of big_setup.cuh (rows a2-a5, W~ to the
// plan workspace), then k_big_apply (rows a6-a7): one CTA per PRB-unit, the
// unit's 168 y vectors bulk-copied at a padded 528-byte stride, thread (RE pair,
// layer quarter) accumulates 2 x 4 complex outputs; with H constant over sym_per_h
// = 7 / 2 / 1 symbols one CTA serves 14 / sym_per_h H-units (the _s7/_s2/_s1
// entries, the default of the C5 shape at those sym_per_h). The C5 configuration itself
// (64 x 16, 64-QAM, int8) runs on the tcgen05 pipeline of k_c5.cu by default.

#include "big_setup.cuh"

namespace mimo {
namespace {

template <int NR, int NL, int SPH>
struct BigSmem {
    static constexpr int G = kSym / SPH;                   // H-units per CTA (168 REs in all)
    static constexpr int YS = NR * 8 + 16;                 // bytes per RE (padded 16 B)
    static constexpr size_t bar = 0;
    static constexpr size_t y = 128;                       // [168][YS]
    static constexpr size_t W = y + (size_t)kRe * YS;      // [G][NR][NL] float2
    static constexpr size_t total = W + (size_t)G * NR * NL * 8;
};

// thread (pair p, quarter h): REs 2p, 2p+1 of the CTA's 168, layers 4h .. 4h+3 (336 threads: four
// threads per RE pair so the FP32 pipe sees 2 x the warps of one per RE at the same shared-memory
// footprint). With H constant over SPH < 14 symbols (NEXT-3) the CTA serves
// G = 14 / SPH consecutive H-units of 12 x SPH REs each, every unit with its own W~ in shared memory.
constexpr int kBigLs = 4;                   // threads per RE pair (layer split)
constexpr int kBigThreads = kRe / 2 * kBigLs;
template <int NR, int NL, int QM, int LT, int SPH>
__global__ void __launch_bounds__(kBigThreads) k_big_apply(DetectArgs a) {
    static_assert(NL == 16 && NR % 2 == 0, "k_big_apply: 16 layers");
    static_assert(kSym % SPH == 0, "k_big_apply: SPH divides 14");
    using SM = BigSmem<NR, NL, SPH>;
    constexpr int WS = BigWs<NR, NL>::stride;
    constexpr int KH = NL / kBigLs;
    constexpr int RU = kSc * SPH;  // REs per H-unit
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::bar);
    unsigned char* sy = smem + SM::y;

    pdl_launch_dependents();
    const int t = threadIdx.x;
    const long long u0 = (long long)blockIdx.x * SM::G;
    const int nv = (int)min((long long)SM::G, a.n_units - u0);  // valid units of this CTA
    if (t == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        mbar_arrive_expect_tx(&bar[0], (uint32_t)(nv * RU) * NR * 8u);
        mbar_arrive_expect_tx(&bar[1], (uint32_t)nv * NR * NL * 8u);
    }
    __syncthreads();
    if (t < kRe && t / RU < nv) {  // thread t copies RE t (symbol (t % RU) / 12, subcarrier t % 12 of its unit)
        const long long uc = u0 + t / RU;
        const int sc = (int)(uc / a.n_fb), fc = (int)(uc % a.n_fb);
        const int s = (t % RU) / kSc, f = t % kSc;
        bulk_g2s(sy + (size_t)t * SM::YS, a.y + ((size_t)(sc * SPH + s) * a.n_sc + fc * kSc + f) * NR, NR * 8u,
                 &bar[0]);
    }
    pdl_wait();  // W~ of this call's setup kernel is complete
    if (t == 0)
        for (int i = 0; i < nv; ++i)
            bulk_g2s(smem + SM::W + (size_t)i * NR * NL * 8, reinterpret_cast<const float*>(a.ws) + (u0 + i) * WS,
                     NR * NL * 8u, &bar[1]);
    const int p = t / kBigLs, h = t % kBigLs;
    const int g = (2 * p) / RU;  // this thread's unit
    if (g >= nv) return;         // ragged last CTA (no later block-wide barrier)
    const long long u = u0 + g;
    const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);  // slot = H time block
    const float2* sW = reinterpret_cast<const float2*>(smem + SM::W + (size_t)g * NR * NL * 8);
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
            const float2 nva = make_float2(-va.y, va.x), nvb = make_float2(-vb.y, vb.x);
            const float4* wr = wq + (2 * r2 + c) * (NL / 2);
#pragma unroll
            for (int k2 = 0; k2 < KH / 2; ++k2) {  // packed FFMA2 (same FMA order as cmac)
                const float4 w2 = wr[k2];
                const float2 wa = make_float2(w2.x, w2.y), wb = make_float2(w2.z, w2.w);
                acc0[2 * k2] = cmac_y(acc0[2 * k2], wa, va, nva);
                acc0[2 * k2 + 1] = cmac_y(acc0[2 * k2 + 1], wb, va, nva);
                acc1[2 * k2] = cmac_y(acc1[2 * k2], wa, vb, nvb);
                acc1[2 * k2 + 1] = cmac_y(acc1[2 * k2 + 1], wb, vb, nvb);
            }
        }
    }
    constexpr int kBytes = KH * QM * LlrTraits<LT>::bytes;  // this thread's quarter of an RE record
    constexpr int kWords = (kBytes + 3) / 4;
    const bool zf = !(a.sigma2 > 0.f);
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int ri = (2 * p + e) % RU;
        const int s = ri / kSc, f = ri % kSc;
        const size_t re = (size_t)(slot * SPH + s) * a.n_sc + fb * kSc + f;
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

template <int NR, int NL, int QM, int LT, int SPH>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    constexpr int UPB = 4;
    constexpr int G = BigSmem<NR, NL, SPH>::G;
    cudaError_t e = launch_kernel(k_big_setup<NR, NL, QM, UPB>, dim3((unsigned)((a.n_units + UPB - 1) / UPB)),
                                  dim3(32 * UPB), UPB * SetupSmem<NR, NL>::per_unit, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    return launch_kernel(k_big_apply<NR, NL, QM, LT, SPH>, dim3((unsigned)((a.n_units + G - 1) / G)), dim3(kBigThreads),
                         BigSmem<NR, NL, SPH>::total, s, a.overlap, a);
}

template <int NR, int NL, int QM, int LT, int SPH>
cudaError_t prepare() {
    cudaError_t e = cudaFuncSetAttribute(k_big_setup<NR, NL, QM, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(4 * SetupSmem<NR, NL>::per_unit));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_big_apply<NR, NL, QM, LT, SPH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)BigSmem<NR, NL, SPH>::total);
}

#define BIG_ENTRY(NAME, NR, NL, QM, LT, SPH)                                                                  \
    KernelEntry {                                                                                             \
        NAME, NR, NL, QM, kSc, SPH, LT, 32, 2, launch<NR, NL, QM, LT, SPH>, prepare<NR, NL, QM, LT, SPH>,     \
            workspace<NR, NL>                                                                                 \
    }

const KernelEntry kEntries[] = {
    BIG_ENTRY("big_64x16_q6_i8", 64, 16, 6, kLlrI8, 14),  // C5 shape on SIMT (alternative to the c5 tcgen05 pipeline)
    BIG_ENTRY("big_64x16_q6_f16", 64, 16, 6, kLlrF16, 14),
    BIG_ENTRY("big_64x16_q6_f32", 64, 16, 6, kLlrF32, 14),
    BIG_ENTRY("big_64x16_q8_i8", 64, 16, 8, kLlrI8, 14),
    BIG_ENTRY("big_64x16_q4_i8", 64, 16, 4, kLlrI8, 14),
    BIG_ENTRY("big_32x16_q6_i8", 32, 16, 6, kLlrI8, 14),
    // time-varying H on the C5 shape (NEXT-3): 14 / SPH H-units per CTA
    BIG_ENTRY("big_64x16_q6_i8_s7", 64, 16, 6, kLlrI8, 7),
    BIG_ENTRY("big_64x16_q6_i8_s2", 64, 16, 6, kLlrI8, 2),
    BIG_ENTRY("big_64x16_q6_i8_s1", 64, 16, 6, kLlrI8, 1),
};

}  // namespace

const KernelEntry* big_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
