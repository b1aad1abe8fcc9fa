// k_prbp.cu -- persistent, TMA-pipelined per-PRB detector (C3: 8 rx x 4
// layers, 64-QAM, int8; any per-PRB shape whose W~ fits one thread).
//
// Mapping (DESIGN.md §"Kernels"): a persistent grid (CTAS_PER_SM per SM) walks
// tiles of P PRB-units of one slot. Each CTA keeps S tile buffers in shared
// memory; thread 0 keeps S-1 future tiles in flight with cp.async.bulk (the
// 14 y rows + the P H matrices of a tile complete on one mbarrier), so every SM
// streams HBM continuously while the CTA computes the current tile:
//   a2-a5  cooperative fp32 setup of the P units in shared memory (Gram entries
//          over threads, one thread per unit for Cholesky / L^-1 / G^-1 /
//          mu / SINR, W~ entries over threads; reading R18);
//   a6-a7  thread (g, f) copies its unit's W~ to registers and handles
//          subcarrier f for symbols g, g+G, ...: x~ = W~ y, exact max-log
//          demap, direct vector stores of the RE's NL*QM LLRs.
// A __syncthreads after each tile releases its buffer; thread 0 then refills it
// with the tile S iterations ahead.
#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;
constexpr int kSc = 12;

template <int NR, int NL, int P, int S>
struct PSmem {
    static constexpr int TF = kSc * P;
    static constexpr size_t ybytes = (size_t)kSym * TF * NR * 8;
    static constexpr size_t hbytes = (size_t)P * NR * NL * 8;
    static constexpr size_t stage = ybytes + hbytes;                     // y [14][TF][NR], H [P][NR][NL]
    static constexpr size_t bars = 0;                                    // S full barriers
    static constexpr size_t stages = 128;
    static constexpr size_t Gi = stages + S * stage;                     // [P][NL][NL] float2
    static constexpr size_t W = Gi + (size_t)P * NL * NL * 8;            // [P][NL][NR] float2
    static constexpr size_t slope = W + (size_t)P * NL * NR * 8;         // [P][NL]
    static constexpr size_t sinr = slope + (size_t)P * NL * 4;
    static constexpr size_t fac = sinr + (size_t)P * NL * 4;
    static constexpr size_t total = fac + (size_t)P * NL * 4;
};

__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}

template <int NR, int NL, int P, int S>
__device__ __forceinline__ void issue_tile(const DetectArgs& a, unsigned char* smem, int st, long long tile, int n_pg) {
    using SM = PSmem<NR, NL, P, S>;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM::bars) + st;
    unsigned char* base = smem + SM::stages + (size_t)st * SM::stage;
    const int slot = (int)(tile / n_pg);
    const int fb0 = (int)(tile % n_pg) * P;
    const int np = min(P, a.n_fb - fb0);
    const uint32_t row = (uint32_t)np * kSc * NR * 8u;
    const uint32_t hb = (uint32_t)np * NR * NL * 8u;
    mbar_arrive_expect_tx(bar, row * kSym + hb);
    bulk_g2s(base + SM::ybytes, a.H + ((size_t)slot * a.n_fb + fb0) * NR * NL, hb, bar);
#pragma unroll 1
    for (int s = 0; s < kSym; ++s)
        bulk_g2s(base + (size_t)s * SM::TF * NR * 8,
                 a.y + ((size_t)(slot * kSym + s) * a.n_sc + (size_t)fb0 * kSc) * NR, row, bar);
}

template <int NR, int NL, int QM, int LT, int P, int G, int S>
__global__ void __launch_bounds__(kSc* P* G) k_prbp(DetectArgs a) {
    using SM = PSmem<NR, NL, P, S>;
    constexpr int TF = SM::TF;
    constexpr int T = TF * G;
    constexpr int NE = NL * (NL + 1) / 2;
    static_assert(NR % 2 == 0, "16-byte y rows");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bars);
    float2* sGi = reinterpret_cast<float2*>(smem + SM::Gi);
    float2* sW = reinterpret_cast<float2*>(smem + SM::W);
    float* sSlope = reinterpret_cast<float*>(smem + SM::slope);
    float* sSinr = reinterpret_cast<float*>(smem + SM::sinr);
    float* sFac = reinterpret_cast<float*>(smem + SM::fac);

    pdl_launch_dependents();
    const int t = threadIdx.x;
    const int f = t % TF, g = t / TF;
    const int p = f / kSc;
    const int n_pg = (a.n_fb + P - 1) / P;
    const long long n_tiles = (long long)n_pg * a.n_slots;
    const float norm = (float)qam_norm(QM);
    const float s2 = a.sigma2;
    const float sqn = sqrtf(norm);
    const float ia = rsqrtf(norm);

    if (t == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
#pragma unroll 1
        for (int s = 0; s < S; ++s) {
            const long long tile = blockIdx.x + (long long)s * gridDim.x;
            if (tile < n_tiles) issue_tile<NR, NL, P, S>(a, smem, s, tile, n_pg);
        }
    }
    bool waited = false;

#pragma unroll 1
    for (int it = 0;; ++it) {
        const long long tile = blockIdx.x + (long long)it * gridDim.x;
        if (tile >= n_tiles) break;
        const int st = it % S;
        const int slot = (int)(tile / n_pg);
        const int fb0 = (int)(tile % n_pg) * P;
        const int np = min(P, a.n_fb - fb0);
        const bool active = f < np * kSc;
        const unsigned char* base = smem + SM::stages + (size_t)st * SM::stage;
        const float2* sy = reinterpret_cast<const float2*>(base);
        const float2* sH = reinterpret_cast<const float2*>(base + SM::ybytes);
        mbar_wait(&bars[st], (it / S) & 1);

        // a2: Gram lower triangle
        for (int idx = t; idx < np * NE; idx += T) {
            const int pu = idx / NE;
            int e = idx % NE, i = 0;
            while (e > i) {
                e -= i + 1;
                ++i;
            }
            const int j = e;
            const float2* h = sH + pu * NR * NL;
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const float2 c = cmulc(h[r * NL + i], h[r * NL + j]);
                acc.x += c.x;
                acc.y += c.y;
            }
            if (i == j) acc = make_float2(acc.x + s2, 0.f);
            sGi[(pu * NL + i) * NL + j] = acc;
        }
        __syncthreads();
        // a3-a5: one thread per unit
        if (t < np) {
            float2 L[NL][NL];
            float gmax = 0.f;
#pragma unroll
            for (int i = 0; i < NL; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j) {
                    L[i][j] = sGi[(t * NL + i) * NL + j];
                    if (i == j) gmax = fmaxf(gmax, L[i][i].x);
                }
            bool fail = !(gmax == gmax);
            float dinv[NL];
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                float pj = L[j][j].x;
#pragma unroll
                for (int k = 0; k < j; ++k) pj = fmaf(-L[j][k].x, L[j][k].x, fmaf(-L[j][k].y, L[j][k].y, pj));
                if (!(pj > (float)kPivotTau * gmax)) {
                    fail = true;
                    pj = 1.f;
                }
                dinv[j] = rsqrtf(pj);
#pragma unroll
                for (int i = j + 1; i < NL; ++i) {
                    float2 sv = L[i][j];
#pragma unroll
                    for (int k = 0; k < j; ++k) {
                        sv.x = fmaf(-L[i][k].x, L[j][k].x, fmaf(-L[i][k].y, L[j][k].y, sv.x));
                        sv.y = fmaf(-L[i][k].y, L[j][k].x, fmaf(L[i][k].x, L[j][k].y, sv.y));
                    }
                    L[i][j] = make_float2(sv.x * dinv[j], sv.y * dinv[j]);
                }
            }
            float2 X[NL][NL];
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                X[j][j] = make_float2(dinv[j], 0.f);
#pragma unroll
                for (int i = j + 1; i < NL; ++i) {
                    float2 sv = make_float2(0.f, 0.f);
#pragma unroll
                    for (int m = j; m < i; ++m) sv = cmac(sv, L[i][m], X[m][j]);
                    X[i][j] = make_float2(-sv.x * dinv[i], -sv.y * dinv[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < NL; ++i)
#pragma unroll
                for (int j = 0; j < NL; ++j) {
                    float2 sv = make_float2(0.f, 0.f);
#pragma unroll
                    for (int m = (i > j ? i : j); m < NL; ++m) {
                        const float2 c = cmulc(X[m][i], X[m][j]);
                        sv.x += c.x;
                        sv.y += c.y;
                    }
                    sGi[(t * NL + i) * NL + j] = sv;
                    if (i == j) {
                        const float A = sv.x;
                        const float mu = fmaf(-s2, A, 1.f);
                        float sinr, fac;
                        if (s2 == 0.f) {
                            sinr = __int_as_float(0x7f800000);
                            fac = sqn;
                        } else {
                            sinr = mu / (s2 * A);
                            fac = sqn / mu;
                        }
                        if (!(mu > 0.f) || fail) {
                            sinr = 0.f;
                            fac = 0.f;
                        }
                        sSinr[t * NL + i] = sinr;
                        sSlope[t * NL + i] = sinr / norm * a.llr_scale;
                        sFac[t * NL + i] = fac;
                    }
                }
            if (fail) sFac[t * NL] = -1.f;
        }
        __syncthreads();
        // W~ = diag(sqrt(norm)/mu) G^-1 H^H
        for (int idx = t; idx < np * NL * NR; idx += T) {
            const int pu = idx / (NL * NR), k = (idx / NR) % NL, r = idx % NR;
            const float2* gi = sGi + (pu * NL + k) * NL;
            const float2* h = sH + (pu * NR + r) * NL;
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                sv.x = fmaf(gi[j].x, h[j].x, fmaf(gi[j].y, h[j].y, sv.x));
                sv.y = fmaf(gi[j].y, h[j].x, fmaf(-gi[j].x, h[j].y, sv.y));
            }
            const float fac = sFac[pu * NL + k];
            const bool dead = !(fac > 0.f) || sFac[pu * NL] < 0.f;
            sW[idx] = dead ? make_float2(0.f, 0.f) : make_float2(sv.x * fac, sv.y * fac);
        }
        __syncthreads();
        float2 w[NL][NR];
        float slope[NL];
        if (active) {
#pragma unroll
            for (int k = 0; k < NL; ++k) {
#pragma unroll
                for (int r = 0; r < NR; ++r) w[k][r] = sW[(p * NL + k) * NR + r];
                slope[k] = sSlope[p * NL + k];
            }
        }
        if (!waited) {  // PDL: first global write only after the previous grid completed
            pdl_wait();
            waited = true;
        }
        if (t < np) {
            const size_t unit = (size_t)slot * a.n_fb + fb0 + t;
            if (sFac[t * NL] < 0.f) atomicAdd(a.fail_count, 1ull);
            if (a.sinr) {
#pragma unroll
                for (int k = 0; k < NL; ++k) a.sinr[unit * NL + k] = sSinr[t * NL + k];
            }
        }
        constexpr int kLlrBytes = NL * QM * LlrTraits<LT>::bytes;
        constexpr int kWords = (kLlrBytes + 3) / 4;
        const int sc = fb0 * kSc + f;
        if (active) {
#pragma unroll 1
            for (int s = g; s < kSym; s += G) {
                float2 yv[NR];
                const float2* ys = sy + (s * TF + f) * NR;
#pragma unroll
                for (int r = 0; r < NR; ++r) yv[r] = ys[r];
                float2 x[NL];
#pragma unroll
                for (int k = 0; k < NL; ++k) {
                    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int r = 0; r < NR; ++r) acc = cmac(acc, w[k][r], yv[r]);
                    x[k] = acc;
                }
                const size_t re = (size_t)(slot * kSym + s) * a.n_sc + sc;
                if (a.llr) {
                    float v[NL * QM];
                    uint32_t wd[kWords];
                    if (s2 > 0.f) {
#pragma unroll
                        for (int k = 0; k < NL; ++k) demap_layer<QM, false, LT>(x[k], slope[k], v + k * QM);
                        pack_llr<LT, NL * QM, false>(v, wd);
                    } else {
#pragma unroll
                        for (int k = 0; k < NL; ++k) demap_layer<QM, true, LT>(x[k], slope[k], v + k * QM);
                        pack_llr<LT, NL * QM, true>(v, wd);
                    }
                    store_bytes<kLlrBytes>((char*)a.llr + re * kLlrBytes, wd);
                }
                if (a.xhat) {
                    uint32_t wd[2 * NL];
#pragma unroll
                    for (int k = 0; k < NL; ++k) {
                        wd[2 * k] = __float_as_uint(x[k].x * ia);
                        wd[2 * k + 1] = __float_as_uint(x[k].y * ia);
                    }
                    store_bytes<NL * 8>(a.xhat + re * NL, wd);
                }
            }
        }
        __syncthreads();  // stage st and the setup scratch are free
        if (t == 0) {
            const long long nt = tile + (long long)S * gridDim.x;
            if (nt < n_tiles) issue_tile<NR, NL, P, S>(a, smem, st, nt, n_pg);
        }
    }
    if (!waited) pdl_wait();
}

template <int NR, int NL, int QM, int LT, int P, int G, int S, int CPS>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_fb <= 0 || a.n_slots <= 0) return cudaSuccess;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const long long n_tiles = (long long)((a.n_fb + P - 1) / P) * a.n_slots;
    const long long grid = n_tiles < (long long)n_sm * CPS ? n_tiles : (long long)n_sm * CPS;
    return launch_kernel(k_prbp<NR, NL, QM, LT, P, G, S>, dim3((unsigned)grid), dim3(kSc * P * G),
                         PSmem<NR, NL, P, S>::total, s, a.overlap, a);
}

template <int NR, int NL, int QM, int LT, int P, int G, int S, int CPS>
cudaError_t prepare() {
    return cudaFuncSetAttribute(k_prbp<NR, NL, QM, LT, P, G, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)PSmem<NR, NL, P, S>::total);
}

#define PRBP_ENTRY(NAME, NR, NL, QM, LT, P, G, S, CPS)                                   \
    KernelEntry {                                                                         \
        NAME, NR, NL, QM, kSc, 14, LT, 32, 1, launch<NR, NL, QM, LT, P, G, S, CPS>,      \
            prepare<NR, NL, QM, LT, P, G, S, CPS>                                         \
    }

const KernelEntry kEntries[] = {
    PRBP_ENTRY("prbp_8x4_q6_i8", 8, 4, 6, kLlrI8, 4, 7, 3, 1),  // C3
    PRBP_ENTRY("prbp_8x4_q6_f32", 8, 4, 6, kLlrF32, 4, 7, 3, 1),
    PRBP_ENTRY("prbp_8x4_q6_f16", 8, 4, 6, kLlrF16, 4, 7, 3, 1),
    // tuning variants
    PRBP_ENTRY("prbp_8x4_q6_i8_p4g7s2c2", 8, 4, 6, kLlrI8, 4, 7, 2, 2),
    PRBP_ENTRY("prbp_8x4_q6_i8_p4g4s3c1", 8, 4, 6, kLlrI8, 4, 4, 3, 1),
    PRBP_ENTRY("prbp_8x4_q6_i8_p2g7s4c2", 8, 4, 6, kLlrI8, 2, 7, 4, 2),
    PRBP_ENTRY("prbp_8x4_q6_i8_p2g14s3c2", 8, 4, 6, kLlrI8, 2, 14, 3, 2),
    PRBP_ENTRY("prbp_8x4_q6_i8_p4g14s3c1", 8, 4, 6, kLlrI8, 4, 14, 3, 1),
};

}  // namespace

const KernelEntry* prbp_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
