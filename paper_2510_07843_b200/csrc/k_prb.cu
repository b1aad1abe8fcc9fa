// k_prb.cu -- per-PRB-channel detector for tall shapes whose W~ fits one
// thread's registers (C3: 8 rx x 4 layers, 64-QAM, int8; NL*NR <= 32).
//
// Mapping (DESIGN.md §"Kernels"): a CTA owns P PRB-units (12 P subcarriers) of
// one slot and G thread groups; thread (g, f) serves subcarrier f for symbols
// g, g+G, ... of the slot.
//   1. thread 0 bulk-copies the P H matrices (one mbarrier) and the 14 y rows
//      of the tile (12 P NR complex each, one mbarrier per row) into shared
//      memory -- everything is in flight at once;
//   2. the CTA runs rows a2-a5 for its P units cooperatively in shared memory
//      in fp32 (reading R18: tall configs meet the x~ bound in fp32 with >= 5x
//      margin): Gram entries over threads, one thread per unit
//      for the Cholesky / L^-1 / G^-1 chain, W~ entries over threads;
//   3. each thread copies its unit's W~ (NL x NR) and slopes into registers and
//      streams its symbols: x~ = W~ y from the y tile (row a6), exact max-log
//      demap (row a7), direct vector stores of its RE's NL*QM LLRs.
#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;
constexpr int kSc = 12;  // subcarriers per PRB (sc_per_h)

template <int NR, int NL, int P>
struct PrbSmem {
    static constexpr int TF = kSc * P;
    static constexpr size_t bars = 0;                                    // 15 mbarriers
    static constexpr size_t y = 128;                                     // [14][TF][NR] float2
    static constexpr size_t H = y + (size_t)kSym * TF * NR * 8;          // [P][NR][NL] float2
    static constexpr size_t Gi = H + (size_t)P * NR * NL * 8;            // [P][NL][NL] float2: G, then G^-1
    static constexpr size_t W = Gi + (size_t)P * NL * NL * 8;            // [P][NL][NR] float2
    static constexpr size_t slope = W + (size_t)P * NL * NR * 8;         // [P][NL] float
    static constexpr size_t sinr = slope + (size_t)P * NL * 4;           // [P][NL] float
    static constexpr size_t fac = sinr + (size_t)P * NL * 4;             // [P][NL] float (sqrt(norm)/mu or 0)
    static constexpr size_t total = fac + (size_t)P * NL * 4;
};

__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}

template <int NR, int NL, int QM, int LT, int P, int G>
__global__ void __launch_bounds__(kSc* P* G) k_prb(DetectArgs a) {
    using SM = PrbSmem<NR, NL, P>;
    constexpr int TF = SM::TF;
    constexpr int T = TF * G;
    constexpr int NE = NL * (NL + 1) / 2;
    static_assert(NR % 2 == 0, "16-byte y rows");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bars);
    float2* sy = reinterpret_cast<float2*>(smem + SM::y);
    float2* sH = reinterpret_cast<float2*>(smem + SM::H);
    float2* sGi = reinterpret_cast<float2*>(smem + SM::Gi);
    float2* sW = reinterpret_cast<float2*>(smem + SM::W);
    float* sSlope = reinterpret_cast<float*>(smem + SM::slope);
    float* sSinr = reinterpret_cast<float*>(smem + SM::sinr);
    float* sFac = reinterpret_cast<float*>(smem + SM::fac);

    pdl_launch_dependents();
    const int slot = blockIdx.y;
    const int fb0 = blockIdx.x * P;
    const int np = min(P, a.n_fb - fb0);
    const int t = threadIdx.x;
    const int f = t % TF, g = t / TF;
    const int p = f / kSc;
    const bool active = f < np * kSc;
    const float norm = (float)qam_norm(QM);
    const float s2 = block_sigma2(a, slot);

    if (t == 0) {
#pragma unroll
        for (int s = 0; s <= kSym; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        const uint32_t hb = (uint32_t)np * NR * NL * 8u;
        mbar_arrive_expect_tx(&bars[kSym], hb);
        bulk_g2s(sH, a.H + ((size_t)slot * a.n_fb + fb0) * NR * NL, hb, &bars[kSym]);
        const uint32_t row = (uint32_t)np * kSc * NR * 8u;
#pragma unroll 1
        for (int s = 0; s < kSym; ++s) {
            mbar_arrive_expect_tx(&bars[s], row);
            bulk_g2s(sy + s * TF * NR, a.y + ((size_t)(slot * kSym + s) * a.n_sc + (size_t)fb0 * kSc) * NR, row,
                     &bars[s]);
        }
    }
    mbar_wait(&bars[kSym], 0);

    // a2: Gram lower triangle, entries over threads: G_ij = sum_r conj(H_ri) H_rj (+ s2 on the diagonal)
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

    // a3-a5: one thread per unit -- Cholesky (guard R17), X = L^-1, G^-1 = X^H X, mu, SINR, slope
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
                for (int k = 0; k < j; ++k) {  // s -= L_ik conj(L_jk)
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
        const float sqn = sqrtf(norm);
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
        if (fail) sFac[t * NL] = -1.f;  // marks the unit as flagged
    }
    __syncthreads();

    // W~ = diag(sqrt(norm)/mu) G^-1 H^H, entries over threads
    for (int idx = t; idx < np * NL * NR; idx += T) {
        const int pu = idx / (NL * NR), k = (idx / NR) % NL, r = idx % NR;
        const float2* gi = sGi + (pu * NL + k) * NL;
        const float2* h = sH + (pu * NR + r) * NL;
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < NL; ++j) {  // G^-1_kj conj(H_rj)
            sv.x = fmaf(gi[j].x, h[j].x, fmaf(gi[j].y, h[j].y, sv.x));
            sv.y = fmaf(gi[j].y, h[j].x, fmaf(-gi[j].x, h[j].y, sv.y));
        }
        const float fac = fmaxf(sFac[pu * NL + k], 0.f);
        const bool dead = !(sFac[pu * NL + k] > 0.f) || sFac[pu * NL] < 0.f;
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
    // PDL: global writes only after the previous grid completed
    pdl_wait();
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
    const float ia = rsqrtf(norm);
    const int sc = fb0 * kSc + f;
#pragma unroll 1
    for (int s = g; s < kSym; s += G) {
        mbar_wait(&bars[s], 0);
        if (!active) continue;
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
            if (s2 > 0.f) {
#pragma unroll
                for (int k = 0; k < NL; ++k) demap_layer<QM, false, LT>(x[k], slope[k], v + k * QM);
                uint32_t wd[kWords];
                pack_llr<LT, NL * QM, false>(v, wd);
                store_bytes<kLlrBytes>((char*)a.llr + re * kLlrBytes, wd);
            } else {
#pragma unroll
                for (int k = 0; k < NL; ++k) demap_layer<QM, true, LT>(x[k], slope[k], v + k * QM);
                uint32_t wd[kWords];
                pack_llr<LT, NL * QM, true>(v, wd);
                store_bytes<kLlrBytes>((char*)a.llr + re * kLlrBytes, wd);
            }
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

template <int NR, int NL, int QM, int LT, int P, int G>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_fb <= 0 || a.n_slots <= 0) return cudaSuccess;
    dim3 grid((a.n_fb + P - 1) / P, a.n_slots);
    return launch_kernel(k_prb<NR, NL, QM, LT, P, G>, grid, dim3(kSc * P * G), PrbSmem<NR, NL, P>::total, s,
                         a.overlap, a);
}

template <int NR, int NL, int QM, int LT, int P, int G>
cudaError_t prepare() {
    constexpr size_t smem = PrbSmem<NR, NL, P>::total;
    if (smem > 48 * 1024)
        return cudaFuncSetAttribute(k_prb<NR, NL, QM, LT, P, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    return cudaSuccess;
}

#define PRB_ENTRY(NAME, NR, NL, QM, LT, P, G) \
    KernelEntry { NAME, NR, NL, QM, kSc, 14, LT, 32, 1, launch<NR, NL, QM, LT, P, G>, prepare<NR, NL, QM, LT, P, G> }

const KernelEntry kEntries[] = {
    PRB_ENTRY("prb_8x4_q6_i8", 8, 4, 6, kLlrI8, 4, 2),  // C3
    PRB_ENTRY("prb_8x4_q6_f32", 8, 4, 6, kLlrF32, 4, 2),
    PRB_ENTRY("prb_8x4_q6_f16", 8, 4, 6, kLlrF16, 4, 2),
    PRB_ENTRY("prb_8x4_q4_i8", 8, 4, 4, kLlrI8, 4, 2),
    PRB_ENTRY("prb_4x4_q6_i8", 4, 4, 6, kLlrI8, 4, 2),
    PRB_ENTRY("prb_8x2_q6_i8", 8, 2, 6, kLlrI8, 4, 2),
};

}  // namespace

const KernelEntry* prb_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
