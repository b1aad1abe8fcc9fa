// k_split.cu -- two-kernel detector for per-PRB channels (C3: 8 rx x 4 layers,
// 64-QAM, int8 -- H shared by 12 subcarriers x 14 symbols = 168 REs).
//
// A per-PRB W~ (NL x NR complex) is reused by 168 REs, so it costs < 2% of the
// y traffic to write it once to a plan-owned workspace and read it back
// (L2-resident) -- which lets each phase run at its own best shape:
//   k_setup_units (rows a2-a5): CTA of UPC units, fp32 setup cooperatively in
//     shared memory (Gram entries over threads, one thread per unit for the
//     Cholesky / L^-1 / G^-1 / mu / SINR chain, W~ entries over threads;
//     reading R18), writes W~ (PAM level units), slopes, SINR, fail count;
//   k_apply_units (rows a6-a7): a pure streaming kernel, one thread per
//     (subcarrier, group of 14/G symbols): its y loads are issued first, then
//     W~ of its unit (L1/L2 broadcast to the 12 lanes of a PRB), x~ = W~ y,
//     exact max-log demap, direct vector stores.
// With MIMO_PLAN_OVERLAP_CALLS (PDL) the setup of call i+1 overlaps the apply
// tail of call i, and the y loads of each apply overlap its setup's tail;
// writes always follow griddepcontrol.wait.
#include <cstdlib>

#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;

// workspace layout per unit: W~ [NL][NR] float2, then slope [NL] float (padded)
template <int NR, int NL>
struct UnitWs {
    static constexpr int w_floats = NL * NR * 2;
    static constexpr int stride = ((w_floats + NL) + 7) / 8 * 8;  // floats per unit, 32-byte multiple
};

__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}

template <int NR, int NL, int QM, int UPC>
__global__ void __launch_bounds__(128) k_setup_units(DetectArgs a) {
    constexpr int T = 128;
    constexpr int NE = NL * (NL + 1) / 2;
    constexpr int WS = UnitWs<NR, NL>::stride;
    __shared__ float2 sH[UPC * NR * NL];
    __shared__ float2 sGi[UPC * NL * NL];
    __shared__ float sFac[UPC * NL];
    __shared__ float sSinr[UPC * NL];
    __shared__ int sFail[UPC];

    pdl_launch_dependents();
    const int t = threadIdx.x;
    const long long u0 = (long long)blockIdx.x * UPC;
    const int nu = (int)min((long long)UPC, a.n_units - u0);
    const float norm = (float)qam_norm(QM);
    const float sqn = sqrtf(norm);
    float* ws = reinterpret_cast<float*>(a.ws);

    // a1: H of the CTA's units (contiguous)
    {
        const float4* src = reinterpret_cast<const float4*>(a.H + u0 * NR * NL);
        float4* dst = reinterpret_cast<float4*>(sH);
        for (int i = t; i < nu * NR * NL / 2; i += T) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    // a2: Gram lower triangle
    for (int idx = t; idx < nu * NE; idx += T) {
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
        if (i == j) acc = make_float2(acc.x + unit_sigma2(a, u0 + pu), 0.f);
        sGi[(pu * NL + i) * NL + j] = acc;
    }
    __syncthreads();
    // a3-a5: one thread per unit
    if (t < nu) {
        const float s2 = unit_sigma2(a, u0 + t);
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
                        sinr = __fdividef(mu, s2 * A);
                        fac = __fdividef(sqn, mu);
                    }
                    if (!(mu > 0.f) || fail) {
                        sinr = 0.f;
                        fac = 0.f;
                    }
                    sSinr[t * NL + i] = sinr;
                    sFac[t * NL + i] = fac;
                }
            }
        sFail[t] = fail;
    }
    __syncthreads();
    // W~ = diag(sqrt(norm)/mu) G^-1 H^H -> registers (written after pdl_wait)
    constexpr int kPer = (UPC * NL * NR + T - 1) / T;
    float2 wv[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int idx = t + q * T;
        wv[q] = make_float2(0.f, 0.f);
        if (idx < nu * NL * NR) {
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
            wv[q] = (fac > 0.f && !sFail[pu]) ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
        }
    }
    pdl_wait();  // the previous call (which may still read the workspace) has completed
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int idx = t + q * T;
        if (idx < nu * NL * NR) {
            const int pu = idx / (NL * NR), kr = idx % (NL * NR);
            reinterpret_cast<float2*>(ws + (u0 + pu) * WS)[kr] = wv[q];
        }
    }
    for (int idx = t; idx < nu * NL; idx += T) {
        const int pu = idx / NL, k = idx % NL;
        const float sinr = sFail[pu] ? 0.f : sSinr[idx];
        ws[(u0 + pu) * WS + NL * NR * 2 + k] = sinr / norm * a.llr_scale;
        if (a.sinr) a.sinr[(u0 + pu) * NL + k] = sinr;
    }
    if (t < nu && sFail[t]) atomicAdd(a.fail_count, 1ull);
}

// One thread per (subcarrier, symbol group g of G): symbols g, g+G, ... of its slot.
template <int NR, int NL, int QM, int LT, int G, int SCPH>
__global__ void __launch_bounds__(128) k_apply_units(DetectArgs a) {
    constexpr int NS = (kSym + G - 1) / G;
    constexpr int WS = UnitWs<NR, NL>::stride;
    pdl_launch_dependents();
    const int sc = blockIdx.x * blockDim.x + threadIdx.x;
    const int slot = blockIdx.y / G, g = blockIdx.y % G;
    const bool active = sc < a.n_sc;
    float2 yv[NS][NR];
    if (active) {
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            const int s = g + i * G;
            if (s < kSym)
                load_bytes<NR * 8>(a.y + ((size_t)(slot * kSym + s) * a.n_sc + sc) * NR,
                                   reinterpret_cast<uint32_t*>(&yv[i][0]));
        }
    }
    pdl_wait();  // W~ of this call's setup kernel is complete
    if (!active) return;
    const size_t unit = (size_t)slot * (a.n_sc / SCPH) + sc / SCPH;
    const float* wsu = reinterpret_cast<const float*>(a.ws) + unit * WS;
    float2 w[NL][NR];
    static_assert((NL * NR * 8) % 32 == 0, "W~ rows in 32-byte chunks");
#pragma unroll
    for (int i = 0; i < NL * NR * 8 / 32; ++i)
        ld_v8_coherent(wsu + 8 * i, reinterpret_cast<uint32_t*>(&w[0][0]) + 8 * i);
    float slope[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) slope[k] = wsu[NL * NR * 2 + k];
    constexpr int kLlrBytes = NL * QM * LlrTraits<LT>::bytes;
    constexpr int kWords = (kLlrBytes + 3) / 4;
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const int s = g + i * G;
        if (s >= kSym) break;
        float2 x[NL];
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc = cmac(acc, w[k][r], yv[i][r]);
            x[k] = acc;
        }
        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + sc;
        if (a.llr) {
            float v[NL * QM];
            uint32_t wd[kWords];
            if (a.sigma2 > 0.f) {
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

// Streaming apply with a register prefetch ring: thread (g, sc) walks symbols
// g, g+G, ... of its slot keeping PF y vectors in flight (continuous HBM
// traffic instead of one burst per thread).
// KS = symbols sharing one H (sym_per_h; 14 = one H per slot): a "slot" of this kernel is one H time block
// of KS symbols (a.n_slots = n_sym / KS blocks), so time-varying channels (KS = 7, 2, 1) take the same code
template <int NR, int NL, int QM, int LT, int G, int PF, int SCPH, int MINB, int KS = kSym>
__global__ void __launch_bounds__(128, MINB) k_apply_stream(DetectArgs a) {
    constexpr int NS = (KS + G - 1) / G;
    constexpr int WS = UnitWs<NR, NL>::stride;
    static_assert(PF >= 1 && PF <= NS, "prefetch distance");
    pdl_launch_dependents();
    const int sc = blockIdx.x * blockDim.x + threadIdx.x;
    const int slot = blockIdx.y / G, g = blockIdx.y % G;
    const bool active = sc < a.n_sc;
    float2 ring[PF][NR];
    if (active) {
#pragma unroll
        for (int i = 0; i < PF; ++i) {
            const int s = g + i * G;
            if (s < KS)
                load_bytes<NR * 8>(a.y + ((size_t)(slot * KS + s) * a.n_sc + sc) * NR,
                                   reinterpret_cast<uint32_t*>(&ring[i][0]));
        }
    }
    pdl_wait();
    if (!active) return;
    const size_t unit = (size_t)slot * (a.n_sc / SCPH) + sc / SCPH;
    const float* wsu = reinterpret_cast<const float*>(a.ws) + unit * WS;
    float2 w[NL][NR];
#pragma unroll
    for (int i = 0; i < NL * NR * 8 / 32; ++i)
        ld_v8_coherent(wsu + 8 * i, reinterpret_cast<uint32_t*>(&w[0][0]) + 8 * i);
    float slope[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) slope[k] = wsu[NL * NR * 2 + k];
    constexpr int kLlrBytes = NL * QM * LlrTraits<LT>::bytes;
    constexpr int kWords = (kLlrBytes + 3) / 4;
    const bool zf = !(a.sigma2 > 0.f);
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const int s = g + i * G;
        if (s >= KS) break;
        float2 yv[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) yv[r] = ring[i % PF][r];
        const int sn = g + (i + PF) * G;
        if (i + PF < NS && sn < KS)
            load_bytes<NR * 8>(a.y + ((size_t)(slot * KS + sn) * a.n_sc + sc) * NR,
                               reinterpret_cast<uint32_t*>(&ring[i % PF][0]));
        float2 x[NL];
#pragma unroll
        for (int k = 0; k < NL; ++k) x[k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < NR; ++r) {  // packed FFMA2, y_r shared by the NL layers
            const float2 ny = make_float2(-yv[r].y, yv[r].x);
#pragma unroll
            for (int k = 0; k < NL; ++k) x[k] = cmac_y(x[k], w[k][r], yv[r], ny);
        }
        const size_t re = (size_t)(slot * KS + s) * a.n_sc + sc;
        if (a.llr) {
            float v[NL * QM];
            uint32_t wd[kWords];
            if (!zf) {
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
            const float ia = rsqrtf((float)qam_norm(QM));
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

// k_apply_bfp: the k_apply_units apply with the y loads replaced by fused
// block-floating-point decompression (reading R25): per
// (symbol, PRB, antenna) one block of roundup4(1 + 3W) bytes (exponent byte,
// then 24 W-bit two's-complement mantissas MSB-first). Per symbol the CTA's
// blocks (<= 12 PRBs x 8 antennas, contiguous) are copied into shared memory with
// coalesced 16-byte cp.async (double-buffered, next symbol in flight); thread
// (subcarrier f of its PRB) reads the exponent and the one or two 32-bit words
// holding its 2W bits (I then Q), byte-swaps them into a big-endian 64-bit window
// and extracts the signed mantissas with arithmetic shifts: y = m * 2^e * scale.
// The raw fp32 y never exists in HBM: y traffic drops from 64 B to
// 8 * roundup4(1 + 3W) / 12 B per RE (18.7 B at W = 9).
template <int NR, int NL, int QM, int LT, int G>
__global__ void __launch_bounds__(128, 4) k_apply_bfp(DetectArgs a, const uint32_t* __restrict__ yb, int W, float scale) {
    constexpr int NS = (kSym + G - 1) / G;
    constexpr int WS = UnitWs<NR, NL>::stride;
    constexpr int kMaxPrb = 12;                     // a 128-subcarrier CTA touches at most 12 PRBs
    __shared__ __align__(16) uint32_t sb[2][kMaxPrb * NR * 13];  // 2 symbols x (PRBs x antennas x <= 52-byte blocks)
    pdl_launch_dependents();
    const int sc0 = blockIdx.x * blockDim.x;
    const int sc = sc0 + threadIdx.x;
    const int slot = blockIdx.y / G, g = blockIdx.y % G;
    const bool active = sc < a.n_sc;
    const int bw = ((1 + 3 * W) + 3) >> 2;         // 32-bit words per block
    const int n_prb = a.n_sc / 12;
    const int p0 = sc0 / 12, p1 = min(n_prb, (sc0 + (int)blockDim.x + 11) / 12);
    const int span16 = (p1 - p0) * NR * bw / 4;     // 16-byte chunks of the CTA's blocks in one symbol
    const int prb = sc / 12, f = sc % 12;
    const int bit0 = 8 + 2 * f * W;                 // stream position of this subcarrier's I mantissa
    const int wi = bit0 >> 5, sh = bit0 & 31;
    const bool two = sh + 2 * W > 32;
    // cooperative, coalesced 16-byte async copies of one symbol's blocks into a shared buffer
    auto fetch = [&](int i, int buf) {
        const int s = g + i * G;
        if (s < kSym) {
            const uint32_t* src = yb + ((size_t)(slot * kSym + s) * n_prb + p0) * NR * bw;
            for (int q = threadIdx.x; q < span16; q += blockDim.x)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&sb[buf][4 * q])),
                             "l"(src + 4 * q) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch(0, 0);
    pdl_wait();  // W~ of this call's setup kernel is complete
    const size_t unit = (size_t)slot * n_prb + (active ? prb : p0);
    const float* wsu = reinterpret_cast<const float*>(a.ws) + unit * WS;
    float2 w[NL][NR];
    static_assert((NL * NR * 8) % 32 == 0, "W~ rows in 32-byte chunks");
#pragma unroll
    for (int i = 0; i < NL * NR * 8 / 32; ++i)
        ld_v8_coherent(wsu + 8 * i, reinterpret_cast<uint32_t*>(&w[0][0]) + 8 * i);
    float slope[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) slope[k] = wsu[NL * NR * 2 + k];
    constexpr int kLlrBytes = NL * QM * LlrTraits<LT>::bytes;
    constexpr int kWords = (kLlrBytes + 3) / 4;
    const bool zf = !(a.sigma2 > 0.f);
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll 1
    for (int i = 0; i < NS; ++i) {
        const int s = g + i * G;
        if (s >= kSym) break;
        fetch(i + 1, (i + 1) & 1);                   // next symbol streams in while this one is decoded
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const uint32_t* rowb = &sb[i & 1][(prb - p0) * NR * bw];
        float2 yv[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const uint32_t* blk = rowb + r * bw;
            const uint32_t e = blk[0] & 0xFu, a0 = blk[wi], a1 = two ? blk[wi + 1] : 0u;
            const unsigned long long win =
                (((unsigned long long)__byte_perm(a0, 0, 0x0123) << 32) | __byte_perm(a1, 0, 0x0123)) << sh;
            const int mi = (int)(((long long)win) >> (64 - W));
            const int mq = (int)(((long long)(win << W)) >> (64 - W));
            const float step = scale * __int_as_float((127 + (int)e) << 23);  // scale * 2^e
            yv[r] = make_float2((float)mi * step, (float)mq * step);
        }
        __syncthreads();                              // buffer i & 1 is refilled two iterations later
        if (!active) continue;
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
            if (!zf) {
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

template <int QM, int LT, int G>
cudaError_t launch_bfp_g(const DetectArgs& a, const uint32_t* yb, int W, float scale, cudaStream_t s) {
    const unsigned g1 = (unsigned)((a.n_units + 15) / 16);
    cudaError_t e = launch_kernel(k_setup_units<8, 4, QM, 16>, dim3(g1), dim3(128), 0, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((a.n_sc + 127) / 128, a.n_slots * G);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_apply_bfp<8, 4, QM, LT, G>, a, yb, W, scale);
}

// symbols per thread = 14 / G (G = 2: measured best of 1, 2, 7, 14 in round 1)
template <int QM, int LT>
cudaError_t launch_bfp_t(const DetectArgs& a, const uint32_t* yb, int W, float scale, cudaStream_t s) {
    return launch_bfp_g<QM, LT, 2>(a, yb, W, scale, s);
}

template <int QM>
cudaError_t launch_bfp_q(const DetectArgs& a, const uint32_t* yb, int W, float scale, cudaStream_t s) {
    switch (a.llr_type) {
    case kLlrF32: return launch_bfp_t<QM, kLlrF32>(a, yb, W, scale, s);
    case kLlrF16: return launch_bfp_t<QM, kLlrF16>(a, yb, W, scale, s);
    default: return launch_bfp_t<QM, kLlrI8>(a, yb, W, scale, s);
    }
}

template <int NR, int NL, int QM, int LT, int UPC, int G, int PF, int SCPH, int MINB, int KS = kSym>
cudaError_t launch_stream(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    const unsigned g1 = (unsigned)((a.n_units + UPC - 1) / UPC);
    cudaError_t e = launch_kernel(k_setup_units<NR, NL, QM, UPC>, dim3(g1), dim3(128), 0, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    dim3 g2((a.n_sc + 127) / 128, a.n_slots * G);
    return launch_kernel(k_apply_stream<NR, NL, QM, LT, G, PF, SCPH, MINB, KS>, g2, dim3(128), 0, s, a.overlap, a);
}

template <int NR, int NL>
size_t workspace(const DetectArgs& a) {
    return (size_t)a.n_units * UnitWs<NR, NL>::stride * 4;
}

template <int NR, int NL, int QM, int LT, int UPC, int G, int SCPH>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    const unsigned g1 = (unsigned)((a.n_units + UPC - 1) / UPC);
    cudaError_t e = launch_kernel(k_setup_units<NR, NL, QM, UPC>, dim3(g1), dim3(128), 0, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    dim3 g2((a.n_sc + 127) / 128, a.n_slots * G);
    return launch_kernel(k_apply_units<NR, NL, QM, LT, G, SCPH>, g2, dim3(128), 0, s, a.overlap, a);
}

#define SPLIT_ENTRY(NAME, NR, NL, QM, LT, SCPH, UPC, G)                                              \
    KernelEntry {                                                                                    \
        NAME, NR, NL, QM, SCPH, 14, LT, 32, 2, launch<NR, NL, QM, LT, UPC, G, SCPH>, nullptr,        \
            workspace<NR, NL>                                                                        \
    }

#define STREAM_ENTRY(NAME, NR, NL, QM, LT, SCPH, UPC, G, PF) STREAM_ENTRY_B(NAME, NR, NL, QM, LT, SCPH, UPC, G, PF, 1)
#define STREAM_ENTRY_B(NAME, NR, NL, QM, LT, SCPH, UPC, G, PF, MINB)                                 \
    KernelEntry {                                                                                    \
        NAME, NR, NL, QM, SCPH, 14, LT, 32, 2, launch_stream<NR, NL, QM, LT, UPC, G, PF, SCPH, MINB>,    \
            nullptr, workspace<NR, NL>                                                               \
    }

// time-varying channels on the C3 shape (SPEC.md:481 leaves per-slot vs per-symbol W open; NEXT-3): one H per
// KS symbols and PRB, the setup per (block, PRB) unit and the streaming apply over blocks of KS symbols
#define STREAM_TV_ENTRY(NAME, NR, NL, QM, LT, SCPH, UPC, G, PF, MINB, KS)                             \
    KernelEntry {                                                                                    \
        NAME, NR, NL, QM, SCPH, KS, LT, 32, 2, launch_stream<NR, NL, QM, LT, UPC, G, PF, SCPH, MINB, KS>, \
            nullptr, workspace<NR, NL>                                                               \
    }

const KernelEntry kEntries[] = {
    STREAM_ENTRY_B("stream_8x4_q6_i8", 8, 4, 6, kLlrI8, 12, 16, 2, 2, 4),  // C3: <= 128 regs -> 4 CTAs/SM
    STREAM_TV_ENTRY("stream_8x4_q6_i8_s7", 8, 4, 6, kLlrI8, 12, 16, 1, 2, 4, 7),
    STREAM_TV_ENTRY("stream_8x4_q6_i8_s2", 8, 4, 6, kLlrI8, 12, 16, 1, 2, 4, 2),
    STREAM_TV_ENTRY("stream_8x4_q6_i8_s1", 8, 4, 6, kLlrI8, 12, 16, 1, 1, 4, 1),
    SPLIT_ENTRY("split_8x4_q6_i8", 8, 4, 6, kLlrI8, 12, 32, 7),
    SPLIT_ENTRY("split_8x4_q6_f32", 8, 4, 6, kLlrF32, 12, 32, 7),
    SPLIT_ENTRY("split_8x4_q6_f16", 8, 4, 6, kLlrF16, 12, 32, 7),
};

}  // namespace

bool bfp_supported(int n_rx, int n_layers, int sc_per_h, int sym_per_h) {
    return n_rx == 8 && n_layers == 4 && sc_per_h == 12 && sym_per_h == kSym;
}

size_t bfp_workspace(const DetectArgs& a) { return (size_t)a.n_units * UnitWs<8, 4>::stride * 4; }

cudaError_t launch_bfp(const DetectArgs& a, const void* y_bfp, int W, float scale, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    const uint32_t* yb = static_cast<const uint32_t*>(y_bfp);
    switch (a.qm) {
    case 2: return launch_bfp_q<2>(a, yb, W, scale, s);
    case 4: return launch_bfp_q<4>(a, yb, W, scale, s);
    case 6: return launch_bfp_q<6>(a, yb, W, scale, s);
    default: return launch_bfp_q<8>(a, yb, W, scale, s);
    }
}

const KernelEntry* split_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
