// big_setup.cuh -- the SIMT per-unit setup of the 16-layer per-PRB families
// (rows a2-a5 for n_rx = 32 / 64, 16 layers): one warp per H-unit, writing the
// W~ workspace [unit][r][k] float2 + slopes that the apply kernels read.
// Included by k_big.cu (SIMT apply, other shapes / LLR types) and k_c5.cu
// (the SIMT-setup variant of the C5 tensor-core pipeline).
#pragma once

#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;
constexpr int kSc = 12;
constexpr int kRe = kSym * kSc;  // 168 REs per PRB-unit

template <int NR, int NL>
struct BigWs {
    static constexpr int w_floats = NR * NL * 2;                 // W~ [r][k] float2
    static constexpr int stride = (w_floats + NL + 3 + 31) / 32 * 32; // + slopes, 3 fp16-apply scales (128-B multiple)
};

__device__ __forceinline__ float2 shfl2(float2 v, int src) {
    return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// One warp per PRB-unit (UPB units per CTA), warp-synchronous, no CTA barriers.
template <int NR, int NL, int ALG = 1>
struct SetupSmem {
    // sH [NR][NL] float2 | sX [NL][NL] float2 | sDinv [NL] float (Cholesky route only) | mbarrier
    static constexpr size_t h = 0;
    static constexpr size_t x = (size_t)NR * NL * 8;
    static constexpr size_t dinv = x + (ALG == 0 ? (size_t)NL * NL * 8 : 0);
    static constexpr size_t bar = (dinv + (ALG == 0 ? NL * 4 : 0) + 7) / 8 * 8;
    static constexpr size_t per_unit = (bar + 8 + 15) / 16 * 16;
};

template <int NR, int NL, int QM, int UPB, int ALG = 1>
__global__ void __launch_bounds__(32 * UPB) k_big_setup(DetectArgs a) {
    static_assert(NL == 16 && NR % 32 == 0, "k_big_setup: 16 layers, NR multiple of 32");
    constexpr int WS = BigWs<NR, NL>::stride;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    using SS = SetupSmem<NR, NL, ALG>;
    unsigned char* base = smem + (size_t)warp * SS::per_unit;
    float2* sH = reinterpret_cast<float2*>(base + SS::h);         // [r][l]
    float2* sX = reinterpret_cast<float2*>(base + SS::x);         // L rows, then X = L^-1 [i][j]
    float* sDinv = reinterpret_cast<float*>(base + SS::dinv);
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + SS::bar);

    pdl_launch_dependents();
    const long long u = (long long)blockIdx.x * UPB + warp;
    const bool valid = u < a.n_units;
    const float s2 = unit_sigma2(a, valid ? u : 0);
    const float norm = (float)qam_norm(QM);
    if (valid && lane == 0) {  // a1: the unit's H (8 KiB) by one bulk copy
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, (uint32_t)(NR * NL * 8));
        bulk_g2s(sH, a.H + u * NR * NL, (uint32_t)(NR * NL * 8), bar);
    }
    __syncwarp();
    if (valid) mbar_wait(bar, 0);
    // a2: lane -> row i = lane/2, columns 8h .. 8h+7 of G (broadcast H reads)
    float2 gq[8];
    {
        const int i = lane >> 1, h = lane & 1;
#pragma unroll
        for (int q = 0; q < 8; ++q) gq[q] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int r = 0; r < NR; ++r) {  // packed FFMA2: gq[q] += conj(H_ri) H_r,8h+q
            const CPack hi = cpack_conj(sH[r * NL + i]);
            const float4* hr = reinterpret_cast<const float4*>(sH + r * NL + 8 * h);
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
                const float4 v = hr[q2];
                gq[2 * q2] = cmac_p(gq[2 * q2], hi, make_float2(v.x, v.y));
                gq[2 * q2 + 1] = cmac_p(gq[2 * q2 + 1], hi, make_float2(v.z, v.w));
            }
        }
    }
    // ||H||_F^2 = trace(H^H H): the mean receive power per antenna is ||H||^2 / NR + s2 (unit-power
    // symbols); the fp16 apply (big11) scales y by a power of two derived from it
    float trH = 0.f;
    {
        const int i = lane >> 1, h = lane & 1;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (8 * h + q == i) trH = gq[q].x;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) trH += __shfl_xor_sync(0xffffffffu, trH, off);
    }
    int k, half;         // W~ lanes: row k of G^-1, antenna half
    float2 gi[NL];       // row k of G^-1
    float sinr, fac;
    bool fail;
    if constexpr (ALG == 1) {
        // a3-a4 (reading R26): in-place Gauss-Jordan inversion of G (Hermitian PD: no pivoting),
        // lane (k, h) = (lane / 2, lane % 2) keeps G[k][8h .. 8h+7] from the Gram. Step j: pivot
        // p_j = G[j][j] (the LDL^H pivot = square of Cholesky's d_jj, guard R17), row j scaled by
        // 1/p_j and broadcast by shuffles, every other row k updated with f = G[k][j].
        k = lane >> 1;
        half = lane & 1;
        const int h = half;
        float gd = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (8 * h + q == k) {
                gq[q] = make_float2(gq[q].x + s2, 0.f);
                gd = gq[q].x;
            }
        float gmax = gd;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
        fail = !(gmax == gmax);
        const float tau = (float)kPivotTau * gmax;
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const int hj = j >> 3, qj = j & 7;
            const float2 f = shfl2(gq[qj], (lane & ~1) | hj);    // G[k][j]
            float p = __shfl_sync(0xffffffffu, gq[qj].x, 2 * j + hj);  // G[j][j]
            if (!(p > tau)) {
                fail = true;
                p = 1.f;
            }
            const float pinv = 1.f / p;
            const bool prow = k == j;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float2 rj = shfl2(gq[q], 2 * j + h);                 // G[j][8h+q]
                if (8 * h + q == j) rj = make_float2(1.f, 0.f);
                rj = make_float2(rj.x * pinv, rj.y * pinv);
                float2 b = (8 * h + q == j) ? make_float2(0.f, 0.f) : gq[q];
                b.x = fmaf(-f.x, rj.x, fmaf(f.y, rj.y, b.x));
                b.y = fmaf(-f.x, rj.y, fmaf(-f.y, rj.x, b.y));
                gq[q] = prow ? rj : b;
            }
        }
        // row k of G^-1: own half + the partner lane's half
        float A = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float2 o = shfl2(gq[q], lane ^ 1);
            gi[q] = h ? o : gq[q];
            gi[8 + q] = h ? gq[q] : o;
        }
#pragma unroll
        for (int j = 0; j < NL; ++j)
            if (j == k) A = gi[j].x;
        const float mu = fmaf(-s2, A, 1.f);
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
    } else {
        // a3: Cholesky, lane k (and its duplicate k+16) holds row k
        k = lane & 15;
        half = lane >> 4;
        float2 g[NL];  // row k of G: columns 0-7 from lane 2k, 8-15 from lane 2k+1
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            g[q] = shfl2(gq[q], 2 * k);
            g[8 + q] = shfl2(gq[q], 2 * k + 1);
        }
#pragma unroll
        for (int j = 0; j < NL; ++j)
            if (j == k) g[j] = make_float2(g[j].x + s2, 0.f);
        float gmax = 0.f;
#pragma unroll
        for (int j = 0; j < NL; ++j)
            if (j == k) gmax = g[j].x;
#pragma unroll
        for (int off = 1; off < NL; off <<= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
        fail = !(gmax == gmax);
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
    }
    // W~[r][k] = fac_k sum_j G^-1_kj conj(H_rj): lane (k, half) covers r in [half*NR/2, (half+1)*NR/2)
    pdl_wait();  // the previous call may still read the workspace
    if (valid) {
        float2* ws = reinterpret_cast<float2*>(reinterpret_cast<float*>(a.ws) + u * WS);
        float wmax = 0.f;
        CPackC gp[NL];  // packed FFMA2: sv += G^-1_kj conj(H_rj)
#pragma unroll
        for (int j = 0; j < NL; ++j) gp[j] = cpackc(gi[j]);
#pragma unroll 2
        for (int rr = 0; rr < NR / 2; ++rr) {
            const int r = half * (NR / 2) + rr;
            const float4* hr = reinterpret_cast<const float4*>(sH + r * NL);
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int j2 = 0; j2 < NL / 2; ++j2) {
                const float4 v = hr[j2];
                sv = cmacc_p(sv, gp[2 * j2], make_float2(v.x, v.y));
                sv = cmacc_p(sv, gp[2 * j2 + 1], make_float2(v.z, v.w));
            }
            const float2 w = fac > 0.f ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
            ws[r * NL + k] = w;
            wmax = fmaxf(wmax, fmaxf(fabsf(w.x), fabsf(w.y)));
        }
        if (half == 0) {
            reinterpret_cast<float*>(ws)[NR * NL * 2 + k] = sinr / norm * a.llr_scale;
            if (a.sinr) a.sinr[u * NL + k] = sinr;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
        if (lane == 0) {  // reading R27: sy = 2^-ey, sw = 2^-ew bring y and W~ to O(1); inv = 2^(ey + ew)
            const float py = sqrtf(trH / (float)NR + s2);
            int ey = 0, ew = 0;
            if (py > 0.f && py < 3.0e38f) frexpf(py, &ey);
            if (wmax > 0.f && wmax < 3.0e38f) frexpf(wmax, &ew);
            float* sc = reinterpret_cast<float*>(ws) + NR * NL * 2 + NL;
            sc[0] = ldexpf(1.f, -ey);
            sc[1] = ldexpf(1.f, -ew);
            sc[2] = ldexpf(1.f, ey + ew);
        }
        if (lane == 0 && fail) atomicAdd(a.fail_count, 1ull);
    }
}

}  // namespace
}  // namespace mimo
