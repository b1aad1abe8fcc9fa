// k_big.cu -- massive-MIMO per-PRB detector (C5: 64 rx x 16 layers, 64-QAM,
// int8, H per PRB). The per-RE filter x~ = W~ y is a dense complex contraction
// (16 x 64 per RE, 1024 cMAC): on the FP32 SIMT pipe C5 is FP32-bound (SURVEY.md
// §8(d)); on the tensor cores (3-pass TF32, reading R21) it becomes HBM-bound.
//
//   k_big_setup (rows a2-a5), one warp per PRB-unit, warp-synchronous, fp32
//     (reading R18; cond(G) <= ~10 on C5): H by one bulk copy, G = H^H H + s2 I
//     (half a row per lane, broadcast 128-bit H reads), then G^-1 by in-place
//     Gauss-Jordan on the same lane layout (ALG = 1, default, reading R26; pivots
//     and rows by __shfl_sync, guard R17) -- or, ALG = 0, rows gathered to lane k,
//     Cholesky, X = L^-1 column per lane and row k of G^-1 = X^H X --, then
//     W~ = diag(sqrt(norm)/mu) G^-1 H^H (lane (k, half) covers half the antennas),
//     written to the plan workspace as [unit][r][k] plus slopes.
//   Apply kernels (rows a6-a7), all reading W~ from the workspace:
//   k_big_apply4: persistent, warp-specialised tcgen05 pipeline (TMA y chunks,
//     single-thread MMA issue, converter and epilogue warps); TA = 1 ("big8";
//     "big8e6" with six epilogue warps is the C5 default) keeps the y operand in
//     TMEM, TA = 2 ("big11") in fp16.
//   k_big_apply3: the same tensor-core computation, one CTA per unit.
//   k_big_apply2: SIMT, K-streamed TMA chunks, 4 x 4 complex register tile.
//   k_big_apply (other shapes / LLR types): SIMT, CTA per PRB-unit, the unit's
//     168 y vectors bulk-copied at a padded 528-byte stride, thread (RE pair,
//     layer half) accumulates 2 x 8 complex outputs.

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

// ------------------------------------------------------------------------
// tcgen05 / TMA building blocks for the tensor-core apply kernels (k_big_apply3/4).
// fp32-accurate products from TF32 units (reading R21): the tensor core reads an
// fp32 operand as TF32 (low 13 mantissa bits ignored, i.e. hi = trunc(x)), so
// A B = A_hi B_hi + A_hi B_lo + A_lo B_hi with B_lo = B - trunc(B) and
// A_lo = A - trunc(A); the dropped lo*lo term and the truncation of the lo
// parts are ~2^-20 relative per product.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    // start address >> 4 | LBO (unused for swizzled K-major) = 1 | SBO = 1024 B | version 1 | SWIZZLE_128B
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// A operand in TMEM (lane = row m, one 32-bit column per K element), B by smem descriptor.
__device__ __forceinline__ void umma_tf32_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_f16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
// fp16 hi/lo split of a pair (reading R27): hi = rn(a), lo = rn(a - hi); packed as one 32-bit word
// (low half = the even K element).
__device__ __forceinline__ void split_h2(float a0, float a1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a0, a1);
    const float2 f = __half22float2(h);
    unsigned long long ua, uf, ud;  // packed (a - f): one sub.f32x2
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(uf) : "f"(f.x), "f"(f.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ud) : "l"(ua), "l"(uf));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(ud));
    const __half2 l = __floats2half2_rn(d.x, d.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
        "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// ------------------------------------------------------------------------
// k_big_apply2: rows a6-a7 as a K-streamed SIMT GEMM.
// One CTA (168 threads) per PRB-unit; X~[16 x 168] = W~[16 x 64] Y[64 x 168]
// complex, K (= rx) streamed in 4 chunks of 16 antennas: each chunk is one TMA
// tile of the unit's 168 y rows x 128 B (3-D map {128 floats, n_sc, n_sym}, box
// {32, 12, 14}, SWIZZLE_128B: the 16-byte chunk c of RE row e sits at c ^ (e & 7),
// so 8 consecutive REs reading the same antennas hit 8 distinct bank groups).
// Two chunk stages (2 x 21 KiB) + W~ (8 KiB) keep 4 CTAs (21 warps) per SM.
// Thread t: layer quad lq = t & 3 (layers 4lq..4lq+3), RE quad q = t >> 2
// (REs q, q+42, q+84, q+126): a 4 x 4 complex register tile, 16 FFMA per
// 128-bit shared load. Epilogue: exact max-log demap of the 4 x 4 outputs,
// 24-byte (int8) LLR pieces per RE (4 threads = one contiguous 96-byte record).
struct Ap2 {
    static constexpr int ROWS = kRe;                        // 168
    static constexpr size_t chunk = (size_t)ROWS * 128;     // 21504 = 21 KiB
    static constexpr size_t y0 = 0;                         // 2 stages, 1024-aligned
    static constexpr size_t W = 2 * chunk;                  // [64][16] float2 + 16 slopes
    static constexpr size_t wbytes = 64 * 16 * 8 + 16 * 4;  // 8256
    static constexpr size_t bars = W + (wbytes + 127) / 128 * 128;  // 3 mbarriers
    static constexpr size_t total = bars + 64 + 1024;       // + alignment slack
    static constexpr int THREADS = 168;
};

template <int NR, int NL, int QM, int LT>
__global__ void __launch_bounds__(Ap2::THREADS, 4) k_big_apply2(DetectArgs a, const __grid_constant__ CUtensorMap ymap) {
    static_assert(NL == 16 && NR == 64, "k_big_apply2: 64 x 16");
    constexpr int WS = BigWs<NR, NL>::stride;
    constexpr int NCH = NR / 16;  // K chunks of 16 antennas
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(g + Ap2::bars);  // [0],[1] y stages, [2] W~
    const float2* sW = reinterpret_cast<const float2*>(g + Ap2::W);
    const float* sSlope = reinterpret_cast<const float*>(g + Ap2::W + 64 * 16 * 8);

    pdl_launch_dependents();
    const int t = threadIdx.x;
    const long long u = blockIdx.x;
    const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ymap)) : "memory");
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            mbar_arrive_expect_tx(&bars[c], (uint32_t)Ap2::chunk);
            tma_load_3d(base + (uint32_t)(Ap2::y0 + c * Ap2::chunk), &ymap, 32 * c, fb * kSc, slot * kSym, &bars[c]);
        }
    }
    __syncthreads();  // barriers initialised before anyone waits on them
    pdl_wait();       // W~ of this call's setup kernel is complete
    if (t == 0) {
        mbar_arrive_expect_tx(&bars[2], (uint32_t)Ap2::wbytes);
        bulk_g2s(g + Ap2::W, reinterpret_cast<const float*>(a.ws) + u * WS, (uint32_t)Ap2::wbytes, &bars[2]);
    }
    const int lq = t & 3, q = t >> 2;
    float2 acc[4][4];  // [RE e][layer kk]
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) acc[e][kk] = make_float2(0.f, 0.f);
    mbar_wait(&bars[2], 0);
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
        const int st = c & 1;
        mbar_wait(&bars[st], (uint32_t)((c >> 1) & 1));
        const unsigned char* ys = g + Ap2::y0 + st * Ap2::chunk;
#pragma unroll 2
        for (int j = 0; j < 8; ++j) {  // 16-byte chunk j = antennas 16c + 2j, 16c + 2j + 1
            float4 yv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = q + 42 * e;
                yv[e] = *reinterpret_cast<const float4*>(ys + row * 128 + ((j ^ (row & 7)) << 4));
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = 16 * c + 2 * j + h;
                const float4 w01 = *reinterpret_cast<const float4*>(sW + r * NL + 4 * lq);
                const float4 w23 = *reinterpret_cast<const float4*>(sW + r * NL + 4 * lq + 2);
                const float2 wk[4] = {make_float2(w01.x, w01.y), make_float2(w01.z, w01.w),
                                      make_float2(w23.x, w23.y), make_float2(w23.z, w23.w)};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 yr = h ? make_float2(yv[e].z, yv[e].w) : make_float2(yv[e].x, yv[e].y);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) acc[e][kk] = cmac(acc[e][kk], wk[kk], yr);
                }
            }
        }
        if (c + 2 < NCH) {
            __syncthreads();  // every thread is done with stage st
            if (t == 0) {
                mbar_arrive_expect_tx(&bars[st], (uint32_t)Ap2::chunk);
                tma_load_3d(base + (uint32_t)(Ap2::y0 + st * Ap2::chunk), &ymap, 32 * (c + 2), fb * kSc, slot * kSym,
                            &bars[st]);
            }
        }
    }
    float slope[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) slope[kk] = sSlope[4 * lq + kk];
    constexpr int kRec = NL * QM * LlrTraits<LT>::bytes;   // one RE record
    constexpr int kPiece = 4 * QM * LlrTraits<LT>::bytes;  // this thread's 4 layers
    const bool zf = !(a.sigma2 > 0.f);
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int ri = q + 42 * e;
        const int s = ri / kSc, f = ri % kSc;
        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
        if (a.llr) {
            float v[4 * QM];
            uint32_t wd[(kPiece + 3) / 4];
            if (!zf) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) demap_layer<QM, false, LT>(acc[e][kk], slope[kk], v + kk * QM);
                pack_llr<LT, 4 * QM, false>(v, wd);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) demap_layer<QM, true, LT>(acc[e][kk], slope[kk], v + kk * QM);
                pack_llr<LT, 4 * QM, true>(v, wd);
            }
            store_bytes<kPiece>((char*)a.llr + re * kRec + lq * kPiece, wd);
        }
        if (a.xhat) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                a.xhat[re * NL + 4 * lq + kk] = make_float2(acc[e][kk].x * ia, acc[e][kk].y * ia);
        }
    }
}

template <int NR, int NL, int QM, int LT>
cudaError_t launch_ap2(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap ymap;
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * NR), (cuuint64_t)a.n_sc, (cuuint64_t)a.n_sym};
    const cuuint64_t gstride[2] = {(cuuint64_t)NR * 8, (cuuint64_t)a.n_sc * NR * 8};
    const cuuint32_t box[3] = {32, (cuuint32_t)kSc, (cuuint32_t)kSym};
    const cuuint32_t estride[3] = {1, 1, 1};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(a.y), gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    constexpr int UPB = 4;
    cudaError_t e = launch_kernel(k_big_setup<NR, NL, QM, UPB>, dim3((unsigned)((a.n_units + UPB - 1) / UPB)),
                                  dim3(32 * UPB), UPB * SetupSmem<NR, NL>::per_unit, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.n_units);
    cfg.blockDim = dim3(Ap2::THREADS);
    cfg.dynamicSmemBytes = Ap2::total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_big_apply2<NR, NL, QM, LT>, a, ymap);
}

template <int NR, int NL, int QM, int LT>
cudaError_t prepare_ap2() {
    cudaError_t e = cudaFuncSetAttribute(k_big_setup<NR, NL, QM, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(4 * SetupSmem<NR, NL>::per_unit));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_big_apply2<NR, NL, QM, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Ap2::total);
}

// ------------------------------------------------------------------------
// k_big_apply3: rows a6-a7 on the tensor cores, one CTA (4 warps) per PRB-unit,
// two CTAs per SM. The 168 x 128 real GEMM  X^T = Y^T B  (reading R21: 3-pass
// TF32 split) is streamed over K in the same 4 TMA chunks as k_big_apply2
// (16 antennas = 128 B per RE row, SWIZZLE_128B = the canonical K-major UMMA
// layout). Per chunk c:
//   MMA1(c): A = y chunk (fp32 read as TF32 = y_hi), B = [B_hi; B_lo] rows of
//            K-tile c (N = 64): columns 0-31 += y_hi B_hi, 32-63 += y_hi B_lo;
//   SIMT   : y_lo = y - trunc(y) into a separate chunk buffer (no in-place
//            rewrite, so the y stage is released as soon as MMA1 has read it);
//   MMA2(c): A = y_lo chunk, B = B_hi rows (N = 32): columns 0-31 += y_lo B_hi.
// Two M = 128 tiles cover the 168 RE rows (rows 0-127 and 40-167), 64 TMEM
// columns each. B is built once per unit from W~ (plan workspace) by the SIMT
// threads: row n < 16 = Re output k = n (Wr, -Wi pairs), n >= 16 = Im output
// (Wi, Wr pairs), B_lo = B - trunc(B) at row n + 32. Epilogue: thread = TMEM
// lane = RE row, 64 columns -> x~_k = hi + lo, exact max-log demap, 96-byte
// record store. Thread 0 issues the MMAs (single-thread tcgen05.mma) and the
// TMA refills.
struct Ap3 {
    static constexpr int THREADS = 128;
    static constexpr size_t chunk = (size_t)kRe * 128;      // 21504
    static constexpr size_t y0 = 0;                         // 2 stages
    static constexpr size_t ylo = 2 * chunk;                // 1 buffer
    static constexpr size_t B = 3 * chunk;                  // 4 K-tiles x 64 rows x 128 B (1024-aligned)
    static constexpr size_t wraw = B + 4 * 64 * 128;        // W~ [64][16] float2 + 16 slopes
    static constexpr size_t wbytes = 64 * 16 * 8 + 16 * 4;  // 8256
    static constexpr size_t bars = wraw + 8320;             // 8 mbarriers
    static constexpr size_t tslot = bars + 64;
    static constexpr size_t total = tslot + 16 + 1024;
};
static_assert(Ap3::B % 1024 == 0, "B set must be 1024-aligned");

template <int NR, int NL, int QM, int LT>
__global__ void __launch_bounds__(Ap3::THREADS, 2) k_big_apply3(DetectArgs a, const __grid_constant__ CUtensorMap ymap) {
    static_assert(NL == 16 && NR == 64, "k_big_apply3: 64 x 16");
    constexpr int WS = BigWs<NR, NL>::stride;
    constexpr int NCH = 4;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    uint64_t* ybar = reinterpret_cast<uint64_t*>(g + Ap3::bars);  // [2]
    uint64_t* wbar = ybar + 2;
    uint64_t* m1bar = ybar + 3;
    uint64_t* m2bar = ybar + 4;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g + Ap3::tslot);
    const float2* sW = reinterpret_cast<const float2*>(g + Ap3::wraw);
    const float* sSlope = reinterpret_cast<const float*>(g + Ap3::wraw + 64 * 16 * 8);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    pdl_launch_dependents();
    const long long u = blockIdx.x;
    const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
    if (t == 0) {
        for (int i = 0; i < 5; ++i) mbar_init(&ybar[i], 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ymap)) : "memory");
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            mbar_arrive_expect_tx(&ybar[c], (uint32_t)Ap3::chunk);
            tma_load_3d(base + (uint32_t)(Ap3::y0 + c * Ap3::chunk), &ymap, 32 * c, fb * kSc, slot * kSym, &ybar[c]);
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    pdl_wait();  // W~ of this call's setup kernel is complete
    if (t == 0) {
        mbar_arrive_expect_tx(wbar, (uint32_t)Ap3::wbytes);
        bulk_g2s(g + Ap3::wraw, reinterpret_cast<const float*>(a.ws) + u * WS, (uint32_t)Ap3::wbytes, wbar);
    }
    mbar_wait(wbar, 0);
    {  // B set: thread -> row n = t >> 2 (output), K-tile kt = t & 3, 8 chunks of 2 antennas
        const int n = t >> 2, kt = t & 3, kk = n & 15;
        const bool im_row = n >= 16;
        float* kb = reinterpret_cast<float*>(g + Ap3::B + (size_t)kt * 64 * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int r0 = 16 * kt + 2 * c;
            const float2 w0 = sW[r0 * NL + kk], w1 = sW[(r0 + 1) * NL + kk];
            const float4 v = im_row ? make_float4(w0.y, w0.x, w1.y, w1.x) : make_float4(w0.x, -w0.y, w1.x, -w1.y);
            const float4 lo = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                          v.w - tf32_trunc(v.w));
            *reinterpret_cast<float4*>(kb + n * 32 + ((c ^ (n & 7)) << 2)) = v;
            *reinterpret_cast<float4*>(kb + (n + 32) * 32 + ((c ^ (n & 7)) << 2)) = lo;
        }
    }
    fence_proxy_async();
    __syncthreads();
    constexpr uint32_t id64 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t id32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t bbase = base + (uint32_t)Ap3::B;
    const uint32_t ylob = base + (uint32_t)Ap3::ylo;
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
        const int st = c & 1;
        const uint32_t ys = base + (uint32_t)(Ap3::y0 + st * Ap3::chunk);
        mbar_wait(&ybar[st], (uint32_t)((c >> 1) & 1));
        if (t == 0) {
            tc_fence_after();
#pragma unroll
            for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    umma_tf32(tmem + 64u * tile, umma_desc_sw128(ys + (tile ? 40u * 128u : 0u) + ks * 32u),
                              umma_desc_sw128(bbase + (uint32_t)c * 8192u + ks * 32u), id64, (c | ks) ? 1u : 0u);
            umma_commit(m1bar);
        }
        if (c >= 1) mbar_wait(m2bar, (uint32_t)((c - 1) & 1));  // y_lo buffer free
        {
            const float4* src = reinterpret_cast<const float4*>(g + Ap3::y0 + st * Ap3::chunk);
            float4* dst = reinterpret_cast<float4*>(g + Ap3::ylo);
            constexpr int n4 = (int)(Ap3::chunk / 16);
#pragma unroll 4
            for (int i = t; i < n4; i += Ap3::THREADS) {
                float4 v = src[i];
                v.x -= tf32_trunc(v.x);
                v.y -= tf32_trunc(v.y);
                v.z -= tf32_trunc(v.z);
                v.w -= tf32_trunc(v.w);
                dst[i] = v;
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            tc_fence_after();
#pragma unroll
            for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    umma_tf32(tmem + 64u * tile, umma_desc_sw128(ylob + (tile ? 40u * 128u : 0u) + ks * 32u),
                              umma_desc_sw128(bbase + (uint32_t)c * 8192u + ks * 32u), id32, 1u);
            umma_commit(m2bar);
            if (c + 2 < NCH) {
                mbar_wait(m1bar, (uint32_t)(c & 1));  // MMA1(c) has read stage st
                mbar_arrive_expect_tx(&ybar[st], (uint32_t)Ap3::chunk);
                tma_load_3d(ys, &ymap, 32 * (c + 2), fb * kSc, slot * kSym, &ybar[st]);
            }
        }
    }
    mbar_wait(m2bar, (uint32_t)((NCH - 1) & 1));
    tc_fence_after();
    // epilogue: tile 0 rows 0-127 (all warps), tile 1 rows 128-167 (= TMEM lanes 88-127 of tile 1)
    constexpr int kRec = NL * QM * LlrTraits<LT>::bytes;
    const bool zf = !(a.sigma2 > 0.f);
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll 1
    for (int tile = 0; tile < 2; ++tile) {
        if (tile == 1 && warp < 2) break;
        uint32_t hv[32], lv[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 64u * tile;
        tmem_ld32(taddr, hv);
        tmem_ld32(taddr + 32u, lv);
        const int row = (tile ? 40 : 0) + 32 * warp + lane;
        if (tile == 1 && row < 128) continue;
        const int s = row / kSc, f = row % kSc;
        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
        float2 x[NL];
#pragma unroll
        for (int k = 0; k < NL; ++k)
            x[k] = make_float2(__uint_as_float(hv[k]) + __uint_as_float(lv[k]),
                               __uint_as_float(hv[16 + k]) + __uint_as_float(lv[16 + k]));
        if (a.llr) {
            float v[NL * QM];
            uint32_t wd[(kRec + 3) / 4];
            if (!zf) {
#pragma unroll
                for (int k = 0; k < NL; ++k) demap_layer<QM, false, LT>(x[k], sSlope[k], v + k * QM);
                pack_llr<LT, NL * QM, false>(v, wd);
            } else {
#pragma unroll
                for (int k = 0; k < NL; ++k) demap_layer<QM, true, LT>(x[k], sSlope[k], v + k * QM);
                pack_llr<LT, NL * QM, true>(v, wd);
            }
            store_bytes<kRec>((char*)a.llr + re * kRec, wd);
        }
        if (a.xhat) {
#pragma unroll
            for (int k = 0; k < NL; ++k) a.xhat[re * NL + k] = make_float2(x[k].x * ia, x[k].y * ia);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

template <int NR, int NL, int QM, int LT>
cudaError_t launch_ap3(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap ymap;
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * NR), (cuuint64_t)a.n_sc, (cuuint64_t)a.n_sym};
    const cuuint64_t gstride[2] = {(cuuint64_t)NR * 8, (cuuint64_t)a.n_sc * NR * 8};
    const cuuint32_t box[3] = {32, (cuuint32_t)kSc, (cuuint32_t)kSym};
    const cuuint32_t estride[3] = {1, 1, 1};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(a.y), gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    constexpr int UPB = 4;
    cudaError_t e = launch_kernel(k_big_setup<NR, NL, QM, UPB>, dim3((unsigned)((a.n_units + UPB - 1) / UPB)),
                                  dim3(32 * UPB), UPB * SetupSmem<NR, NL>::per_unit, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)a.n_units);
    cfg.blockDim = dim3(Ap3::THREADS);
    cfg.dynamicSmemBytes = Ap3::total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_big_apply3<NR, NL, QM, LT>, a, ymap);
}

template <int NR, int NL, int QM, int LT>
cudaError_t prepare_ap3() {
    cudaError_t e = cudaFuncSetAttribute(k_big_setup<NR, NL, QM, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(4 * SetupSmem<NR, NL>::per_unit));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_big_apply3<NR, NL, QM, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Ap3::total);
}

// ------------------------------------------------------------------------
// k_big_apply4: the k_big_apply3 computation as a persistent, warp-specialised
// pipeline (one CTA per SM, 288 threads) so that loads, tensor-core passes,
// y_lo conversion and the demap epilogue of different chunks / units overlap:
//   warp 8 lane 0  control: TMA producer (y chunks S = 4 stages ahead, W~ of
//                  unit i+2) and single-thread tcgen05.mma issuer;
//   warps 0-3      converters: B(i) from W~ (hi/lo, double-buffered), y -> y_lo
//                  per chunk (2 y_lo buffers);
//   warps 4-7      epilogue: TMEM (2 accumulator buffers x 128 columns) ->
//                  x~ -> exact max-log demap -> LLR stores.
// Chunk g = 4 i + c of the CTA's i-th unit (u = blockIdx.x + i gridDim.x).
// mbarrier k-th completion is waited with parity k & 1.
template <int S_, int NLO_, int TR_ = 0, int TRW_ = 96, int TA_ = 0>
struct Ap4 {
    static constexpr int S = S_;                             // y stages
    static constexpr int TRW = TRW_;                         // TR: transpose-buffer width (REs)
    static constexpr int TRS = TRW + 4;                      // TR: floats per accumulator row in the stage (pad: banks)
    static constexpr int NLO = NLO_;                         // y_lo buffers
    static constexpr size_t chunk = (size_t)kRe * 128;       // 21504 = 21 x 1024
    static constexpr size_t y0 = 0;
    static constexpr size_t ylo = S * chunk;
    static constexpr size_t B = ylo + (TA_ ? 0 : NLO * chunk);  // 2 x 32 KiB (1024-aligned)
    static constexpr size_t bset = 4 * 64 * 128;
    static constexpr size_t slope = B + 2 * bset;            // [4][16] float (unit i -> slot i & 3)
    static constexpr size_t tb = slope + 512;                // TR: [TRW][TRS] float (slope area: [4][16] + [4] inv)
    static constexpr size_t bars = tb + (TR_ ? (size_t)64 * TRS * 4 : 0);  // mbarriers
    static constexpr int NBAR = 2 * S + 2 * NLO + 2 * 3;     // yfull, yfree | ylofull, ylofree | bready, accfull, tfree
    static constexpr size_t tslot = bars + NBAR * 8;
    static constexpr size_t total = tslot + 16 + 1024;
    static_assert(B % 1024 == 0 && ylo % 1024 == 0, "UMMA operand alignment");
    static_assert(total <= 227 * 1024, "shared memory");
};

// TR = 1 ("big5"): the transposed product  X[64 x 168] = [B_hi; B_lo][64 x 128] Y^T[128 x 168]
// with the W~ set as the M = 64 A operand and the unit's 168 y rows as one N = 168 B operand:
// 4 + 4 tcgen05.mma per chunk instead of 16 (two M = 128 tiles x hi|lo and lo passes), no
// duplicated rows. The M = 64 accumulator puts row m in TMEM lane (m % 16) + 32 (m / 16),
// column n = RE, so the epilogue transposes through shared memory (96 REs at a time; with
// EW = 8 all 168 at once, two warps per TMEM lane quadrant).
// TA = 1 ("big8"): the A operand (y rows, hi and lo) lives in TMEM instead of shared memory.
// The converter warps read each y row once from the TMA stage (warp w serves TMEM lane quadrant
// w: rows 32w + lane of tile 0 and 40 + 32w + lane of tile 1; a compact tile 1 -- REs 128-167
// in lanes 0-39 only -- measured slower, 383 vs 352 us: it piles converter and epilogue work on
// the same two SM sub-partitions), store it raw (the tensor core reads
// its TF32 truncation = y_hi) and as y_lo = y - trunc(y) with tcgen05.st, so the MMAs read only
// the small W~ operand from shared memory; the TMA stage is released as soon as it is read.
// TMEM: columns 0-255 accumulators (2 x 128), 256-511 the A ring (NLO = 2 chunks x 2 tiles x hi|lo
// x 32 columns). Measured per step (C5): 352 us against big4's 402 us. Not better: a hybrid that keeps
// the y_hi pass in shared memory (only y_lo in TMEM, 4-deep ring) 372 us; three N = 32 passes into
// one 32-column accumulator (3-deep ring) 430 us -- an A-in-TMEM tf32 MMA costs ~81 cycles against
// ~50 for an SS one (tools/tcbench.cu), so the MMA count matters more than the ring depth.
template <int NR, int NL, int QM, int LT, int EW, int S_, int NLO_, int ABL, int TR, int TA = 0>
__global__ void __launch_bounds__(32 * (6 + EW), 1) k_big_apply4(DetectArgs a, const __grid_constant__ CUtensorMap ymap) {
    using A4 = Ap4<S_, NLO_, TR, (TR && EW == 8) ? kRe : 96, TA>;
    static_assert(!TA || (!TR && NLO_ == 2), "TA: untransposed, two A buffers");
    // EW = 6 (TA only): warps 4-7 take tile 0 of their lane quadrant, warps 8-9 tile 1, which is
    // compact (REs 128-167 in lanes 0-39 of quadrants 0, 1): one epilogue pass per warp per unit
    constexpr bool CT = EW == 6;
    static_assert(!CT || TA, "EW 6: TMEM A operand only");
    constexpr uint32_t kTmemCols = (TR || TA) ? 512u : 256u;
    constexpr uint32_t kAccStride = TR ? 256u : 128u;
    constexpr uint32_t kAring = 256u;  // TA: first TMEM column of the A ring
    constexpr int CW = 4 + EW;  // control warp (MMA issuer); CW + 1: TMA producer
    constexpr int NLO = NLO_;
    static_assert(NL == 16 && NR == 64, "k_big_apply4: 64 x 16");
    constexpr int WS = BigWs<NR, NL>::stride;
    constexpr int S = A4::S;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(g + A4::bars);
    uint64_t* yfull = bar;            // [S]  TMA tx
    uint64_t* yfree = bar + S;        // [S]  MMA1 commit + converters (count 2)
    uint64_t* ylofull = bar + 2 * S;  // [NLO]  converters
    uint64_t* ylofree = ylofull + NLO;  // [NLO]  MMA2 commit
    uint64_t* bready = ylofree + NLO;  // [2]  converters
    uint64_t* accfull = bready + 2;   // [2]  commit after the unit's last MMA
    uint64_t* tfree = accfull + 2;    // [2]  epilogue done with the TMEM buffer
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g + A4::tslot);
    float* sslope = reinterpret_cast<float*>(g + A4::slope);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long u0 = blockIdx.x, du = gridDim.x;
    const long long n_my = u0 < a.n_units ? (a.n_units - u0 + du - 1) / du : 0;
    const long long G = 4 * n_my;

    pdl_launch_dependents();
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&yfull[i], 1);
            mbar_init(&yfree[i], TA ? 1 : 2);
        }
        for (int i = 0; i < NLO; ++i) {
            mbar_init(&ylofull[i], 1);
            mbar_init(&ylofree[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bready[i], 1);
            mbar_init(&accfull[i], 1);
            mbar_init(&tfree[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == CW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    auto issue_y = [&](long long gg) {
        const long long uu = u0 + (gg >> 2) * du;
        const int slot = (int)(uu / a.n_fb), fb = (int)(uu % a.n_fb), st = (int)(gg % S);
        mbar_arrive_expect_tx(&yfull[st], (uint32_t)A4::chunk);
        tma_load_3d(base + (uint32_t)(A4::y0 + st * A4::chunk), &ymap, 32 * (int)(gg & 3), fb * kSc, slot * kSym,
                    &yfull[st]);
    };

    if (warp == CW + 1) {
        // ================= TMA producer: y chunks, S stages ahead =================
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ymap)) : "memory");
#pragma unroll 1
            for (long long gg = 0; gg < G; ++gg) {
                const int st = (int)(gg % S);
                if (gg >= S) mbar_wait(&yfree[st], (uint32_t)(((gg / S) + 1) & 1));  // MMA1 + conversion of gg - S
                issue_y(gg);
            }
        }
    } else if (warp == CW) {
        // ================= control: MMA issuer =================
        if (lane == 0) {
            constexpr uint32_t id64 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
            constexpr uint32_t id32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
#pragma unroll 1
            for (long long i = 0; i < n_my; ++i) {
                const int b = (int)(i & 1);
                mbar_wait(&bready[b], (uint32_t)((i >> 1) & 1));
                if (i >= 2) mbar_wait(&tfree[b], (uint32_t)(((i >> 1) + 1) & 1));
                constexpr uint32_t idT = (1u << 4) | (2u << 7) | (2u << 10) | (((uint32_t)kRe >> 3) << 17) | ((64u >> 4) << 24);
                const uint32_t acc = tmem + kAccStride * (uint32_t)b;
                const uint32_t bb = base + (uint32_t)(A4::B + b * A4::bset);
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    const long long gg = 4 * i + c;
                    const int st = (int)(gg % S), lb = (int)(gg % NLO);
                    if constexpr (TA == 2) {  // fp16 hi/lo (R27): 2 K-steps of 16 per chunk, 8 MMAs
                        constexpr uint32_t h64 = (1u << 4) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
                        constexpr uint32_t h32 = (1u << 4) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
                        const uint32_t ab = tmem + kAring + 64u * (uint32_t)lb;  // A ring buffer lb
                        mbar_wait(&ylofull[lb], (uint32_t)((gg / NLO) & 1));
                        tc_fence_after();
                        const uint32_t wb = bb + (uint32_t)(c >> 1) * 8192u + (uint32_t)(c & 1) * 64u;
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 2; ++ks) {
                                umma_f16_ta(acc + 64u * tile, ab + 32u * tile + 8u * ks, umma_desc_sw128(wb + ks * 32u),
                                            h64, (c | ks) ? 1u : 0u);
                                umma_f16_ta(acc + 64u * tile, ab + 32u * tile + 16u + 8u * ks,
                                            umma_desc_sw128(wb + ks * 32u), h32, 1u);
                            }
                        umma_commit(&ylofree[lb]);
                        if (c == 3) umma_commit(&accfull[b]);
                        continue;
                    }
                    if constexpr (TA) {
                        const uint32_t ab = tmem + kAring + 128u * (uint32_t)lb;  // A ring buffer lb
                        mbar_wait(&ylofull[lb], (uint32_t)((gg / NLO) & 1));
                        tc_fence_after();
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                umma_tf32_ta(acc + 64u * tile, ab + 64u * tile + 8u * ks,
                                             umma_desc_sw128(bb + (uint32_t)c * 8192u + ks * 32u), id64, (c | ks) ? 1u : 0u);
#pragma unroll
                        for (int tile = 0; tile < (ABL & 4 ? 0 : 2); ++tile)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                umma_tf32_ta(acc + 64u * tile, ab + 64u * tile + 32u + 8u * ks,
                                             umma_desc_sw128(bb + (uint32_t)c * 8192u + ks * 32u), id32, 1u);
                        umma_commit(&ylofree[lb]);
                        if (c == 3) umma_commit(&accfull[b]);
                        continue;
                    }
                    const uint32_t ys = base + (uint32_t)(A4::y0 + st * A4::chunk);
                    mbar_wait(&yfull[st], (uint32_t)((gg / S) & 1));
                    tc_fence_after();
                    if constexpr (TR) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            umma_tf32(acc, umma_desc_sw128(bb + (uint32_t)c * 8192u + ks * 32u),
                                      umma_desc_sw128(ys + ks * 32u), idT, (c | ks) ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                umma_tf32(acc + 64u * tile, umma_desc_sw128(ys + (tile ? 40u * 128u : 0u) + ks * 32u),
                                          umma_desc_sw128(bb + (uint32_t)c * 8192u + ks * 32u), id64,
                                          (c | ks) ? 1u : 0u);
                    }
                    umma_commit(&yfree[st]);
                    mbar_wait(&ylofull[lb], (uint32_t)((gg / NLO) & 1));
                    tc_fence_after();
                    const uint32_t yl = base + (uint32_t)(A4::ylo + lb * A4::chunk);
                    if constexpr (TR) {  // A = [B_hi; B_lo]: also adds the (tiny) lo*lo term
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            umma_tf32(acc, umma_desc_sw128(bb + (uint32_t)c * 8192u + ks * 32u),
                                      umma_desc_sw128(yl + ks * 32u), idT, 1u);
                    } else if constexpr (!(ABL & 4)) {
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                umma_tf32(acc + 64u * tile, umma_desc_sw128(yl + (tile ? 40u * 128u : 0u) + ks * 32u),
                                          umma_desc_sw128(bb + (uint32_t)c * 8192u + ks * 32u), id32, 1u);
                    }
                    umma_commit(&ylofree[lb]);
                    if (c == 3) umma_commit(&accfull[b]);
                }
            }
        }
    } else if (warp < 4) {
        // ================= converters =================
        // W~ of the next unit is prefetched into registers (plain coherent loads; the setup kernel wrote it)
        // while the current unit's chunks are converted.
        const int tc = t;  // 0..127
        const int n = tc >> 2, kt = tc & 3, kk = n & 15;
        const bool im_row = n >= 16;
        pdl_wait();  // W~ of this call's setup kernel is complete and visible
        float2 wv[16];
        float slv = 0.f;
        float3 scl = make_float3(1.f, 1.f, 1.f);  // TA 2: (sy, sw, inv) of the prefetched unit
        auto fetch = [&](long long i) {
            const float2* src = reinterpret_cast<const float2*>(reinterpret_cast<const float*>(a.ws) + (u0 + i * du) * WS);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int r0 = 16 * kt + 2 * c;
                wv[2 * c] = src[r0 * NL + kk];
                wv[2 * c + 1] = src[(r0 + 1) * NL + kk];
            }
            if (tc < NL) slv = reinterpret_cast<const float*>(src + NR * NL)[tc];
            if constexpr (TA == 2) {
                const float* sc = reinterpret_cast<const float*>(src + NR * NL) + NL;
                scl = make_float3(sc[0], sc[1], sc[2]);
            }
        };
        if (n_my > 0) fetch(0);
#pragma unroll 1
        for (long long i = 0; i < n_my; ++i) {
            const int b = (int)(i & 1);
            // B buffer b is free once unit i-2's MMAs completed; slopes use a 4-deep ring (unit i+4 reuses
            // slot i & 3 only after accfull(i+2), which the control issues after tfree(i): epilogue(i) done)
            if (i >= 2) mbar_wait(&accfull[b], (uint32_t)(((i >> 1) + 1) & 1));
            const float sy = scl.x;  // this unit's y scale (scl is overwritten by the prefetch below)
            if constexpr (TA == 2) {
                // B (fp16, SW128 K-major): K-tile kt2 = kt / 2 holds chunks 2 kt2, 2 kt2 + 1 (64 fp16 per row);
                // this thread's 16 antennas are 16-byte chunks 4 (kt & 1) + j, j = 0..3, of rows n and n + 32
                unsigned char* kb = g + A4::B + b * A4::bset + (size_t)(kt >> 1) * 8192;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t hv[4], lv[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const float2 w = make_float2(wv[4 * j + m].x * scl.y, wv[4 * j + m].y * scl.y);
                        if (im_row) split_h2(w.y, w.x, hv[m], lv[m]);
                        else split_h2(w.x, -w.y, hv[m], lv[m]);
                    }
                    const int q = 4 * (kt & 1) + j;
                    *reinterpret_cast<uint4*>(kb + n * 128 + ((q ^ (n & 7)) << 4)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
                    *reinterpret_cast<uint4*>(kb + (n + 32) * 128 + ((q ^ (n & 7)) << 4)) =
                        make_uint4(lv[0], lv[1], lv[2], lv[3]);
                }
                if (tc < NL) sslope[(i & 3) * 16 + tc] = slv;
                if (tc == 0) sslope[64 + (i & 3)] = scl.z;
            } else {
                float* kb = reinterpret_cast<float*>(g + A4::B + b * A4::bset + (size_t)kt * 64 * 128);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float2 w0 = wv[2 * c], w1 = wv[2 * c + 1];
                    const float4 v = im_row ? make_float4(w0.y, w0.x, w1.y, w1.x) : make_float4(w0.x, -w0.y, w1.x, -w1.y);
                    const float4 lo = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                                  v.w - tf32_trunc(v.w));
                    *reinterpret_cast<float4*>(kb + n * 32 + ((c ^ (n & 7)) << 2)) = v;
                    *reinterpret_cast<float4*>(kb + (n + 32) * 32 + ((c ^ (n & 7)) << 2)) = lo;
                }
                if (tc < NL) sslope[(i & 3) * 16 + tc] = slv;
            }
            fence_proxy_async();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (tc == 0) mbar_arrive(&bready[b]);
            if (i + 1 < n_my) fetch(i + 1);
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                const long long gg = 4 * i + c;
                const int st = (int)(gg % S), lb = (int)(gg % NLO);
                mbar_wait(&yfull[st], (uint32_t)((gg / S) & 1));
                if (gg >= NLO) mbar_wait(&ylofree[lb], (uint32_t)(((gg / NLO) + 1) & 1));
                if constexpr (TA) {
                    // tile 0: REs 32 w + lane; tile 1: REs 40 + 32 w + lane -> TMEM lane quadrant w
                    tc_fence_after();
                    const unsigned char* ysm = g + A4::y0 + st * A4::chunk;
#pragma unroll
                    for (int tile = 0; tile < (ABL & 1 ? 0 : 2); ++tile) {
                        if (CT && tile == 1 && warp >= 2) break;  // compact tile 1: REs 128-167 in lanes 0-39
                        const int r = tile ? (CT ? min(128 + 32 * warp + lane, kRe - 1) : 40 + 32 * warp + lane)
                                           : 32 * warp + lane;
                        const float4* row = reinterpret_cast<const float4*>(ysm + (size_t)r * 128);
                        float v[32], lo[32];
#pragma unroll
                        for (int cc = 0; cc < 8; ++cc) {
                            const float4 q = row[cc ^ (r & 7)];  // SWIZZLE_128B: 16-byte chunk cc of row r
                            v[4 * cc] = q.x;
                            v[4 * cc + 1] = q.y;
                            v[4 * cc + 2] = q.z;
                            v[4 * cc + 3] = q.w;
                        }
                        if constexpr (TA == 2) {  // fp16 pairs: columns 0-15 y_hi, 16-31 y_lo (scaled by sy)
                            uint32_t pk[32];
                            if (sy != 1.f) {  // uniform per unit; 1 for O(1)-scaled inputs
#pragma unroll
                                for (int k = 0; k < 32; ++k) v[k] *= sy;
                            }
#pragma unroll
                            for (int k2 = 0; k2 < 16; ++k2) split_h2(v[2 * k2], v[2 * k2 + 1], pk[k2], pk[16 + k2]);
                            tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + kAring + 64u * (uint32_t)lb + 32u * tile,
                                      reinterpret_cast<const float*>(pk));
                        } else {
#pragma unroll
                            for (int k = 0; k < 32; ++k) lo[k] = v[k] - tf32_trunc(v[k]);
                            const uint32_t ta =
                                tmem + ((uint32_t)(32 * warp) << 16) + kAring + 128u * (uint32_t)lb + 64u * tile;
                            tmem_st32(ta, v);
                            tmem_st32(ta + 32u, lo);
                        }
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (tc == 0) {
                        mbar_arrive(&ylofull[lb]);
                        mbar_arrive(&yfree[st]);
                    }
                    continue;
                }
                const float4* src = reinterpret_cast<const float4*>(g + A4::y0 + st * A4::chunk);
                float4* dst = reinterpret_cast<float4*>(g + A4::ylo + lb * A4::chunk);
                constexpr int n4 = (int)(A4::chunk / 16);
                if constexpr (!(ABL & 1)) {  // ABL: timing ablations (wrong results), never selected by default
#pragma unroll 4
                    for (int q = tc; q < n4; q += 128) {
                        float4 v = src[q];
                        v.x -= tf32_trunc(v.x);
                        v.y -= tf32_trunc(v.y);
                        v.z -= tf32_trunc(v.z);
                        v.w -= tf32_trunc(v.w);
                        dst[q] = v;
                    }
                }
                fence_proxy_async();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (tc == 0) {
                    mbar_arrive(&ylofull[lb]);
                    mbar_arrive(&yfree[st]);
                }
            }
        }
    } else {
        // ================= epilogue =================
        // EW = 4: warp 4+q reads TMEM lane quadrant q, all 16 layers of its RE rows;
        // EW = 8: warps 4+q and 8+q share quadrant q, layers 8h .. 8h+7 each (h = e >> 2).
        const int e = warp - 4, we = e & 3, h = EW == 8 ? (e >> 2) : 0;
        constexpr int KL = EW == 8 ? NL / 2 : NL;  // layers per thread
        constexpr int kRec = NL * QM * LlrTraits<LT>::bytes;
        constexpr int kPiece = KL * QM * LlrTraits<LT>::bytes;
        const bool zf = !(a.sigma2 > 0.f);
        const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll 1
        for (long long i = 0; i < n_my; ++i) {
            const int b = (int)(i & 1);
            const long long u = u0 + i * du;
            const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
            mbar_wait(&accfull[b], (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            if constexpr (TR) {
                // rows 16q..16q+15 of quadrant q = (Re hi | Im hi | Re lo | Im lo) x 16 layers, column = RE
                // (EW = 8: the two warps of a quadrant take alternate 32-column blocks, and TRW = 168
                // so one pass covers the unit with one RE per epilogue thread)
                float* T = reinterpret_cast<float*>(g + A4::tb);
                const int tid = t - 128;
                const uint32_t tq = tmem + ((uint32_t)(32 * we) << 16) + kAccStride * (uint32_t)b;
                constexpr int NPASS = (kRe + A4::TRW - 1) / A4::TRW;
#pragma unroll 1
                for (int p = 0; p < NPASS; ++p) {
                    const int n0 = p * A4::TRW, wcol = (kRe - n0 < A4::TRW) ? kRe - n0 : A4::TRW;
#pragma unroll 1
                    for (int c0 = 32 * h; c0 < wcol; c0 += 32 * (EW / 4)) {
                        uint32_t v[32];
                        if (wcol - c0 >= 32) {
                            tmem_ld32(tq + (uint32_t)(n0 + c0), v);
                        } else {
                            tmem_ld8(tq + (uint32_t)(n0 + c0), v);
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        }
                        if (lane < 16) {  // accumulator row m = 16 we + lane, 128-bit stores along the REs
                            const int nc = wcol - c0 >= 32 ? 32 : 8;
                            float* trow = T + (16 * we + lane) * A4::TRS + c0;
#pragma unroll
                            for (int j4 = 0; j4 < 8; ++j4)
                                if (4 * j4 < nc)
                                    *reinterpret_cast<float4*>(trow + 4 * j4) =
                                        make_float4(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1]),
                                                    __uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3]));
                        }
                    }
                    asm volatile("bar.sync 2, %0;" ::"r"(32 * EW) : "memory");
                    if (tid < wcol) {
                        const int row = n0 + tid;
                        const int s = row / kSc, f = row % kSc;
                        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
                        float q[64];  // column tid of the 64 accumulator rows (consecutive threads: conflict-free)
#pragma unroll
                        for (int m = 0; m < 64; ++m) q[m] = T[m * A4::TRS + tid];
                        float2 x[NL];
#pragma unroll
                        for (int k = 0; k < NL; ++k) x[k] = make_float2(q[k] + q[32 + k], q[16 + k] + q[48 + k]);
                        const float* sl = sslope + (i & 3) * 16;
                        if (a.llr && !(ABL & 2)) {
                            float vv[NL * QM];
                            uint32_t wd[(kRec + 3) / 4];
                            if (!zf) {
#pragma unroll
                                for (int k = 0; k < NL; ++k) demap_layer<QM, false, LT>(x[k], sl[k], vv + k * QM);
                                pack_llr<LT, NL * QM, false>(vv, wd);
                            } else {
#pragma unroll
                                for (int k = 0; k < NL; ++k) demap_layer<QM, true, LT>(x[k], sl[k], vv + k * QM);
                                pack_llr<LT, NL * QM, true>(vv, wd);
                            }
                            store_bytes<kRec>((char*)a.llr + re * kRec, wd);
                        }
                        if (a.xhat) {
#pragma unroll
                            for (int k = 0; k < NL; ++k) a.xhat[re * NL + k] = make_float2(x[k].x * ia, x[k].y * ia);
                        }
                    }
                    asm volatile("bar.sync 2, %0;" ::"r"(32 * EW) : "memory");
                }
            }
#pragma unroll 1
            for (int tile = CT ? (e >> 2) : 0; tile < (TR ? 0 : (CT ? (e >> 2) + 1 : 2)); ++tile) {
                if (!CT && tile == 1 && we < 2) break;
                uint32_t hr[KL], hi[KL], lr[KL], li[KL];
                const uint32_t taddr = tmem + ((uint32_t)(32 * we) << 16) + kAccStride * (uint32_t)b + 64u * tile + KL * h;
                if constexpr (KL == 16) {
                    uint32_t hv[32], lv[32];
                    tmem_ld32(taddr, hv);
                    tmem_ld32(taddr + 32u, lv);
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        hr[k] = hv[k];
                        hi[k] = hv[16 + k];
                        lr[k] = lv[k];
                        li[k] = lv[16 + k];
                    }
                } else {
                    tmem_ld8(taddr, hr);
                    tmem_ld8(taddr + 16u, hi);
                    tmem_ld8(taddr + 32u, lr);
                    tmem_ld8(taddr + 48u, li);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                }
                const int row = (tile ? (CT ? 128 : 40) : 0) + 32 * we + lane;
                if (tile == 1 && (CT ? row >= kRe : row < 128)) continue;
                const int s = row / kSc, f = row % kSc;
                const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
                float2 x[KL];
#pragma unroll
                for (int k = 0; k < KL; ++k)
                    x[k] = make_float2(__uint_as_float(hr[k]) + __uint_as_float(lr[k]),
                                       __uint_as_float(hi[k]) + __uint_as_float(li[k]));
                if constexpr (TA == 2) {  // undo the fp16 path's scales (exact; 1 for O(1)-scaled units)
                    const float xs = sslope[64 + (i & 3)];
                    if (xs != 1.f) {
#pragma unroll
                        for (int k = 0; k < KL; ++k) x[k] = make_float2(x[k].x * xs, x[k].y * xs);
                    }
                }
                const float* sl = sslope + (i & 3) * 16 + KL * h;
                if (a.llr && !(ABL & 2)) {
                    float v[KL * QM];
                    uint32_t wd[(kPiece + 3) / 4];
                    if (!zf) {
#pragma unroll
                        for (int k = 0; k < KL; ++k) demap_layer<QM, false, LT>(x[k], sl[k], v + k * QM);
                        pack_llr<LT, KL * QM, false>(v, wd);
                    } else {
#pragma unroll
                        for (int k = 0; k < KL; ++k) demap_layer<QM, true, LT>(x[k], sl[k], v + k * QM);
                        pack_llr<LT, KL * QM, true>(v, wd);
                    }
                    store_bytes<kPiece>((char*)a.llr + re * kRec + h * kPiece, wd);
                }
                if (a.xhat) {
#pragma unroll
                    for (int k = 0; k < KL; ++k)
                        a.xhat[re * NL + KL * h + k] = make_float2(x[k].x * ia, x[k].y * ia);
                }
            }
            tc_fence_before();
            asm volatile("bar.sync 2, %0;" ::"r"(32 * EW) : "memory");
            if (t == 128) mbar_arrive(&tfree[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == CW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

template <int NR, int NL, int QM, int LT, int EW, int S_, int NLO_, int ABL = 0, int TR = 0, int SALG = 1, int TA = 0>
cudaError_t launch_ap4(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap ymap;
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * NR), (cuuint64_t)a.n_sc, (cuuint64_t)a.n_sym};
    const cuuint64_t gstride[2] = {(cuuint64_t)NR * 8, (cuuint64_t)a.n_sc * NR * 8};
    const cuuint32_t box[3] = {32, (cuuint32_t)kSc, (cuuint32_t)kSym};
    const cuuint32_t estride[3] = {1, 1, 1};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(a.y), gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    constexpr int UPB = 4;
    cudaError_t e = launch_kernel(k_big_setup<NR, NL, QM, UPB, SALG>, dim3((unsigned)((a.n_units + UPB - 1) / UPB)),
                                  dim3(32 * UPB), UPB * SetupSmem<NR, NL, SALG>::per_unit, s, a.overlap, a);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.n_units < n_sm ? a.n_units : n_sm));
    cfg.blockDim = dim3(32 * (6 + EW));
    cfg.dynamicSmemBytes = Ap4<S_, NLO_, TR, (TR && EW == 8) ? kRe : 96, TA>::total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_big_apply4<NR, NL, QM, LT, EW, S_, NLO_, ABL, TR, TA>, a, ymap);
}

template <int NR, int NL, int QM, int LT, int EW, int S_, int NLO_, int ABL = 0, int TR = 0, int SALG = 1, int TA = 0>
cudaError_t prepare_ap4() {
    cudaError_t e = cudaFuncSetAttribute(k_big_setup<NR, NL, QM, 4, SALG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(4 * SetupSmem<NR, NL, SALG>::per_unit));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_big_apply4<NR, NL, QM, LT, EW, S_, NLO_, ABL, TR, TA>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Ap4<S_, NLO_, TR, (TR && EW == 8) ? kRe : 96, TA>::total);
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

#define BIGAP2_ENTRY(NAME, NR, NL, QM, LT)                                                               \
    KernelEntry {                                                                                         \
        NAME, NR, NL, QM, kSc, 14, LT, 32, 2, launch_ap2<NR, NL, QM, LT>, prepare_ap2<NR, NL, QM, LT>,   \
            workspace<NR, NL>                                                                             \
    }

const KernelEntry kEntries[] = {
#define BIG4_ENTRY(NAME, EW, S, NLO)                                                                       \
    KernelEntry {                                                                                          \
        NAME, 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, EW, S, NLO>,                \
            prepare_ap4<64, 16, 6, kLlrI8, EW, S, NLO>, workspace<64, 16>                                  \
    }
    // C5 default: big4's tcgen05 3-pass TF32 pipeline with the y operand (hi, lo) in TMEM and six epilogue
    // warps (tile 0 on warps 4-7, compact tile 1 on warps 8-9)
    KernelEntry{"big8e6_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 6, 4, 2, 0, 0, 1, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 6, 4, 2, 0, 0, 1, 1>, workspace<64, 16>},
    KernelEntry{"big8_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 0, 1, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 0, 1, 1>, workspace<64, 16>},
    BIG4_ENTRY("big4_64x16_q6_i8", 4, 4, 2),  // y_lo through a shared-memory ring
    // big11: big8 with fp16 hi/lo operands (reading R27): K = 16 per MMA, 8 MMAs per chunk instead of 16
    KernelEntry{"big11_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 0, 1, 2>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 0, 1, 2>, workspace<64, 16>},
    BIG4_ENTRY("big4e8_64x16_q6_i8", 8, 4, 2),
    // big4 with the Cholesky / L^-1 / X^H X setup route instead of Gauss-Jordan (reading R26)
    KernelEntry{"big4c_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 0, 0>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 0, 0>, workspace<64, 16>},
    KernelEntry{"big5_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 0, 1>, workspace<64, 16>},
    KernelEntry{"ablation_big8_noconv", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 1, 0, 1, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 1, 0, 1, 1>, workspace<64, 16>},
    KernelEntry{"ablation_big8_none", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3, 0, 1, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3, 0, 1, 1>, workspace<64, 16>},
    KernelEntry{"big11e6_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 6, 4, 2, 0, 0, 1, 2>,
                prepare_ap4<64, 16, 6, kLlrI8, 6, 4, 2, 0, 0, 1, 2>, workspace<64, 16>},
    KernelEntry{"ablation_big11_noepi", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 2, 0, 1, 2>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 2, 0, 1, 2>, workspace<64, 16>},
    KernelEntry{"ablation_big11_none", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3, 0, 1, 2>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3, 0, 1, 2>, workspace<64, 16>},
    KernelEntry{"ablation_big11_noconv", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 1, 0, 1, 2>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 1, 0, 1, 2>, workspace<64, 16>},
    KernelEntry{"ablation_big8_noepi", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 2, 0, 1, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 2, 0, 1, 1>, workspace<64, 16>},
    KernelEntry{"ablation_big8_mma1", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 4, 0, 1, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 4, 0, 1, 1>, workspace<64, 16>},
    KernelEntry{"big5e8_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 8, 3, 2, 0, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 8, 3, 2, 0, 1>, workspace<64, 16>},
    KernelEntry{"ablation_big5_none", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3, 1>, workspace<64, 16>},
    // timing ablations (results are wrong on purpose; only reachable through MIMO_FORCE_KERNEL)
    KernelEntry{"ablation_big4_noconv", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 1>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 1>, workspace<64, 16>},
    KernelEntry{"ablation_big4_noepi", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 2>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 2>, workspace<64, 16>},
    KernelEntry{"ablation_big4_none", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 3>, workspace<64, 16>},
    KernelEntry{"ablation_big4_mma1", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 7>,
                prepare_ap4<64, 16, 6, kLlrI8, 4, 4, 2, 7>, workspace<64, 16>},
    BIGAP2_ENTRY("big2_64x16_q6_i8", 64, 16, 6, kLlrI8),  // SIMT K-streamed apply
    BIG_ENTRY("big_64x16_q6_i8", 64, 16, 6, kLlrI8),
    KernelEntry{"big3_64x16_q6_i8", 64, 16, 6, kSc, 14, kLlrI8, 32, 2, launch_ap3<64, 16, 6, kLlrI8>,
                prepare_ap3<64, 16, 6, kLlrI8>, workspace<64, 16>},
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
