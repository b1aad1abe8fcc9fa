// k_lg.cu -- "lane group per H-unit" detector for per-subcarrier channels with
// many layers (C4: 16 rx x 8 layers, 256-QAM, fp16). W~ (NL x NR) does not fit
// one thread, so NL lanes of a warp share a unit: lane k owns layer k.
//
// Mapping (DESIGN.md §"Kernels"): a CTA owns TU = (32/NL) * NW consecutive
// subcarriers of one slot. Thread 0 bulk-copies the CTA's H tile (one
// mbarrier) and its 14 y rows (one mbarrier per row). Per unit, rows a2-a5 run
// in fp32 (reading R18) inside the lane group, warp-synchronously:
//   a2  lane k forms row k of G = H^H H + s2 I from the H tile;
//   a3  right-looking Cholesky: lane k keeps row k of the trailing matrix, the
//       pivot and column j are broadcast by __shfl_sync (guard R17);
//   a4  lane j forms column j of X = L^-1 (L rows via shared memory) and
//       A_jj = sum_i |X_ij|^2, then row j of G^-1 = X^H X and of W = G^-1 H^H;
//   a5  mu_k, SINR_k, W~_k = W_k sqrt(norm) / mu_k kept in lane k's registers.
// Per symbol, each lane reads the RE's y from the row tile (broadcast within
// the group), forms x~_k = W~_k y (row a6), demaps its layer (row a7) and
// writes its QM LLRs; the NL lanes of a unit write one contiguous RE record.
#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;

template <int NR, int NL, int NW, int KS = kSym>
struct LgSmem {
    static constexpr int UPW = 32 / NL;
    static constexpr int TU = UPW * NW;
    // per-unit strides padded by 16-32 B so the UPW units of a warp hit distinct banks
    static constexpr int YS = NR + 2;                                   // float2 per unit in a y row
    static constexpr int HS = NR * NL + 4;                              // float2 per unit H
    static constexpr int LS = NL * NL + 4;                              // float2 per unit L / X
    static constexpr size_t bars = 0;                                   // 15 mbarriers
    static constexpr size_t y = 128;                                    // [14][TU][YS]
    static constexpr size_t H = y + (size_t)KS * TU * YS * 8;           // [TU][HS]
    static constexpr size_t LX = H + (size_t)TU * HS * 8;               // [TU][LS]  L rows, then X
    static constexpr size_t dinv = LX + (size_t)TU * LS * 8;            // [TU][NL] float
    static constexpr size_t total = dinv + (size_t)TU * NL * 4;
};

__device__ __forceinline__ float2 shfl2(float2 v, int src) {
    return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// KS = symbols sharing one H (sym_per_h): a "slot" of this kernel is one H time block of KS symbols
// (a.n_slots = n_sym / KS), so time-varying channels (KS = 7, 2, 1) take the same code
template <int NR, int NL, int QM, int LT, int NW, int KS = kSym>
__global__ void __launch_bounds__(32 * NW) k_lg(DetectArgs a) {
    using SM = LgSmem<NR, NL, NW, KS>;
    constexpr int UPW = SM::UPW;
    constexpr int TU = SM::TU;
    static_assert(32 % NL == 0, "NL must divide 32");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bars);
    float2* sy = reinterpret_cast<float2*>(smem + SM::y);
    float2* sH = reinterpret_cast<float2*>(smem + SM::H);
    float2* sLX = reinterpret_cast<float2*>(smem + SM::LX);
    float* sDinv = reinterpret_cast<float*>(smem + SM::dinv);

    pdl_launch_dependents();
    const int slot = blockIdx.y;
    const int sc0 = blockIdx.x * TU;
    const int nvalid = min(TU, a.n_sc - sc0);
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int k = lane % NL;                     // this lane's layer
    const int gbase = lane - k;                  // first lane of the group
    const int ul = warp * UPW + lane / NL;       // unit within the tile
    const bool active = ul < nvalid;
    const int sc = sc0 + ul;
    const float s2 = block_sigma2(a, slot);
    const float norm = (float)qam_norm(QM);

    if (t == 0) {
#pragma unroll
        for (int s = 0; s <= KS; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        mbar_arrive_expect_tx(&bars[KS], (uint32_t)nvalid * NR * NL * 8u);
#pragma unroll 1
        for (int s = 0; s < KS; ++s) mbar_arrive_expect_tx(&bars[s], (uint32_t)nvalid * NR * 8u);
    }
    __syncthreads();
    // the group leader of each unit copies its H and its 14 y vectors into padded slots
    if (k == 0 && active) {
        bulk_g2s(sH + ul * SM::HS, a.H + ((size_t)slot * a.n_sc + sc) * NR * NL, NR * NL * 8u, &bars[KS]);
#pragma unroll 1
        for (int s = 0; s < KS; ++s)
            bulk_g2s(sy + (s * TU + ul) * SM::YS, a.y + ((size_t)(slot * KS + s) * a.n_sc + sc) * NR, NR * 8u,
                     &bars[s]);
    }
    mbar_wait(&bars[KS], 0);

    const float2* hU = sH + ul * SM::HS;  // H[r][l] of this lane's unit (garbage but in-bounds if !active)
    // a2: row k of G
    float2 g[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) g[j] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int r = 0; r < NR; ++r) {
        const float2 hk = hU[r * NL + k];
#pragma unroll
        for (int j = 0; j < NL; ++j) {  // conj(H_rk) H_rj
            const float2 hj = hU[r * NL + j];
            g[j].x = fmaf(hk.x, hj.x, fmaf(hk.y, hj.y, g[j].x));
            g[j].y = fmaf(hk.x, hj.y, fmaf(-hk.y, hj.x, g[j].y));
        }
    }
    // diagonal: real, + s2
#pragma unroll
    for (int j = 0; j < NL; ++j)
        if (j == k) g[j] = make_float2(g[j].x + s2, 0.f);
    // max_i G_ii over the group (guard scale)
    float gmax = 0.f;
#pragma unroll
    for (int j = 0; j < NL; ++j)
        if (j == k) gmax = g[j].x;
#pragma unroll
    for (int off = 1; off < NL; off <<= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));

    // a3: right-looking Cholesky, lane k holds row k (entries j <= k meaningful)
    bool fail = !(gmax == gmax);
    float my_dinv = 0.f;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        float p = __shfl_sync(0xffffffffu, g[j].x, gbase + j);  // G_jj of the trailing matrix
        if (!(p > (float)kPivotTau * gmax)) {
            fail = true;
            p = 1.f;
        }
        const float dinv = rsqrtf(p);
        if (k == j) my_dinv = dinv;
        if (k > j) g[j] = make_float2(g[j].x * dinv, g[j].y * dinv);  // L_kj
#pragma unroll
        for (int m = j + 1; m < NL; ++m) {
            const float2 lmj = shfl2(g[j], gbase + m);  // L_mj from lane m
            if (k >= m) {                              // G_km -= L_kj conj(L_mj)
                g[m].x = fmaf(-g[j].x, lmj.x, fmaf(-g[j].y, lmj.y, g[m].x));
                g[m].y = fmaf(-g[j].y, lmj.x, fmaf(g[j].x, lmj.y, g[m].y));
            }
        }
    }
    // L rows to shared memory (strictly lower part), 1/L_kk
    float2* lU = sLX + ul * SM::LS;
#pragma unroll
    for (int j = 0; j < NL; ++j) lU[k * NL + j] = (j < k) ? g[j] : make_float2(0.f, 0.f);
    sDinv[ul * NL + k] = my_dinv;
    __syncwarp();
    // a4: column k of X = L^-1:  X_kk = 1/L_kk, X_ik = -(1/L_ii) sum_{m<i} L_im X_mk
    float2 x[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < i; ++m) sv = cmac(sv, lU[i * NL + m], x[m]);
        const float di = sDinv[ul * NL + i];
        x[i] = (i == k) ? make_float2(my_dinv, 0.f)
                        : (i < k ? make_float2(0.f, 0.f) : make_float2(-sv.x * di, -sv.y * di));
    }
    float A = 0.f;
#pragma unroll
    for (int i = 0; i < NL; ++i) A = fmaf(x[i].x, x[i].x, fmaf(x[i].y, x[i].y, A));
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NL; ++i) lU[i * NL + k] = x[i];  // X column k (X_ik)
    __syncwarp();
    // row k of G^-1 = X^H X: Gi_kj = sum_{m >= max(k,j)} conj(X_mk) X_mj (X_mk = x[m] here)
    float2 gi[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = j; m < NL; ++m) {  // x[m] = 0 for m < k
            const float2 xm = x[m], xmj = lU[m * NL + j];
            sv.x = fmaf(xm.x, xmj.x, fmaf(xm.y, xmj.y, sv.x));
            sv.y = fmaf(xm.x, xmj.y, fmaf(-xm.y, xmj.x, sv.y));
        }
        gi[j] = sv;
    }
    // a5
    float sinr, fac;
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
    const float slope = sinr / norm * a.llr_scale;
    // row k of W = G^-1 H^H: W_kr = sum_j Gi_kj conj(H_rj), scaled to W~ (level units)
    float2 w[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const float2 h = hU[r * NL + j];
            sv.x = fmaf(gi[j].x, h.x, fmaf(gi[j].y, h.y, sv.x));
            sv.y = fmaf(gi[j].y, h.x, fmaf(-gi[j].x, h.y, sv.y));
        }
        w[r] = (fac > 0.f) ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
    }

    pdl_wait();  // global writes only after the previous grid completed
    if (active) {
        const size_t unit = (size_t)slot * a.n_sc + sc;
        if (k == 0 && fail) atomicAdd(a.fail_count, 1ull);
        if (a.sinr) a.sinr[unit * NL + k] = sinr;
    }
    constexpr int kLlrBytes = QM * LlrTraits<LT>::bytes;  // this lane's layer
    constexpr int kWords = (kLlrBytes + 3) / 4;
    const float ia = rsqrtf(norm);
    const bool zf = !(s2 > 0.f);
#pragma unroll 1
    for (int s = 0; s < KS; ++s) {
        mbar_wait(&bars[s], 0);
        if (!active) continue;
        const float2* ys = sy + (s * TU + ul) * SM::YS;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc = cmac(acc, w[r], ys[r]);
        const size_t re = (size_t)(slot * KS + s) * a.n_sc + sc;
        if (a.llr) {
            float v[QM];
            uint32_t wd[kWords];
            if (!zf) {
                demap_layer<QM, false, LT>(acc, slope, v);
                pack_llr<LT, QM, false>(v, wd);
            } else {
                demap_layer<QM, true, LT>(acc, slope, v);
                pack_llr<LT, QM, true>(v, wd);
            }
            store_bytes<kLlrBytes>((char*)a.llr + (re * NL + k) * kLlrBytes, wd);
        }
        if (a.xhat) a.xhat[re * NL + k] = make_float2(acc.x * ia, acc.y * ia);
    }
}

// k_lg3: k_lg with the CTA's whole y tile (14 symbols x TU subcarriers x NR
// antennas) fetched by ONE TMA tensor-box copy (3-D map {2 NR floats, n_sc,
// n_sym}, box {2 NR, TU, 14}, SWIZZLE_128B) instead of 14 small bulk copies per
// unit: the copy engine generates the 128-byte rows itself (tools/tmabench.cu:
// tensor boxes stream at ~7 TB/s, per-row bulk copies are request-rate bound).
// Row = 14-symbol index x TU + unit; the 16-byte chunk c of a row sits at
// c ^ (row & 7), so the UPW units of a warp reading the same antennas hit
// different bank groups (no padding needed). Ragged tails are zero-filled by TMA.
template <int NR, int NL, int NW, int HT = 0>
struct Lg3Smem {
    static constexpr int UPW = 32 / NL;
    static constexpr int TU = UPW * NW;
    static constexpr int HS = NR * NL + 4;                                  // float2 per unit H (padded)
    static constexpr int LS = NL * NL + 4;                                  // float2 per unit L / X
    static constexpr size_t y = 0;                                          // [14][TU][NR] float2, SW128
    // HT 4: y lands after the setup, over the H / L / X area (which is dead by then)
    static constexpr size_t ybytes = (size_t)kSym * TU * NR * 8;
    static constexpr size_t H = HT == 4 ? 0 : ybytes;                       // [TU][HS], or HT: [NR*NL/16][TU][128 B] SW128
    static constexpr size_t LX = H + (HT ? (size_t)TU * NR * NL * 8 : (size_t)TU * HS * 8);  // [TU][LS]
    static constexpr size_t dinv = LX + (size_t)TU * LS * 8;                // [TU][NL]
    static constexpr size_t setup_end = dinv + (size_t)TU * NL * 4;
    static constexpr size_t bars = ((setup_end > ybytes ? setup_end : ybytes) + 7) / 8 * 8;  // y, H
    static constexpr size_t total = bars + 16 + 1024;                       // + 1024-alignment slack
};

// HT = 2: as HT = 1 with the per-RE apply as packed FFMA2, acc += (w.x, w.y) y.x + (-w.y, w.x) y.y
// (y components broadcast; 80.3 vs 80.9 us per C4 step -- the same packing in the Gram and W~
// loops of the setup made the step slower, 82.4 us, so they stay scalar).
// HT = 1: H also by one TMA tensor box per CTA: H viewed as (32 floats = one 128-byte row of
// 2 rx x 8 layers, unit, row-within-unit) -- unit as the middle dimension -- so the box lands
// as [row][unit][128 B] and SWIZZLE_128B spreads the UPW units of a warp over distinct banks.
template <int NR, int NL, int QM, int LT, int NW, int PFD, int HT = 0>
// HT 4, 4 warps: at most 80 registers (6 CTAs per SM instead of 5; 12 bytes of spill): 141k vs 150k
// cycles per C4 step (81.7 vs 83.1 us at the power-capped clock); 7 CTAs (72 registers) spill more
__global__ void __launch_bounds__(32 * NW, (HT == 4 && NW == 4) ? 6 : 1) k_lg3(DetectArgs a, const __grid_constant__ CUtensorMap ymap,
                                                 const __grid_constant__ CUtensorMap hmap) {
    using SM = Lg3Smem<NR, NL, NW, HT>;
    constexpr int UPW = SM::UPW;
    constexpr int TU = SM::TU;
    static_assert(32 % NL == 0 && NR * 8 == 128, "k_lg3: one 128-byte row per (symbol, unit)");
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (base - raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::bars);
    float2* sH = reinterpret_cast<float2*>(smem + SM::H);
    float2* sLX = reinterpret_cast<float2*>(smem + SM::LX);
    float* sDinv = reinterpret_cast<float*>(smem + SM::dinv);

    pdl_launch_dependents();
    const int slot = blockIdx.y;
    const int sc0 = blockIdx.x * TU;
    const int nvalid = min(TU, a.n_sc - sc0);
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int k = lane % NL;                     // this lane's layer
    const int gbase = lane - k;                  // first lane of the group
    const int ul = warp * UPW + lane / NL;       // unit within the tile
    const bool active = ul < nvalid;
    const int sc = sc0 + ul;
    const float s2 = block_sigma2(a, slot);
    const float norm = (float)qam_norm(QM);

    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        if constexpr (HT == 4) {  // y is copied after the setup; warm L2 with it now
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                             reinterpret_cast<uint64_t>(&ymap)),
                         "r"(0), "r"(sc0), "r"(slot * kSym) : "memory");
        } else {
            mbar_arrive_expect_tx(&bars[0], (uint32_t)(kSym * TU * NR * 8));
            tma_load_3d(base + (uint32_t)SM::y, &ymap, 0, sc0, slot * kSym, &bars[0]);
        }
        if constexpr (HT) {
            mbar_arrive_expect_tx(&bars[1], (uint32_t)(TU * NR * NL * 8));
            tma_load_3d(base + (uint32_t)SM::H, &hmap, 0, slot * a.n_sc + sc0, 0, &bars[1]);
        } else {
            mbar_arrive_expect_tx(&bars[1], (uint32_t)nvalid * NR * NL * 8u);
        }
        if constexpr (PFD > 0) {
            // warm L2 with the H and y tiles of the CTA PFD launches ahead (about one wave later),
            // so its start-up loads hit L2 instead of exposing DRAM latency
            const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + PFD;
            if (lin < (long long)gridDim.x * gridDim.y) {
                const int ps = (int)(lin / gridDim.x), psc0 = (int)(lin % gridDim.x) * TU;
                const int pn = min(TU, a.n_sc - psc0);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.H + ((size_t)ps * a.n_sc + psc0) * NR * NL),
                             "r"((uint32_t)pn * NR * NL * 8u) : "memory");
                asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                                 reinterpret_cast<uint64_t>(&ymap)),
                             "r"(0), "r"(psc0), "r"(ps * kSym) : "memory");
            }
        }
    }
    __syncthreads();
    if (!HT && k == 0 && active)
        bulk_g2s(sH + ul * SM::HS, a.H + ((size_t)slot * a.n_sc + sc) * NR * NL, NR * NL * 8u, &bars[1]);
    mbar_wait(&bars[1], 0);

    const float2* hU = sH + ul * SM::HS;
    const unsigned char* hT = smem + SM::H;
    auto hat = [&](int r, int j) -> float2 {  // H[r][j] of this lane's unit
        if constexpr (HT) {
            constexpr int RPR = 128 / (NL * 8);  // rx rows per 128-byte row
            const int row = (r / RPR) * TU + ul;
            const int byte = (r % RPR) * NL * 8 + j * 8;
            return *reinterpret_cast<const float2*>(hT + row * 128 + (((byte >> 4) ^ (row & 7)) << 4) + (byte & 15));
        } else {
            return hU[r * NL + j];
        }
    };
    // HT 3: the NL entries H[r][0 .. NL-1] of one antenna as NL / 2 16-byte loads (one swizzled half row)
    auto hrow = [&](int r, float2* hr) {
        constexpr int RPR = 128 / (NL * 8);
        const int row = (r / RPR) * TU + ul;
#pragma unroll
        for (int q = 0; q < NL / 2; ++q) {
            const int c = (r % RPR) * (NL / 2) + q;
            const float4 v = *reinterpret_cast<const float4*>(hT + row * 128 + ((c ^ (row & 7)) << 4));
            hr[2 * q] = make_float2(v.x, v.y);
            hr[2 * q + 1] = make_float2(v.z, v.w);
        }
    };
    float2 g[NL];
    if constexpr (HT >= 3) {
        // G_kj = sum_r conj(H_rk) H_rj as two packed accumulators with free operand forms (broadcast,
        // swapped pair): a += H_rk.x (H_rj.x, H_rj.y), b += H_rk.y (H_rj.y, H_rj.x), G = (a.x + b.x, a.y - b.y)
        float2 ga[NL], gb[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) ga[j] = gb[j] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int r = 0; r < NR; ++r) {
            const float2 hk = hat(r, k);
            float2 hr[NL];
            hrow(r, hr);
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                ga[j] = ffma2(make_float2(hk.x, hk.x), hr[j], ga[j]);
                gb[j] = ffma2(make_float2(hk.y, hk.y), make_float2(hr[j].y, hr[j].x), gb[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < NL; ++j) g[j] = make_float2(ga[j].x + gb[j].x, ga[j].y - gb[j].y);
    } else {
#pragma unroll
        for (int j = 0; j < NL; ++j) g[j] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int r = 0; r < NR; ++r) {
            const float2 hk = hat(r, k);
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const float2 hj = hat(r, j);
                g[j].x = fmaf(hk.x, hj.x, fmaf(hk.y, hj.y, g[j].x));
                g[j].y = fmaf(hk.x, hj.y, fmaf(-hk.y, hj.x, g[j].y));
            }
        }
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

    bool fail = !(gmax == gmax);
    float my_dinv = 0.f;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        float p = __shfl_sync(0xffffffffu, g[j].x, gbase + j);
        if (!(p > (float)kPivotTau * gmax)) {
            fail = true;
            p = 1.f;
        }
        const float dinv = rsqrtf(p);
        if (k == j) my_dinv = dinv;
        if (k > j) g[j] = make_float2(g[j].x * dinv, g[j].y * dinv);
        if constexpr (HT >= 3) {  // G_km -= L_kj conj(L_mj) = L_mj.x (-L_kj) + L_mj.y (-L_kj.y, L_kj.x)
            const float2 na = make_float2(-g[j].x, -g[j].y), ra = make_float2(-g[j].y, g[j].x);
#pragma unroll
            for (int m = j + 1; m < NL; ++m) {
                const float2 lmj = shfl2(g[j], gbase + m);
                if (k >= m) {
                    g[m] = ffma2(make_float2(lmj.x, lmj.x), na, g[m]);
                    g[m] = ffma2(make_float2(lmj.y, lmj.y), ra, g[m]);
                }
            }
        } else {
#pragma unroll
            for (int m = j + 1; m < NL; ++m) {
                const float2 lmj = shfl2(g[j], gbase + m);
                if (k >= m) {
                    g[m].x = fmaf(-g[j].x, lmj.x, fmaf(-g[j].y, lmj.y, g[m].x));
                    g[m].y = fmaf(-g[j].y, lmj.x, fmaf(g[j].x, lmj.y, g[m].y));
                }
            }
        }
    }
    float2* lU = sLX + ul * SM::LS;
#pragma unroll
    for (int j = 0; j < NL; ++j) lU[k * NL + j] = (j < k) ? g[j] : make_float2(0.f, 0.f);
    sDinv[ul * NL + k] = my_dinv;
    __syncwarp();
    float2 x[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        float2 sv = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < i; ++m) sv = cmac(sv, lU[i * NL + m], x[m]);
        const float di = sDinv[ul * NL + i];
        x[i] = (i == k) ? make_float2(my_dinv, 0.f)
                        : (i < k ? make_float2(0.f, 0.f) : make_float2(-sv.x * di, -sv.y * di));
    }
    float A = 0.f;
#pragma unroll
    for (int i = 0; i < NL; ++i) A = fmaf(x[i].x, x[i].x, fmaf(x[i].y, x[i].y, A));
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NL; ++i) lU[i * NL + k] = x[i];
    __syncwarp();
    float2 gi[NL];
    if constexpr (HT >= 3) {  // Gi_kj += conj(X_mk) X_mj = X_mj.x (x.x, -x.y) + X_mj.y (x.y, x.x), x = X_mk
        float2 cx[NL];
#pragma unroll
        for (int m = 0; m < NL; ++m) cx[m] = make_float2(x[m].x, -x[m].y);
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = j; m < NL; ++m) {
                const float2 xmj = lU[m * NL + j];
                sv = ffma2(make_float2(xmj.x, xmj.x), cx[m], sv);
                sv = ffma2(make_float2(xmj.y, xmj.y), make_float2(x[m].y, x[m].x), sv);
            }
            gi[j] = sv;
        }
    } else {
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = j; m < NL; ++m) {
                const float2 xm = x[m], xmj = lU[m * NL + j];
                sv.x = fmaf(xm.x, xmj.x, fmaf(xm.y, xmj.y, sv.x));
                sv.y = fmaf(xm.x, xmj.y, fmaf(-xm.y, xmj.x, sv.y));
            }
            gi[j] = sv;
        }
    }
    float sinr, fac;
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
    const float slope = sinr / norm * a.llr_scale;
    float2 w[NR];
    if constexpr (HT >= 3) {  // W_kr = sum_j h.x (Gi.x, Gi.y) + h.y (Gi.y, -Gi.x), h = H_rj (broadcast halves)
        float2 gs[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) gs[j] = make_float2(gi[j].y, -gi[j].x);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            float2 hr[NL];
            hrow(r, hr);
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                sv = ffma2(make_float2(hr[j].x, hr[j].x), gi[j], sv);
                sv = ffma2(make_float2(hr[j].y, hr[j].y), gs[j], sv);
            }
            w[r] = (fac > 0.f) ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
        }
    } else {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            float2 sv = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const float2 h = hat(r, j);
                sv.x = fmaf(gi[j].x, h.x, fmaf(gi[j].y, h.y, sv.x));
                sv.y = fmaf(gi[j].y, h.x, fmaf(-gi[j].x, h.y, sv.y));
            }
            w[r] = (fac > 0.f) ? make_float2(sv.x * fac, sv.y * fac) : make_float2(0.f, 0.f);
        }
    }

    float2 wq[HT >= 2 ? NR : 1];  // HT 2-4: (-w.y, w.x) for the packed apply
    if constexpr (HT >= 2) {
#pragma unroll
        for (int r = 0; r < NR; ++r) wq[r] = make_float2(-w[r].y, w[r].x);
    }
    if constexpr (HT == 4) {  // H, L, X are dead in every warp: y over them (the L2-warm tile)
        __syncthreads();
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(&bars[0], (uint32_t)(kSym * TU * NR * 8));
            tma_load_3d(base + (uint32_t)SM::y, &ymap, 0, sc0, slot * kSym, &bars[0]);
        }
    }
    pdl_wait();  // global writes only after the previous grid completed
    if (active) {
        const size_t unit = (size_t)slot * a.n_sc + sc;
        if (k == 0 && fail) atomicAdd(a.fail_count, 1ull);
        if (a.sinr) a.sinr[unit * NL + k] = sinr;
    }
    constexpr int kLlrBytes = QM * LlrTraits<LT>::bytes;
    constexpr int kWords = (kLlrBytes + 3) / 4;
    const float ia = rsqrtf(norm);
    const bool zf = !(s2 > 0.f);
    mbar_wait(&bars[0], 0);
    if (!active) return;
    const unsigned char* ybase = smem + SM::y;
#pragma unroll 1
    for (int s = 0; s < kSym; ++s) {
        const int row = s * TU + ul;
        const unsigned char* yr = ybase + row * 128;
        const int sw = row & 7;
        float2 acc = make_float2(0.f, 0.f);
        if constexpr (HT >= 2) {  // packed FFMA2: acc += w y as (w.x, w.y) y.x + (-w.y, w.x) y.y
#pragma unroll
            for (int c = 0; c < NR / 2; ++c) {
                const float4 v = *reinterpret_cast<const float4*>(yr + ((c ^ sw) << 4));
                acc = ffma2(w[2 * c], make_float2(v.x, v.x), acc);
                acc = ffma2(wq[2 * c], make_float2(v.y, v.y), acc);
                acc = ffma2(w[2 * c + 1], make_float2(v.z, v.z), acc);
                acc = ffma2(wq[2 * c + 1], make_float2(v.w, v.w), acc);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NR / 2; ++c) {
                const float4 v = *reinterpret_cast<const float4*>(yr + ((c ^ sw) << 4));
                acc = cmac(acc, w[2 * c], make_float2(v.x, v.y));
                acc = cmac(acc, w[2 * c + 1], make_float2(v.z, v.w));
            }
        }
        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + sc;
        if (a.llr) {
            float v[QM];
            uint32_t wd[kWords];
            if (!zf) {
                if constexpr (HT >= 3 && QM >= 6 && LT != kLlrI8) {
                    demap_layer_x2<QM, LT>(acc, slope, wd);  // I and Q axes as packed pairs
                } else {
                    demap_layer<QM, false, LT>(acc, slope, v);
                    pack_llr<LT, QM, false>(v, wd);
                }
            } else {
                demap_layer<QM, true, LT>(acc, slope, v);
                pack_llr<LT, QM, true>(v, wd);
            }
            store_bytes<kLlrBytes>((char*)a.llr + (re * NL + k) * kLlrBytes, wd);
        }
        if (a.xhat) a.xhat[re * NL + k] = make_float2(acc.x * ia, acc.y * ia);
    }
}

template <int NR, int NL, int QM, int LT, int NW, int PFD, int HT = 0>
cudaError_t launch3(const DetectArgs& a, cudaStream_t s) {
    if (a.n_sc <= 0 || a.n_slots <= 0) return cudaSuccess;
    constexpr int TU = Lg3Smem<NR, NL, NW>::TU;
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap ymap;
    const cuuint64_t gdim[3] = {(cuuint64_t)(2 * NR), (cuuint64_t)a.n_sc, (cuuint64_t)a.n_sym};
    const cuuint64_t gstride[2] = {(cuuint64_t)NR * 8, (cuuint64_t)a.n_sc * NR * 8};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * NR), (cuuint32_t)TU, (cuuint32_t)kSym};
    const cuuint32_t estride[3] = {1, 1, 1};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(a.y), gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    CUtensorMap hmap = ymap;  // unused unless HT
    if (HT) {
        const cuuint64_t hdim[3] = {32, (cuuint64_t)a.n_slots * a.n_sc, (cuuint64_t)(NR * NL * 8 / 128)};
        const cuuint64_t hstride[2] = {(cuuint64_t)NR * NL * 8, 128};
        const cuuint32_t hbox[3] = {32, (cuuint32_t)TU, (cuuint32_t)(NR * NL * 8 / 128)};
        if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(a.H), hdim, hstride, hbox, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((a.n_sc + TU - 1) / TU, a.n_slots);
    cfg.blockDim = dim3(32 * NW);
    cfg.dynamicSmemBytes = Lg3Smem<NR, NL, NW, HT>::total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_lg3<NR, NL, QM, LT, NW, PFD, HT>, a, ymap, hmap);
}

template <int NR, int NL, int QM, int LT, int NW, int PFD, int HT = 0>
cudaError_t prepare3() {
    constexpr size_t smem = Lg3Smem<NR, NL, NW, HT>::total;
    if (smem > 48 * 1024)
        return cudaFuncSetAttribute(k_lg3<NR, NL, QM, LT, NW, PFD, HT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    return cudaSuccess;
}

template <int NR, int NL, int QM, int LT, int NW, int KS = kSym>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_sc <= 0 || a.n_slots <= 0) return cudaSuccess;
    constexpr int TU = LgSmem<NR, NL, NW, KS>::TU;
    dim3 grid((a.n_sc + TU - 1) / TU, a.n_slots);
    return launch_kernel(k_lg<NR, NL, QM, LT, NW, KS>, grid, dim3(32 * NW), LgSmem<NR, NL, NW, KS>::total, s, a.overlap, a);
}

template <int NR, int NL, int QM, int LT, int NW, int KS = kSym>
cudaError_t prepare() {
    constexpr size_t smem = LgSmem<NR, NL, NW, KS>::total;
    if (smem > 48 * 1024)
        return cudaFuncSetAttribute(k_lg<NR, NL, QM, LT, NW, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaSuccess;
}

#define LG_ENTRY(NAME, NR, NL, QM, LT, NW) \
    KernelEntry { NAME, NR, NL, QM, 1, 14, LT, 32, 1, launch<NR, NL, QM, LT, NW>, prepare<NR, NL, QM, LT, NW> }
// time-varying channels on the 16 x 8 per-subcarrier shape (NEXT-3): one H per KS symbols
#define LG_TV_ENTRY(NAME, NR, NL, QM, LT, NW, KS) \
    KernelEntry { NAME, NR, NL, QM, 1, KS, LT, 32, 1, launch<NR, NL, QM, LT, NW, KS>, prepare<NR, NL, QM, LT, NW, KS> }

#define LG3_ENTRY(NAME, NR, NL, QM, LT, NW) LG3P_ENTRY(NAME, NR, NL, QM, LT, NW, 0)
#define LG3P_ENTRY(NAME, NR, NL, QM, LT, NW, PFD)                                                      \
    KernelEntry {                                                                                      \
        NAME, NR, NL, QM, 1, 14, LT, 32, 1, launch3<NR, NL, QM, LT, NW, PFD>, prepare3<NR, NL, QM, LT, NW, PFD> \
    }

const KernelEntry kEntries[] = {
    // C4 default (lg3hl, HT = 4): H by one TMA box, the Gram, Cholesky update, G^-1 and W~ products and
    // the max-log demap as packed FFMA2 / FADD2 pairs with free operand forms (HT >= 3), and the y tile
    // copied only after the setup, over the dead H / L / X area (L2-warm by a prefetch at CTA start):
    // 29.7 instead of 54 KiB of shared memory lifts residency from 4 to 5 CTAs of 4 warps per SM.
    // Measured per C4 step (bench, power-capped clocks): lg3hl 78.6 us at 1.78 GHz (139.7k cycles),
    // lg3hq (HT 3, y early) 80.7 at 1.82 (147k), lg3hp (HT 2) 82.4 at 1.85 (152.6k), lg3hl2 (2 warps) 79.8.
    KernelEntry{"lg3hl_16x8_q8_f16", 16, 8, 8, 1, 14, kLlrF16, 32, 1, launch3<16, 8, 8, kLlrF16, 4, 0, 4>,
                prepare3<16, 8, 8, kLlrF16, 4, 0, 4>},
    KernelEntry{"lg3hl2_16x8_q8_f16", 16, 8, 8, 1, 14, kLlrF16, 32, 1, launch3<16, 8, 8, kLlrF16, 2, 0, 4>,
                prepare3<16, 8, 8, kLlrF16, 2, 0, 4>},
    KernelEntry{"lg3hq_16x8_q8_f16", 16, 8, 8, 1, 14, kLlrF16, 32, 1, launch3<16, 8, 8, kLlrF16, 4, 0, 3>,
                prepare3<16, 8, 8, kLlrF16, 4, 0, 3>},
    // HT = 2: y and H as TMA boxes, the per-RE apply as packed FFMA2 (round 1 default)
    KernelEntry{"lg3hp_16x8_q8_f16", 16, 8, 8, 1, 14, kLlrF16, 32, 1, launch3<16, 8, 8, kLlrF16, 4, 0, 2>,
                prepare3<16, 8, 8, kLlrF16, 4, 0, 2>},
    LG3_ENTRY("lg3_16x8_q8_f16", 16, 8, 8, kLlrF16, 2),  // y by TMA, H by per-unit bulk copies
    LG_ENTRY("lg_16x8_q8_f16", 16, 8, 8, kLlrF16, 2),
    LG_TV_ENTRY("lg_16x8_q8_f16_s7", 16, 8, 8, kLlrF16, 2, 7),
    LG_TV_ENTRY("lg_16x8_q8_f16_s2", 16, 8, 8, kLlrF16, 2, 2),
    LG_TV_ENTRY("lg_16x8_q8_f16_s1", 16, 8, 8, kLlrF16, 2, 1),
    LG_ENTRY("lg_16x8_q8_f32", 16, 8, 8, kLlrF32, 2),
    LG_ENTRY("lg_16x8_q8_i8", 16, 8, 8, kLlrI8, 2),
    LG_ENTRY("lg_16x8_q6_f16", 16, 8, 6, kLlrF16, 2),
    LG_ENTRY("lg_8x8_q6_f16", 8, 8, 6, kLlrF16, 2),
    LG_ENTRY("lg_16x16_q8_f16", 16, 16, 8, kLlrF16, 2),
};

}  // namespace

const KernelEntry* lg_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
