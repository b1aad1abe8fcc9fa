// k_c5.cu -- the C5 detector (64 rx x 16 layers, 64-QAM, int8 LLRs, H per PRB)
// on the 5th-generation tensor cores.
//
// Per call: a setup kernel writes, per H-unit, W~ = diag(sqrt(norm)/mu) G^-1 H^H
// ([unit][r][k] float2) and the LLR slopes to the plan workspace (rows a2-a5),
// then the persistent apply kernel k_c5_apply runs rows a6-a7 for all REs:
//
//   x~ (168 x 16 complex) = Y (168 x 64 complex) W~^T
//
// as the real product  X (168 x 32) = Y (168 x 128) B (128 x 32), with the fp32
// accuracy of three split passes (reading R21 TF32 / R28 BF16):
//   X = Y_hi [B_hi | B_lo] (N = 64)  +  Y_lo B_hi (N = 32, into columns 0-31),
// x~_k = X[:, k] + X[:, 32 + k] (re), X[:, 16 + k] + X[:, 48 + k] (im).
// One CTA per SM, warp-specialised:
//   producer warp (lane 0): TMA 3-D tensor boxes of y, one 16-antenna K chunk of the
//                 unit's 168 RE rows (168 x 128 B, SWIZZLE_128B) per stage, S stages;
//   MMA warp (lane 0):  tcgen05.mma, A = y rows from TMEM, B = the unit's W~ set from smem;
//   converter warps 0-3: B = [B_hi; B_lo] per unit from the W~ workspace (double-buffered),
//                 and each y row of a stage split into hi/lo and stored to the TMEM A ring
//                 with tcgen05.st (warp w serves TMEM lane quadrant w);
//   epilogue warps: TMEM accumulators (2 x 128 columns) -> x~ -> exact max-log demap ->
//                 int8 -> 96-byte LLR record per RE.
// Two M = 128 row tiles cover a unit's 168 REs: tile 0 = REs 0-127; tile 1 = REs 128-167 in
// TMEM lanes 0-39 (EW = 6, "compact") or REs 40-167 (EW = 4).
// TA = 1: kind::tf32 (y raw = y_hi as read by the tensor core, y_lo = y - trunc(y));
// TA = 3: kind::f16 with BF16 hi/lo operands (K = 16 per instruction: half the MMAs and half
// the TMEM A bytes of TA = 1).

#include "big_setup.cuh"
#include "tc.cuh"

namespace mimo {
namespace {

template <int S_, int NLO_, int TA_>
struct C5Smem {
    static constexpr int S = S_;                              // y stages
    static constexpr int NLO = NLO_;                          // TMEM A ring slots (chunks)
    static constexpr size_t chunk = (size_t)kRe * 128;        // 21504 = 21 x 1024
    static constexpr size_t y0 = 0;
    static constexpr size_t B = S * chunk;                    // 2 B sets (1024-aligned)
    static constexpr size_t bset = TA_ == 1 ? 4 * 64 * 128 : 2 * 64 * 128;  // K atoms x 64 rows x 128 B
    static constexpr size_t slope = B + 2 * bset;             // [4][16] slope | [4][16] sqrt(slope / 127)
    static constexpr size_t bars = slope + 512;
    static constexpr int NBAR = 2 * S + 2 * NLO + 2 * 3;      // yfull, yfree | afull, afree | bready, accfull, tfree
    static constexpr size_t tslot = bars + NBAR * 8;
    static constexpr size_t total = tslot + 16 + 1024;        // + 1024-B alignment slack
    static_assert(B % 1024 == 0, "UMMA operand alignment");
    static_assert(total <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ float fma_sat(float a, float b, float c) {
    float d;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// Exact max-log LLRs of one axis, int8 (sigma2 > 0, the fold form of
// common.cuh demap_axis, pinned by P10): with rs = sqrt(slope / 127),
//   t_0 = u, t_i = 2^(M-i) - |t_{i-1}|,  e = rs (|t_{M-1}| - 1),
//   m_i = sat_[0,1]( (rs (|t_i| + 1))^2 - e^2 )  = min(slope ((|t_i|+1)^2 - D), 127) / 127,
//   q_i = rint(sgn(t_i) 127 m_i)   (1.5 * 2^23 magic: the low byte of the float is the int8).
template <int M>
__device__ __forceinline__ void demap_axis_i8(float u, float rs, uint32_t* q, int stride) {
    float t[M];
    t[0] = u;
#pragma unroll
    for (int i = 1; i < M; ++i) t[i] = float(1 << (M - i)) - fabsf(t[i - 1]);
    const float e = fmaf(fabsf(t[M - 1]), rs, -rs);
    const float D = e * e;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const float at = fmaf(fabsf(t[i]), rs, rs);
        const float m = fma_sat(at, at, -D);
        const float s127 = __uint_as_float((__float_as_uint(t[i]) & 0x80000000u) | 0x42FE0000u);  // copysign(127, t)
        q[i * stride] = __float_as_uint(fmaf(m, s127, 12582912.f));
    }
}

template <int QM, int LT, int EW, int S_, int NLO_, int TA>
__global__ void __launch_bounds__(32 * (6 + EW), 1) k_c5_apply(DetectArgs a, const __grid_constant__ CUtensorMap ymap) {
    constexpr int NR = 64, NL = 16;
    using SM = C5Smem<S_, NLO_, TA>;
    constexpr int S = S_, NLO = NLO_;
    constexpr bool CT = EW == 6;  // compact tile 1 (REs 128-167 in lanes 0-39)
    static_assert(EW == 4 || EW == 6, "4 or 6 epilogue warps");
    static_assert(TA == 1 || TA == 3, "TF32 or BF16 operands");
    constexpr uint32_t kAring = 256u;                // TMEM columns 0-255: 2 accumulators x 128
    constexpr uint32_t kAcols = TA == 1 ? 128u : 64u;  // TMEM columns per A ring slot (one chunk, 2 tiles)
    static_assert(kAring + NLO * kAcols <= 512u, "TMEM");
    constexpr int CW = 4 + EW;                       // MMA warp; CW + 1: TMA producer
    constexpr int WS = BigWs<NR, NL>::stride;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(g + SM::bars);
    uint64_t* yfull = bar;             // [S]    TMA tx
    uint64_t* yfree = bar + S;         // [S]    converters done with the stage
    uint64_t* afull = bar + 2 * S;     // [NLO]  converters stored the chunk's A rows
    uint64_t* afree = afull + NLO;     // [NLO]  MMAs of the chunk completed
    uint64_t* bready = afree + NLO;    // [2]    converters built B
    uint64_t* accfull = bready + 2;    // [2]    the unit's last MMA completed
    uint64_t* tfree = accfull + 2;     // [2]    epilogue done with the accumulator
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g + SM::tslot);
    float* sslope = reinterpret_cast<float*>(g + SM::slope);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long u0 = blockIdx.x, du = gridDim.x;
    const long long n_my = u0 < a.n_units ? (a.n_units - u0 + du - 1) / du : 0;
    const long long G = 4 * n_my;

    pdl_launch_dependents();
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&yfull[i], 1);
            mbar_init(&yfree[i], 1);
        }
        for (int i = 0; i < NLO; ++i) {
            mbar_init(&afull[i], 1);
            mbar_init(&afree[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bready[i], 1);
            mbar_init(&accfull[i], 1);
            mbar_init(&tfree[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == CW) tc::alloc<512>(tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tslot;

    if (warp == CW + 1) {
        // ================= TMA producer: y chunks, S stages ahead =================
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ymap)) : "memory");
#pragma unroll 1
            for (long long gg = 0; gg < G; ++gg) {
                const int st = (int)(gg % S);
                if (gg >= S) mbar_wait_sleep(&yfree[st], (uint32_t)(((gg / S) + 1) & 1));
                const long long uu = u0 + (gg >> 2) * du;
                const int slot = (int)(uu / a.n_fb), fb = (int)(uu % a.n_fb);
                mbar_arrive_expect_tx(&yfull[st], (uint32_t)SM::chunk);
                tma_load_3d(base + (uint32_t)(SM::y0 + st * SM::chunk), &ymap, 32 * (int)(gg & 3), fb * kSc,
                            slot * kSym, &yfull[st]);
            }
        }
    } else if (warp == CW) {
        // ================= MMA issuer =================
        if (lane == 0) {
            constexpr uint32_t f = TA == 1 ? tc::kFmtTF32 : tc::kFmtBF16;
            constexpr uint32_t id64 = tc::idesc(f, 128, 64), id32 = tc::idesc(f, 128, 32);
            const uint64_t dB = tc::desc_sw128(base + (uint32_t)SM::B);
#pragma unroll 1
            for (long long i = 0; i < n_my; ++i) {
                const int b = (int)(i & 1);
                mbar_wait_sleep(&bready[b], (uint32_t)((i >> 1) & 1));
                if (i >= 2) mbar_wait_sleep(&tfree[b], (uint32_t)(((i >> 1) + 1) & 1));
                const uint32_t acc = tmem + 128u * (uint32_t)b;
                const uint64_t db = tc::desc_add(dB, (uint32_t)(b * SM::bset));
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    const long long gg = 4 * i + c;
                    const int lb = (int)(gg % NLO);
                    const uint32_t ab = tmem + kAring + kAcols * (uint32_t)lb;
                    mbar_wait_sleep(&afull[lb], (uint32_t)((gg / NLO) & 1));
                    tc::fence_after();
                    if constexpr (TA == 1) {  // 4 K-steps of 8 per chunk; K atom c of the B set
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks) {
                                const uint64_t dk = tc::desc_add(db, (uint32_t)(c * 8192 + ks * 32));
                                tc::mma_tf32_ts(acc + 64u * tile, ab + 64u * tile + 8u * ks, dk, id64, (c | ks) ? 1u : 0u);
                                tc::mma_tf32_ts(acc + 64u * tile, ab + 64u * tile + 32u + 8u * ks, dk, id32, 1u);
                            }
                    } else {  // 2 K-steps of 16; chunk c = half (c & 1) of K atom c >> 1
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 2; ++ks) {
                                const uint64_t dk = tc::desc_add(db, (uint32_t)((c >> 1) * 8192 + (c & 1) * 64 + ks * 32));
                                tc::mma_f16_ts(acc + 64u * tile, ab + 32u * tile + 8u * ks, dk, id64, (c | ks) ? 1u : 0u);
                                tc::mma_f16_ts(acc + 64u * tile, ab + 32u * tile + 16u + 8u * ks, dk, id32, 1u);
                            }
                    }
                    tc::commit(&afree[lb]);
                    if (c == 3) tc::commit(&accfull[b]);
                }
            }
        }
    } else if (warp < 4) {
        // ================= converters =================
        const int tc_ = t;  // 0..127
        const int n = tc_ >> 2, kt = tc_ & 3, kk = n & 15;
        const bool im_row = n >= 16;
        pdl_wait();  // W~ of this call's setup kernel is complete and visible
        float2 wv[16];
        float slv = 0.f;
        auto fetch = [&](long long i) {  // this thread's 16 antennas of W~ row kk of unit i
            const float2* src = reinterpret_cast<const float2*>(reinterpret_cast<const float*>(a.ws) + (u0 + i * du) * WS);
#pragma unroll
            for (int c = 0; c < 16; ++c) wv[c] = src[(16 * kt + c) * NL + kk];
            if (tc_ < NL) slv = reinterpret_cast<const float*>(src + NR * NL)[tc_];
        };
        if (n_my > 0) fetch(0);
#pragma unroll 1
        for (long long i = 0; i < n_my; ++i) {
            const int b = (int)(i & 1);
            // B set b is free once unit i-2's MMAs completed; the slope ring slot i & 3 was last read
            // by epilogue(i-4), which finished before tfree(i-4) < accfull(i-2)
            if (i >= 2) mbar_wait_sleep(&accfull[b], (uint32_t)(((i >> 1) + 1) & 1));
            if constexpr (TA == 1) {
                float* kb = reinterpret_cast<float*>(g + SM::B + b * SM::bset + (size_t)kt * 64 * 128);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float2 w0 = wv[2 * c], w1 = wv[2 * c + 1];
                    const float4 v = im_row ? make_float4(w0.y, w0.x, w1.y, w1.x) : make_float4(w0.x, -w0.y, w1.x, -w1.y);
                    const float4 lo = make_float4(v.x - tc::tf32_trunc(v.x), v.y - tc::tf32_trunc(v.y),
                                                  v.z - tc::tf32_trunc(v.z), v.w - tc::tf32_trunc(v.w));
                    *reinterpret_cast<float4*>(kb + n * 32 + ((c ^ (n & 7)) << 2)) = v;
                    *reinterpret_cast<float4*>(kb + (n + 32) * 32 + ((c ^ (n & 7)) << 2)) = lo;
                }
            } else {
                // BF16, SW128 K-major: K atom kt >> 1 holds chunks 2 (kt >> 1), +1 (64 bf16 per row);
                // this thread's 16 antennas are 16-byte pieces 4 (kt & 1) + j of rows n and n + 32
                unsigned char* kb = g + SM::B + b * SM::bset + (size_t)(kt >> 1) * 8192;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t hv[4], lv[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const float2 w = wv[4 * j + m];
                        if (im_row) tc::split_bf2(w.y, w.x, hv[m], lv[m]);
                        else tc::split_bf2(w.x, -w.y, hv[m], lv[m]);
                    }
                    const int q = 4 * (kt & 1) + j;
                    *reinterpret_cast<uint4*>(kb + n * 128 + ((q ^ (n & 7)) << 4)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
                    *reinterpret_cast<uint4*>(kb + (n + 32) * 128 + ((q ^ (n & 7)) << 4)) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
                }
            }
            if (tc_ < NL) {
                sslope[(i & 3) * 16 + tc_] = slv;
                sslope[64 + (i & 3) * 16 + tc_] = sqrtf(slv * (1.f / 127.f));
            }
            tc::fence_proxy_async();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (tc_ == 0) mbar_arrive(&bready[b]);
            if (i + 1 < n_my) fetch(i + 1);
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                const long long gg = 4 * i + c;
                const int st = (int)(gg % S), lb = (int)(gg % NLO);
                mbar_wait_sleep(&yfull[st], (uint32_t)((gg / S) & 1));
                if (gg >= NLO) mbar_wait_sleep(&afree[lb], (uint32_t)(((gg / NLO) + 1) & 1));
                tc::fence_after();
                const unsigned char* ysm = g + SM::y0 + st * SM::chunk;
#pragma unroll
                for (int tile = 0; tile < 2; ++tile) {
                    if (CT && tile == 1 && warp >= 2) break;
                    const int r = tile ? (CT ? min(128 + 32 * warp + lane, kRe - 1) : 40 + 32 * warp + lane) : 32 * warp + lane;
                    const float4* row = reinterpret_cast<const float4*>(ysm + (size_t)r * 128);
                    float v[32];
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const float4 q = row[cc ^ (r & 7)];  // SWIZZLE_128B: 16-byte piece cc of row r
                        v[4 * cc] = q.x;
                        v[4 * cc + 1] = q.y;
                        v[4 * cc + 2] = q.z;
                        v[4 * cc + 3] = q.w;
                    }
                    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + kAring + kAcols * (uint32_t)lb;
                    if constexpr (TA == 1) {
                        uint32_t lo[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) lo[k] = __float_as_uint(v[k] - tc::tf32_trunc(v[k]));
                        tc::st32(ta + 64u * tile, reinterpret_cast<const uint32_t*>(v));
                        tc::st32(ta + 64u * tile + 32u, lo);
                    } else {
                        uint32_t pk[32];
#pragma unroll
                        for (int k2 = 0; k2 < 16; ++k2) tc::split_bf2(v[2 * k2], v[2 * k2 + 1], pk[k2], pk[16 + k2]);
                        tc::st32(ta + 32u * tile, pk);
                    }
                }
                tc::wait_st();
                tc::fence_before();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (tc_ == 0) {
                    mbar_arrive(&afull[lb]);
                    mbar_arrive(&yfree[st]);
                }
            }
        }
    } else {
        // ================= epilogue =================
        const int e = warp - 4, we = e & 3;
        constexpr int kRec = NL * QM * LlrTraits<LT>::bytes;
        const bool zf = !(a.sigma2 > 0.f);
        const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll 1
        for (long long i = 0; i < n_my; ++i) {
            const int b = (int)(i & 1);
            const long long u = u0 + i * du;
            const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
            mbar_wait_sleep(&accfull[b], (uint32_t)((i >> 1) & 1));
            tc::fence_after();
#pragma unroll 1
            for (int tile = CT ? (e >> 2) : 0; tile < (CT ? (e >> 2) + 1 : 2); ++tile) {
                if (!CT && tile == 1 && we < 2) break;
                uint32_t hv[32], lv[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * we) << 16) + 128u * (uint32_t)b + 64u * tile;
                tc::ld32(taddr, hv);
                tc::ld32(taddr + 32u, lv);
                tc::wait_ld();
                const int row = (tile ? (CT ? 128 : 40) : 0) + 32 * we + lane;
                if (tile == 1 && (CT ? row >= kRe : row < 128)) continue;
                const int s = row / kSc, f = row % kSc;
                const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
                float2 x[NL];
#pragma unroll
                for (int k = 0; k < NL; ++k)
                    x[k] = make_float2(__uint_as_float(hv[k]) + __uint_as_float(lv[k]),
                                       __uint_as_float(hv[16 + k]) + __uint_as_float(lv[16 + k]));
                const float* sl = sslope + (i & 3) * 16;
                if (a.llr) {
                    uint32_t wd[(kRec + 3) / 4];
                    if (LT == kLlrI8 && !zf) {
                        uint32_t q[NL * QM];
                        const float* rs = sslope + 64 + (i & 3) * 16;
#pragma unroll
                        for (int k = 0; k < NL; ++k) {
                            demap_axis_i8<QM / 2>(x[k].x, rs[k], q + k * QM, 2);
                            demap_axis_i8<QM / 2>(x[k].y, rs[k], q + k * QM + 1, 2);
                        }
#pragma unroll
                        for (int w4 = 0; w4 < NL * QM / 4; ++w4)
                            wd[w4] = __byte_perm(__byte_perm(q[4 * w4], q[4 * w4 + 1], 0x0040),
                                                 __byte_perm(q[4 * w4 + 2], q[4 * w4 + 3], 0x0040), 0x5410);
                    } else {
                        float v[NL * QM];
                        if (!zf) {
#pragma unroll
                            for (int k = 0; k < NL; ++k) demap_layer<QM, false, LT>(x[k], sl[k], v + k * QM);
                            pack_llr<LT, NL * QM, false>(v, wd);
                        } else {
#pragma unroll
                            for (int k = 0; k < NL; ++k) demap_layer<QM, true, LT>(x[k], sl[k], v + k * QM);
                            pack_llr<LT, NL * QM, true>(v, wd);
                        }
                    }
                    store_bytes<kRec>((char*)a.llr + re * kRec, wd);
                }
                if (a.xhat) {
#pragma unroll
                    for (int k = 0; k < NL; ++k) a.xhat[re * NL + k] = make_float2(x[k].x * ia, x[k].y * ia);
                }
            }
            tc::fence_before();
            asm volatile("bar.sync 2, %0;" ::"r"(32 * EW) : "memory");
            if (t == 128) mbar_arrive(&tfree[b]);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == CW) tc::dealloc<512>(tmem);
}

// ------------------------------------------------------------------------
// k_c5_setup: rows a2-a5 with the two contractions on the tensor cores and the
// factorisation on the FP32 pipe, two H-units per batch per CTA (4 warps):
//   a1  H_u (64 x 16 complex = 64 x 32 real X, row r = antenna) by a 2-D TMA box
//       (SWIZZLE_128B); X_lo = X - trunc(X) beside it (reading R21, TF32 split);
//   a2  C = Xe^T Xe with Xe = X + X_lo: 16 kind::tf32 MMAs (M = 64 = [X | X_lo]
//       columns, N = 32, K = 64 antennas), both operands MN-major views of the
//       same smem tile; G_kl = (C[2k][2l] + C[2k+1][2l+1]) + i (C[2k][2l+1] -
//       C[2k+1][2l]) + sigma2 delta_kl;
//   a3  G = L L^H, right-looking Cholesky in registers, one lane per row, the two
//       units in the two half-warps of warp 0, guard R17 on every pivot;
//   a4  X = L^-1 by forward substitution (lane k: column k), [G^-1]_kl = sum_i
//       conj(X_ik) X_il, A_kk = sum_i |X_ik|^2;
//   a5  mu, SINR, fac = sqrt(norm)/mu (readings R3/R4), B = real form of fac G^-1;
//   a4  W~^T = X B on the tensor cores: 8 kind::tf32 MMAs (M = 128 = [X; X_lo]
//       rows, N = 32, K = 32), W~[r] = D[r] + D[64 + r] -> workspace [r][k].
// The 64-row accumulators span all four TMEM lane quadrants, so every warp reads
// its quadrant and the halves meet in shared memory.
namespace su {
constexpr int UPB = 2;                        // units per batch
constexpr size_t X = 0;                       // [UPB] x (X 8 KiB | X_lo 8 KiB)
constexpr size_t BG = UPB * 16384;            // [UPB] x (B_hi 4 KiB | B_lo 4 KiB); also the exchange buffers
constexpr size_t CS = BG + 8192;              // [UPB][32][32] float C (G assembly), then X^-T rows; dead when
                                              // B is written (aliases unit 1's B set)
constexpr size_t BAR = BG + UPB * 8192;
constexpr size_t TSLOT = BAR + 16;
constexpr size_t TOTAL = TSLOT + 16 + 1024;   // + alignment slack
constexpr int CTAS_PER_SM = 4;
static_assert(TOTAL * CTAS_PER_SM <= 227 * 1024, "shared memory");
}  // namespace su

__device__ __forceinline__ float2 cmul_conj_a(float2 a, float2 b) {  // conj(a) * b
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}

template <int QM>
__global__ void __launch_bounds__(128, su::CTAS_PER_SM) k_c5_setup(DetectArgs a, const __grid_constant__ CUtensorMap hmap) {
    constexpr int NR = 64, NL = 16;
    constexpr int WS = BigWs<NR, NL>::stride;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    uint64_t* bar_tma = reinterpret_cast<uint64_t*>(g + su::BAR);
    uint64_t* bar_mma = bar_tma + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g + su::TSLOT);
    float* Cs = reinterpret_cast<float*>(g + su::CS);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const float norm = (float)qam_norm(QM);
    const long long n_batch = (a.n_units + su::UPB - 1) / su::UPB;

    pdl_launch_dependents();
    if (t == 0) {
        mbar_init(bar_tma, 1);
        mbar_init(bar_mma, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&hmap)) : "memory");
    }
    if (warp == 0) tc::alloc<64>(tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tslot;
    bool waited = false;  // PDL: wait for the previous grid before the first workspace write
    uint32_t it = 0;
#pragma unroll 1
    for (long long bt = blockIdx.x; bt < n_batch; bt += gridDim.x, ++it) {
        const long long ub = bt * su::UPB;
        const int nv = (int)min((long long)su::UPB, a.n_units - ub);  // valid units in this batch
        // ---- a1: H of the batch's units
        if (t == 0) {
            mbar_arrive_expect_tx(bar_tma, (uint32_t)(nv * NR * NL * 8));
            for (int s = 0; s < nv; ++s)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                    ::"r"(base + (uint32_t)(su::X + s * 16384)), "l"(reinterpret_cast<uint64_t>(&hmap)), "r"(0),
                    "r"((int)((ub + s) * NR)), "r"(smem_u32(bar_tma))
                    : "memory");
        }
        mbar_wait(bar_tma, it & 1);
        {  // X_lo = X - trunc(X) (same offsets: the SWIZZLE_128B pattern depends on address bits < 1024)
            for (int q = t; q < su::UPB * 512; q += 128) {
                const int s = q >> 9, o = q & 511;
                const float4 v = reinterpret_cast<const float4*>(g + su::X + s * 16384)[o];
                reinterpret_cast<float4*>(g + su::X + s * 16384 + 8192)[o] =
                    make_float4(v.x - tc::tf32_trunc(v.x), v.y - tc::tf32_trunc(v.y), v.z - tc::tf32_trunc(v.z),
                                v.w - tc::tf32_trunc(v.w));
            }
        }
        tc::fence_proxy_async();
        tc::fence_before();
        __syncthreads();
        // ---- a2: Gram on the tensor cores
        if (t == 0) {
            tc::fence_after();
            constexpr uint32_t idg = tc::idesc(tc::kFmtTF32, 64, 32, 1, 1);
            for (int s = 0; s < su::UPB; ++s) {
                const uint32_t xs = base + (uint32_t)(su::X + s * 16384);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {  // K = antennas 8 ks .. 8 ks + 7 = one 1024-B atom
                    const uint64_t dA = tc::desc_sw128(xs + 1024u * ks, 8192, 1024);  // M atoms: X cols | X_lo cols
                    tc::mma_tf32_ss(tmem + 32u * s, dA, tc::desc_sw128(xs + 1024u * ks, 8192, 1024), idg, ks ? 1u : 0u);
                    tc::mma_tf32_ss(tmem + 32u * s, dA, tc::desc_sw128(xs + 8192u + 1024u * ks, 8192, 1024), idg, 1u);
                }
            }
            tc::commit(bar_mma);
        }
        mbar_wait(bar_mma, 0);
        tc::fence_after();
        {  // M = 64 accumulator: row m in TMEM lane 32 (m / 16) + m % 16; C = D[0:32] + D[32:64]
            float* ex = reinterpret_cast<float*>(g + su::BG);  // [UPB][32][32]
#pragma unroll 1
            for (int s = 0; s < su::UPB; ++s) {
                uint32_t v[32];
                tc::ld32(tmem + ((uint32_t)(32 * warp) << 16) + 32u * s, v);
                tc::wait_ld();
                if (warp >= 2 && lane < 16) {
                    float4* dst = reinterpret_cast<float4*>(ex + (s * 32 + 16 * (warp - 2) + lane) * 32);
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        dst[c ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                                                          __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
                }
                __syncthreads();
                if (warp < 2 && lane < 16) {
                    const int m = 16 * warp + lane;
                    const float4* src = reinterpret_cast<const float4*>(ex + (s * 32 + m) * 32);
                    float4* dst = reinterpret_cast<float4*>(Cs + (s * 32 + m) * 32);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 e = src[c ^ (lane & 7)];
                        dst[c] = make_float4(__uint_as_float(v[4 * c]) + e.x, __uint_as_float(v[4 * c + 1]) + e.y,
                                             __uint_as_float(v[4 * c + 2]) + e.z, __uint_as_float(v[4 * c + 3]) + e.w);
                    }
                }
            }
        }
        tc::fence_before();
        __syncthreads();
        // ---- a3-a5: Cholesky, inverse, SINR and the B operand (warp 0; unit h = lane / 16, row k = lane % 16)
        if (warp == 0) {
            if (!waited) {
                pdl_wait();  // the previous call may still read the workspace
                waited = true;
            }
            const int h = lane >> 4, k = lane & 15, hb = lane & 16;
            const long long u = ub + h;
            const bool valid = h < nv;
            const float s2 = unit_sigma2(a, valid ? u : ub);
            float2 gr[NL];
            {
                const float* c0 = Cs + (h * 32 + 2 * k) * 32;
                const float* c1 = c0 + 32;
#pragma unroll
                for (int l = 0; l < NL; ++l) gr[l] = make_float2(c0[2 * l] + c1[2 * l + 1], c0[2 * l + 1] - c1[2 * l]);
            }
#pragma unroll
            for (int l = 0; l < NL; ++l)
                if (l == k) gr[l] = make_float2(gr[l].x + s2, 0.f);
            float gmax = 0.f;
#pragma unroll
            for (int l = 0; l < NL; ++l)
                if (l == k) gmax = gr[l].x;
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
            bool fail = !(gmax == gmax);
            const float tau = (float)kPivotTau * gmax;
            // a3: right-looking Cholesky; lane k's gr[m] (m <= k) becomes L[k][m]
            float dinv = 0.f;
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                float p = __shfl_sync(0xffffffffu, gr[j].x, hb | j);
                if (!(p > tau)) {
                    fail = true;
                    p = 1.f;
                }
                const float r = rsqrtf(p);
                if (k == j) dinv = r;
                if (k >= j) gr[j] = make_float2(gr[j].x * r, gr[j].y * r);
#pragma unroll
                for (int m = j + 1; m < NL; ++m) {
                    const float2 lm = shfl2(gr[j], hb | m);  // L[m][j]
                    if (k >= m) {  // G[k][m] -= L[k][j] conj(L[m][j])
                        gr[m].x = fmaf(-gr[j].x, lm.x, fmaf(-gr[j].y, lm.y, gr[m].x));
                        gr[m].y = fmaf(-gr[j].y, lm.x, fmaf(gr[j].x, lm.y, gr[m].y));
                    }
                }
            }
            // a4: column k of X = L^-1 by forward substitution: X_ik = -(1/L_ii) sum_{m<i} L_im X_mk
            float2 x[NL];
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                float2 sv = make_float2(0.f, 0.f);
#pragma unroll
                for (int m = 0; m < i; ++m) sv = cmac(sv, shfl2(gr[m], hb | i), x[m]);
                const float di = __shfl_sync(0xffffffffu, dinv, hb | i);
                x[i] = (i == k) ? make_float2(di, 0.f) : (i < k ? make_float2(0.f, 0.f) : make_float2(-sv.x * di, -sv.y * di));
            }
            float A = 0.f;
#pragma unroll
            for (int i = 0; i < NL; ++i) A = fmaf(x[i].x, x[i].x, fmaf(x[i].y, x[i].y, A));
            // columns of X through shared memory (row k of Xt = column k of X), then row k of G^-1
            float2* Xt = reinterpret_cast<float2*>(Cs) + h * NL * NL;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < NL; i += 2)
                *reinterpret_cast<float4*>(Xt + k * NL + i) = make_float4(x[i].x, x[i].y, x[i + 1].x, x[i + 1].y);
            __syncwarp();
            float2 gi[NL];
#pragma unroll
            for (int l = 0; l < NL; ++l) {
                float2 sv = make_float2(0.f, 0.f);
#pragma unroll
                for (int i = l & ~1; i < NL; i += 2) {  // X_il = 0 for i < l
                    const float4 v = *reinterpret_cast<const float4*>(Xt + l * NL + i);
                    const float2 c0 = cmul_conj_a(x[i], make_float2(v.x, v.y));
                    const float2 c1 = cmul_conj_a(x[i + 1], make_float2(v.z, v.w));
                    sv.x += c0.x + c1.x;
                    sv.y += c0.y + c1.y;
                }
                gi[l] = sv;
            }
            // a5
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
            // B operand of W~^T = X B: rows k (Re W~_k) and 16 + k (Im W~_k), K = (Re, Im) of layer j
            __syncwarp();  // every lane is done with Xt / C (aliased by the B sets)
            unsigned char* bg = g + su::BG + h * 8192;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float2 g0 = make_float2(fac * gi[2 * c].x, fac * gi[2 * c].y);
                const float2 g1 = make_float2(fac * gi[2 * c + 1].x, fac * gi[2 * c + 1].y);
                const float4 vr = make_float4(g0.x, g0.y, g1.x, g1.y);
                const float4 vi = make_float4(g0.y, -g0.x, g1.y, -g1.x);
                const int nr = k, ni = 16 + k;
                *reinterpret_cast<float4*>(bg + nr * 128 + ((c ^ (nr & 7)) << 4)) = vr;
                *reinterpret_cast<float4*>(bg + ni * 128 + ((c ^ (ni & 7)) << 4)) = vi;
                *reinterpret_cast<float4*>(bg + 4096 + nr * 128 + ((c ^ (nr & 7)) << 4)) =
                    make_float4(vr.x - tc::tf32_trunc(vr.x), vr.y - tc::tf32_trunc(vr.y), vr.z - tc::tf32_trunc(vr.z),
                                vr.w - tc::tf32_trunc(vr.w));
                *reinterpret_cast<float4*>(bg + 4096 + ni * 128 + ((c ^ (ni & 7)) << 4)) =
                    make_float4(vi.x - tc::tf32_trunc(vi.x), vi.y - tc::tf32_trunc(vi.y), vi.z - tc::tf32_trunc(vi.z),
                                vi.w - tc::tf32_trunc(vi.w));
            }
            if (valid) {
                float* wsu = reinterpret_cast<float*>(a.ws) + u * WS;
                wsu[NR * NL * 2 + k] = sinr / norm * a.llr_scale;
                if (a.sinr) a.sinr[u * NL + k] = sinr;
                if (k == 0 && fail) atomicAdd(a.fail_count, 1ull);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();
        // ---- a4: W~^T = [X; X_lo] (B_hi + B_lo) on the tensor cores
        if (t == 0) {
            tc::fence_after();
            constexpr uint32_t idw = tc::idesc(tc::kFmtTF32, 128, 32);
            for (int s = 0; s < su::UPB; ++s) {
                const uint32_t xs = base + (uint32_t)(su::X + s * 16384), bs = base + (uint32_t)(su::BG + s * 8192);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t dA = tc::desc_sw128(xs + 32u * ks);
                    tc::mma_tf32_ss(tmem + 32u * s, dA, tc::desc_sw128(bs + 32u * ks), idw, ks ? 1u : 0u);
                    tc::mma_tf32_ss(tmem + 32u * s, dA, tc::desc_sw128(bs + 4096u + 32u * ks), idw, 1u);
                }
            }
            tc::commit(bar_mma);
        }
        mbar_wait(bar_mma, 1);
        tc::fence_after();
        {  // M = 128 accumulator: row m in lane m. W~[r] = D[r] + D[64 + r]; rows 64-127 meet rows 0-63 in smem
            float* ex = reinterpret_cast<float*>(g + su::BG);  // [UPB][64][32] (B no longer needed)
#pragma unroll 1
            for (int s = 0; s < su::UPB; ++s) {
                uint32_t v[32];
                tc::ld32(tmem + ((uint32_t)(32 * warp) << 16) + 32u * s, v);
                tc::wait_ld();
                if (warp >= 2) {
                    float4* dst = reinterpret_cast<float4*>(ex + (s * 64 + 32 * (warp - 2) + lane) * 32);
#pragma unroll
                    for (int c = 0; c < 8; ++c)  // 16-byte piece c at c ^ (row & 7): conflict-free
                        dst[c ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                                                          __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
                }
                __syncthreads();
                if (warp < 2 && s < nv) {
                    const int r = 32 * warp + lane;
                    const float4* src = reinterpret_cast<const float4*>(ex + (s * 64 + r) * 32);
                    float w[32];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 e = src[c ^ (lane & 7)];
                        w[4 * c] = __uint_as_float(v[4 * c]) + e.x;
                        w[4 * c + 1] = __uint_as_float(v[4 * c + 1]) + e.y;
                        w[4 * c + 2] = __uint_as_float(v[4 * c + 2]) + e.z;
                        w[4 * c + 3] = __uint_as_float(v[4 * c + 3]) + e.w;
                    }
                    // row r of W~^T: columns 0-15 = Re W~_kr, 16-31 = Im W~_kr -> ws[u][r][k] float2
                    uint32_t o[32];
#pragma unroll
                    for (int kq = 0; kq < NL; ++kq) {
                        o[2 * kq] = __float_as_uint(w[kq]);
                        o[2 * kq + 1] = __float_as_uint(w[16 + kq]);
                    }
                    char* dst = reinterpret_cast<char*>(reinterpret_cast<float*>(a.ws) + (ub + s) * WS) + (size_t)r * NL * 8;
#pragma unroll
                    for (int q = 0; q < 4; ++q) st_v8(dst + 32 * q, o + 8 * q);
                }
            }
        }
        tc::fence_before();
        __syncthreads();
    }
    if (!waited) pdl_wait();
    if (warp == 0) tc::dealloc<64>(tmem);
}

// Setup kernels: SETUP = 0 SIMT Cholesky route (big_setup.cuh ALG 0), 1 SIMT Gauss-Jordan (ALG 1),
// 2 tensor-core contractions + register Cholesky (k_c5_setup).
template <int QM, int SETUP>
cudaError_t launch_setup(const DetectArgs& a, cudaStream_t s) {
    if constexpr (SETUP == 2) {
        static int n_sm = 0;
        if (!n_sm) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        }
        auto enc = tensor_map_encoder();
        if (!enc) return cudaErrorNotSupported;
        CUtensorMap hmap;  // H as {32 floats (16 layers re/im), n_units * 64 rows}; box = one unit (8 KiB)
        const cuuint64_t gdim[2] = {32, (cuuint64_t)a.n_units * 64};
        const cuuint64_t gstride[1] = {128};
        const cuuint32_t box[2] = {32, 64};
        const cuuint32_t estride[2] = {1, 1};
        if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(a.H), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
        const long long nb = (a.n_units + su::UPB - 1) / su::UPB;
        const long long cap = (long long)n_sm * su::CTAS_PER_SM;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(nb < cap ? nb : cap));
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = su::TOTAL;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = a.overlap ? 1 : 0;
        return cudaLaunchKernelEx(&cfg, k_c5_setup<QM>, a, hmap);
    } else {
        constexpr int UPB = 4;
        return launch_kernel(k_big_setup<64, 16, QM, UPB, SETUP == 0 ? 0 : 1>, dim3((unsigned)((a.n_units + UPB - 1) / UPB)),
                             dim3(32 * UPB), UPB * SetupSmem<64, 16, SETUP == 0 ? 0 : 1>::per_unit, s, a.overlap, a);
    }
}
template <int QM, int SETUP>
cudaError_t prepare_setup() {
    if constexpr (SETUP == 2)
        return cudaFuncSetAttribute(k_c5_setup<QM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)su::TOTAL);
    else
        return cudaFuncSetAttribute(k_big_setup<64, 16, QM, 4, SETUP == 0 ? 0 : 1>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(4 * SetupSmem<64, 16, SETUP == 0 ? 0 : 1>::per_unit));
}

template <int QM, int LT, int EW, int S, int NLO, int TA, int SETUP>
cudaError_t launch_c5(const DetectArgs& a, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap ymap;  // y as {128 floats (64 rx re/im), n_sc, n_sym}; box = one K chunk of a unit
    const cuuint64_t gdim[3] = {128, (cuuint64_t)a.n_sc, (cuuint64_t)a.n_sym};
    const cuuint64_t gstride[2] = {(cuuint64_t)64 * 8, (cuuint64_t)a.n_sc * 64 * 8};
    const cuuint32_t box[3] = {32, (cuuint32_t)kSc, (cuuint32_t)kSym};
    const cuuint32_t estride[3] = {1, 1, 1};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(a.y), gdim, gstride, box, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    cudaError_t e = launch_setup<QM, SETUP>(a, s);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.n_units < n_sm ? a.n_units : n_sm));
    cfg.blockDim = dim3(32 * (6 + EW));
    cfg.dynamicSmemBytes = C5Smem<S, NLO, TA>::total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_c5_apply<QM, LT, EW, S, NLO, TA>, a, ymap);
}

template <int QM, int LT, int EW, int S, int NLO, int TA, int SETUP>
cudaError_t prepare_c5() {
    cudaError_t e = prepare_setup<QM, SETUP>();
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_c5_apply<QM, LT, EW, S, NLO, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)C5Smem<S, NLO, TA>::total);
}

size_t c5_workspace(const DetectArgs& a) { return (size_t)a.n_units * BigWs<64, 16>::stride * 4; }

#define C5_ENTRY(NAME, QM, LT, EW, S, NLO, TA, SETUP)                                                     \
    KernelEntry {                                                                                          \
        NAME, 64, 16, QM, kSc, 14, LT, 32, 2, launch_c5<QM, LT, EW, S, NLO, TA, SETUP>,                    \
            prepare_c5<QM, LT, EW, S, NLO, TA, SETUP>, c5_workspace                                        \
    }

// First entry of a shape = its default (mimo_api.cu select_fast); the others are selectable by name.
const KernelEntry kEntries[] = {
    C5_ENTRY("c5_bf16_64x16_q6_i8", 6, kLlrI8, 6, 6, 4, 3, 1),  // C5 default
    C5_ENTRY("c5_tf32_64x16_q6_i8", 6, kLlrI8, 6, 4, 2, 1, 1),  // round-1 big8e6 operands
    C5_ENTRY("c5_bf16_chol_64x16_q6_i8", 6, kLlrI8, 6, 6, 4, 3, 0),
    C5_ENTRY("c5_bf16_tcs_64x16_q6_i8", 6, kLlrI8, 6, 6, 4, 3, 2),  // tensor-core setup
};

}  // namespace

const KernelEntry* c5_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
