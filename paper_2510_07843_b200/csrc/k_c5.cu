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

#include <type_traits>

#include "big_setup.cuh"
#include "tc.cuh"

// Optional per-role cycle accounting for tuning builds (tools/dbg/build_prof.sh compiles this
// file with -DC5_PROFILE into a separate library); compiled out of libmimo.so.
#ifdef C5_PROFILE
__device__ unsigned long long g_c5_prof[148 * 32];
extern "C" int mimo_c5_prof_read(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, g_c5_prof, sizeof(g_c5_prof));
}
extern "C" int mimo_c5_prof_reset() {
    static unsigned long long z[148 * 32] = {};
    return (int)cudaMemcpyToSymbol(g_c5_prof, z, sizeof(z));
}
#define PROF_T(v) const long long v = clock64()
#define PROF_ADD(acc, slot, t0) acc[slot] += (unsigned long long)(clock64() - (t0))
#define PROF_DECL unsigned long long prof[32] = {}
#define PROF_FLUSH(cond)                                                                   \
    if (cond)                                                                              \
        for (int _i = 0; _i < 32; ++_i)                                                    \
            if (prof[_i]) atomicAdd(&g_c5_prof[(blockIdx.x % 148) * 32 + _i], prof[_i]);
__device__ unsigned long long g_c5_sprof[148 * 32];
extern "C" int mimo_c5_sprof_read(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, g_c5_sprof, sizeof(g_c5_sprof));
}
#define PROF_SFLUSH(cond)                                                                  \
    if (cond)                                                                              \
        for (int _i = 0; _i < 32; ++_i)                                                    \
            if (prof[_i]) atomicAdd(&g_c5_sprof[(blockIdx.x % 148) * 32 + _i], prof[_i]);
#else
#define PROF_SFLUSH(cond)
#define PROF_T(v)
#define PROF_ADD(acc, slot, t0)
#define PROF_DECL
#define PROF_FLUSH(cond)
#endif

namespace mimo {
namespace {

template <int S_, int NLO_, int TA_, bool FUSED_ = false, int NB_ = 2, bool BI_ = false>
struct C5Smem {
    static constexpr int S = S_;                              // y stages
    static constexpr int NLO = NLO_;                          // TMEM A ring slots (chunks)
    static constexpr size_t chunk = (size_t)kRe * 128;        // 21504 = 21 x 1024
    static constexpr size_t y0 = 0;
    static constexpr size_t B = S * chunk;                    // NB_ B sets (1024-aligned)
    static constexpr size_t bset = TA_ == 1 ? 4 * 64 * 128 : 2 * 64 * 128;  // K atoms x 64 rows x 128 B
    static constexpr size_t slope = B + NB_ * bset;           // [8][16] slope | [8][16] sqrt(slope / 127)
    static constexpr size_t wst = slope + 1024;               // [2] W~ workspace records staged by TMA
    static constexpr size_t wrec = (size_t)BigWs<64, 16>::stride * 4;
    static constexpr size_t setup = (wst + (BI_ ? 0 : 2 * wrec) + 1023) / 1024 * 1024;  // FUSED: the setup group's 64 KiB
    static constexpr size_t bars = setup + (FUSED_ ? 65536 : 0);
    static constexpr int NBAR = 2 * S + 2 * NLO + NB_ * 3 + 4 + 2;  // yfull, yfree | afull, afree | bready, accfull, tfree | wfull, wfree | setup tma, mma
    static constexpr size_t ready = bars + NBAR * 8;           // FUSED: [0] units whose W~ records are written,
                                                               //        [1] units whose B sets are built
    static constexpr size_t tslot = ready + 8;
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

// demap_axis_i8 for the I and Q axes of one layer as packed pairs (FADD2 / FFMA2 / FMUL2 with the free
// |.| operand forms; only the saturating FMA and the sign select stay scalar): the same operations in the
// same order, so bit-identical to two demap_axis_i8 calls; q[2 i] = I LLR i, q[2 i + 1] = Q LLR i
template <int M>
__device__ __forceinline__ void demap_pair_i8(float2 u, float rs, uint32_t* q) {
    float2 t[M];
    t[0] = u;
#pragma unroll
    for (int i = 1; i < M; ++i)
        t[i] = fadd2_(make_float2(float(1 << (M - i)), float(1 << (M - i))),
                      make_float2(-fabsf(t[i - 1].x), -fabsf(t[i - 1].y)));
    const float2 rs2 = make_float2(rs, rs);
    const float2 e = ffma2(make_float2(fabsf(t[M - 1].x), fabsf(t[M - 1].y)), rs2, make_float2(-rs, -rs));
    const float2 nD = fmul2_(e, make_float2(-e.x, -e.y));  // -D, exactly
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const float2 at = ffma2(make_float2(fabsf(t[i].x), fabsf(t[i].y)), rs2, rs2);
        const float mx = fma_sat(at.x, at.x, nD.x), my = fma_sat(at.y, at.y, nD.y);
        const float2 s127 = make_float2(__uint_as_float((__float_as_uint(t[i].x) & 0x80000000u) | 0x42FE0000u),
                                        __uint_as_float((__float_as_uint(t[i].y) & 0x80000000u) | 0x42FE0000u));
        const float2 qq = ffma2(make_float2(mx, my), s127, make_float2(12582912.f, 12582912.f));
        q[2 * i] = __float_as_uint(qq.x);
        q[2 * i + 1] = __float_as_uint(qq.y);
    }
}

// ------------------------------------------------------------------------
// k_c5_setup: rows a2-a5 with both contractions on the tensor cores (BF16 split
// operands, reading R28) and the 16 x 16 inversion on the FP32 pipe. One CTA =
// 4 warps = 4 H-units per batch (warp w owns unit w of the batch):
//   a1  H_u (64 x 16 complex = 64 x 32 real X, row r = antenna) by a 2-D TMA box
//       (fp32, SWIZZLE_128B), converted to XB = [X_hi | X_lo] (bf16, 128-B row r,
//       same swizzle), X_hi = rn_bf16(X), X_lo = rn_bf16(X - X_hi);
//   a2  C = (X_hi + X_lo)^T (X_hi + X_lo): 16 kind::f16 MMAs with BOTH operands the
//       MN-major view of XB (M = 64 from the hi, then the lo columns, N = 32 hi then 32
//       lo, K = 64 antennas), C in D rows 0-31; G_kl = (C[2k][2l] + C[2k+1][2l+1]) +
//       i (C[2k][2l+1] - C[2k+1][2l]) + sigma2 delta_kl;
//   a3-a5  G^-1 by in-place Gauss-Jordan (no pivoting: G is Hermitian PD; its
//       pivots are the LDL^H pivots, so guard R17 reads the same quantities as
//       Cholesky's d_jj^2 -- reading R26), mu, SINR, fac = sqrt(norm) / mu,
//       B = real form of fac G^-1, split into bf16 hi / lo and duplicated along K;
//   a4  W~^T = XB B'^T: 8 kind::f16 MMAs, A = the K-major view of the SAME XB tile
//       (K = 64 = hi | lo halves of the 32 real inputs), B' = [B | B] (hi, lo).
// TMEM: 32 columns per unit (the Gram accumulator, reused for W~). M = 64
// accumulators put row m in lane 32 (m / 16) + m % 16, so every warp reads its
// lane quadrant of W~, and warps 0-1 read C.
// (A persistent warp-specialised variant -- producer, MMA, readout and 12 worker warps
// over a ring of unit slots -- measured 107-124 us against this kernel's 90, the
// per-slot chain of H load, Gram round trip and inversion being sequential.)
// Fused kernel: W~ records per CTA in the workspace ring (4 setup batches; the setup group waits for a
// slot only when it is that far ahead of the B builder, which consumes the records in order. 8 slots
// coupled the two and cost 15 us per C5 step; 16 are as fast as one record per unit and 4.6x smaller)
constexpr int kC5Ring = 16;
constexpr int kSetupConvUnroll = 2;  // 4 and 8 measured slower
// B-image records (the `bi` fused kernel): the setup group writes each unit's apply B operand itself -- the
// bf16 hi / lo split of the real form of W~, MN-major SWIZZLE_128B, K = 128 rows of 128 B -- followed by the
// 16 slopes and the 16 sqrt(slope / 127); the apply bulk-copies it straight into its B set (no B build)
constexpr int kBiImg = 128 * 128;
constexpr int kBiRec = kBiImg + 128;

// L2 eviction-priority helpers (BI == 4): y tiles and LLR records are streamed once; marking them
// evict-first keeps the B-image records (written a few units ahead of their copy) resident until consumed
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void st_v8_hint(void* p, const uint32_t* w, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "l"(pol)
                 : "memory");
}

// K row R of a B image from 32 words (8 chunks of 16 B: hi pairs n 0..31, then lo), SWIZZLE_128B positions
// (chunk q of row R at q ^ (R & 7)), as four 32-byte stores of chunk pairs; ODD = R & 1 (an odd row puts
// chunk q0 + 1 before chunk q0)
template <bool ODD>
__device__ __forceinline__ void bi_store_row(char* img, int R, const uint32_t* w) {
    const int sw = R & 7;
#pragma unroll
    for (int qp = 0; qp < 4; ++qp) {
        const int q0 = 2 * qp, p = q0 ^ sw;
        uint32_t o[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            o[e] = ODD ? w[4 * (q0 + 1) + e] : w[4 * q0 + e];
            o[4 + e] = ODD ? w[4 * q0 + e] : w[4 * (q0 + 1) + e];
        }
        st_v8(img + R * 128 + ((p & ~1) << 4), o);
    }
}

namespace su {
constexpr int UPB = 4;                   // units per batch (= warps)
constexpr size_t XB = 0;                 // [UPB] x 8 KiB  bf16 [64 r][hi c 0..31 | lo c 0..31], SW128
constexpr size_t BG = UPB * 8192;        // [UPB] x 8 KiB  H landing (fp32) -> exchange | C -> B'_hi | B'_lo
constexpr size_t BAR = BG + UPB * 8192;
constexpr size_t TSLOT = BAR + 16;
constexpr size_t TOTAL = TSLOT + 16 + 1024;  // + 1024-B alignment slack
constexpr int CTAS_PER_SM = 3;
static_assert(TOTAL * CTAS_PER_SM <= 227 * 1024, "shared memory");
}  // namespace su

// TMA of the H tiles of one setup batch (fp32, SWIZZLE_128B) into the group's B regions.
template <typename UnitF>
__device__ __forceinline__ void setup_issue_h(const CUtensorMap* hmapp, uint32_t gaddr, uint64_t* bar_tma, int nv,
                                              UnitF unit_of) {
    mbar_arrive_expect_tx(bar_tma, (uint32_t)(nv * 64 * 16 * 8));
    for (int s = 0; s < nv; ++s)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(gaddr + (uint32_t)(su::BG + s * 8192)), "l"(reinterpret_cast<uint64_t>(hmapp)), "r"(0),
            "r"((int)(unit_of(s) * 64)), "r"(smem_u32(bar_tma))
            : "memory");
}

// One batch of up to su::UPB = 4 H-units through rows a2-a5 (a1-a5 steps documented at k_c5_setup),
// run by a 4-warp group: gt = thread 0..127 of the group, gw = its warp 0..3 (= TMEM lane quadrant
// of the group's warps), g / gaddr = generic / shared address of the group's 64-KiB region (XB at
// su::XB, B sets at su::BG), tmem = the group's 128 TMEM columns, it = the group's batch count (TMA
// barrier parity), unit_of(s) = global H-unit of batch slot s < nv, sync() = the group's barrier.
// The batch's H tiles were issued by the previous batch (or the caller, for the first one);
// issue_next() issues the next batch's as soon as this batch's W~ MMAs have released the B regions,
// so that the H load overlaps the W~ readout.
//
// PUB (the fused kernel): the W~ records are read back by TMA inside the same kernel, so every writer
// thread makes its record stores visible at GPU scope and to the async proxy before they are published.
// That fence is deferred to the NEXT batch, after its conversion (the stores have drained by then and
// the fence costs nothing), and publish_prev() (after the group barrier) announces the previous batch;
// the caller fences and publishes the last batch itself.
// WIDE (the fused kernel, 256 TMEM columns): the Gram and W~ products as N = 64 MMAs (hi | lo halves side
// by side, summed at readout): 4 + 4 instead of 8 + 8 MMAs per unit; otherwise 128 columns.
//
// rec_of(s) = the workspace record (W~ + slopes) of batch slot s: the unit itself, or (fused) a slot of
// the CTA's ring of records, which ring_wait() (called by every thread before the batch's first record
// write) makes sure the apply has finished reading.
template <int QM, bool PUB, bool WIDE, int BI, typename UnitF, typename SyncF, typename NextF, typename PubF, typename RecF,
          typename RingF>
__device__ __forceinline__ void setup_batch(const DetectArgs& a, const CUtensorMap* hmapp, unsigned char* g,
                                            uint32_t gaddr, uint64_t* bar_tma, uint64_t* bar_mma, uint32_t tmem,
                                            uint32_t it, int nv, int gt, int gw, int lane, bool& waited,
                                            UnitF unit_of, SyncF sync, NextF issue_next, PubF publish_prev,
                                            RecF rec_of, RingF ring_wait) {
    constexpr int NR = 64, NL = 16;
    constexpr int WS = BigWs<NR, NL>::stride;
    const float norm = (float)qam_norm(QM);
    PROF_DECL;
        PROF_T(p0);
        // ---- a1: H of the batch (fp32, SW128) in the B regions -> XB = bf16 hi | lo
        mbar_wait(bar_tma, it & 1);
        PROF_ADD(prof, 0, p0);
        PROF_T(p1);
#pragma unroll (kSetupConvUnroll)
        for (int q = gt; q < su::UPB * 256; q += 128) {  // item = (unit, row r, 8 columns 8 cp .. 8 cp + 7)
            const int s = q >> 8, r = (q >> 2) & 63, cp = q & 3, sw = r & 7;
            const unsigned char* src = g + su::BG + s * 8192 + r * 128;
            const float4 v0 = *reinterpret_cast<const float4*>(src + (((2 * cp) ^ sw) << 4));
            const float4 v1 = *reinterpret_cast<const float4*>(src + (((2 * cp + 1) ^ sw) << 4));
            uint32_t hi[4], lo[4];
            tc::split_bf2(v0.x, v0.y, hi[0], lo[0]);
            tc::split_bf2(v0.z, v0.w, hi[1], lo[1]);
            tc::split_bf2(v1.x, v1.y, hi[2], lo[2]);
            tc::split_bf2(v1.z, v1.w, hi[3], lo[3]);
            unsigned char* dst = g + su::XB + s * 8192 + r * 128;
            *reinterpret_cast<uint4*>(dst + ((cp ^ sw) << 4)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(dst + (((4 + cp) ^ sw) << 4)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
        tc::fence_proxy_async();
        if constexpr (PUB) {
            if (it > 0) {  // the previous batch's W~ records (deferred, see above)
                __threadfence();
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
        }
        tc::fence_before();
        sync();
        if constexpr (PUB) publish_prev();
        PROF_ADD(prof, 1, p1);
        PROF_T(p2);
        // ---- a2: Gram, MN-major XB as both operands. A (M = 64) spans the whole 128-byte XB row = the hi
        // columns (D rows 0-31) and the lo columns (D rows 32-63); B (N = 32) is the hi, then (start + 64 B)
        // the lo columns: D = [hi | lo]^T (hi + lo), and C = (hi + lo)^T (hi + lo) = D[0:32] + D[32:64]
        // (two MMAs per K step instead of four N = 32, M = 32-useful ones)
        if (gt == 0) {
            tc::fence_after();
            constexpr uint32_t idg = tc::idesc(tc::kFmtBF16, 64, WIDE ? 64 : 32, 1, 1);
            for (int s = 0; s < su::UPB; ++s) {
                const uint32_t xs = gaddr + (uint32_t)(su::XB + s * 8192);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {  // K = antennas 16 ks .. 16 ks + 15 = two 8-row atoms
                    const uint64_t dh = tc::desc_sw128(xs + 2048u * ks, 16, 1024);
                    if constexpr (WIDE) {  // B = [hi | lo] (N = 64): D = [hi | lo]^T [hi | lo]
                        tc::mma_f16_ss(tmem + 64u * s, dh, dh, idg, ks ? 1u : 0u);
                    } else {
                        const uint64_t dl = tc::desc_sw128(xs + 64u + 2048u * ks, 16, 1024);
                        tc::mma_f16_ss(tmem + 32u * s, dh, dh, idg, ks ? 1u : 0u);
                        tc::mma_f16_ss(tmem + 32u * s, dh, dl, idg, 1u);
                    }
                }
            }
            tc::commit(bar_mma);
        }
        mbar_wait(bar_mma, 0);
        PROF_ADD(prof, 2, p2);
        PROF_T(p3);
        tc::fence_after();
        // M = 64 accumulator: D row m in TMEM lane 32 (m / 16) + m % 16, so warp w < 2 holds D rows 16 w + lane
        // (-> C_hi at BG + 4 KiB) and warp w >= 2 D rows 32 + 16 (w - 2) + lane (-> C_lo at BG); the inversion
        // sums the two
#pragma unroll 1
        for (int s = 0; s < su::UPB; ++s) {
            uint32_t v[32];
            if constexpr (WIDE) {  // columns n (B = hi) + n + 32 (B = lo)
                uint32_t v2[32];
                tc::ld32(tmem + ((uint32_t)(32 * gw) << 16) + 64u * s, v);
                tc::ld32(tmem + ((uint32_t)(32 * gw) << 16) + 64u * s + 32u, v2);
                tc::wait_ld();
#pragma unroll
                for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) + __uint_as_float(v2[c]));
            } else {
                tc::ld32(tmem + ((uint32_t)(32 * gw) << 16) + 32u * s, v);
                tc::wait_ld();
            }
            if (lane < 16) {
                const int m = 16 * (gw & 1) + lane;
                float* cs = reinterpret_cast<float*>(g + su::BG + s * 8192 + (gw < 2 ? 4096 : 0));
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    reinterpret_cast<float4*>(cs + m * 32)[c ^ (m & 7)] =
                        make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                                    __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
            }
        }
        tc::fence_before();
        sync();
        PROF_ADD(prof, 3, p3);
        PROF_T(p4);
        // ---- a3-a5: warp w inverts unit w; lane (k, h) = (lane / 2, lane % 2) holds G[k][8h .. 8h+7]
        if (!waited) {
            pdl_wait();
            waited = true;
        }
        PROF_ADD(prof, 8, p4);
        PROF_T(p4r);
        ring_wait();
        PROF_ADD(prof, 9, p4r);
        PROF_T(p4g);
        {
            const int s = gw, k = lane >> 1, h = lane & 1;
            const bool valid = s < nv;
            const long long u = valid ? unit_of(s) : unit_of(0);
            const float s2 = unit_sigma2(a, u);
            const float* cs = reinterpret_cast<const float*>(g + su::BG + s * 8192 + 4096);
            float2 gq[8];
            {
                const int m0 = 2 * k, m1 = 2 * k + 1;
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // columns 16h + 4i .. +3 = layers 8h + 2i, 8h + 2i + 1
                    const float4 a0 = reinterpret_cast<const float4*>(cs + m0 * 32)[(4 * h + i) ^ (m0 & 7)];
                    const float4 a1 = reinterpret_cast<const float4*>(cs + m1 * 32)[(4 * h + i) ^ (m1 & 7)];
                    const float4 b0 = reinterpret_cast<const float4*>(cs - 1024 + m0 * 32)[(4 * h + i) ^ (m0 & 7)];
                    const float4 b1 = reinterpret_cast<const float4*>(cs - 1024 + m1 * 32)[(4 * h + i) ^ (m1 & 7)];
                    const float4 c0 = make_float4(a0.x + b0.x, a0.y + b0.y, a0.z + b0.z, a0.w + b0.w);
                    const float4 c1 = make_float4(a1.x + b1.x, a1.y + b1.y, a1.z + b1.z, a1.w + b1.w);
                    gq[2 * i] = make_float2(c0.x + c1.y, c0.y - c1.x);
                    gq[2 * i + 1] = make_float2(c0.z + c1.w, c0.w - c1.z);
                }
            }
            float gd = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const bool d = 8 * h + q == k;
                gq[q].x += d ? s2 : 0.f;
                gq[q].y = d ? 0.f : gq[q].y;
                gd = fmaxf(gd, d ? gq[q].x : 0.f);
            }
            float gmax = gd;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
            bool fail = !(gmax == gmax);
            const float tau = (float)kPivotTau * gmax;
            // pivot loop rolled over the two column halves (hj), unrolled inside (qj): a fully unrolled
            // elimination starves the warps on instruction fetch. Pivot row j is published through shared memory (ping-pong 128-B row buffers in the unit's
            // free H landing area) instead of 16 shuffles per lane; the update b - (G[k][j] / p) r is two
            // packed FFMA2 per entry, the pivot row's own lanes take b = 0, fs = -1/p (so r / p exactly)
            float2* rowbuf = reinterpret_cast<float2*>(g + su::BG + s * 8192);
            __syncwarp();  // every lane has read its C rows (C2 lives here)
#pragma unroll 1
            for (int hj = 0; hj < 2; ++hj)
#pragma unroll
            for (int qj = 0; qj < 8; ++qj) {
                const int j = 8 * hj + qj;
                const bool prow = k == j;
                float4* rb = reinterpret_cast<float4*>(rowbuf + 16 * (qj & 1) + 8 * h);
                if (prow) {
#pragma unroll
                    for (int q2 = 0; q2 < 4; ++q2)
                        rb[q2] = make_float4(gq[2 * q2].x, gq[2 * q2].y, gq[2 * q2 + 1].x, gq[2 * q2 + 1].y);
                }
                const float2 f = shfl2(gq[qj], (lane & ~1) | hj);          // G[k][j]
                float p = __shfl_sync(0xffffffffu, gq[qj].x, 2 * j + hj);  // G[j][j]
                __syncwarp();
                if (!(p > tau)) {
                    fail = true;
                    p = 1.f;
                }
                float pinv;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(pinv) : "f"(p));
                const float2 fs = prow ? make_float2(-pinv, 0.f) : make_float2(f.x * pinv, f.y * pinv);
                const float m = prow ? 0.f : 1.f;
                const float2 nfx = make_float2(-fs.x, -fs.x), fyy = make_float2(fs.y, -fs.y), mm = make_float2(m, m);
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2) {
                    const float4 r4 = rb[q2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int q = 2 * q2 + e;
                        const float2 r = e ? make_float2(r4.z, r4.w) : make_float2(r4.x, r4.y);
                        float2 b = ffma2(gq[q], mm, make_float2(0.f, 0.f));
                        b = ffma2(nfx, r, b);
                        b = ffma2(fyy, make_float2(r.y, r.x), b);
                        if (q == qj && h == hj) b = prow ? make_float2(pinv, 0.f) : make_float2(-fs.x, -fs.y);
                        gq[q] = b;
                    }
                }
            }
            PROF_ADD(prof, 10, p4g);
            PROF_T(p4b);
            // A_kk = [G^-1]_kk lives in lane (k, k / 8)
            float Ad = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) Ad += (8 * h + q == k) ? gq[q].x : 0.f;
            const float A = Ad + __shfl_xor_sync(0xffffffffu, Ad, 1);
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
            __syncwarp();  // C is read; its region becomes B'_lo
            // B' rows k (Re W~_k) and 16 + k (Im W~_k): K pair (2l, 2l+1) = (Re, Im) parts, duplicated over
            // the hi | lo halves of K (chunks c and 4 + c); this lane's layers l = 8h .. 8h+7 = chunks 2h, 2h+1
            unsigned char* bh = g + su::BG + s * 8192;
            unsigned char* bl = bh + 4096;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                uint32_t rh[4], rl[4], ih[4], il[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 w = make_float2(fac * gq[4 * cc + e].x, fac * gq[4 * cc + e].y);
                    tc::split_bf2(w.x, w.y, rh[e], rl[e]);
                    tc::split_bf2(w.y, -w.x, ih[e], il[e]);
                }
                const int c = 2 * h + cc, nr = k, ni = 16 + k;
#pragma unroll
                for (int dup = 0; dup < 2; ++dup) {
                    const int cd = c + 4 * dup;
                    *reinterpret_cast<uint4*>(bh + nr * 128 + ((cd ^ (nr & 7)) << 4)) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
                    *reinterpret_cast<uint4*>(bl + nr * 128 + ((cd ^ (nr & 7)) << 4)) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
                    *reinterpret_cast<uint4*>(bh + ni * 128 + ((cd ^ (ni & 7)) << 4)) = make_uint4(ih[0], ih[1], ih[2], ih[3]);
                    *reinterpret_cast<uint4*>(bl + ni * 128 + ((cd ^ (ni & 7)) << 4)) = make_uint4(il[0], il[1], il[2], il[3]);
                }
            }
            if (valid && h == 0) {
                if constexpr (BI) {  // B-image record: slopes and sqrt(slope / 127) after the 16-KiB image
                    float* wsu = reinterpret_cast<float*>(reinterpret_cast<char*>(a.ws) + rec_of(s) * kBiRec + kBiImg);
                    const float slv = sinr / norm * a.llr_scale;
                    wsu[k] = slv;
                    wsu[16 + k] = sqrtf(slv * (1.f / 127.f));
                } else {
                    float* wsu = reinterpret_cast<float*>(a.ws) + rec_of(s) * WS;
                    wsu[NR * NL * 2 + k] = sinr / norm * a.llr_scale;
                }
                if (a.sinr) a.sinr[u * NL + k] = sinr;
                if (k == 0 && fail) atomicAdd(a.fail_count, 1ull);
            }
            PROF_ADD(prof, 11, p4b);
        }
        tc::fence_proxy_async();
        tc::fence_before();
        PROF_T(p4s);
        sync();
        PROF_ADD(prof, 12, p4s);
        PROF_ADD(prof, 4, p4);
        PROF_T(p5);
        // ---- a4: W~^T = XB B'^T (K-major view of XB: K = 64 = hi | lo halves)
        if (gt == 0) {
            tc::fence_after();
            constexpr uint32_t idw = tc::idesc(tc::kFmtBF16, 64, WIDE ? 64 : 32);
            for (int s = 0; s < su::UPB; ++s) {
                const uint32_t xs = gaddr + (uint32_t)(su::XB + s * 8192), bs = gaddr + (uint32_t)(su::BG + s * 8192);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint64_t dA = tc::desc_sw128(xs + 32u * ks);
                    if constexpr (WIDE) {  // B = [B'_hi rows; B'_lo rows] (N = 64, contiguous): D = [W_hi | W_lo]
                        tc::mma_f16_ss(tmem + 64u * s, dA, tc::desc_sw128(bs + 32u * ks), idw, ks ? 1u : 0u);
                    } else {
                        tc::mma_f16_ss(tmem + 32u * s, dA, tc::desc_sw128(bs + 32u * ks), idw, ks ? 1u : 0u);
                        tc::mma_f16_ss(tmem + 32u * s, dA, tc::desc_sw128(bs + 4096u + 32u * ks), idw, 1u);
                    }
                }
            }
            tc::commit(bar_mma);
        }
        mbar_wait(bar_mma, 1);
        if (gt == 0) issue_next();  // the B regions are free: the next batch's H loads under the W~ readout
        PROF_ADD(prof, 5, p5);
        PROF_T(p6);
        tc::fence_after();
#pragma unroll 1
        for (int s = 0; s < nv; ++s) {  // row r = 16 warp + lane of W~^T: cols k = Re W~_kr, 16 + k = Im W~_kr
            if constexpr (BI == 2 && WIDE) {
                // the whole warp: lane l < 16 takes antenna r = 16 warp + l, columns k (Re W~_kr), lane l + 16 the
                // same antenna's columns 16 + k (Im W~_kr); hi + lo products summed, split into bf16 hi / lo, and
                // each lane stores its halves of B-image rows 2r and 2r + 1 (Re lanes: row 2r chunks 0-1 | 4-5,
                // row 2r + 1 chunks 2-3 | 6-7; Im lanes: the others, negated in row 2r + 1)
                uint32_t v[16], v2[16];
                const uint32_t ta = tmem + ((uint32_t)(32 * gw) << 16) + 64u * s;
                tc::ld16x2_16<16>(ta, v);
                tc::ld16x2_16<16>(ta + 32u, v2);
                tc::wait_ld();
                const bool im = lane >= 16;
                const int r = 16 * gw + (lane & 15);
                uint32_t h[8], l[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    tc::split_bf2(__uint_as_float(v[2 * j]) + __uint_as_float(v2[2 * j]),
                                  __uint_as_float(v[2 * j + 1]) + __uint_as_float(v2[2 * j + 1]), h[j], l[j]);
                char* img = reinterpret_cast<char*>(a.ws) + rec_of(s) * kBiRec;
                // row 2r: this lane's chunk pair q0 = 0 (Re) / 2 (Im) for hi, + 4 for lo
                {
                    const int R = 2 * r, sw = R & 7, q0 = im ? 2 : 0;
                    st_v8(img + R * 128 + ((q0 ^ sw) << 4), h);
                    st_v8(img + R * 128 + (((4 + q0) ^ sw) << 4), l);
                }
                {
                    const int R = 2 * r + 1, sw = R & 7, q0 = im ? 0 : 2;  // odd row: chunk q0 + 1 lands first
                    const uint32_t sg = im ? 0x80008000u : 0u;
                    uint32_t oh[8], ol[8];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        oh[e] = h[4 + e] ^ sg;
                        oh[4 + e] = h[e] ^ sg;
                        ol[e] = l[4 + e] ^ sg;
                        ol[4 + e] = l[e] ^ sg;
                    }
                    st_v8(img + R * 128 + (((q0 ^ sw) & ~1) << 4), oh);
                    st_v8(img + R * 128 + ((((4 + q0) ^ sw) & ~1) << 4), ol);
                }
                continue;
            }
            uint32_t v[32];
            if constexpr (WIDE) {
                uint32_t v2[32];
                tc::ld32(tmem + ((uint32_t)(32 * gw) << 16) + 64u * s, v);
                tc::ld32(tmem + ((uint32_t)(32 * gw) << 16) + 64u * s + 32u, v2);
                tc::wait_ld();
#pragma unroll
                for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) + __uint_as_float(v2[c]));
            } else {
                tc::ld32(tmem + ((uint32_t)(32 * gw) << 16) + 32u * s, v);
                tc::wait_ld();
            }
            if (BI && lane < 16) {
                // B image (MN-major SW128 bf16, K row = real input 2r | 2r + 1 of antenna r, 128 B = [hi n 0..31 |
                // lo n 0..31]): K row 2r (x Re y_r) holds (Re W~_nr | Im W~_(n-16)r), K row 2r + 1 (x Im y_r)
                // holds (-Im W~_nr | Re W~_(n-16)r) = row 2r's halves swapped, the first negated (RN split is odd)
                const int r = 16 * gw + lane;
                uint32_t w0[32], w1[32];
#pragma unroll
                for (int j = 0; j < 16; ++j) tc::split_bf2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]), w0[j], w0[16 + j]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    w1[j] = w0[8 + j] ^ 0x80008000u;
                    w1[16 + j] = w0[24 + j] ^ 0x80008000u;
                    w1[8 + j] = w0[j];
                    w1[24 + j] = w0[16 + j];
                }
                char* dst = reinterpret_cast<char*>(a.ws) + rec_of(s) * kBiRec;
                bi_store_row<false>(dst, 2 * r, w0);
                bi_store_row<true>(dst, 2 * r + 1, w1);
            } else if (lane < 16) {
                const int r = 16 * gw + lane;
                uint32_t o[32];
#pragma unroll
                for (int kq = 0; kq < NL; ++kq) {
                    o[2 * kq] = v[kq];
                    o[2 * kq + 1] = v[16 + kq];
                }
                char* dst = reinterpret_cast<char*>(reinterpret_cast<float*>(a.ws) + rec_of(s) * WS) + (size_t)r * NL * 8;
#pragma unroll
                for (int q = 0; q < 4; ++q) st_v8(dst + 32 * q, o + 8 * q);
            }
        }
        PROF_ADD(prof, 6, p6);
        PROF_T(p7);
        tc::fence_before();
        sync();
        PROF_ADD(prof, 7, p7);
    PROF_SFLUSH(gt == 0);
}

// NACC = accumulators in TMEM = B sets in shared memory: unit i uses slot i % NACC, and its MMAs wait
// for the epilogue of unit i - NACC (and for B set i % NACC, built after unit i - NACC's MMAs).
template <int QM, int LT, int EW, int S_, int NLO_, int TA, bool BEPI, bool FUSED, int NACC = 2, int BI = 0>
__global__ void __launch_bounds__(32 * (6 + EW) + (FUSED ? 128 : 0), 1)
    k_c5_apply(DetectArgs a, const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap hmap) {
    constexpr int NR = 64, NL = 16;
    using SM = C5Smem<S_, NLO_, TA, FUSED, NACC, BI != 0>;
    static_assert(!BI || (FUSED && TA == 4), "B-image records: fused kernel, single-accumulator bf16 split");
    constexpr int S = S_, NLO = NLO_;
    static_assert(EW == 6, "6 epilogue warps (4 for tile 0, 2 for the compact tile 1)");

    static_assert(TA == 1 || TA == 3 || TA == 4, "TF32 or BF16 operands");
    // TA = 4: BF16 with the three split products accumulated into ONE 32-column accumulator per tile
    // (A = y_hi with B_hi and B_lo, then y_lo with B_hi, all N = 32): x~ needs no hi + lo sum, and the
    // two accumulators take 128 TMEM columns instead of 256
    constexpr bool KC = TA == 4;
    constexpr uint32_t kAccCols = KC ? 64u : 128u;   // TMEM columns per accumulator (2 row tiles)
    constexpr uint32_t kAring = NACC * kAccCols;     // TMEM columns 0 .. kAring-1: NACC accumulators
    constexpr uint32_t kAcols = TA == 1 ? 128u : 64u;  // TMEM columns per A ring slot (one chunk, 2 tiles)
    constexpr bool kWide = kAring + NLO * kAcols + 256u <= 512u;  // FUSED: room for the wide setup products
    static_assert(kAring + NLO * kAcols + (FUSED ? 128u : 0u) <= 512u, "TMEM");
    static_assert(!FUSED || BEPI, "fused setup: the epilogue warps build the B sets");
    constexpr uint32_t kSetupCols = kAring + NLO * kAcols;  // FUSED: the setup group's 128 / 256 TMEM columns
    constexpr int CW = 4 + EW;                       // MMA warp; CW + 1: TMA producer
    constexpr int WS = BigWs<NR, NL>::stride;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    // workspace record of local unit i: FUSED = slot i % kC5Ring of this CTA's ring (reused: 20 MB instead of 91),
    // otherwise the unit's own record (written by the setup kernel)
    auto rec_of = [&](long long i) -> long long {
        if constexpr (FUSED) return (long long)blockIdx.x * kC5Ring + i % kC5Ring;
        else return (long long)blockIdx.x + i * (long long)gridDim.x;
    };
    uint64_t* bar = reinterpret_cast<uint64_t*>(g + SM::bars);
    uint64_t* yfull = bar;             // [S]    TMA tx
    uint64_t* yfree = bar + S;         // [S]    converters done with the stage
    uint64_t* afull = bar + 2 * S;     // [NLO]  converters stored the chunk's A rows
    uint64_t* afree = afull + NLO;     // [NLO]  MMAs of the chunk completed
    uint64_t* bready = afree + NLO;    // [NACC] B set built
    uint64_t* accfull = bready + NACC; // [NACC] the unit's last MMA completed
    uint64_t* tfree = accfull + NACC;  // [NACC] epilogue done with the accumulator
    uint64_t* wfull = tfree + NACC;    // [2]    W~ record of unit i staged (TMA tx)
    uint64_t* wfree = wfull + 2;       // [2]    B set built from it
    uint64_t* stma = wfree + 2;        //        FUSED: setup group's H TMA
    uint64_t* smma = stma + 1;         //        FUSED: setup group's MMAs
    volatile int* units_ready = reinterpret_cast<volatile int*>(g + SM::ready);  // FUSED
    volatile int* units_built = units_ready + 1;                                 // FUSED
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g + SM::tslot);
    float* sslope = reinterpret_cast<float*>(g + SM::slope);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long u0 = blockIdx.x, du = gridDim.x;
    const long long n_my = u0 < a.n_units ? (a.n_units - u0 + du - 1) / du : 0;
    const long long G = 4 * n_my;

    pdl_launch_dependents();
    if (t == 0) {
        constexpr uint32_t ngrp = 1;
        for (int i = 0; i < S; ++i) {
            mbar_init(&yfull[i], 1);
            mbar_init(&yfree[i], ngrp);
        }
        for (int i = 0; i < NLO; ++i) {
            mbar_init(&afull[i], ngrp);
            mbar_init(&afree[i], 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(&bready[i], 1);
            mbar_init(&accfull[i], 1);
            mbar_init(&tfree[i], ngrp);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wfree[i], 1);
        }
        mbar_init(stma, 1);
        mbar_init(smma, 1);
        *units_ready = 0;
        *units_built = 0;
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
            PROF_DECL;
            PROF_T(tk0);
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ymap)) : "memory");
            // !BEPI: W~ records (rows a2-a5 of the setup kernel) of units i = j + 2 are staged when the y
            // chunks of unit j start (BEPI: by the B builder, so that the y stream never waits on them); y
            // itself is this call's input and streams before the setup completes
            auto issue_w = [&](long long i) {
                const int ws_ = (int)(i & 1);
                if (i >= 2) mbar_wait_sleep(&wfree[ws_], (uint32_t)(((i >> 1) + 1) & 1));
                if constexpr (FUSED) {  // the setup group of this CTA has written unit i's W~ record
                    PROF_T(tsw);
                    while (*units_ready <= i) __nanosleep(64);
                    PROF_ADD(prof, 1, tsw);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                mbar_arrive_expect_tx(&wfull[ws_], (uint32_t)SM::wrec);
                bulk_g2s(g + SM::wst + ws_ * SM::wrec, reinterpret_cast<const float*>(a.ws) + rec_of(i) * WS,
                         (uint32_t)SM::wrec, &wfull[ws_]);
            };
            bool waited = false;
#pragma unroll 1
            for (long long gg = 0; gg < G; ++gg) {
                const int st = (int)(gg % S);
                if (!BEPI && (gg & 3) == 0) {
                    if (!waited) {
                        pdl_wait();  // the setup kernel of this call has written the workspace
                        waited = true;
                        issue_w(0);
                        if (n_my > 1) issue_w(1);
                    }
                    if ((gg >> 2) + 2 < n_my) issue_w((gg >> 2) + 2);
                }
                PROF_T(tw);
                if (gg >= S) mbar_wait_sleep(&yfree[st], (uint32_t)(((gg / S) + 1) & 1));
                PROF_ADD(prof, 0, tw);
                const long long uu = u0 + (gg >> 2) * du;
                const int slot = (int)(uu / a.n_fb), fb = (int)(uu % a.n_fb);
                mbar_arrive_expect_tx(&yfull[st], (uint32_t)SM::chunk);
                if constexpr (BI == 4)
                    tma_load_3d_hint(base + (uint32_t)(SM::y0 + st * SM::chunk), &ymap, 32 * (int)(gg & 3), fb * kSc,
                                     slot * kSym, &yfull[st], l2_evict_first_policy());
                else
                    tma_load_3d(base + (uint32_t)(SM::y0 + st * SM::chunk), &ymap, 32 * (int)(gg & 3), fb * kSc,
                                slot * kSym, &yfull[st]);
            }
            PROF_ADD(prof, 31, tk0);
            PROF_FLUSH(true);
        }
    } else if (FUSED && warp >= CW + 2) {
        // ================= fused setup group (warps 12-15 = lane quadrants 0-3): rows a2-a5 of this CTA's
        // units, four at a time, ahead of the apply pipeline; W~ records to the workspace (L2-resident
        // by the time the producer stages them), progress published through units_ready =================
        const int gw = warp - (CW + 2), gt = t - 32 * (CW + 2);
        bool waited = false;
        uint32_t it = 0;
        if (gt == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&hmap)) : "memory");
        auto nv_of = [&](long long j0) { return (int)min((long long)su::UPB, n_my - j0); };
        if (gt == 0 && n_my > 0)
            setup_issue_h(&hmap, base + (uint32_t)SM::setup, stma, nv_of(0), [&](int s_) { return u0 + s_ * du; });
#pragma unroll 1
        for (long long j0 = 0; j0 < n_my; j0 += su::UPB, ++it) {
            const int nv = nv_of(j0);
            const long long jn = j0 + su::UPB;
            setup_batch<QM, true, kWide, (BI == 3 || BI == 4) ? 2 : (BI != 0 ? 1 : 0)>(a, &hmap, g + SM::setup, base + (uint32_t)SM::setup, stma, smma, tmem + kSetupCols, it,
                                  nv, gt, gw, lane, waited, [&](int s_) { return u0 + (j0 + s_) * du; },
                                  [] { asm volatile("bar.sync 5, 128;" ::: "memory"); },
                                  [&] {
                                      if (jn < n_my)
                                          setup_issue_h(&hmap, base + (uint32_t)SM::setup, stma, nv_of(jn),
                                                        [&](int s_) { return u0 + (jn + s_) * du; });
                                  },
                                  [&] {
                                      if (gt == 0) *units_ready = (int)j0;  // batches before this one are visible
                                  },
                                  [&](int s_) { return rec_of(j0 + s_); },
                                  [&] {  // ring slots of units j0 .. j0 + nv - 1 held units j0 - kC5Ring ..: built?
                                      while (*units_built < (int)(j0 + nv - kC5Ring)) __nanosleep(32);
                                      if constexpr (BI >= 2) __threadfence_block();  // acquire: after the L2 discards
                                  });
            if (j0 == 0 && nv < n_my) {
                // the first batch is published at once (the others one batch late, see setup_batch): the apply
                // pipeline idles until it is
                __threadfence();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                asm volatile("bar.sync 5, 128;" ::: "memory");
                if (gt == 0) *units_ready = nv;
            }
        }
        if (n_my > 0) {  // the last batch
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("bar.sync 5, 128;" ::: "memory");
            if (gt == 0) *units_ready = (int)n_my;
        }
        if (!waited) pdl_wait();
    } else if (warp == CW) {
        // ================= MMA issuer =================
        if (lane == 0) {
            constexpr uint32_t f = TA == 1 ? tc::kFmtTF32 : tc::kFmtBF16;
            // BI: B is the MN-major image (K row = real input, [hi n 0..31 | lo n 0..31])
            constexpr uint32_t id64 = tc::idesc(f, 128, 64), id32 = tc::idesc(f, 128, 32, 0, BI ? 1 : 0);
            const uint64_t dB = tc::desc_sw128(base + (uint32_t)SM::B);
            PROF_DECL;
#pragma unroll 1
            for (long long i = 0; i < n_my; ++i) {
                const int b = (int)(i % NACC);
                const uint32_t ph = (uint32_t)(i / NACC);  // completion index of this unit on slot b
                PROF_T(t0);
                mbar_wait_sleep(&bready[b], ph & 1u);
                PROF_ADD(prof, 8, t0);
                PROF_T(t1);
                if (i >= NACC) mbar_wait_sleep(&tfree[b], (ph + 1u) & 1u);
                PROF_ADD(prof, 9, t1);
                const uint32_t acc = tmem + kAccCols * (uint32_t)b;
                const uint64_t db = tc::desc_add(dB, (uint32_t)(b * SM::bset));
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    const long long gg = 4 * i + c;
                    const int lb = (int)(gg % NLO);
                    const uint32_t ab = tmem + kAring + kAcols * (uint32_t)lb;
                    PROF_T(t2);
                    mbar_wait_sleep(&afull[lb], (uint32_t)((gg / NLO) & 1));
                    PROF_ADD(prof, 10, t2);
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
                    } else if constexpr (KC) {  // 2 K-steps of 16, three N = 32 products into one accumulator
#pragma unroll
                        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                            for (int ks = 0; ks < 2; ++ks) {
                                const uint64_t dk = BI ? tc::desc_add(db, (uint32_t)(c * 4096 + ks * 2048))
                                                       : tc::desc_add(db, (uint32_t)((c >> 1) * 8192 + (c & 1) * 64 + ks * 32));
                                const uint64_t dkl = tc::desc_add(dk, BI ? 64u : 4096u);  // B_lo (BI: the lo half of each K row)
                                tc::mma_f16_ts(acc + 32u * tile, ab + 32u * tile + 8u * ks, dk, id32, (c | ks) ? 1u : 0u);
                                tc::mma_f16_ts(acc + 32u * tile, ab + 32u * tile + 8u * ks, dkl, id32, 1u);
                                tc::mma_f16_ts(acc + 32u * tile, ab + 32u * tile + 16u + 8u * ks, dk, id32, 1u);
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
            PROF_FLUSH(true);
        }
    } else {
        // ---- shared pieces of the converter and epilogue roles
        // convert RE row r of stage st into TMEM A-ring slot lb, row tile `tile`, this warp's lane quadrant
        auto convert_row = [&](int st, int lb, int tile, int r, int quad) {
            const float4* row = reinterpret_cast<const float4*>(g + SM::y0 + st * SM::chunk + (size_t)r * 128);
            float v[32];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const float4 q = row[cc ^ (r & 7)];  // SWIZZLE_128B: 16-byte piece cc of row r
                v[4 * cc] = q.x;
                v[4 * cc + 1] = q.y;
                v[4 * cc + 2] = q.z;
                v[4 * cc + 3] = q.w;
            }
            const uint32_t ta = tmem + ((uint32_t)(32 * quad) << 16) + kAring + kAcols * (uint32_t)lb;
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
        };
        constexpr int kRec = NL * QM * LlrTraits<LT>::bytes;
        const bool zf = !(a.sigma2 > 0.f);
        const float ia = rsqrtf((float)qam_norm(QM));
        // x~ of RE `row` (TMEM lane quadrant `quad`, accumulator b, row tile `tile`) -> LLR record
        auto epilogue_row = [&](long long i, int b, int tile, int row, int quad, bool active) {
            uint32_t hv[32], lv[KC ? 1 : 32];
            const uint32_t taddr = tmem + ((uint32_t)(32 * quad) << 16) + kAccCols * (uint32_t)b + (kAccCols / 2) * tile;
            tc::ld32(taddr, hv);
            if constexpr (!KC) tc::ld32(taddr + 32u, lv);
            tc::wait_ld();
            if (!active) return;
            const long long u = u0 + i * du;
            const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
            const int s = row / kSc, f = row % kSc;
            const size_t re = (size_t)(slot * kSym + s) * a.n_sc + fb * kSc + f;
            float2 x[NL];
#pragma unroll
            for (int k = 0; k < NL; ++k) {
                if constexpr (KC) x[k] = make_float2(__uint_as_float(hv[k]), __uint_as_float(hv[16 + k]));
                else x[k] = make_float2(__uint_as_float(hv[k]) + __uint_as_float(lv[k]),
                                        __uint_as_float(hv[16 + k]) + __uint_as_float(lv[16 + k]));
            }
            const float* sl = sslope + (i & 7) * (BI ? 32 : 16);  // BI: [8][slope 16 | rs 16] (one copy per unit)
            if (a.llr) {
                uint32_t wd[(kRec + 3) / 4];
                if (LT == kLlrI8 && !zf) {
                    uint32_t q[NL * QM];
                    const float* rs = BI ? sl + 16 : sslope + 128 + (i & 7) * 16;
#pragma unroll
                    for (int k = 0; k < NL; ++k) demap_pair_i8<QM / 2>(x[k], rs[k], q + k * QM);
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
                if constexpr (BI == 4 && kRec % 32 == 0) {
                    const uint64_t pol = l2_evict_first_policy();
#pragma unroll
                    for (int q = 0; q < kRec / 32; ++q) st_v8_hint((char*)a.llr + re * kRec + 32 * q, wd + 8 * q, pol);
                } else {
                    store_bytes<kRec>((char*)a.llr + re * kRec, wd);
                }
            }
            if (a.xhat) {
#pragma unroll
                for (int k = 0; k < NL; ++k) a.xhat[re * NL + k] = make_float2(x[k].x * ia, x[k].y * ia);
            }
        };

        // B = [B_hi; B_lo] of unit i (bf16 or tf32 split of the real form of W~) into B set i % NACC, and the
        // unit's slopes into slope ring slot i & 7; tid in 0..127 of the building warp group
        auto build_B = [&](long long i, int tid) {
            // thread = (B row n = lane, K quarter kt = warp): the 32 lanes of a warp read 16 distinct W~ entries
            // of one antenna row (no bank conflicts; n and n + 16 share theirs) and store one 16-byte piece each
            const int n = tid & 31, kt = tid >> 5, kk = n & 15, b = (int)(i % NACC);
            const bool im_row = n >= 16;
            mbar_wait_sleep(&wfull[i & 1], (uint32_t)((i >> 1) & 1));
            const float2* src = reinterpret_cast<const float2*>(g + SM::wst + (i & 1) * SM::wrec);
            float2 wv[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) wv[c] = src[(16 * kt + c) * NL + kk];  // this thread's 16 antennas of row kk
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
            if (tid < NL) {
                const float slv = reinterpret_cast<const float*>(src + NR * NL)[tid];
                sslope[(i & 7) * 16 + tid] = slv;
                sslope[128 + (i & 7) * 16 + tid] = sqrtf(slv * (1.f / 127.f));
            }
            tc::fence_proxy_async();
        };

        if (warp < 4) {
            // ================= converter group: y rows -> TMEM A ring (+ the B sets unless BEPI) =================
            const int tc_ = t;  // 0..127
            PROF_DECL;
#pragma unroll 1
            for (long long i = 0; i < n_my; ++i) {
                const int b = (int)(i % NACC);
                if constexpr (!BEPI) {
                    // B set b is free once unit i-NACC's MMAs completed; the slope ring slot i & 7 was last read
                    // by epilogue(i-8), which finished before tfree(i-8) < accfull(i-NACC)
                    PROF_T(t0);
                    if (i >= NACC) mbar_wait_sleep(&accfull[b], (uint32_t)(((i / NACC) + 1) & 1));
                    PROF_ADD(prof, 16, t0);
                    PROF_T(t1);
                    build_B(i, tc_);
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (tc_ == 0) {
                        mbar_arrive(&bready[b]);
                        mbar_arrive(&wfree[i & 1]);
                    }
                    PROF_ADD(prof, 17, t1);
                }
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    const long long gg = 4 * i + c;
                    const int st = (int)(gg % S), lb = (int)(gg % NLO);
                    PROF_T(t2);
                    mbar_wait_sleep(&yfull[st], (uint32_t)((gg / S) & 1));
                    PROF_ADD(prof, 18, t2);
                    PROF_T(t3);
                    if (gg >= NLO) mbar_wait_sleep(&afree[lb], (uint32_t)(((gg / NLO) + 1) & 1));
                    PROF_ADD(prof, 19, t3);
                    PROF_T(t4);
                    tc::fence_after();
                    convert_row(st, lb, 0, 32 * warp + lane, warp);
                    if (warp < 2) convert_row(st, lb, 1, min(128 + 32 * warp + lane, kRe - 1), warp);  // REs 128-167
                    tc::wait_st();
                    PROF_ADD(prof, 20, t4);
                    PROF_T(t5);
                    tc::fence_before();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (tc_ == 0) {
                        mbar_arrive(&afull[lb]);
                        mbar_arrive(&yfree[st]);
                    }
                    PROF_ADD(prof, 21, t5);
                }
            }
            PROF_FLUSH(t == 0);
        } else {
            // ================= epilogue: tile 0 on warps 4-7, compact tile 1 on warps 8-9 =================
            // (BEPI: warps 4-7 also build the B set of unit i + 2 as soon as unit i's MMAs completed)
            const int e = warp - 4, we = e & 3, tile = e >> 2;
            PROF_DECL;
            // BEPI: thread 128 stages the W~ record of unit i into W stage i & 1 (after the B set that last
            // read the stage was built); FUSED: once this CTA's setup group has published unit i
            auto issue_w = [&](long long i) {
                if constexpr (FUSED) {
                    while (*units_ready <= i) __nanosleep(64);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                mbar_arrive_expect_tx(&wfull[i & 1], (uint32_t)SM::wrec);
                bulk_g2s(g + SM::wst + (i & 1) * SM::wrec, reinterpret_cast<const float*>(a.ws) + rec_of(i) * WS,
                         (uint32_t)SM::wrec, &wfull[i & 1]);
            };
            // BI: thread 128 bulk-copies unit j's B image into B set j % NACC and its slopes into slope slot j & 7
            // (once this CTA's setup group has published it; the B set's previous unit j - NACC has completed
            // its MMAs, the slope slot's unit j - 8 its epilogue)
            auto issue_b = [&](long long j) {
                while (*units_ready <= j) __nanosleep(64);
                asm volatile("fence.proxy.async.global;" ::: "memory");
                const char* src = reinterpret_cast<const char*>(a.ws) + rec_of(j) * kBiRec;
                uint64_t* bb = &bready[j % NACC];
                mbar_arrive_expect_tx(bb, (uint32_t)kBiRec);
                bulk_g2s(g + SM::B + (j % NACC) * SM::bset, src, (uint32_t)kBiImg, bb);
                bulk_g2s(sslope + (j & 7) * 32, src + kBiImg, 128u, bb);
            };
            if constexpr (BI) {
                if (t == 128) {
                    PROF_T(ts);
                    pdl_wait();
                    for (long long j = 0; j < NACC && j < n_my; ++j) issue_b(j);
                    PROF_ADD(prof, 30, ts);
                }
            } else if constexpr (BEPI) {
                if (warp < 8) {  // B sets of units 0 .. NACC-1; W stage j & 1 is refilled with unit j + 2's record
                    if (t == 128) {
                        pdl_wait();  // the setup (kernel or group) of this call writes the workspace
                        for (long long i0 = 0; i0 < 2 && i0 < n_my; ++i0) issue_w(i0);
                    }
                    for (long long j = 0; j < NACC && j < n_my; ++j) {
                        build_B(j, t - 128);
                        asm volatile("bar.sync 4, 128;" ::: "memory");
                        if (t == 128) {
                            mbar_arrive(&bready[j]);
                            if constexpr (FUSED) *units_built = (int)(j + 1);
                            if (j + 2 < n_my) issue_w(j + 2);
                        }
                    }
                }
            }
#pragma unroll 1
            for (long long i = 0; i < n_my; ++i) {
                const int b = (int)(i % NACC);
                PROF_T(t0);
                mbar_wait_sleep(&accfull[b], (uint32_t)((i / NACC) & 1));
                PROF_ADD(prof, 24, t0);
                tc::fence_after();
                if constexpr (BI) {
                    if (t == 128 && i + NACC < n_my) {  // B set b is free: unit i's MMAs completed
                        PROF_T(ti);
                        issue_b(i + NACC);
                        PROF_ADD(prof, 29, ti);
                    }
                    if (warp == 8) {
                        // unit i's record has been copied (its MMAs read the B set): drop its L2 lines without
                        // the write-back, then hand the ring slot back to the setup group
                        if constexpr (BI >= 2) {
                            const char* rec = reinterpret_cast<const char*>(a.ws) + rec_of(i) * kBiRec;
                            for (int l = lane; l < kBiRec / 128; l += 32)
                                asm volatile("discard.global.L2 [%0], 128;" ::"l"(rec + 128 * l) : "memory");
                        }
                        __syncwarp();  // orders the warp's discards before lane 0's release (CTA scope: the
                        if (lane == 0) {  // setup group that rewrites the slot is in this CTA)
                            if constexpr (BI >= 2) __threadfence_block();
                            *units_built = (int)(i + 1);
                        }
                    }
                } else if constexpr (BEPI) {
                    if (warp < 8 && i + NACC < n_my) {  // B set b is free: unit i's MMAs completed
                        PROF_T(tb);
#ifdef C5_PROFILE
                        {
                            PROF_T(tw);
                            mbar_wait_sleep(&wfull[(i + NACC) & 1], (uint32_t)(((i + NACC) >> 1) & 1));
                            PROF_ADD(prof, 28, tw);
                        }
#endif
                        build_B(i + NACC, t - 128);
                        asm volatile("bar.sync 4, 128;" ::: "memory");
                        if (t == 128) {
                            mbar_arrive(&bready[b]);
                            if constexpr (FUSED) *units_built = (int)(i + NACC + 1);
                            PROF_T(ti);
                            if (i + NACC + 2 < n_my) issue_w(i + NACC + 2);  // its W stage is read
                            PROF_ADD(prof, 29, ti);
                        }
                        PROF_ADD(prof, 27, tb);
                    }
                }
                PROF_T(t1);
                const int row = (tile ? 128 : 0) + 32 * we + lane;
                epilogue_row(i, b, tile, row, we, row < kRe);
                PROF_ADD(prof, 25, t1);
                PROF_T(t2);
                tc::fence_before();
                asm volatile("bar.sync 2, %0;" ::"r"(32 * EW) : "memory");
                if (t == 128) mbar_arrive(&tfree[b]);
                PROF_ADD(prof, 26, t2);
            }
            PROF_FLUSH(t == 128);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == CW) tc::dealloc<512>(tmem);
}

template <int QM>
__global__ void __launch_bounds__(128, su::CTAS_PER_SM) k_c5_setup(DetectArgs a, const __grid_constant__ CUtensorMap hmap) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    unsigned char* g = smem_raw + (base - raw);
    uint64_t* bar_tma = reinterpret_cast<uint64_t*>(g + su::BAR);
    uint64_t* bar_mma = bar_tma + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g + su::TSLOT);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long n_batch = (a.n_units + su::UPB - 1) / su::UPB;

    pdl_launch_dependents();
    if (t == 0) {
        mbar_init(bar_tma, 1);
        mbar_init(bar_mma, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&hmap)) : "memory");
    }
    if (warp == 0) tc::alloc<128>(tslot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tslot;
    bool waited = false;  // PDL: the previous call may still read the workspace
    uint32_t it = 0;
    auto nv_of = [&](long long bt) { return (int)min((long long)su::UPB, a.n_units - bt * su::UPB); };
    if (t == 0 && blockIdx.x < n_batch)
        setup_issue_h(&hmap, base, bar_tma, nv_of(blockIdx.x), [&](int s) { return (long long)blockIdx.x * su::UPB + s; });
#pragma unroll 1
    for (long long bt = blockIdx.x; bt < n_batch; bt += gridDim.x, ++it) {
        const long long ub = bt * su::UPB, bn = bt + gridDim.x;
        setup_batch<QM, false, false, 0>(a, &hmap, g, base, bar_tma, bar_mma, tmem, it, nv_of(bt), t, warp, lane, waited,
                               [&](int s) { return ub + s; }, [] { __syncthreads(); },
                               [&] {
                                   if (bn < n_batch)
                                       setup_issue_h(&hmap, base, bar_tma, nv_of(bn), [&](int s) { return bn * su::UPB + s; });
                               },
                               [] {}, [&](int s) { return (long long)(ub + s); }, [] {});
    }
    if (!waited) pdl_wait();
    if (warp == 0) tc::dealloc<128>(tmem);
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
        cudaLaunchConfig_t cfg = {};
        const long long nb = (a.n_units + su::UPB - 1) / su::UPB;
        const long long cap = (long long)n_sm * su::CTAS_PER_SM;
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

template <int QM, int LT, int EW, int S, int NLO, int TA, int SETUP, bool BEPI, bool FUSED = false, int NACC = 2, int BI = 0>
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
    CUtensorMap hmap = ymap;  // FUSED: H as {32 floats (16 layers re/im), n_units * 64 rows}; box = one unit
    if constexpr (FUSED) {
        const cuuint64_t hdim[2] = {32, (cuuint64_t)a.n_units * 64};
        const cuuint64_t hstride[1] = {128};
        const cuuint32_t hbox[2] = {32, 64};
        if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(a.H), hdim, hstride, hbox, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    } else {
        cudaError_t e = launch_setup<QM, SETUP>(a, s);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.n_units < n_sm ? a.n_units : n_sm));
    cfg.blockDim = dim3(32 * (6 + EW) + (FUSED ? 128 : 0));
    cfg.dynamicSmemBytes = C5Smem<S, NLO, TA, FUSED, NACC, BI != 0>::total;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.overlap ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_c5_apply<QM, LT, EW, S, NLO, TA, BEPI, FUSED, NACC, BI>, a, ymap, hmap);
}

template <int QM, int LT, int EW, int S, int NLO, int TA, int SETUP, bool BEPI, bool FUSED = false, int NACC = 2, int BI = 0>
cudaError_t prepare_c5() {
    if constexpr (!FUSED) {
        cudaError_t e = prepare_setup<QM, SETUP>();
        if (e != cudaSuccess) return e;
    }
    return cudaFuncSetAttribute(k_c5_apply<QM, LT, EW, S, NLO, TA, BEPI, FUSED, NACC, BI>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C5Smem<S, NLO, TA, FUSED, NACC, BI != 0>::total);
}

size_t c5_workspace(const DetectArgs& a) { return (size_t)a.n_units * BigWs<64, 16>::stride * 4; }
// fused kernel: a ring of kC5Ring records per CTA
size_t c5f_workspace(const DetectArgs& a) {
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const long long ctas = a.n_units < n_sm ? a.n_units : n_sm;
    return (size_t)ctas * kC5Ring * BigWs<64, 16>::stride * 4;
}
// fused kernel with B-image records
size_t c5fb_workspace(const DetectArgs& a) {
    return c5f_workspace(a) / ((size_t)BigWs<64, 16>::stride * 4) * (size_t)kBiRec;
}

#define C5_ENTRY(NAME, QM, LT, S, NLO, TA, SETUP, BEPI)                                                   \
    KernelEntry {                                                                                          \
        NAME, 64, 16, QM, kSc, 14, LT, 32, 2, launch_c5<QM, LT, 6, S, NLO, TA, SETUP, BEPI>,               \
            prepare_c5<QM, LT, 6, S, NLO, TA, SETUP, BEPI>, c5_workspace                                   \
    }
// BI = 1: B-image records; 2: + the consumed records discarded from L2 (no dirty write-back) by the tile-1
// epilogue warp; 3: 2 + the setup group's image readout by whole warps (16x32bx2 TMEM loads); 4: 3 + y tiles and
// LLR stores with an L2 evict-first policy
#define C5FB_ENTRY(NAME, QM, LT, S, BI)                                                                     \
    KernelEntry {                                                                                          \
        NAME, 64, 16, QM, kSc, 14, LT, 32, 1, launch_c5<QM, LT, 6, S, 2, 4, 2, true, true, 2, BI>,         \
            prepare_c5<QM, LT, 6, S, 2, 4, 2, true, true, 2, BI>, c5fb_workspace                           \
    }
#define C5F_ENTRY(NAME, QM, LT, S, NACC)                                                                    \
    KernelEntry {                                                                                          \
        NAME, 64, 16, QM, kSc, 14, LT, 32, 1, launch_c5<QM, LT, 6, S, 2, 4, 2, true, true, NACC>,          \
            prepare_c5<QM, LT, 6, S, 2, 4, 2, true, true, NACC>, c5f_workspace                             \
    }

// First entry of a shape = its default (mimo_api.cu select_fast); the others are selectable by name.
// Name parts: fused = one kernel (setup warp group inside the apply); otherwise a setup kernel + the
// apply: operand split (bf16 / bf16kc = one accumulator per tile / tf32), setup (tcs = tensor-core
// contractions; gj = SIMT Gauss-Jordan; chol = SIMT Cholesky), be = the B sets built by the
// (under-loaded) epilogue warps instead of the converter warps, which set the pace of the pipeline.
const KernelEntry kEntries[] = {
    // C5 default: setup warp group inside the apply kernel, writing B-image records (read out of TMEM by whole
    // warps) that the apply copies straight into its B sets; consumed records discarded from L2; the streamed
    // y tiles and LLR stores marked L2 evict-first so that the records stay resident until they are copied
    C5FB_ENTRY("c5_fusedbie_64x16_q6_i8", 6, kLlrI8, 5, 4),
    C5FB_ENTRY("c5_fusedbiw_64x16_q6_i8", 6, kLlrI8, 5, 3),  // without the evict-first hints
    C5FB_ENTRY("c5_fusedbid_64x16_q6_i8", 6, kLlrI8, 5, 2),  // image readout by half warps (lanes 0-15)
    C5FB_ENTRY("c5_fusedbi_64x16_q6_i8", 6, kLlrI8, 5, 1),  // B-image records, no discards
    C5F_ENTRY("c5_fused_64x16_q6_i8", 6, kLlrI8, 5, 2),  // W~ records, B sets built by epilogue warps 4-7
    C5F_ENTRY("c5_fused3_64x16_q6_i8", 6, kLlrI8, 4, 3),  // 3 accumulators / B sets, 4 y stages, narrow setup
    C5_ENTRY("c5_bf16_tcs_be_64x16_q6_i8", 6, kLlrI8, 6, 4, 3, 2, true),  // two kernels: tensor-core setup + apply
    C5_ENTRY("c5_bf16kc_tcs_be_64x16_q6_i8", 6, kLlrI8, 6, 4, 4, 2, true),
    C5_ENTRY("c5_bf16_tcs_64x16_q6_i8", 6, kLlrI8, 6, 4, 3, 2, false),
    C5_ENTRY("c5_bf16_gj_64x16_q6_i8", 6, kLlrI8, 6, 4, 3, 1, false),
    C5_ENTRY("c5_bf16_chol_64x16_q6_i8", 6, kLlrI8, 6, 4, 3, 0, false),
    C5_ENTRY("c5_tf32_gj_64x16_q6_i8", 6, kLlrI8, 4, 2, 1, 1, false),  // round-1 big8e6 configuration
};

}  // namespace

const KernelEntry* c5_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
