// common.cuh -- device building blocks shared by the sm_100a detector kernels.
//
// Complex fp32/fp64 helpers, the exact per-axis max-log demapper (SURVEY.md
// §8(a) row a7), saturating quantisers (reading R10), wide vector stores and
// the mbarrier / cp.async.bulk wrappers used to stage y tiles in shared memory.
// Nothing here is shared with oracle/ (DESIGN.md §"Oracle").
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mimo {

constexpr int kLlrF32 = 0;
constexpr int kLlrF16 = 1;
constexpr int kLlrI8 = 2;

// Reading R17: Cholesky guard p_j > kPivotTau * max_i G_ii, kPivotTau = 16 * 2^-24.
constexpr double kPivotTau = 16.0 * 5.9604644775390625e-08;

// Arguments of one detect call (plain pointers; layouts in include/mimo.h).
struct DetectArgs {
    const float2* H;      // [n_slots][n_fb][nr][nl]
    const float2* y;      // [n_sym][n_sc][nr]
    void* llr;            // [n_sym][n_sc][nl][qm] of llr_type (may be null)
    float2* xhat;         // [n_sym][n_sc][nl] (may be null)
    float* sinr;          // [n_units][nl] (may be null)
    unsigned long long* fail_count;
    float sigma2;
    float llr_scale;
    int n_rx, n_layers, qm;
    int n_sc, n_sym;
    int sc_per_h, sym_per_h;
    int n_fb, n_slots;    // n_fb = n_sc / sc_per_h; n_slots = n_sym / sym_per_h
    long long n_units;
    int llr_type;
    int overlap;          // launch with programmatic dependent launch (MIMO_PLAN_OVERLAP_CALLS)
    void* ws;             // plan-owned workspace (kernel families that need one)
    const float* sigma2_v;  // mimo_detect_mmse_sv: one noise variance per H time block [n_slots] (else null)
};

// Noise variance of H time block `blk` (= slot for sym_per_h = 14): the scalar sigma2, or the
// per-block array entry, which must be finite and > 0 -- anything else becomes NaN so that the
// unit fails the pivot guard (R17) and is counted / zeroed like a non-PD unit.
__device__ __forceinline__ float block_sigma2(const DetectArgs& a, long long blk) {
    if (!a.sigma2_v) return a.sigma2;
    const float v = __ldg(a.sigma2_v + blk);
    return (v > 0.f && v <= 3.4e38f) ? v : __int_as_float(0x7fc00000);
}
__device__ __forceinline__ float unit_sigma2(const DetectArgs& a, long long u) { return block_sigma2(a, u / a.n_fb); }

// Per-axis PAM normalisation of the 38.211 constellations: a = 1/sqrt(norm).
__host__ __device__ constexpr int qam_norm(int qm) { return qm == 2 ? 2 : qm == 4 ? 10 : qm == 6 ? 42 : 170; }

// ------------------------------------------------------------ complex ----
__device__ __forceinline__ float2 cmac(float2 acc, float2 a, float2 b) {   // acc + a*b
    acc.x = fmaf(a.x, b.x, acc.x);
    acc.x = fmaf(-a.y, b.y, acc.x);
    acc.y = fmaf(a.x, b.y, acc.y);
    acc.y = fmaf(a.y, b.x, acc.y);
    return acc;
}
// ---- packed fp32x2 (FFMA2, sm_100): two fp32 FMAs per instruction. A plain 3-register
// FFMA issues at half the FMA pipe's rate on Blackwell, so complex MACs written as two
// FFMA2 (with broadcast / half-swapped operands, which the ISA encodes for free) halve
// the FMA-pipe instruction count of the SIMT GEMM-like loops.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {  // (a.x b.x + c.x, a.y b.y + c.y)
    unsigned long long ua, ub, uc, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(uc) : "f"(c.x), "f"(c.y));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ua), "l"(ub), "l"(uc));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
    return r;
}
// A complex coefficient w pre-packed for acc += w * y:  (w.x, w.x) * y + (-w.y, w.y) * swap(y)
struct CPack {
    float2 xx, ny;
};
__device__ __forceinline__ CPack cpack(float2 w) { return CPack{make_float2(w.x, w.x), make_float2(-w.y, w.y)}; }
// ... and for acc += conj(w) * y:  (w.x, w.x) * y + (w.y, -w.y) * swap(y)
__device__ __forceinline__ CPack cpack_conj(float2 w) { return CPack{make_float2(w.x, w.x), make_float2(w.y, -w.y)}; }
__device__ __forceinline__ float2 cmac_p(float2 acc, const CPack& w, float2 y) {
    acc = ffma2(w.xx, y, acc);
    return ffma2(w.ny, make_float2(y.y, y.x), acc);
}
// acc + w * conj(y):  (w.x, w.y) * y.x + (w.y, -w.x) * y.y  ==  (w.x, w.x)... written for a fixed w:
// acc.x += w.x y.x + w.y y.y ; acc.y += w.y y.x - w.x y.y
struct CPackC {
    float2 a, b;  // a = (w.x, w.y) * y.x ; b = (w.y, -w.x) * y.y
};
__device__ __forceinline__ CPackC cpackc(float2 w) { return CPackC{w, make_float2(w.y, -w.x)}; }
__device__ __forceinline__ float2 cmacc_p(float2 acc, const CPackC& w, float2 y) {  // acc + w * conj(y)
    acc = ffma2(w.a, make_float2(y.x, y.x), acc);
    return ffma2(w.b, make_float2(y.y, y.y), acc);
}

// acc + w * y with y shared by several w: ny = (-y.y, y.x) computed once per y,
// w's halves used as broadcast scalars (free operand forms of FFMA2).
__device__ __forceinline__ float2 cmac_y(float2 acc, float2 w, float2 y, float2 ny) {
    acc = ffma2(make_float2(w.x, w.x), y, acc);
    return ffma2(make_float2(w.y, w.y), ny, acc);
}

__device__ __forceinline__ double2 dmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 dmac(double2 acc, double2 a, double2 b) {      // acc + a*b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ double2 dmacc(double2 acc, double2 a, double2 b) {     // acc + conj(a)*b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ double2 dsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 dscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double dnorm2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// ------------------------------------------------------------ demapper ----
// Output-type magnitude clamp folded into the demapper (reading R10): int8
// saturates at 127; fp16 saturates in the packing conversion (satfinite);
// fp32 needs no clamp unless slopes are infinite (sigma2 = 0).
template <int LT>
__device__ __forceinline__ float clamp_mag(float v) {  // v >= 0
    if constexpr (LT == kLlrI8) return fminf(v, 127.f);
    else return v;
}
template <int LT>
__device__ __forceinline__ float clamp_signed(float v) {
    if constexpr (LT == kLlrI8) return fminf(fmaxf(v, -127.f), 127.f);
    else return v;
}

// Exact max-log per axis (equals brute force, pins P10).
// u: equalised coordinate in PAM level units (levels at odd integers, i.e.
// Re/Im(x~) * sqrt(norm)); slope = SINR * a^2 * llr_scale. Writes the LLRs of
// the M bits on this axis (axis bit i is symbol bit 2i on I, 2i+1 on Q):
//   t_0 = u, t_i = 2^(M-i) - |t_{i-1}|   (Gray folding)
//   D = (|t_{M-1}| - 1)^2                 (squared distance to the nearest level,
//                                          = (u - clamp(2 floor(u/2)+1))^2)
//   LLR_i = sgn(t_i) * slope * ((|t_i| + 1)^2 - D)
// (|t|+1)^2 - D is one FMA. QPSK / 16-QAM use the equal linear-region forms
// (D_1 - D_0 = (b - a)(2u - a - b) between fixed nearest points a, b):
//   QPSK bit 0: 4u;  16-QAM bit 0: 4(u + sgn(u) max(|u| - 2, 0)), bit 1: 4(2 - |u|).
// ZF = true is the sigma2 = 0 variant (reading R11): slope = +inf, a zero
// distance gap gives 0 instead of NaN, and packing saturates.
template <int M, bool ZF, int LT>
__device__ __forceinline__ void demap_axis(float u, float slope, float* out, int stride) {
    if constexpr (!ZF && M <= 2) {
        const float s4 = 4.f * slope;
        if constexpr (M == 1) {
            out[0] = clamp_signed<LT>(s4 * u);
        } else {
            out[0] = clamp_signed<LT>(s4 * (u + copysignf(fmaxf(fabsf(u) - 2.f, 0.f), u)));
            out[stride] = clamp_signed<LT>(s4 * (2.f - fabsf(u)));
        }
        return;
    }
    float t[M];
    t[0] = u;
#pragma unroll
    for (int i = 1; i < M; ++i) t[i] = float(1 << (M - i)) - fabsf(t[i - 1]);
    const float e = fabsf(t[M - 1]) - 1.f;
    const float D = e * e;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const float at = fabsf(t[i]) + 1.f;
        const float mag = fmaf(at, at, -D);
        float v;
        if constexpr (ZF) v = mag > 0.f ? slope * mag : 0.f;
        else v = clamp_mag<LT>(slope * mag);
        out[i * stride] = copysignf(v, t[i]);
    }
}

// Demap one layer: x = x~ / a (level units), qm bits into out[0..QM).
template <int QM, bool ZF = false, int LT = kLlrF32>
__device__ __forceinline__ void demap_layer(float2 x, float slope, float* out) {
    demap_axis<QM / 2, ZF, LT>(x.x, slope, out, 2);
    demap_axis<QM / 2, ZF, LT>(x.y, slope, out + 1, 2);
}

// ---------------------------------------------------------- quantisers ----
// Reading R10: fp32 saturating at +-FLT_MAX; fp16 RNE saturating at +-65504;
// int8 rint (half-even) saturating at +-127.
__device__ __forceinline__ float sat_f32(float v) { return fminf(fmaxf(v, -3.402823466e38f), 3.402823466e38f); }
__device__ __forceinline__ __half q_f16(float v) { return __float2half_rn(fminf(fmaxf(v, -65504.f), 65504.f)); }
__device__ __forceinline__ int8_t q_i8(float v) { return (int8_t)__float2int_rn(fminf(fmaxf(v, -127.f), 127.f)); }

// two floats -> binary16 x2 (RNE, saturating at +-65504: F2FP.SATFINITE)
__device__ __forceinline__ uint32_t pack_f16x2_sat(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// v in [-127, 127] -> float whose low byte is rint(v) as int8 (1.5 * 2^23 magic)
__device__ __forceinline__ uint32_t i8_magic(float v) { return __float_as_uint(v + 12582912.f); }

// demap_layer for sigma2 > 0 with the I and Q axes as one packed pair (FADD2 / FFMA2 / FMUL2, the |.|
// and immediate operand forms are free): the same per-axis arithmetic as demap_axis for M >= 3, in the
// same order, two axes per instruction. Writes the QM LLRs as QM / 2 (I, Q) pairs: f16 -> one binary16x2
// word per pair, f32 -> two words.
__device__ __forceinline__ float2 fadd2_(float2 a, float2 b) {
    unsigned long long ua, ub, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(ua), "l"(ub));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
    return r;
}
__device__ __forceinline__ float2 fmul2_(float2 a, float2 b) {
    unsigned long long ua, ub, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ua) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ub) : "f"(b.x), "f"(b.y));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(ua), "l"(ub));
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
    return r;
}
template <int QM, int LT>
__device__ __forceinline__ void demap_layer_x2(float2 x, float slope, uint32_t* w) {
    constexpr int M = QM / 2;
    static_assert(M >= 3 && (LT == kLlrF16 || LT == kLlrF32), "packed demap: 64/256-QAM, float LLRs");
    float2 t[M];
    t[0] = x;
#pragma unroll
    for (int i = 1; i < M; ++i)
        t[i] = fadd2_(make_float2(float(1 << (M - i)), float(1 << (M - i))),
                      make_float2(-fabsf(t[i - 1].x), -fabsf(t[i - 1].y)));
    const float2 e = fadd2_(make_float2(fabsf(t[M - 1].x), fabsf(t[M - 1].y)), make_float2(-1.f, -1.f));
    const float2 D = fmul2_(e, e);
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const float2 at = fadd2_(make_float2(fabsf(t[i].x), fabsf(t[i].y)), make_float2(1.f, 1.f));
        const float2 mag = ffma2(at, at, make_float2(-D.x, -D.y));
        const float2 v = fmul2_(make_float2(slope, slope), mag);
        const float vi = copysignf(v.x, t[i].x), vq = copysignf(v.y, t[i].y);
        if constexpr (LT == kLlrF16) {
            w[i] = pack_f16x2_sat(vi, vq);
        } else {
            w[2 * i] = __float_as_uint(vi);
            w[2 * i + 1] = __float_as_uint(vq);
        }
    }
}

template <int LT> struct LlrTraits;
template <> struct LlrTraits<kLlrF32> { static constexpr int bytes = 4; };
template <> struct LlrTraits<kLlrF16> { static constexpr int bytes = 2; };
template <> struct LlrTraits<kLlrI8> { static constexpr int bytes = 1; };

// Pack N float LLRs into little-endian 32-bit words of the output type.
// SAT = true: values may be out of range / infinite (sigma2 = 0 path) and are
// saturated here; SAT = false: the demapper already clamped them.
template <int LT, int N, bool SAT = true>
__device__ __forceinline__ void pack_llr(const float* v, uint32_t* w) {
    if constexpr (LT == kLlrF32) {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = __float_as_uint(SAT ? sat_f32(v[i]) : v[i]);
    } else if constexpr (LT == kLlrF16) {
#pragma unroll
        for (int i = 0; i < (N + 1) / 2; ++i) w[i] = pack_f16x2_sat(v[2 * i], (2 * i + 1 < N) ? v[2 * i + 1] : 0.f);
    } else {
#pragma unroll
        for (int i = 0; i < (N + 3) / 4; ++i) {
            uint32_t q[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const float x = (4 * i + b < N) ? v[4 * i + b] : 0.f;
                q[b] = i8_magic(SAT ? fminf(fmaxf(x, -127.f), 127.f) : x);
            }
            w[i] = __byte_perm(__byte_perm(q[0], q[1], 0x0040), __byte_perm(q[2], q[3], 0x0040), 0x5410);
        }
    }
}

// ------------------------------------------------------- vector stores ----
__device__ __forceinline__ void st_v8(void* p, const uint32_t* w) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
}
__device__ __forceinline__ void st_v4(void* p, const uint32_t* w) {
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
}
__device__ __forceinline__ void st_v2(void* p, const uint32_t* w) {
    asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(w[0]), "r"(w[1]) : "memory");
}
__device__ __forceinline__ void st_v1(void* p, uint32_t w) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(w) : "memory");
}

// Store NB bytes held in words w to p, with the widest vectors the byte count
// and the (RE-stride-implied) alignment allow. p must be aligned to
// min(32, largest power of two dividing NB).
template <int NB>
__device__ __forceinline__ void store_bytes(void* p, const uint32_t* w) {
    if constexpr (NB % 32 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 32; ++i) st_v8((char*)p + 32 * i, w + 8 * i);
    } else if constexpr (NB % 16 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 16; ++i) st_v4((char*)p + 16 * i, w + 4 * i);
    } else if constexpr (NB % 8 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 8; ++i) st_v2((char*)p + 8 * i, w + 2 * i);
    } else if constexpr (NB % 4 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 4; ++i) st_v1((char*)p + 4 * i, w[i]);
    } else if constexpr (NB % 2 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 2; ++i)
            *(uint16_t*)((char*)p + 2 * i) = (uint16_t)(w[i / 2] >> (16 * (i & 1)));
    } else {
#pragma unroll
        for (int i = 0; i < NB; ++i) *((uint8_t*)p + i) = (uint8_t)(w[i / 4] >> (8 * (i & 3)));
    }
}

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256).
__device__ __forceinline__ void ld_v8(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld_v4(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p));
}

// Coherent (non-.nc) 256-bit load, for data written by an earlier kernel of the same call.
__device__ __forceinline__ void ld_v8_coherent(const void* p, uint32_t* w) {
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p)
                 : "memory");
}

// Load NB bytes (NB % 16 == 0, p 16- or 32-aligned accordingly) into words.
template <int NB>
__device__ __forceinline__ void load_bytes(const void* p, uint32_t* w) {
    static_assert(NB % 8 == 0, "load_bytes needs 8-byte multiples");
    if constexpr (NB % 32 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 32; ++i) ld_v8((const char*)p + 32 * i, w + 8 * i);
    } else if constexpr (NB % 16 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 16; ++i) ld_v4((const char*)p + 16 * i, w + 4 * i);
    } else {
#pragma unroll
        for (int i = 0; i < NB / 8; ++i) {
            uint2 v = __ldg((const uint2*)((const char*)p + 8 * i));
            w[2 * i] = v.x;
            w[2 * i + 1] = v.y;
        }
    }
}

// ------------------------------------------ programmatic dependent launch ----
// Kernels call pdl_launch_dependents() first (the next detect call on the
// stream may start its read-only prologue) and pdl_wait() before their first
// global write (the previous grid has completed and its writes are visible).
// Both are no-ops unless the launch carried the programmatic-serialization
// attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------- mbarrier + bulk async copy ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Global -> shared bulk copy (TMA unit, non-tensor): bytes % 16 == 0, both
// addresses 16-byte aligned; completes `bytes` tx on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------ TMA tensor copies ----
// 3-D tensor-map tile load global -> shared (completes the box's bytes as tx on bar).
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

}  // namespace mimo
