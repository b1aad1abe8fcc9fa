// k_lu.cu -- the paper-literal LMMSE pipeline as five unfused stage kernels
// (SURVEY.md §8(f) NEXT-1): the route the paper describes and times,
//   "LU decomposition, forward/backward substitution, and matrix inversion"
//   (Fig. 4 caption; §IV) of "the received signal
//   covariance matrix R",
// kept stage-separated on purpose so that the per-stage device time can be
// measured -- the B200 analogue of Fig. 5b's breakdown (PAPER.md:108-109,
// :119 "matrix inversion ... dominates"). The fused Gram/Cholesky kernels
// (k_tpu / k_lg / k_big ...) are the production path; this route exists to
// reproduce the paper's structure, in "PS" (fp32) or "PD" (fp64) arithmetic
// (PAPER.md:117, :119).
//
// Stages (each its own kernel; intermediate results go through the plan's
// workspace in HBM, one record per H-unit):
//   S0 cov      R = H H^H + s2 I  (nr x nr)               thread per (unit, row i)
//   S1 lu       P R = L U, partial pivoting                NR lanes per unit, lane i owns row i
//               (largest |a_ik|, lowest index on ties; guard |u_kk| > 16 u max|a_ij|)
//   S2 inv      R^-1 e_c by forward (L z = P e_c) and backward (U x = z)
//               substitution                                thread per (unit, column c)
//   S3 weights  W = H^H R^-1, mu_k = [W H]_kk (pin P7), SINR_k = mu_k / (1 - mu_k),
//               W~ = W sqrt(norm) / mu_k (rounded once to fp32), slope = SINR / norm * llr_scale
//                                                           thread per (unit, layer k)
//   S4 apply    x~ = W~ y, exact max-log demap, quantise     thread per RE
// Failure (singular R, e.g. sigma2 = 0 with n_rx > n_layers, or NaN): the unit
// is counted in the plan's failure counter and its outputs are erasures.
#include <float.h>

#include "kernels.h"

namespace mimo {
namespace {

template <typename T> struct Cx { T x, y; };
template <typename T> __device__ __forceinline__ Cx<T> cx(T x, T y) { return Cx<T>{x, y}; }
template <typename T> __device__ __forceinline__ Cx<T> cmul(Cx<T> a, Cx<T> b) {
    return cx<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename T> __device__ __forceinline__ Cx<T> cmacT(Cx<T> acc, Cx<T> a, Cx<T> b) {  // acc + a b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
    return acc;
}
template <typename T> __device__ __forceinline__ Cx<T> cmscT(Cx<T> acc, Cx<T> a, Cx<T> b) {  // acc - a b
    acc.x = fma(-a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(-a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
    return acc;
}
template <typename T> __device__ __forceinline__ Cx<T> cmaccT(Cx<T> acc, Cx<T> a, Cx<T> b) {  // acc + conj(a) b
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
    return acc;
}
template <typename T> __device__ __forceinline__ Cx<T> cdiv(Cx<T> a, Cx<T> b) {  // a / b
    const T inv = T(1) / fma(b.x, b.x, b.y * b.y);
    return cx<T>((a.x * b.x + a.y * b.y) * inv, (a.y * b.x - a.x * b.y) * inv);
}
template <typename T> __device__ __forceinline__ T cabsT(Cx<T> a) { return hypot(a.x, a.y); }
__device__ __forceinline__ float cabsT(Cx<float> a) { return hypotf(a.x, a.y); }

// LU pivot guard: 16 unit roundoffs of the stage's working precision (the
// scale-invariant guard of SPEC.md:266, reading R17 applied to LU).
template <typename T> struct Prec;
template <> struct Prec<float> { static constexpr double tau = 16.0 * 5.9604644775390625e-08; };
template <> struct Prec<double> { static constexpr double tau = 16.0 * 1.1102230246251565e-16; };

// Workspace records (per unit u), laid out as separate arrays:
//   LU   Cx<T> [n_units][NR][NR]   (R after S0, L\U after S1)
//   Ri   Cx<T> [n_units][NR][NR]   (R^-1, row-major)
//   perm int   [n_units][NR]       (row i of P R = row perm[i] of R)
//   ok   int   [n_units]           (1 = factorised)
//   Wt   float2[n_units][NR][NR]   (W~ rows k < n_layers, level units)
//   slope float[n_units][NR]
template <int NR, typename T>
struct LuWs {
    static constexpr size_t align(size_t b) { return (b + 255) & ~(size_t)255; }
    static size_t lu_bytes(long long n) { return align((size_t)n * NR * NR * sizeof(Cx<T>)); }
    static size_t perm_bytes(long long n) { return align((size_t)n * NR * sizeof(int)); }
    static size_t ok_bytes(long long n) { return align((size_t)n * sizeof(int)); }
    static size_t w_bytes(long long n) { return align((size_t)n * NR * NR * sizeof(float2)); }
    static size_t s_bytes(long long n) { return align((size_t)n * NR * sizeof(float)); }
    static size_t total(long long n) {
        return 2 * lu_bytes(n) + perm_bytes(n) + ok_bytes(n) + w_bytes(n) + s_bytes(n);
    }
    static Cx<T>* LU(void* ws, long long) { return (Cx<T>*)ws; }
    static Cx<T>* Ri(void* ws, long long n) { return (Cx<T>*)((char*)ws + lu_bytes(n)); }
    static int* perm(void* ws, long long n) { return (int*)((char*)ws + 2 * lu_bytes(n)); }
    static int* ok(void* ws, long long n) { return (int*)((char*)ws + 2 * lu_bytes(n) + perm_bytes(n)); }
    static float2* Wt(void* ws, long long n) {
        return (float2*)((char*)ws + 2 * lu_bytes(n) + perm_bytes(n) + ok_bytes(n));
    }
    static float* slope(void* ws, long long n) {
        return (float*)((char*)ws + 2 * lu_bytes(n) + perm_bytes(n) + ok_bytes(n) + w_bytes(n));
    }
};

struct LuPtrs {
    void* LU;
    void* Ri;
    int* perm;
    int* ok;
    float2* Wt;
    float* slope;
};

// ---------------------------------------------------------------- S0 ----
// R_ij = sum_l H_il conj(H_jl) + s2 delta_ij (Fig. 3b's FMA
// covariance accumulation).
template <int NR, typename T>
__global__ void __launch_bounds__(128) k_lu_cov(DetectArgs a, LuPtrs w) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.n_units * NR) return;
    const long long u = g / NR;
    const int i = (int)(g % NR);
    const int nl = a.n_layers;
    const float2* Hu = a.H + u * NR * nl;
    Cx<T> row[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) row[j] = cx<T>(0, 0);
    for (int l = 0; l < nl; ++l) {
        const float2 hi = __ldg(Hu + i * nl + l);
        const Cx<T> hiT = cx<T>((T)hi.x, (T)hi.y);
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const float2 hj = __ldg(Hu + j * nl + l);
            row[j] = cmaccT(row[j], cx<T>((T)hj.x, (T)hj.y), hiT);  // H_il conj(H_jl)
        }
    }
    row[i].x += (T)a.sigma2;
    Cx<T>* dst = (Cx<T>*)w.LU + (u * NR + i) * NR;
#pragma unroll
    for (int j = 0; j < NR; ++j) dst[j] = row[j];
}

// ---------------------------------------------------------------- S1 ----
// Doolittle LU with partial pivoting, NR
// lanes per unit: lane i owns row i; the pivot search is an arg-max over the
// lanes, the row exchange and the pivot row broadcast are shuffles.
template <int NR, typename T>
__global__ void __launch_bounds__(128) k_lu_factor(DetectArgs a, LuPtrs w) {
    static_assert(32 % NR == 0, "NR must divide 32");
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long u_raw = g / NR;
    const bool valid = u_raw < a.n_units;
    const long long u = valid ? u_raw : a.n_units - 1;  // whole warps stay converged
    const int i = (int)(g % NR);
    Cx<T>* src = (Cx<T>*)w.LU + (u * NR + i) * NR;
    Cx<T> r[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) r[j] = src[j];
    int pi = i;  // original row index held by this lane
    T amax = 0;
#pragma unroll
    for (int j = 0; j < NR; ++j) amax = fmax(amax, cabsT(r[j]));
#pragma unroll
    for (int off = 1; off < NR; off <<= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off, NR));
    bool ok = (amax == amax);
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        // pivot: largest |a_ik| over i >= k, lowest i on ties
        T best = (i >= k) ? cabsT(r[k]) : T(-1);
        int bi = i;
#pragma unroll
        for (int off = 1; off < NR; off <<= 1) {
            const T ob = __shfl_xor_sync(0xffffffffu, best, off, NR);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off, NR);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if (!(best > (T)Prec<T>::tau * amax)) ok = false;
        // exchange rows k and bi
        const int srcl = (i == k) ? bi : (i == bi ? k : i);
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            r[j].x = __shfl_sync(0xffffffffu, r[j].x, srcl, NR);
            r[j].y = __shfl_sync(0xffffffffu, r[j].y, srcl, NR);
        }
        pi = __shfl_sync(0xffffffffu, pi, srcl, NR);
        // eliminate below the pivot
        const Cx<T> piv = cx<T>(__shfl_sync(0xffffffffu, r[k].x, k, NR), __shfl_sync(0xffffffffu, r[k].y, k, NR));
        Cx<T> l = cx<T>(0, 0);
        if (i > k && ok) {
            l = cdiv(r[k], piv);
            r[k] = l;
        }
#pragma unroll
        for (int j = k + 1; j < NR; ++j) {
            const Cx<T> ukj = cx<T>(__shfl_sync(0xffffffffu, r[j].x, k, NR), __shfl_sync(0xffffffffu, r[j].y, k, NR));
            if (i > k) r[j] = cmscT(r[j], l, ukj);
        }
    }
    if (!valid) return;
#pragma unroll
    for (int j = 0; j < NR; ++j) src[j] = r[j];
    w.perm[u * NR + i] = pi;
    if (i == 0) {
        w.ok[u] = ok ? 1 : 0;
        if (!ok) atomicAdd(a.fail_count, 1ull);
    }
}

// ---------------------------------------------------------------- S2 ----
// Column c of R^-1: L z = P e_c (forward), U x = z (backward) -- PAPER.md:115
// "forward substitution and backward substitution", :93 "matrix inversion".
template <int NR, typename T>
__global__ void __launch_bounds__(128) k_lu_invert(DetectArgs a, LuPtrs w) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.n_units * NR) return;
    const long long u = g / NR;
    const int c = (int)(g % NR);
    if (!w.ok[u]) return;
    const Cx<T>* A = (const Cx<T>*)w.LU + u * NR * NR;
    const int* perm = w.perm + u * NR;
    Cx<T> z[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        Cx<T> s = cx<T>(perm[i] == c ? T(1) : T(0), 0);
#pragma unroll
        for (int k = 0; k < i; ++k) s = cmscT(s, A[i * NR + k], z[k]);
        z[i] = s;
    }
    Cx<T> x[NR];
#pragma unroll
    for (int i = NR - 1; i >= 0; --i) {
        Cx<T> s = z[i];
#pragma unroll
        for (int k = i + 1; k < NR; ++k) s = cmscT(s, A[i * NR + k], x[k]);
        x[i] = cdiv(s, A[i * NR + i]);
    }
    Cx<T>* Ri = (Cx<T>*)w.Ri + u * NR * NR;
#pragma unroll
    for (int i = 0; i < NR; ++i) Ri[i * NR + c] = x[i];
}

// ---------------------------------------------------------------- S3 ----
// W = H^H R^-1 (the paper-literal covariance form), unbiasing and SINR
// (readings R3, R4; mu_k = [W H]_kk is pin P7's identity).
template <int NR, int QM, typename T>
__global__ void __launch_bounds__(128) k_lu_weights(DetectArgs a, LuPtrs w) {
    const int nl = a.n_layers;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.n_units * nl) return;
    const long long u = g / nl;
    const int k = (int)(g % nl);
    const float2* Hu = a.H + u * NR * nl;
    float2* Wt = w.Wt + (u * NR + k) * NR;
    const T norm = (T)qam_norm(QM);
    if (!w.ok[u]) {
#pragma unroll
        for (int c = 0; c < NR; ++c) Wt[c] = make_float2(0.f, 0.f);
        w.slope[u * NR + k] = 0.f;
        if (a.sinr) a.sinr[u * nl + k] = 0.f;
        return;
    }
    const Cx<T>* Ri = (const Cx<T>*)w.Ri + u * NR * NR;
    Cx<T> Wk[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) Wk[c] = cx<T>(0, 0);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const float2 h = __ldg(Hu + r * nl + k);
        const Cx<T> hT = cx<T>((T)h.x, (T)h.y);
#pragma unroll
        for (int c = 0; c < NR; ++c) Wk[c] = cmaccT(Wk[c], hT, Ri[r * NR + c]);  // conj(H_rk) Ri_rc
    }
    T mu = 0;
#pragma unroll
    for (int c = 0; c < NR; ++c) {
        const float2 h = __ldg(Hu + c * nl + k);
        mu = fma(Wk[c].x, (T)h.x, fma(-Wk[c].y, (T)h.y, mu));  // Re(W_kc H_ck)
    }
    T sinr;
    if (a.sigma2 == 0.f) {
        mu = 1;
        sinr = (T)INFINITY;
    } else {
        sinr = mu / (T(1) - mu);
    }
    T f = 0;
    if (!(mu > 0)) sinr = 0;
    else f = sqrt(norm) / mu;
#pragma unroll
    for (int c = 0; c < NR; ++c) Wt[c] = make_float2((float)(Wk[c].x * f), (float)(Wk[c].y * f));
    w.slope[u * NR + k] = (float)(sinr / norm) * a.llr_scale;
    if (a.sinr) a.sinr[u * nl + k] = (float)sinr;
}

// ---------------------------------------------------------------- S4 ----
template <int QM, int LT>
__device__ __forceinline__ void store_llr_layer(void* llr, size_t idx, const float* v) {
    uint32_t wd[(QM * LlrTraits<LT>::bytes + 3) / 4];
    pack_llr<LT, QM, true>(v, wd);
    constexpr int NB = QM * LlrTraits<LT>::bytes;
    char* p = (char*)llr + idx * LlrTraits<LT>::bytes;
    if constexpr (NB % 4 == 0) {
#pragma unroll
        for (int i = 0; i < NB / 4; ++i) *(uint32_t*)(p + 4 * i) = wd[i];
    } else {
#pragma unroll
        for (int i = 0; i < NB / 2; ++i) *(uint16_t*)(p + 2 * i) = (uint16_t)(wd[i / 2] >> (16 * (i & 1)));
    }
}

template <int NR, int QM, int LT, bool ZF>
__global__ void __launch_bounds__(128) k_lu_apply(DetectArgs a, LuPtrs w) {
    const long long re = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n_re = (long long)a.n_sym * a.n_sc;
    if (re >= n_re) return;
    const int sym = (int)(re / a.n_sc), sc = (int)(re % a.n_sc);
    const long long u = (long long)(sym / a.sym_per_h) * a.n_fb + sc / a.sc_per_h;
    const int nl = a.n_layers;
    float2 yv[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) yv[r] = __ldg(a.y + re * NR + r);
    const float ia = rsqrtf((float)qam_norm(QM));
    for (int k = 0; k < nl; ++k) {
        const float2* Wk = w.Wt + (u * NR + k) * NR;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < NR; ++r) acc = cmac(acc, Wk[r], yv[r]);
        if (a.llr) {
            float v[QM];
            demap_layer<QM, ZF>(acc, w.slope[u * NR + k], v);
            store_llr_layer<QM, LT>(a.llr, (size_t)(re * nl + k) * QM, v);
        }
        if (a.xhat) a.xhat[re * nl + k] = make_float2(acc.x * ia, acc.y * ia);
    }
}

inline unsigned blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

template <int NR, int QM, int LT, typename T>
cudaError_t run_stages(const DetectArgs& a, cudaStream_t s, cudaEvent_t* ev) {
    using WS = LuWs<NR, T>;
    LuPtrs w{WS::LU(a.ws, a.n_units), WS::Ri(a.ws, a.n_units), WS::perm(a.ws, a.n_units),
             WS::ok(a.ws, a.n_units), WS::Wt(a.ws, a.n_units), WS::slope(a.ws, a.n_units)};
    constexpr int TB = 128;
    auto rec = [&](int i) { return ev ? cudaEventRecord(ev[i], s) : cudaSuccess; };
    cudaError_t e = rec(0);
    if (e == cudaSuccess) k_lu_cov<NR, T><<<blocks(a.n_units * NR, TB), TB, 0, s>>>(a, w), e = cudaGetLastError();
    if (e == cudaSuccess) e = rec(1);
    if (e == cudaSuccess) k_lu_factor<NR, T><<<blocks(a.n_units * NR, TB), TB, 0, s>>>(a, w), e = cudaGetLastError();
    if (e == cudaSuccess) e = rec(2);
    if (e == cudaSuccess) k_lu_invert<NR, T><<<blocks(a.n_units * NR, TB), TB, 0, s>>>(a, w), e = cudaGetLastError();
    if (e == cudaSuccess) e = rec(3);
    if (e == cudaSuccess)
        k_lu_weights<NR, QM, T><<<blocks(a.n_units * a.n_layers, TB), TB, 0, s>>>(a, w), e = cudaGetLastError();
    if (e == cudaSuccess) e = rec(4);
    if (e == cudaSuccess) {
        const long long n_re = (long long)a.n_sym * a.n_sc;
        if (a.sigma2 > 0.f) k_lu_apply<NR, QM, LT, false><<<blocks(n_re, TB), TB, 0, s>>>(a, w);
        else k_lu_apply<NR, QM, LT, true><<<blocks(n_re, TB), TB, 0, s>>>(a, w);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = rec(5);
    return e;
}

template <int NR, int QM, typename T>
cudaError_t by_llr(const DetectArgs& a, cudaStream_t s, cudaEvent_t* ev) {
    switch (a.llr_type) {
    case kLlrF32: return run_stages<NR, QM, kLlrF32, T>(a, s, ev);
    case kLlrF16: return run_stages<NR, QM, kLlrF16, T>(a, s, ev);
    default: return run_stages<NR, QM, kLlrI8, T>(a, s, ev);
    }
}

template <int NR, typename T>
cudaError_t by_qm(const DetectArgs& a, cudaStream_t s, cudaEvent_t* ev) {
    switch (a.qm) {
    case 2: return by_llr<NR, 2, T>(a, s, ev);
    case 4: return by_llr<NR, 4, T>(a, s, ev);
    case 6: return by_llr<NR, 6, T>(a, s, ev);
    default: return by_llr<NR, 8, T>(a, s, ev);
    }
}

template <typename T>
cudaError_t by_nr(const DetectArgs& a, cudaStream_t s, cudaEvent_t* ev) {
    switch (a.n_rx) {
    case 1: return by_qm<1, T>(a, s, ev);
    case 2: return by_qm<2, T>(a, s, ev);
    case 4: return by_qm<4, T>(a, s, ev);
    case 8: return by_qm<8, T>(a, s, ev);
    default: return by_qm<16, T>(a, s, ev);
    }
}

template <typename T>
size_t ws_t(int nr, long long n) {
    switch (nr) {
    case 1: return LuWs<1, T>::total(n);
    case 2: return LuWs<2, T>::total(n);
    case 4: return LuWs<4, T>::total(n);
    case 8: return LuWs<8, T>::total(n);
    default: return LuWs<16, T>::total(n);
    }
}

}  // namespace

bool lu_route_supported(int n_rx) { return n_rx == 1 || n_rx == 2 || n_rx == 4 || n_rx == 8 || n_rx == 16; }

size_t lu_route_workspace(int n_rx, long long n_units, int precision_bits) {
    return precision_bits == 64 ? ws_t<double>(n_rx, n_units) : ws_t<float>(n_rx, n_units);
}

cudaError_t launch_lu_route(const DetectArgs& a, int precision_bits, cudaStream_t s, cudaEvent_t* ev) {
    if (a.n_units <= 0) return cudaSuccess;
    return precision_bits == 64 ? by_nr<double>(a, s, ev) : by_nr<float>(a, s, ev);
}

}  // namespace mimo
