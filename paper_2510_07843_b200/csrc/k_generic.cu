// k_generic.cu -- the shape-generic detector kernel (any n_rx <= 64,
// n_layers <= 16, qm in {2,4,6,8}, any sc_per_h / sym_per_h, any LLR type).
//
// One CTA per H-unit (grid-stride). The per-unit setup (SURVEY.md §8(a) rows
// a2-a5) runs cooperatively in shared memory in fp64:
//   G = H^H H + s2 I           (threads over lower-triangle entries)
//   G = L L^H                  (right-looking Cholesky, one column per step)
//   X = L^-1                   (forward substitution, one column per thread)
//   G^-1 = X^H X,  A_kk = [G^-1]_kk
//   W = G^-1 H^H,  W~ = W * sqrt(norm) / mu  (rounded once to fp32)
// then rows a6-a7 run with one thread per RE: x~ = W~ y (fp32, W~ broadcast
// from shared memory), exact max-log demap, quantise, store.
//
// This is the correctness path for shapes without a specialised kernel; the
// BASELINE configs use the specialised kernels (k_tpu.cu, k_prb.cu, k_lg.cu).
#include <float.h>

#include "kernels.h"

namespace mimo {
namespace {

constexpr int kThreads = 128;
constexpr int MR = kGenericMaxRx;
constexpr int ML = kGenericMaxLayers;

template <int QM, int LT>
__device__ __forceinline__ void store_layer_llr(void* llr, size_t idx, const float* v) {
    // idx = element index of the layer's first LLR
    if constexpr (LT == kLlrF32) {
        float* p = (float*)llr + idx;
#pragma unroll
        for (int j = 0; j < QM; ++j) p[j] = sat_f32(v[j]);
    } else if constexpr (LT == kLlrF16) {
        __half* p = (__half*)llr + idx;
#pragma unroll
        for (int j = 0; j < QM; ++j) p[j] = q_f16(v[j]);
    } else {
        int8_t* p = (int8_t*)llr + idx;
#pragma unroll
        for (int j = 0; j < QM; ++j) p[j] = q_i8(v[j]);
    }
}

template <int QM, int LT, bool ZF>
__device__ void apply_unit(const DetectArgs& a, const float2* __restrict__ sW, const float* __restrict__ sSlope,
                           int slot, int fb, bool failed) {
    const int nr = a.n_rx, nl = a.n_layers;
    const int n_re = a.sc_per_h * a.sym_per_h;
    for (int e = threadIdx.x; e < n_re; e += blockDim.x) {
        const int sym = slot * a.sym_per_h + e / a.sc_per_h;
        const int sc = fb * a.sc_per_h + e % a.sc_per_h;
        const size_t re = (size_t)sym * a.n_sc + sc;
        float2 acc[ML];
#pragma unroll
        for (int k = 0; k < ML; ++k) acc[k] = make_float2(0.f, 0.f);
        if (!failed) {
            const float2* yp = a.y + re * nr;
            for (int r = 0; r < nr; ++r) {
                const float2 yr = __ldg(yp + r);
#pragma unroll
                for (int k = 0; k < ML; ++k)
                    if (k < nl) acc[k] = cmac(acc[k], sW[r * ML + k], yr);
            }
        }
#pragma unroll
        for (int k = 0; k < ML; ++k) {
            if (k >= nl) break;
            if (a.llr) {
                float v[QM];
                demap_layer<QM, ZF>(acc[k], sSlope[k], v);
                store_layer_llr<QM, LT>(a.llr, (re * nl + k) * QM, v);
            }
            if (a.xhat) {
                const float ia = rsqrtf((float)qam_norm(QM));  // back from level units
                a.xhat[re * nl + k] = make_float2(acc[k].x * ia, acc[k].y * ia);
            }
        }
    }
}

template <int QM, int LT>
__global__ void __launch_bounds__(kThreads) k_generic(DetectArgs a) {
    __shared__ double2 sH[MR * ML];   // H[r][l]
    __shared__ double2 sL[ML * ML];   // G, then L (lower)
    __shared__ double2 sX[ML * ML];   // L^-1 (lower)
    __shared__ double2 sGi[ML * ML];  // G^-1
    __shared__ float2 sW[MR * ML];    // W~[r][k], level units
    __shared__ float sSlope[ML];
    __shared__ double sMu[ML];
    __shared__ int sFail;

    // PDL: no overlap here (grid-stride loop writes early), just order after the previous grid
    pdl_launch_dependents();
    pdl_wait();
    const int nr = a.n_rx, nl = a.n_layers, tid = threadIdx.x;
    const double norm = (double)qam_norm(QM);
    const double sq_norm = sqrt(norm);

    for (long long u = blockIdx.x; u < a.n_units; u += gridDim.x) {
        const int slot = (int)(u / a.n_fb);
        const int fb = (int)(u % a.n_fb);
        const double s2 = (double)block_sigma2(a, slot);
        // a1: stage H_u
        for (int i = tid; i < nr * nl; i += blockDim.x) {
            const float2 h = __ldg(a.H + (size_t)u * nr * nl + i);
            sH[(i / nl) * ML + (i % nl)] = make_double2(h.x, h.y);
        }
        if (tid == 0) sFail = 0;
        __syncthreads();
        // a2: Gram lower triangle, G_ij = sum_r conj(H_ri) H_rj (+ s2 on the diagonal)
        for (int p = tid; p < nl * nl; p += blockDim.x) {
            const int i = p / nl, j = p % nl;
            if (j > i) continue;
            double2 acc = make_double2(0.0, 0.0);
            for (int r = 0; r < nr; ++r) acc = dmacc(acc, sH[r * ML + i], sH[r * ML + j]);
            if (i == j) acc = make_double2(acc.x + s2, 0.0);
            sL[i * ML + j] = acc;
        }
        __syncthreads();
        // a3: right-looking Cholesky with the pivot guard (reading R17)
        double gmax = 0.0;
        for (int i = 0; i < nl; ++i) gmax = fmax(gmax, sL[i * ML + i].x);
        for (int j = 0; j < nl; ++j) {
            if (tid == 0) {
                const double p = sL[j * ML + j].x;
                if (!(p > kPivotTau * gmax)) sFail = 1;
                else sL[j * ML + j] = make_double2(sqrt(p), 0.0);
            }
            __syncthreads();
            if (sFail) break;
            const double dinv = 1.0 / sL[j * ML + j].x;
            for (int i = j + 1 + tid; i < nl; i += blockDim.x) sL[i * ML + j] = dscale(sL[i * ML + j], dinv);
            __syncthreads();
            const int m = nl - j - 1;
            for (int p = tid; p < m * m; p += blockDim.x) {
                const int i = j + 1 + p / m, k = j + 1 + p % m;
                if (k > i) continue;
                const double2 li = sL[i * ML + j], lk = sL[k * ML + j];
                // G_ik -= L_ij conj(L_kj)
                sL[i * ML + k] = dsub(sL[i * ML + k], dmul(li, make_double2(lk.x, -lk.y)));
            }
            __syncthreads();
        }
        const bool failed = sFail != 0;
        if (!failed) {
            // a4: X = L^-1 by forward substitution, column k per thread
            if (tid < nl) {
                const int k = tid;
                for (int i = 0; i < k; ++i) sX[i * ML + k] = make_double2(0.0, 0.0);
                sX[k * ML + k] = make_double2(1.0 / sL[k * ML + k].x, 0.0);
                for (int i = k + 1; i < nl; ++i) {
                    double2 s = make_double2(0.0, 0.0);
                    for (int m2 = k; m2 < i; ++m2) s = dmac(s, sL[i * ML + m2], sX[m2 * ML + k]);
                    sX[i * ML + k] = dscale(s, -1.0 / sL[i * ML + i].x);
                }
            }
            __syncthreads();
            // G^-1 = X^H X
            for (int p = tid; p < nl * nl; p += blockDim.x) {
                const int i = p / nl, j = p % nl;
                double2 s = make_double2(0.0, 0.0);
                for (int m2 = (i > j ? i : j); m2 < nl; ++m2) s = dmacc(s, sX[m2 * ML + i], sX[m2 * ML + j]);
                sGi[i * ML + j] = s;
            }
            __syncthreads();
            // a5: mu, SINR, slope (readings R3, R4, R11)
            if (tid < nl) {
                const int k = tid;
                const double A = sGi[k * ML + k].x;
                double mu, sinr;
                if (s2 == 0.0) {
                    mu = 1.0;
                    sinr = (double)INFINITY;
                } else {
                    mu = 1.0 - s2 * A;
                    sinr = 1.0 / (s2 * A) - 1.0;
                }
                if (!(mu > 0.0)) sinr = 0.0;
                sMu[k] = mu;
                sSlope[k] = (float)(sinr / norm) * a.llr_scale;
                if (a.sinr) a.sinr[u * nl + k] = (float)sinr;
            }
            __syncthreads();
            // W~ = diag(sqrt(norm)/mu) G^-1 H^H
            for (int p = tid; p < nl * nr; p += blockDim.x) {
                const int r = p / nl, k = p % nl;
                double2 s = make_double2(0.0, 0.0);
                for (int j = 0; j < nl; ++j) {
                    const double2 h = sH[r * ML + j];
                    s = dmac(s, sGi[k * ML + j], make_double2(h.x, -h.y));
                }
                const double mu = sMu[k];
                const double f = mu > 0.0 ? sq_norm / mu : 0.0;
                sW[r * ML + k] = make_float2((float)(s.x * f), (float)(s.y * f));
            }
        } else {
            if (tid == 0) atomicAdd(a.fail_count, 1ull);
            if (tid < nl) {
                sSlope[tid] = 0.f;
                if (a.sinr) a.sinr[u * nl + tid] = 0.f;
            }
        }
        __syncthreads();
        if (a.sigma2 > 0.f) apply_unit<QM, LT, false>(a, sW, sSlope, slot, fb, failed);
        else apply_unit<QM, LT, true>(a, sW, sSlope, slot, fb, failed);
        __syncthreads();
    }
}

template <int QM, int LT>
cudaError_t launch_q(const DetectArgs& a, cudaStream_t s) {
    long long grid = a.n_units < 148LL * 16 ? a.n_units : 148LL * 16;
    if (grid <= 0) return cudaSuccess;
    return launch_kernel(k_generic<QM, LT>, dim3((unsigned)grid), dim3(kThreads), 0, s, a.overlap, a);
}

template <int QM>
cudaError_t launch_l(const DetectArgs& a, cudaStream_t s) {
    switch (a.llr_type) {
    case kLlrF32: return launch_q<QM, kLlrF32>(a, s);
    case kLlrF16: return launch_q<QM, kLlrF16>(a, s);
    default: return launch_q<QM, kLlrI8>(a, s);
    }
}

}  // namespace

cudaError_t launch_generic(const DetectArgs& a, cudaStream_t s) {
    switch (a.qm) {
    case 2: return launch_l<2>(a, s);
    case 4: return launch_l<4>(a, s);
    case 6: return launch_l<6>(a, s);
    default: return launch_l<8>(a, s);
    }
}

}  // namespace mimo
