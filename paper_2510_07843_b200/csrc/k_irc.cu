// k_irc.cu -- coloured-noise LMMSE detection (interference-rejection combining,
// SURVEY.md §8(f) NEXT-3; reading R24): y = H x + n with n ~ CN(0, R_nn), R_nn
// Hermitian positive definite per H-unit (e.g. known interferer covariance plus
// noise). The filter W = H^H (H H^H + R_nn)^-1 is formed by whitening, which
// keeps the per-RE cost of the white-noise detector:
//   R_nn = L_R L_R^H (Cholesky),  H~ = L_R^-1 H            (forward substitution)
//   G = H~^H H~ + I = L L^H,  A_kk = [G^-1]_kk             (the white route with sigma2 = 1)
//   mu_k = 1 - A_kk,  SINR_k = 1/A_kk - 1
//   W = G^-1 H~^H L_R^-1  (row-vector back-substitution against L_R), W~ = W sqrt(norm) / mu
// so that x~ = W~ y acts on the UN-whitened y. One CTA per H-unit, setup in fp64
// shared memory (like k_generic), W~ rounded once to fp32, then thread per RE.
// R_nn = sigma2 I reduces to mimo_detect_mmse exactly (pinned in the tests).
// Failure (R_nn or G not positive definite by the R17 guard, or NaN): the unit
// is counted and its outputs are erasures.
#include "kernels.h"

namespace mimo {
namespace {

constexpr int kThreads = 128;
constexpr int MR = 16;  // n_rx <= 16
constexpr int ML = 16;

template <int QM, int LT>
__device__ __forceinline__ void store_layer(void* llr, size_t idx, const float* v) {
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

// in-place right-looking Cholesky of the lower triangle of A (n x n, row stride ld) with the
// R17 guard; returns false on failure. Cooperative over the CTA.
__device__ bool chol_inplace(double2* A, int n, int ld, int* sFail) {
    const int tid = threadIdx.x;
    double amax = 0.0;
    for (int i = 0; i < n; ++i) amax = fmax(amax, A[i * ld + i].x);
    if (tid == 0) *sFail = !(amax == amax);
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (tid == 0) {
            const double p = A[j * ld + j].x;
            if (!(p > kPivotTau * amax)) *sFail = 1;
            else A[j * ld + j] = make_double2(sqrt(p), 0.0);
        }
        __syncthreads();
        if (*sFail) return false;
        const double dinv = 1.0 / A[j * ld + j].x;
        for (int i = j + 1 + tid; i < n; i += blockDim.x) A[i * ld + j] = dscale(A[i * ld + j], dinv);
        __syncthreads();
        const int m = n - j - 1;
        for (int p = tid; p < m * m; p += blockDim.x) {
            const int i = j + 1 + p / m, k = j + 1 + p % m;
            if (k > i) continue;
            const double2 li = A[i * ld + j], lk = A[k * ld + j];
            A[i * ld + k] = dsub(A[i * ld + k], dmul(li, make_double2(lk.x, -lk.y)));
        }
        __syncthreads();
    }
    return true;
}

template <int QM, int LT>
__global__ void __launch_bounds__(kThreads) k_irc(DetectArgs a, const float2* __restrict__ Rnn) {
    __shared__ double2 sR[MR * MR];   // R_nn, then L_R (lower)
    __shared__ double2 sH[MR * ML];   // H~ = L_R^-1 H  [r][l]
    __shared__ double2 sG[ML * ML];   // G, then L (lower)
    __shared__ double2 sX[ML * ML];   // L^-1 (lower)
    __shared__ double2 sGi[ML * ML];  // G^-1
    __shared__ double2 sWh[ML * MR];  // G^-1 H~^H, then W = ... L_R^-1  [k][r]
    __shared__ float2 sW[MR * ML];    // W~ [r][k]
    __shared__ float sSlope[ML];
    __shared__ double sMu[ML];
    __shared__ int sFail;

    pdl_launch_dependents();
    pdl_wait();
    const int nr = a.n_rx, nl = a.n_layers, tid = threadIdx.x;
    const double norm = (double)qam_norm(QM);
    const double sq_norm = sqrt(norm);
    for (long long u = blockIdx.x; u < a.n_units; u += gridDim.x) {
        const int slot = (int)(u / a.n_fb), fb = (int)(u % a.n_fb);
        for (int i = tid; i < nr * nr; i += blockDim.x) {
            const float2 v = __ldg(Rnn + (size_t)u * nr * nr + i);
            sR[(i / nr) * MR + (i % nr)] = make_double2(v.x, v.y);
        }
        for (int i = tid; i < nr * nl; i += blockDim.x) {
            const float2 h = __ldg(a.H + (size_t)u * nr * nl + i);
            sH[(i / nl) * ML + (i % nl)] = make_double2(h.x, h.y);
        }
        __syncthreads();
        bool ok = chol_inplace(sR, nr, MR, &sFail);
        if (ok) {
            // H~ = L_R^-1 H: forward substitution, column l per thread
            if (tid < nl) {
                const int l = tid;
                for (int i = 0; i < nr; ++i) {
                    double2 s = sH[i * ML + l];
                    for (int m = 0; m < i; ++m) s = dsub(s, dmul(sR[i * MR + m], sH[m * ML + l]));
                    sH[i * ML + l] = dscale(s, 1.0 / sR[i * MR + i].x);
                }
            }
            __syncthreads();
            // G = H~^H H~ + I (lower triangle)
            for (int p = tid; p < nl * nl; p += blockDim.x) {
                const int i = p / nl, j = p % nl;
                if (j > i) continue;
                double2 acc = make_double2(0.0, 0.0);
                for (int r = 0; r < nr; ++r) acc = dmacc(acc, sH[r * ML + i], sH[r * ML + j]);
                if (i == j) acc = make_double2(acc.x + 1.0, 0.0);
                sG[i * ML + j] = acc;
            }
            __syncthreads();
            ok = chol_inplace(sG, nl, ML, &sFail);
        }
        if (ok) {
            if (tid < nl) {  // X = L^-1, column k per thread
                const int k = tid;
                for (int i = 0; i < k; ++i) sX[i * ML + k] = make_double2(0.0, 0.0);
                sX[k * ML + k] = make_double2(1.0 / sG[k * ML + k].x, 0.0);
                for (int i = k + 1; i < nl; ++i) {
                    double2 s = make_double2(0.0, 0.0);
                    for (int m2 = k; m2 < i; ++m2) s = dmac(s, sG[i * ML + m2], sX[m2 * ML + k]);
                    sX[i * ML + k] = dscale(s, -1.0 / sG[i * ML + i].x);
                }
            }
            __syncthreads();
            for (int p = tid; p < nl * nl; p += blockDim.x) {  // G^-1 = X^H X
                const int i = p / nl, j = p % nl;
                double2 s = make_double2(0.0, 0.0);
                for (int m2 = (i > j ? i : j); m2 < nl; ++m2) s = dmacc(s, sX[m2 * ML + i], sX[m2 * ML + j]);
                sGi[i * ML + j] = s;
            }
            __syncthreads();
            if (tid < nl) {  // mu, SINR (whitened domain: sigma2 = 1)
                const int k = tid;
                const double A = sGi[k * ML + k].x;
                const double mu = 1.0 - A;
                double sinr = 1.0 / A - 1.0;
                if (!(mu > 0.0)) sinr = 0.0;
                sMu[k] = mu;
                sSlope[k] = (float)(sinr / norm) * a.llr_scale;
                if (a.sinr) a.sinr[u * nl + k] = (float)sinr;
            }
            for (int p = tid; p < nl * nr; p += blockDim.x) {  // Wh = G^-1 H~^H
                const int k = p / nr, r = p % nr;
                double2 s = make_double2(0.0, 0.0);
                for (int j = 0; j < nl; ++j) {
                    const double2 h = sH[r * ML + j];
                    s = dmac(s, sGi[k * ML + j], make_double2(h.x, -h.y));
                }
                sWh[k * MR + r] = s;
            }
            __syncthreads();
            if (tid < nl) {  // W_k L_R = Wh_k  ->  W_k = Wh_k L_R^-1 (back-substitution over columns)
                const int k = tid;
                for (int j = nr - 1; j >= 0; --j) {
                    double2 s = sWh[k * MR + j];
                    for (int i = j + 1; i < nr; ++i) s = dsub(s, dmul(sWh[k * MR + i], sR[i * MR + j]));
                    sWh[k * MR + j] = dscale(s, 1.0 / sR[j * MR + j].x);
                }
            }
            __syncthreads();
            for (int p = tid; p < nl * nr; p += blockDim.x) {
                const int r = p / nl, k = p % nl;
                const double2 w = sWh[k * MR + r];
                const double f = sMu[k] > 0.0 ? sq_norm / sMu[k] : 0.0;
                sW[r * ML + k] = make_float2((float)(w.x * f), (float)(w.y * f));
            }
        } else {
            if (tid == 0) atomicAdd(a.fail_count, 1ull);
            if (tid < nl) {
                sSlope[tid] = 0.f;
                if (a.sinr) a.sinr[u * nl + tid] = 0.f;
            }
            for (int p = tid; p < nl * nr; p += blockDim.x) sW[(p / nl) * ML + (p % nl)] = make_float2(0.f, 0.f);
        }
        __syncthreads();
        // apply: x~ = W~ y per RE, exact max-log, quantise
        const int n_re = a.sc_per_h * a.sym_per_h;
        const float ia = rsqrtf((float)norm);
        for (int e = tid; e < n_re; e += blockDim.x) {
            const int sym = slot * a.sym_per_h + e / a.sc_per_h;
            const int sc = fb * a.sc_per_h + e % a.sc_per_h;
            const size_t re = (size_t)sym * a.n_sc + sc;
            float2 acc[ML];
#pragma unroll
            for (int k = 0; k < ML; ++k) acc[k] = make_float2(0.f, 0.f);
            const float2* yp = a.y + re * nr;
            for (int r = 0; r < nr; ++r) {
                const float2 yr = __ldg(yp + r);
#pragma unroll
                for (int k = 0; k < ML; ++k)
                    if (k < nl) acc[k] = cmac(acc[k], sW[r * ML + k], yr);
            }
#pragma unroll
            for (int k = 0; k < ML; ++k) {
                if (k >= nl) break;
                if (a.llr) {
                    float v[QM];
                    demap_layer<QM, false>(acc[k], sSlope[k], v);
                    store_layer<QM, LT>(a.llr, (re * nl + k) * QM, v);
                }
                if (a.xhat) a.xhat[re * nl + k] = make_float2(acc[k].x * ia, acc[k].y * ia);
            }
        }
        __syncthreads();
    }
}

template <int QM>
cudaError_t by_llr(const DetectArgs& a, const float2* R, cudaStream_t s) {
    const long long grid = a.n_units < 148LL * 16 ? a.n_units : 148LL * 16;
    switch (a.llr_type) {
    case kLlrF32: k_irc<QM, kLlrF32><<<(unsigned)grid, kThreads, 0, s>>>(a, R); break;
    case kLlrF16: k_irc<QM, kLlrF16><<<(unsigned)grid, kThreads, 0, s>>>(a, R); break;
    default: k_irc<QM, kLlrI8><<<(unsigned)grid, kThreads, 0, s>>>(a, R); break;
    }
    return cudaGetLastError();
}

}  // namespace

bool irc_supported(int n_rx, int n_layers) { return n_rx >= 1 && n_rx <= MR && n_layers >= 1 && n_layers <= n_rx; }

cudaError_t launch_irc(const DetectArgs& a, const float2* Rnn, cudaStream_t s) {
    if (a.n_units <= 0) return cudaSuccess;
    switch (a.qm) {
    case 2: return by_llr<2>(a, Rnn, s);
    case 4: return by_llr<4>(a, Rnn, s);
    case 6: return by_llr<6>(a, Rnn, s);
    default: return by_llr<8>(a, Rnn, s);
    }
}

}  // namespace mimo
