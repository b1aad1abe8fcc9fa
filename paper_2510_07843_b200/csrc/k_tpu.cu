// k_tpu.cu -- "thread per H-unit" detector for small per-subcarrier channels
// (C1 2x2 QPSK, C2 4x4 16-QAM; any NR <= 4 even, NL <= NR).
//
// Mapping (DESIGN.md §"Kernels"): a CTA owns TU consecutive subcarriers of one
// slot (TU H-units, 14 x TU REs). One thread per H-unit:
//   1. thread 0 issues 14 cp.async.bulk copies (one per OFDM symbol row, TU*NR*8
//      contiguous bytes each) of the CTA's y tile into shared memory, each
//      completing on its own mbarrier -- the whole tile is in flight at once,
//      with no register cost;
//   2. meanwhile every thread loads its H (NR*NL*8 B, 256-bit loads) and runs
//      the setup (rows a2-a5) fully unrolled in fp64 registers (reading R18: an
//      fp32 setup misses the 1e-4 x~ bound on square 4x4 channels, SURVEY.md
//      §8(c)), rounding W~ (in PAM level units) and the LLR slopes once to fp32;
//   3. for each symbol s it waits on mbarrier s, reads its y from shared
//      memory, computes x~ = W~ y (row a6), demaps exactly (row a7) and writes
//      the RE's NL*QM LLRs with 256-bit stores (full 32-byte sectors).
// The 14 REs of a unit reuse one W~ held in registers.
#include "kernels.h"

namespace mimo {
namespace {

constexpr int kSym = 14;

template <int NR, int NL>
struct SetupOut {
    float2 w[NL][NR];  // W~ * sqrt(norm), fp32
    float slope[NL];   // SINR * llr_scale / norm
    float sinr[NL];
    bool fail;
};

// Rows a2-a5 in fp64 registers, fully unrolled.
template <int NR, int NL>
__device__ __forceinline__ void setup_f64(const float2 (&hf)[NR][NL], double s2, double norm, float llr_scale,
                                          SetupOut<NR, NL>& o) {
    double2 h[NR][NL];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int l = 0; l < NL; ++l) h[r][l] = make_double2(hf[r][l].x, hf[r][l].y);

    // a2: G = H^H H + s2 I (lower triangle)
    double2 L[NL][NL];
    double gmax = 0.0;
#pragma unroll
    for (int i = 0; i < NL; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc = dmacc(acc, h[r][i], h[r][j]);
            L[i][j] = acc;
        }
        L[i][i] = make_double2(L[i][i].x + s2, 0.0);
        gmax = fmax(gmax, L[i][i].x);
    }
    // a3: Cholesky (column by column, in place), keep 1/L_jj
    double dinv[NL];
    bool fail = false;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        double p = L[j][j].x;
#pragma unroll
        for (int k = 0; k < j; ++k) p -= dnorm2(L[j][k]);
        if (!(p > kPivotTau * gmax)) {
            fail = true;
            p = 1.0;
        }
        dinv[j] = rsqrt(p);
#pragma unroll
        for (int i = j + 1; i < NL; ++i) {
            double2 s = L[i][j];
#pragma unroll
            for (int k = 0; k < j; ++k) {
                // s -= L_ik conj(L_jk)
                const double2 a = L[i][k], b = L[j][k];
                s.x -= fma(a.x, b.x, a.y * b.y);
                s.y -= fma(a.y, b.x, -a.x * b.y);
            }
            L[i][j] = dscale(s, dinv[j]);
        }
    }
    // a4: X = L^-1 (lower), X_jj = 1/L_jj, X_ij = -(1/L_ii) sum_{m=j}^{i-1} L_im X_mj
    double2 X[NL][NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        X[j][j] = make_double2(dinv[j], 0.0);
#pragma unroll
        for (int i = j + 1; i < NL; ++i) {
            double2 s = make_double2(0.0, 0.0);
#pragma unroll
            for (int m = j; m < i; ++m) s = dmac(s, L[i][m], X[m][j]);
            X[i][j] = dscale(s, -dinv[i]);
        }
    }
    // A_kk = [G^-1]_kk = sum_{i>=k} |X_ik|^2
    // B = X H^H (NL x NR), B_ir = sum_{m<=i} X_im conj(H_rm)
    double2 B[NL][NR];
#pragma unroll
    for (int i = 0; i < NL; ++i)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            double2 s = make_double2(0.0, 0.0);
#pragma unroll
            for (int m = 0; m <= i; ++m) s = dmac(s, X[i][m], make_double2(h[r][m].x, -h[r][m].y));
            B[i][r] = s;
        }
    const double sqn = sqrt(norm);
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        double A = 0.0;
#pragma unroll
        for (int i = k; i < NL; ++i) A += dnorm2(X[i][k]);
        // a5 (readings R3, R4, R11)
        double mu, sinr;
        if (s2 == 0.0) {
            mu = 1.0;
            sinr = (double)INFINITY;
        } else {
            mu = 1.0 - s2 * A;
            sinr = 1.0 / (s2 * A) - 1.0;
        }
        double f = sqn / mu;
        if (!(mu > 0.0) || fail) {
            sinr = 0.0;
            f = 0.0;
        }
        o.sinr[k] = (float)sinr;
        o.slope[k] = (float)(sinr / norm) * llr_scale;
        // W_kr = sum_{i>=k} conj(X_ik) B_ir
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            double2 s = make_double2(0.0, 0.0);
#pragma unroll
            for (int i = k; i < NL; ++i) s = dmacc(s, X[i][k], B[i][r]);
            o.w[k][r] = make_float2((float)(s.x * f), (float)(s.y * f));
        }
    }
    o.fail = fail;
}

template <int NR, int NL, int QM, int LT, int TU>
__global__ void __launch_bounds__(TU) k_tpu(DetectArgs a) {
    static_assert(NR % 2 == 0, "bulk rows need 16-byte multiples");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    float2* sy = reinterpret_cast<float2*>(smem + 128);

    const int slot = blockIdx.y;
    const int sc0 = blockIdx.x * TU;
    const int nvalid = min(TU, a.n_sc - sc0);
    const int t = threadIdx.x;

    if (t == 0) {
#pragma unroll
        for (int s = 0; s < kSym; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        const uint32_t row_bytes = (uint32_t)nvalid * NR * 8u;
#pragma unroll 1
        for (int s = 0; s < kSym; ++s) {
            mbar_arrive_expect_tx(&bars[s], row_bytes);
            bulk_g2s(sy + s * TU * NR, a.y + ((size_t)(slot * kSym + s) * a.n_sc + sc0) * NR, row_bytes, &bars[s]);
        }
    }

    const bool active = t < nvalid;
    const int sc = sc0 + t;
    const size_t unit = (size_t)slot * a.n_sc + sc;
    SetupOut<NR, NL> o;
    if (active) {
        float2 hf[NR][NL];
        load_bytes<NR * NL * 8>(a.H + unit * NR * NL, reinterpret_cast<uint32_t*>(&hf[0][0]));
        setup_f64<NR, NL>(hf, (double)a.sigma2, (double)qam_norm(QM), a.llr_scale, o);
        if (o.fail) atomicAdd(a.fail_count, 1ull);
        if (a.sinr) {
#pragma unroll
            for (int k = 0; k < NL; ++k) a.sinr[unit * NL + k] = o.sinr[k];
        }
    }

    constexpr int kLlrBytes = NL * QM * LlrTraits<LT>::bytes;
    constexpr int kWords = (kLlrBytes + 3) / 4;
    const float ia = rsqrtf((float)qam_norm(QM));
#pragma unroll 1
    for (int s = 0; s < kSym; ++s) {
        mbar_wait(&bars[s], 0);
        if (!active) continue;
        float2 yv[NR];
        const float2* ys = sy + (s * TU + t) * NR;
#pragma unroll
        for (int r = 0; r < NR; ++r) yv[r] = ys[r];
        float2 x[NL];
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc = cmac(acc, o.w[k][r], yv[r]);
            x[k] = acc;
        }
        const size_t re = (size_t)(slot * kSym + s) * a.n_sc + sc;
        if (a.llr) {
            float v[NL * QM];
#pragma unroll
            for (int k = 0; k < NL; ++k) demap_layer<QM>(x[k], o.slope[k], v + k * QM);
            uint32_t w[kWords];
            pack_llr<LT, NL * QM>(v, w);
            store_bytes<kLlrBytes>((char*)a.llr + re * kLlrBytes, w);
        }
        if (a.xhat) {
            uint32_t w[2 * NL];
#pragma unroll
            for (int k = 0; k < NL; ++k) {
                w[2 * k] = __float_as_uint(x[k].x * ia);
                w[2 * k + 1] = __float_as_uint(x[k].y * ia);
            }
            store_bytes<NL * 8>(a.xhat + re * NL, w);
        }
    }
}

template <int NR, int NL, int QM, int LT, int TU>
cudaError_t launch(const DetectArgs& a, cudaStream_t s) {
    if (a.n_sc <= 0 || a.n_slots <= 0) return cudaSuccess;
    const size_t smem = 128 + (size_t)kSym * TU * NR * 8;
    dim3 grid((a.n_sc + TU - 1) / TU, a.n_slots);
    k_tpu<NR, NL, QM, LT, TU><<<grid, TU, smem, s>>>(a);
    return cudaGetLastError();
}

template <int NR, int NL, int QM, int LT, int TU>
cudaError_t prepare() {
    const int smem = 128 + kSym * TU * NR * 8;
    if (smem > 48 * 1024)
        return cudaFuncSetAttribute(k_tpu<NR, NL, QM, LT, TU>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaSuccess;
}

#define TPU_ENTRY(NR, NL, QM, LT, TU)                                                                       \
    KernelEntry {                                                                                           \
        "tpu_" #NR "x" #NL "_q" #QM "_l" #LT "_tu" #TU, NR, NL, QM, 1, 14, LT, 32, 1,                     \
            launch<NR, NL, QM, LT, TU>, prepare<NR, NL, QM, LT, TU>                                        \
    }

const KernelEntry kEntries[] = {
    TPU_ENTRY(2, 2, 2, kLlrF32, 32),  // C1
    TPU_ENTRY(4, 4, 4, kLlrF32, 32),  // C2 (and the paper's own 4x4 shape)
    TPU_ENTRY(2, 2, 4, kLlrF32, 32),
    TPU_ENTRY(2, 1, 2, kLlrF32, 32),
    TPU_ENTRY(4, 2, 4, kLlrF32, 32),
    TPU_ENTRY(4, 4, 4, kLlrF16, 32),
    TPU_ENTRY(4, 4, 4, kLlrI8, 32),
    TPU_ENTRY(4, 4, 2, kLlrF32, 32),
    TPU_ENTRY(4, 4, 6, kLlrF32, 32),
    TPU_ENTRY(4, 4, 8, kLlrF32, 32),
};

}  // namespace

const KernelEntry* tpu_entries(int* n) {
    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));
    return kEntries;
}

}  // namespace mimo
