// k_bfp.cu -- block-floating-point fronthaul y (reading R25) for every
// detector shape: one kernel expands the blocks into complex64 y, which the shape's own detector
// then reads. (The 8 rx x 4 layer per-PRB family decodes inside its apply loads instead, k_split.cu.)
//
// Block (symbol, PRB, antenna) = ceil4(1 + 3W) bytes: byte 0 = exponent e (bits 0..3), then the 24
// two's-complement W-bit mantissas I0, Q0, ..., I11, Q11 of the PRB's 12 subcarriers, MSB-first;
// value = m * 2^e * scale (exact in fp32: |m| < 2^15, a power-of-two factor).
// Thread = one block; consecutive threads = consecutive antennas, so each of the 12 complex stores
// of a warp is one contiguous run of the y row. Mantissa bit offsets are compile-time per W.
#include "kernels.h"

namespace mimo {
namespace {

template <int W>
__global__ void __launch_bounds__(256) k_bfp_decode(const uint8_t* __restrict__ yb, float2* __restrict__ y, int n_rx,
                                                    int n_prb, long long n_blocks, float scale) {
    constexpr int BB = ((1 + 3 * W) + 3) & ~3;  // block bytes
    constexpr int NW = BB / 4;
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n_blocks) return;
    const int r = (int)(b % n_rx);
    const long long sp = b / n_rx;  // symbol * n_prb + prb
    const int prb = (int)(sp % n_prb);
    const long long sym = sp / n_prb;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(yb + b * BB);
    uint32_t be[NW + 1];  // the block as a big-endian bit stream
#pragma unroll
    for (int i = 0; i < NW; ++i) be[i] = __byte_perm(__ldg(src + i), 0, 0x0123);
    be[NW] = 0;
    const int e = (int)(be[0] >> 24) & 15;
    const float f = ldexpf(scale, e);
    float v[24];
#pragma unroll
    for (int i = 0; i < 24; ++i) {
        const int o = 8 + i * W;  // bit offset of mantissa i
        const int wd = o >> 5, sh = o & 31;
        const uint32_t win = sh ? (be[wd] << sh) | (be[wd + 1] >> (32 - sh)) : be[wd];
        v[i] = (float)((int32_t)win >> (32 - W)) * f;
    }
    const int n_sc = 12 * n_prb;
    float2* dst = y + ((size_t)sym * n_sc + 12 * prb) * n_rx + r;
#pragma unroll
    for (int k = 0; k < 12; ++k) dst[(size_t)k * n_rx] = make_float2(v[2 * k], v[2 * k + 1]);
}

template <int W>
cudaError_t launch_w(const void* yb, float2* y, int n_rx, int n_sc, int n_sym, float scale, cudaStream_t s) {
    const int n_prb = n_sc / 12;
    const long long nb = (long long)n_sym * n_prb * n_rx;
    if (nb == 0) return cudaSuccess;
    k_bfp_decode<W><<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(static_cast<const uint8_t*>(yb), y, n_rx, n_prb, nb,
                                                                scale);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_bfp_decode(const void* y_bfp, float2* y, int n_rx, int n_sc, int n_sym, int iq_width, float scale,
                              cudaStream_t s) {
    switch (iq_width) {
    case 8: return launch_w<8>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 9: return launch_w<9>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 10: return launch_w<10>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 11: return launch_w<11>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 12: return launch_w<12>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 13: return launch_w<13>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 14: return launch_w<14>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 15: return launch_w<15>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    case 16: return launch_w<16>(y_bfp, y, n_rx, n_sc, n_sym, scale, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace mimo
