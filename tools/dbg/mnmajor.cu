// Probe: tcgen05.mma kind::tf32 M=64 N=32 K=8 with MN-major (A and B) SW128 operands.
// Prints where each D row lands in TMEM (lane) and its values.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_07843_b200/csrc/tc.cuh"
using namespace mimo;

__global__ void k(float* out, int amn, uint32_t lbo, uint32_t sbo, int m) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    float* X = reinterpret_cast<float*>(sm);          // 8 K rows x 32 floats (SW128), then X_lo at +8192
    // element (k, c) of atom a: logical value; stored swizzled: chunk (c/4) ^ (k & 7)
    for (int i = t; i < 2 * 8 * 32; i += blockDim.x) {
        const int a = i / 256, k = (i / 32) % 8, c = i % 32;
        const float v = (a ? 1000.f : 0.f) + k * 32 + c;   // A[m = 32 a + c][k]
        const int off = a * 2048 + k * 32 + (((c >> 2) ^ (k & 7)) << 2) + (c & 3);
        X[off] = v;
    }
    if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tc::alloc<64>(&tslot);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tslot, xs = smem_u32(sm);
    if (t == 0) {
        uint32_t id = tc::idesc(tc::kFmtTF32, m, 32, amn, amn);
        uint64_t dA = tc::desc_sw128(xs, lbo, sbo), dB = tc::desc_sw128(xs, lbo, sbo);
        tc::mma_tf32_ss(tm, dA, dB, id, 0u);
        tc::commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc::fence_after();
    uint32_t v[32];
    tc::ld32(tm + ((uint32_t)(32 * warp) << 16), v);
    tc::wait_ld();
    for (int c = 0; c < 32; ++c) out[(32 * warp + lane) * 32 + c] = __uint_as_float(v[c]);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::dealloc<64>(tm);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 32 * 4);
    static float h[128 * 32];
    struct C { int amn; uint32_t lbo, sbo; int m; } cs[] = {{1, 8192, 1024, 64}, {1, 1024, 8192, 64}, {1, 8192, 128, 64},
        {1, 128, 8192, 64}, {1, 16, 1024, 64}, {1, 8192, 1024, 128}, {1, 1024, 8192, 128}};
    for (auto c : cs) {
        cudaMemset(d, 0, 128 * 32 * 4);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        k<<<1, 128, 32768>>>(d, c.amn, c.lbo, c.sbo, c.m);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("major=%s lbo=%u sbo=%u M=%d err=%s\n", c.amn ? "MN" : "K", c.lbo, c.sbo, c.m, cudaGetErrorString(e));
        int shown = 0;
        for (int lane = 0; lane < 128; ++lane) {
            double s = 0; for (int cc = 0; cc < 32; ++cc) s += fabs(h[lane * 32 + cc]);
            if (s == 0) continue;
            if (shown++ < 6 || lane % 16 == 0) printf("  lane %3d: %.0f %.0f %.0f\n", lane, h[lane * 32], h[lane * 32 + 1], h[lane * 32 + 31]);
        }
        printf("  nonzero lanes: %d\n", shown);
    }
    // host reference: for MN-major A[m][k] = (m>=32?1000:0) + k*32 + m%32, B[n][k] = k*32 + n
    for (int m : {0, 1, 15, 16, 31, 32, 33, 63}) {
        double r0 = 0, r1 = 0, r31 = 0;
        for (int kk = 0; kk < 8; ++kk) {
            double a = (m >= 32 ? 1000 : 0) + kk * 32 + m % 32;
            r0 += a * (kk * 32 + 0); r1 += a * (kk * 32 + 1); r31 += a * (kk * 32 + 31);
        }
        printf("ref row %2d: %.0f %.0f %.0f\n", m, r0, r1, r31);
    }
    return 0;
}
