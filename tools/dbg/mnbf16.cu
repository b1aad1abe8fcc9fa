// Probe: tcgen05.mma kind::f16 (BF16) M=64 N=64 K=16 with MN-major SW128 operands (A = B = X^T view).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_2510_07843_b200/csrc/tc.cuh"
using namespace mimo;

__host__ __device__ inline float val(int k, int m) { return (k == (m & 15)) ? (float)(m + 1) : 0.f; }

__global__ void k(float* out, uint32_t lbo, uint32_t sbo, int n) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    __nv_bfloat16* X = reinterpret_cast<__nv_bfloat16*>(sm);  // 16 K rows x 64 bf16 (128 B), SW128
    for (int i = t; i < 16 * 64; i += blockDim.x) {
        const int kk = i / 64, m = i % 64;
        const int off = (kk / 8) * 512 + (kk % 8) * 64 + (((m >> 3) ^ (kk & 7)) << 3) + (m & 7);
        X[off] = __float2bfloat16(val(kk, m));
    }
    if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tc::alloc<64>(&tslot);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tslot, xs = smem_u32(sm);
    if (t == 0) {
        uint32_t id = tc::idesc(tc::kFmtBF16, 64, n, 1, 1);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(tc::desc_sw128(xs, lbo, sbo)), "l"(tc::desc_sw128(xs + (n == 32 ? 64u : 0u), lbo, sbo)), "r"(id), "r"(0));
        tc::commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc::fence_after();
    uint32_t v[32];
    tc::ld32(tm + ((uint32_t)(32 * warp) << 16), v);
    tc::wait_ld();
    for (int c = 0; c < 32; ++c) out[(32 * warp + lane) * 64 + c] = __uint_as_float(v[c]);
    tc::ld32(tm + ((uint32_t)(32 * warp) << 16) + 32, v);
    tc::wait_ld();
    for (int c = 0; c < 32; ++c) out[(32 * warp + lane) * 64 + 32 + c] = __uint_as_float(v[c]);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::dealloc<64>(tm);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 64 * 4);
    static float h[128 * 64];
    double ref[64][64];
    for (int m = 0; m < 64; ++m)
        for (int nn = 0; nn < 64; ++nn) {
            double s = 0;
            for (int kk = 0; kk < 16; ++kk) s += (double)val(kk, m) * val(kk, nn);
            ref[m][nn] = s;
        }
    struct C { uint32_t lbo, sbo; int n; } cs[] = {{16, 1024, 64}, {16, 1024, 32}};
    for (auto c : cs) {
        cudaMemset(d, 0, sizeof(h));
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        k<<<1, 128, 32768>>>(d, c.lbo, c.sbo, c.n);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("BF16 MN lbo=%u sbo=%u N=%d err=%s\n", c.lbo, c.sbo, c.n, cudaGetErrorString(e));
        int nz = 0, bad = 0;
        for (int lane = 0; lane < 128; ++lane) {
            const int m = (lane & 15) + 16 * (lane >> 5);
            if ((lane & 31) >= 16) continue;
            ++nz;
            for (int cc = 0; cc < c.n; ++cc) {
                const int nn = c.n == 32 ? 32 + cc : cc;  // N = 32 with B start + 64 B -> B rows 32..63
                if (fabs(h[lane * 64 + cc] - ref[m][nn]) > 1e-3) ++bad;
            }
        }
        printf("  checked lanes %d, mismatches %d\n", nz, bad);
        printf("  nonzero lanes %d\n", nz);
    }
    return 0;
}
