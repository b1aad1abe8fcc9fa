// tools/tcbench.cu -- tcgen05 kind::tf32 issue/completion timing (M=128, K=8, N in {32,64,128}).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tcbench tools/tcbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int N, int F16 = 0, int TA = 0, int M = 128, int ND = 1>
__global__ void k(int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = F16 ? ((1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24))
                               : ((1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | (((uint32_t)M >> 4) << 24));
    const uint32_t a = su32(sm), b = su32(sm + 65536);
    const uint64_t da0 = desc(a), db0 = desc(b);
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 96; ++kk) {
                // advance the 14-bit start-address field (16-byte units) of precomputed descriptors
                const uint64_t da = da0 + (uint64_t)((kk & 3) * 2 + (kk >> 2) * 64), db = db0 + (uint64_t)((kk & 3) * 2);
                const uint32_t dcol = tb + (uint32_t)((kk % ND) * (TA ? 0 : N));  // ND distinct accumulators
                if (TA)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(tb + (uint32_t)((kk % ND) * 32)), "r"(tb + 128u + 8u * (kk & 3)), "l"(db), "r"(idesc), "r"(kk));
                else if (F16)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tb), "l"(da), "l"(db), "r"(idesc), "r"(kk));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(dcol), "l"(da), "l"(db), "r"(idesc), "r"(kk));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                             : "=r"(ok) : "r"(su32(&bar)), "r"(it & 1));
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    long long h[148];
    for (int n : {32, 64, 128, 32, -32, -64, -128, 1032, 1064, 1128, 2032, 2064, 3032, 3064, 4032, 4064, 5032, 5064}) {
        auto f = n == 32 ? k<32> : n == 64 ? k<64> : n == 128 ? k<128> : n == -32 ? k<32, 1> : n == -64 ? k<64, 1>
               : n == -128 ? k<128, 1> : n == 1032 ? k<32, 0, 1> : n == 1064 ? k<64, 0, 1> : n == 1128 ? k<128, 0, 1>
               : n == 2032 ? k<32, 0, 1, 64> : n == 2064 ? k<64, 0, 1, 64> : n == 3032 ? k<32, 0, 0, 64>
               : n == 3064 ? k<64, 0, 0, 64> : n == 4032 ? k<32, 0, 0, 128, 2> : n == 4064 ? k<64, 0, 0, 128, 2>
               : n == 5032 ? k<32, 0, 1, 128, 2> : k<64, 0, 1, 128, 2>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
        f<<<148, 128, 140 * 1024>>>(10, d);
        cudaDeviceSynchronize();
        f<<<148, 128, 140 * 1024>>>(200, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
        printf("%s N=%3d: %s  %.1f cycles per 96-MMA batch (%.2f per MMA)\n", n < 0 ? "f16 " : n > 5000 ? "tf32 A-in-TMEM 2 acc" : n > 4000 ? "tf32 SS 2 acc" : n > 3000 ? "tf32 M=64 SS" : n > 2000 ? "tf32 M=64 A-in-TMEM" : n > 1000 ? "tf32 A-in-TMEM" : "tf32",
               n < 0 ? -n : n % 1000, cudaGetErrorString(e), h[0] / 200.0,
               h[0] / 200.0 / 96);
    }
    return 0;
}
