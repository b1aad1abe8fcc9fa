// tools/tmabench.cu -- read throughput of the C5 y access patterns (not part of libmimo.so).
// y viewed as [n_sym = 560][n_sc = 3276][128 floats] (939 MB); one "unit" = 14 symbols x 12
// subcarriers x 512 B. Persistent kernel, one CTA (one issuing thread) per SM, units
// round-robin over CTAs, a ring of stages consumed as soon as they land:
//   mode 0: 4 tensor boxes {32 floats, 12, 14} SWIZZLE_128B per unit (k_big_apply4's chunks)
//   mode 1: 1 tensor box {128 floats, 12, 14} SWIZZLE_NONE per unit (86 KiB)
//   mode 2: 168 bulk copies of 512 B per unit (cp.async.bulk, one per RE row)
//   mode 3: 14 bulk copies of 6 KiB per unit (one per symbol: 12 contiguous RE rows)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tmabench tools/tmabench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(s32(b)),
                 "r"(ph) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* b) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(s32(b)) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(n), "r"(s32(b)) : "memory");
}

constexpr int NSC = 3276, NSYM = 560, NFB = NSC / 12, NSLOT = NSYM / 14, NUNIT = NFB * NSLOT;
constexpr uint32_t UNIT = 168 * 512;

__global__ void bench(const float* y, const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                      int mode, int S, uint32_t* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[16];
    if (threadIdx.x != 0) return;
    const uint32_t base = (s32(sm) + 1023u) & ~1023u;
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    // items: mode 0 -> 4 per unit (chunks), else 1 per unit
    const int per = mode == 0 ? 4 : 1;
    const long long n_my = (NUNIT - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const long long G = n_my * per;
    const uint32_t stage = mode == 0 ? 21504u : UNIT;
    auto issue = [&](long long g) {
        const int st = (int)(g % S);
        const long long u = blockIdx.x + (g / per) * gridDim.x;
        const int slot = (int)(u / NFB), fb = (int)(u % NFB);
        uint64_t* b = &bar[st];
        const uint32_t dst = base + st * stage;
        if (mode == 0) {
            expect(b, 21504u);
            tma3(dst, &m0, 32 * (int)(g % 4), fb * 12, slot * 14, b);
        } else if (mode == 1) {
            expect(b, UNIT);
            tma3(dst, &m1, 0, fb * 12, slot * 14, b);
        } else if (mode == 2) {
            expect(b, UNIT);
            for (int r = 0; r < 168; ++r)
                bulk(dst + r * 512, y + ((size_t)(slot * 14 + r / 12) * NSC + fb * 12 + r % 12) * 128, 512, b);
        } else {
            expect(b, UNIT);
            for (int s = 0; s < 14; ++s)
                bulk(dst + s * 6144, y + ((size_t)(slot * 14 + s) * NSC + fb * 12) * 128, 6144, b);
        }
    };
    for (long long g = 0; g < S && g < G; ++g) issue(g);
    uint32_t acc = 0;
    for (long long g = 0; g < G; ++g) {
        const int st = (int)(g % S);
        wait(&bar[st], (uint32_t)((g / S) & 1));
        acc ^= *(volatile uint32_t*)(sm + (base - s32(sm)) + st * stage);
        if (g + S < G) issue(g + S);
    }
    if (acc == 0x1234567u) sink[0] = acc;
}

int main() {
    const size_t bytes = (size_t)NSYM * NSC * 512;
    float* y;
    uint32_t* sink;
    cudaMalloc(&y, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(y, 0, bytes);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m0, m1;
    const cuuint64_t gdim[3] = {128, NSC, NSYM};
    const cuuint64_t gstride[2] = {512, (cuuint64_t)NSC * 512};
    const cuuint32_t box0[3] = {32, 12, 14}, box1[3] = {128, 12, 14}, es[3] = {1, 1, 1};
    enc(&m0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, y, gdim, gstride, box0, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r1 = enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, y, gdim, gstride, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box {128,12,14} no-swizzle encode: %d\n", (int)r1);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { int mode, S; const char* name; } cfgs[] = {
        {0, 4, "4 x SW128 boxes {32,12,14}, 4 stages (86 KB)"},
        {0, 8, "4 x SW128 boxes {32,12,14}, 8 stages (172 KB)"},
        {1, 2, "1 x box {128,12,14} no swizzle, 2 stages"},
        {2, 2, "168 x 512 B bulk copies, 2 stages"},
        {3, 2, "14 x 6 KB bulk copies, 2 stages"},
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto& c : cfgs) {
        if (c.mode == 1 && r1 != CUDA_SUCCESS) continue;
        const size_t smem = (c.mode == 0 ? 21504u : UNIT) * c.S + 1024;
        for (int it = 0; it < 2; ++it) bench<<<148, 32, smem>>>(y, m0, m1, c.mode, c.S, sink);
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) bench<<<148, 32, smem>>>(y, m0, m1, c.mode, c.S, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-50s %8.1f us  %7.1f GB/s  (%s)\n", c.name, ms * 1000 / 5, bytes / (ms / 5 * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
