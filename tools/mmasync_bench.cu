// mmasync_bench.cu -- throughput of the legacy warp-level tensor path (mma.sync) on sm_100a:
// tf32 m16n8k8 and bf16 m16n8k16, independent accumulator chains, full occupancy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mmasync_bench tools/mmasync_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(256) k_mma(float* out, int iters) {
    float c[4][4] = {};
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + threadIdx.x * 1e-3f + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (KIND == 0)
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0.f;
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) s += c[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters) {
    float c[8];
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i;
    const float a = 1.0001f, b = 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) c[i] = fmaf(c[i], a, b);
    }
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, n_sm = 0, clk = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = n_sm * 8, threads = 256, iters = 4096;
    float* out;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, void (*k)(float*, int), double mac_per_warp_iter) {
        k<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double macs = mac_per_warp_iter * iters * blocks * (threads / 32);
        const double per_clk_sm = macs / (ms * 1e-3) / n_sm / (clk * 1e3);
        printf("%-24s %8.3f ms  %8.1f TMAC/s  %7.1f MAC/clk/SM (at %d MHz max)  %s\n", name, ms,
               macs / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000, cudaGetErrorString(cudaGetLastError()));
    };
    run("mma.sync tf32 m16n8k8", k_mma<0>, 4.0 * 16 * 8 * 8);
    run("mma.sync bf16 m16n8k16", k_mma<1>, 4.0 * 16 * 8 * 16);
    run("FFMA (fp32 SIMT)", k_ffma, 16.0 * 8 * 32);
    return 0;
}
