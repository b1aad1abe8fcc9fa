// kernels.h -- internal registry of the detector kernels (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace mimo {

using LaunchFn = cudaError_t (*)(const DetectArgs&, cudaStream_t);

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute when
// `pdl` is set (the kernel must use pdl_launch_dependents / pdl_wait).
template <typename K>
inline cudaError_t launch_kernel(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, int pdl,
                                 const DetectArgs& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

// A specialised kernel serves exactly one (n_rx, n_layers, qm, sc_per_h,
// sym_per_h, llr_type) tuple; `align` is the byte alignment it needs of H, y,
// llr and xhat (else the dispatcher falls back to the generic kernel).
struct KernelEntry {
    const char* name;
    int n_rx, n_layers, qm, sc_per_h, sym_per_h, llr_type;
    int align;
    int launches;
    LaunchFn launch;
    // Optional: configure function attributes once at plan creation.
    cudaError_t (*prepare)();
    // Optional: bytes of plan-owned workspace one call needs (DetectArgs::ws).
    size_t (*workspace)(const DetectArgs&);
};

// Tables provided by each kernel family (k_*.cu).
const KernelEntry* tpu_entries(int* n);
const KernelEntry* prb_entries(int* n);
const KernelEntry* split_entries(int* n);
const KernelEntry* lg_entries(int* n);
const KernelEntry* big_entries(int* n);
const KernelEntry* c5_entries(int* n);

// Generic kernel: any n_rx <= 64, n_layers <= min(16, n_rx), qm, sc_per_h,
// sym_per_h, llr_type; 8-byte alignment.
cudaError_t launch_generic(const DetectArgs& a, cudaStream_t s);
constexpr int kGenericMaxRx = 64;

// Paper-literal covariance/LU route (k_lu.cu): five
// stage kernels over a workspace of lu_route_workspace() bytes (DetectArgs::ws).
// precision_bits 32 ("PS") or 64 ("PD"); ev (nullable) = 6 events recorded
// before stage 0 and after each stage.
bool lu_route_supported(int n_rx);
// Coloured-noise (interference-rejection) detector (k_irc.cu): Rnn device complex64 [n_units][n_rx][n_rx].
bool irc_supported(int n_rx, int n_layers);
// BFP-compressed y, fused decompression (k_split.cu; C3 family: 8 x 4, H per PRB).
bool bfp_supported(int n_rx, int n_layers, int sc_per_h, int sym_per_h);
size_t bfp_workspace(const DetectArgs& a);
cudaError_t launch_bfp(const DetectArgs& a, const void* y_bfp, int iq_width, float scale, cudaStream_t s);
// Any shape: BFP blocks [n_sym][n_sc/12][n_rx][block] -> complex64 y [n_sym][n_sc][n_rx] (k_bfp.cu).
cudaError_t launch_bfp_decode(const void* y_bfp, float2* y, int n_rx, int n_sc, int n_sym, int iq_width, float scale,
                              cudaStream_t s);
cudaError_t launch_irc(const DetectArgs& a, const float2* Rnn, cudaStream_t s);
size_t lu_route_workspace(int n_rx, long long n_units, int precision_bits);
cudaError_t launch_lu_route(const DetectArgs& a, int precision_bits, cudaStream_t s, cudaEvent_t* ev);
constexpr int kGenericMaxLayers = 16;

}  // namespace mimo
