// mimo_api.cu -- the C ABI of include/mimo.h: plan lifecycle, argument
// validation, kernel dispatch and the host-buffer end-to-end path.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "kernels.h"
#include "mimo.h"

namespace {

thread_local char g_last_error[512] = "";

struct DeviceGuard {
    int prev = -1;
    cudaError_t err;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool aligned(const void* p, size_t a) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int llr_bytes(int t) { return t == mimo::kLlrF32 ? 4 : t == mimo::kLlrF16 ? 2 : 1; }

}  // namespace

struct mimo_plan_s {
    mimo_plan_desc_t d{};
    cudaStream_t stream = nullptr;
    unsigned long long* d_fail = nullptr;
    const mimo::KernelEntry* fast = nullptr;
    char err[512] = "";
    // mimo_detect_mmse_host staging
    char* ws = nullptr;
    size_t ws_bytes = 0;
    static constexpr int kNB = 3;          // host path: buffer ring depth
    cudaStream_t hs[3] = {nullptr, nullptr, nullptr};  // H2D, kernels, D2H
    cudaEvent_t ev = nullptr;
    unsigned long long host_chunk = 0;  // host-path buffer ring position
    size_t host_bh = 0, host_by = 0, host_bd = 0, host_bl = 0;  // host-path buffer layout of the ring in use
    cudaEvent_t e_in[kNB] = {}, e_k[kNB] = {}, e_out[kNB] = {};
    // kernel workspaces: slot 0 for the plan's stream, 1..2 for the host path's streams
    void* kws[3] = {nullptr, nullptr, nullptr};
    size_t kws_bytes[3] = {0, 0, 0};
    // BFP y on shapes without the fused decode: the expanded complex64 y (mimo_detect_mmse_bfp)
    void* ydec = nullptr;
    size_t ydec_bytes = 0;
    // paper-literal LU route (mimo_detect_lmmse_lu)
    void* lu_ws = nullptr;
    size_t lu_ws_bytes = 0;
    cudaEvent_t lu_ev[MIMO_LU_STAGES + 1] = {};
};

namespace {

mimo_status_t cuda_fail(mimo_plan_t p, cudaError_t e, const char* what) {
    char* dst = p ? p->err : g_last_error;
    snprintf(dst, 512, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    if (p) snprintf(g_last_error, sizeof(g_last_error), "%s", p->err);
    return e == cudaErrorMemoryAllocation ? MIMO_ERR_OOM : MIMO_ERR_CUDA;
}

mimo_status_t arg_fail(mimo_plan_t p, const char* what) {
    char* dst = p ? p->err : g_last_error;
    snprintf(dst, 512, "invalid argument: %s", what);
    return MIMO_ERR_INVALID_ARG;
}

// The kernel specialisation serving the descriptor: the first table entry of the
// shape (the default), or the entry desc.kernel names. Sets *generic for
// desc.kernel == "generic"; returns nullptr with *unknown set for a name that
// no compiled entry of this shape carries.
const mimo::KernelEntry* select_fast(const mimo_plan_desc_t& d, bool* generic, bool* unknown) {
    using LF = const mimo::KernelEntry* (*)(int*);
    const LF tables[] = {mimo::tpu_entries, mimo::split_entries, mimo::lg_entries, mimo::c5_entries,
                         mimo::big_entries, mimo::prb_entries};
    const char* want = (d.kernel && *d.kernel) ? d.kernel : nullptr;
    *generic = want && strcmp(want, "generic") == 0;
    *unknown = false;
    if (*generic) return nullptr;
    for (LF f : tables) {
        int n = 0;
        const mimo::KernelEntry* t = f(&n);
        for (int i = 0; i < n; ++i)
            if (t[i].n_rx == d.n_rx && t[i].n_layers == d.n_layers && t[i].qm == d.qam_order &&
                t[i].sc_per_h == d.sc_per_h && t[i].sym_per_h == d.sym_per_h && t[i].llr_type == d.llr_type &&
                (!want || strcmp(want, t[i].name) == 0))
                return &t[i];
    }
    *unknown = want != nullptr;
    return nullptr;
}

// Device-pointer sanity check: reject host pointers and pointers on another
// device before a kernel could fault on them.
bool is_device_ptr(const void* p, int dev) {
    if (!p) return true;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) && at.device == dev;
}

mimo_status_t check_dims(mimo_plan_t p, float sigma2, int n_rx, int n_layers, int n_sc, int n_sym, int qm) {
    if (n_rx != p->d.n_rx || n_layers != p->d.n_layers || qm != p->d.qam_order)
        return arg_fail(p, "n_rx / n_layers / qam_order differ from the plan");
    if (n_sc < 0 || n_sym < 0) return arg_fail(p, "n_sc and n_sym must be >= 0");
    if (n_sc % p->d.sc_per_h) return arg_fail(p, "n_sc is not a multiple of sc_per_h");
    if (n_sym % p->d.sym_per_h) return arg_fail(p, "n_sym is not a multiple of sym_per_h");
    if (!(sigma2 >= 0.f) || !std::isfinite(sigma2)) return arg_fail(p, "sigma2 must be finite and >= 0");
    return MIMO_OK;
}

mimo::DetectArgs make_args(mimo_plan_t p, const void* H, const void* y, float sigma2, int n_sc, int n_sym,
                           void* llr, void* xhat, float* sinr) {
    mimo::DetectArgs a{};
    a.H = static_cast<const float2*>(H);
    a.y = static_cast<const float2*>(y);
    a.llr = llr;
    a.xhat = static_cast<float2*>(xhat);
    a.sinr = sinr;
    a.fail_count = p->d_fail;
    a.sigma2 = sigma2;
    a.llr_scale = p->d.llr_scale;
    a.n_rx = p->d.n_rx;
    a.n_layers = p->d.n_layers;
    a.qm = p->d.qam_order;
    a.n_sc = n_sc;
    a.n_sym = n_sym;
    a.sc_per_h = p->d.sc_per_h;
    a.sym_per_h = p->d.sym_per_h;
    a.n_fb = n_sc / p->d.sc_per_h;
    a.n_slots = n_sym / p->d.sym_per_h;
    a.n_units = (long long)a.n_fb * a.n_slots;
    a.llr_type = p->d.llr_type;
    a.overlap = (p->d.flags & MIMO_PLAN_OVERLAP_CALLS) ? 1 : 0;
    return a;
}

// Make sure workspace slot `slot` holds `need` bytes. Growing is refused while
// the stream is being captured (call mimo_plan_reserve before capturing).
mimo_status_t ensure_ws(mimo_plan_t p, int slot, size_t need, cudaStream_t s) {
    if (p->kws_bytes[slot] >= need) return MIMO_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (s) cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone)
        return arg_fail(p, "workspace too small while capturing a graph: call mimo_plan_reserve first");
    cudaError_t e = cudaSuccess;
    if (p->kws[slot]) {
        e = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        cudaFree(p->kws[slot]);
        p->kws[slot] = nullptr;
        p->kws_bytes[slot] = 0;
        if (e != cudaSuccess) return cuda_fail(p, e, "workspace resize");
    }
    e = cudaMalloc(&p->kws[slot], need);
    if (e != cudaSuccess) {
        p->kws[slot] = nullptr;
        return cuda_fail(p, e, "cudaMalloc(kernel workspace)");
    }
    p->kws_bytes[slot] = need;
    return MIMO_OK;
}

mimo_status_t launch(mimo_plan_t p, mimo::DetectArgs a, cudaStream_t s, int ws_slot = 0) {
    if (a.n_units == 0) return MIMO_OK;
    const mimo::KernelEntry* k = p->fast;
    if (k) {
        const size_t al = (size_t)k->align;
        if (!aligned(a.H, al) || !aligned(a.y, al) || !aligned(a.llr, al) || !aligned(a.xhat, al)) k = nullptr;
    }
    if (k && k->workspace) {
        mimo_status_t st = ensure_ws(p, ws_slot, k->workspace(a), s);
        if (st != MIMO_OK) return st;
        a.ws = p->kws[ws_slot];
    }
    cudaError_t e = k ? k->launch(a, s) : mimo::launch_generic(a, s);
    if (e != cudaSuccess) return cuda_fail(p, e, k ? k->name : "generic");
    return MIMO_OK;
}

}  // namespace

extern "C" {

int mimo_abi_version(void) { return MIMO_ABI_VERSION; }

const char* mimo_status_string(mimo_status_t s) {
    switch (s) {
    case MIMO_OK: return "MIMO_OK";
    case MIMO_ERR_INVALID_ARG: return "MIMO_ERR_INVALID_ARG: invalid argument";
    case MIMO_ERR_UNSUPPORTED: return "MIMO_ERR_UNSUPPORTED: no kernel for this shape";
    case MIMO_ERR_CUDA: return "MIMO_ERR_CUDA: CUDA runtime error";
    case MIMO_ERR_NOT_PD: return "MIMO_ERR_NOT_PD: Gram matrix not positive definite for >= 1 unit";
    case MIMO_ERR_OOM: return "MIMO_ERR_OOM: allocation failed";
    }
    return "unknown mimo_status_t";
}

const char* mimo_last_error(void) { return g_last_error; }

const char* mimo_plan_last_error(mimo_plan_t p) { return p ? p->err : ""; }

const char* mimo_plan_kernel_name(mimo_plan_t p) {
    if (!p) return "";
    return p->fast ? p->fast->name : "generic";
}

int mimo_plan_launches_per_call(mimo_plan_t p) {
    if (!p) return 0;
    return p->fast ? p->fast->launches : 1;
}

mimo_status_t mimo_plan_create(const mimo_plan_desc_t* desc, mimo_plan_t* out) {
    g_last_error[0] = 0;
    if (!desc || !out) return arg_fail(nullptr, "null descriptor or output");
    const mimo_plan_desc_t& d = *desc;
    if (d.n_rx < 1 || d.n_rx > mimo::kGenericMaxRx) return arg_fail(nullptr, "n_rx must be in 1..64");
    if (d.n_layers < 1 || d.n_layers > d.n_rx || d.n_layers > mimo::kGenericMaxLayers)
        return arg_fail(nullptr, "n_layers must be in 1..min(16, n_rx)");
    if (d.qam_order != 2 && d.qam_order != 4 && d.qam_order != 6 && d.qam_order != 8)
        return arg_fail(nullptr, "qam_order must be Qm in {2,4,6,8}");
    if (d.sc_per_h < 1 || d.sym_per_h < 1) return arg_fail(nullptr, "sc_per_h and sym_per_h must be >= 1");
    if (d.llr_type < 0 || d.llr_type > 2) return arg_fail(nullptr, "llr_type must be 0, 1 or 2");
    if (!(d.llr_scale > 0.f) || !std::isfinite(d.llr_scale)) return arg_fail(nullptr, "llr_scale must be finite > 0");
    if (d.device < 0) return arg_fail(nullptr, "device must be >= 0");
    if (d.flags & ~MIMO_PLAN_OVERLAP_CALLS) return arg_fail(nullptr, "unknown plan flags");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(nullptr, e, "cudaGetDeviceCount");
    }
    if (d.device >= ndev) return arg_fail(nullptr, "device ordinal out of range");
    DeviceGuard g(d.device);
    if (g.err != cudaSuccess) return cuda_fail(nullptr, g.err, "cudaSetDevice");

    mimo_plan_t p = new (std::nothrow) mimo_plan_s;
    if (!p) return MIMO_ERR_OOM;
    p->d = d;
    p->stream = static_cast<cudaStream_t>(d.stream);
    bool generic = false, unknown = false;
    p->fast = select_fast(d, &generic, &unknown);
    p->d.kernel = nullptr;  // the caller's string is not kept
    if (unknown) {
        snprintf(g_last_error, sizeof(g_last_error), "no compiled kernel named '%s' serves this shape", d.kernel);
        delete p;
        return MIMO_ERR_UNSUPPORTED;
    }
    if (d.host_chunk_bytes < 0) {
        delete p;
        return arg_fail(nullptr, "host_chunk_bytes must be >= 0");
    }
    if (p->fast && p->fast->prepare) {
        e = p->fast->prepare();
        if (e != cudaSuccess) {
            mimo_status_t st = cuda_fail(nullptr, e, "kernel prepare");
            delete p;
            return st;
        }
    }
    e = cudaMalloc(&p->d_fail, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(p->d_fail, 0, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        mimo_status_t st = cuda_fail(nullptr, e, "cudaMalloc(fail counter)");
        if (p->d_fail) cudaFree(p->d_fail);
        delete p;
        return st;
    }
    *out = p;
    return MIMO_OK;
}

mimo_status_t mimo_plan_set_stream(mimo_plan_t p, void* stream) {
    if (!p) return arg_fail(nullptr, "null plan");
    p->stream = static_cast<cudaStream_t>(stream);
    return MIMO_OK;
}

mimo_status_t mimo_detect_mmse_ex(mimo_plan_t p, const void* H, const void* y, float sigma2, int n_rx,
                                  int n_layers, int n_sc, int n_sym, int qm, void* llr_out, void* xhat_out,
                                  float* sinr_out) {
    if (!p) return arg_fail(nullptr, "null plan");
    mimo_status_t st = check_dims(p, sigma2, n_rx, n_layers, n_sc, n_sym, qm);
    if (st != MIMO_OK) return st;
    if ((long long)n_sc * n_sym == 0) return MIMO_OK;
    if (!H || !y) return arg_fail(p, "null H or y");
    if (!llr_out && !xhat_out && !sinr_out) return arg_fail(p, "no output requested");
    if (!aligned(H, 16) || !aligned(y, 16) || !aligned(llr_out, 16) || !aligned(xhat_out, 16) ||
        !aligned(sinr_out, 4))
        return arg_fail(p, "pointer not 16-byte aligned");
    const int dev = p->d.device;
    if (!is_device_ptr(H, dev) || !is_device_ptr(y, dev) || !is_device_ptr(llr_out, dev) ||
        !is_device_ptr(xhat_out, dev) || !is_device_ptr(sinr_out, dev))
        return arg_fail(p, "pointer is not device memory on the plan's device");
    DeviceGuard g(dev);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    mimo::DetectArgs a = make_args(p, H, y, sigma2, n_sc, n_sym, llr_out, xhat_out, sinr_out);
    return launch(p, a, p->stream);
}

mimo_status_t mimo_detect_mmse_sv(mimo_plan_t p, const void* H, const void* y, const float* sigma2_v, int n_rx,
                                  int n_layers, int n_sc, int n_sym, int qm, void* llr_out, void* xhat_out,
                                  float* sinr_out) {
    if (!p) return arg_fail(nullptr, "null plan");
    mimo_status_t st = check_dims(p, 1.0f, n_rx, n_layers, n_sc, n_sym, qm);
    if (st != MIMO_OK) return st;
    if ((long long)n_sc * n_sym == 0) return MIMO_OK;
    if (!sigma2_v) return arg_fail(p, "null sigma2_v");
    if (!aligned(sigma2_v, 4)) return arg_fail(p, "sigma2_v not 4-byte aligned");
    if (!is_device_ptr(sigma2_v, p->d.device)) return arg_fail(p, "sigma2_v is not device memory on the plan's device");
    if (!H || !y) return arg_fail(p, "null H or y");
    if (!llr_out && !xhat_out && !sinr_out) return arg_fail(p, "no output requested");
    if (!aligned(H, 16) || !aligned(y, 16) || !aligned(llr_out, 16) || !aligned(xhat_out, 16) ||
        !aligned(sinr_out, 4))
        return arg_fail(p, "pointer not 16-byte aligned");
    const int dev = p->d.device;
    if (!is_device_ptr(H, dev) || !is_device_ptr(y, dev) || !is_device_ptr(llr_out, dev) ||
        !is_device_ptr(xhat_out, dev) || !is_device_ptr(sinr_out, dev))
        return arg_fail(p, "pointer is not device memory on the plan's device");
    DeviceGuard g(dev);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    // the scalar sigma2 = 1 keeps every apply kernel on its sigma2 > 0 (non zero-forcing) path; the
    // setups read each unit's variance from sigma2_v (block_sigma2 in common.cuh)
    mimo::DetectArgs a = make_args(p, H, y, 1.0f, n_sc, n_sym, llr_out, xhat_out, sinr_out);
    a.sigma2_v = sigma2_v;
    return launch(p, a, p->stream);
}

mimo_status_t mimo_detect_mmse(mimo_plan_t p, const void* H, const void* y, float sigma2, int n_rx, int n_layers,
                               int n_sc, int n_sym, int qm, void* llr_out) {
    if (p && (long long)n_sc * n_sym > 0 && !llr_out) return arg_fail(p, "null llr_out");
    return mimo_detect_mmse_ex(p, H, y, sigma2, n_rx, n_layers, n_sc, n_sym, qm, llr_out, nullptr, nullptr);
}

// y as block floating point (mimo_detect_mmse_bfp_host*): iq_width = 0 means complex64 y.
struct BfpY {
    int iq_width = 0;
    float scale = 1.f;
};

static mimo_status_t host_path(mimo_plan_t p, const void* H_host, const void* y_host, float sigma2, int n_rx, int n_layers,
                        int n_sc, int n_sym, int qm, void* llr_host, bool wait, BfpY bfp = BfpY{}) {
    if (!p) return arg_fail(nullptr, "null plan");
    mimo_status_t st = check_dims(p, sigma2, n_rx, n_layers, n_sc, n_sym, qm);
    if (st != MIMO_OK) return st;
    // BFP y: decoded inside the apply loads (8 rx x 4 layers per PRB) or expanded by k_bfp_decode into
    // the chunk's complex64 y buffer (every other shape)
    bool bfp_fused = false;
    if (bfp.iq_width) {
        if (bfp.iq_width < 8 || bfp.iq_width > 16) return arg_fail(p, "iq_width must be in 8..16");
        if (!(bfp.scale > 0.f) || !std::isfinite(bfp.scale)) return arg_fail(p, "bfp_scale must be finite > 0");
        if (n_sc % 12) return arg_fail(p, "BFP y: n_sc must be a multiple of 12 (one block per PRB)");
        bfp_fused = mimo::bfp_supported(n_rx, n_layers, p->d.sc_per_h, p->d.sym_per_h);
    }
    if ((long long)n_sc * n_sym == 0) return MIMO_OK;
    if (!H_host || !y_host || !llr_host) return arg_fail(p, "null host buffer");
    DeviceGuard g(p->d.device);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");

    const int symph = p->d.sym_per_h;
    const int n_slots = n_sym / symph;
    const int n_fb = n_sc / p->d.sc_per_h;
    const size_t h_slot = (size_t)n_fb * n_rx * n_layers * 8;
    const size_t bfp_block = bfp.iq_width ? (size_t)((1 + 3 * bfp.iq_width + 3) & ~3) : 0;
    const size_t y_slot = bfp.iq_width ? (size_t)symph * (n_sc / 12) * n_rx * bfp_block
                                       : (size_t)symph * n_sc * n_rx * 8;
    const size_t l_slot = (size_t)symph * n_sc * n_layers * qm * llr_bytes(p->d.llr_type);
    // Chunks of whole slots, ~4 MiB of input each, on a 3-deep buffer ring over
    // three streams (H2D | kernels | D2H) so both PCIe directions and the
    // kernels run concurrently; events order buffer reuse.
    constexpr int NB = mimo_plan_s::kNB;
    // measured best on the B200 box for C2 (tools/e2e_chunks.py): 4 MiB for a synchronous call (its
    // own fill and drain are exposed), 16 MiB for a stream of asynchronous calls (they overlap)
    size_t chunk_bytes = p->d.host_chunk_bytes > 0 ? (size_t)p->d.host_chunk_bytes : wait ? (4u << 20) : (16u << 20);
    int cs = (int)(chunk_bytes / (h_slot + y_slot));
    if (cs < 1) cs = 1;
    if (cs > n_slots) cs = n_slots;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t bh = up(h_slot * cs), by = up(y_slot * cs), bl = up(l_slot * cs);
    const size_t bd = (bfp.iq_width && !bfp_fused) ? up((size_t)symph * n_sc * n_rx * 8 * cs) : 0;
    const size_t need = NB * (bh + by + bd + bl);
    cudaError_t e;
    for (int i = 0; i < 3; ++i)
        if (!p->hs[i] && (e = cudaStreamCreateWithFlags(&p->hs[i], cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(p, e, "cudaStreamCreate");
    if (!p->ev) {
        if ((e = cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(p, e, "cudaEventCreate");
        for (int i = 0; i < NB; ++i) {
            cudaEventCreateWithFlags(&p->e_in[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&p->e_k[i], cudaEventDisableTiming);
            if ((e = cudaEventCreateWithFlags(&p->e_out[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(p, e, "cudaEventCreate");
        }
    }
    // The ring position carries over between calls, so consecutive calls must share one buffer
    // layout: when it changes (other chunk size or call shape), drain every pending use of the
    // old layout and restart the ring before any buffer is reused (an earlier asynchronous call
    // may still be copying into / out of the region a new layout would overlap).
    if (bh != p->host_bh || by != p->host_by || bd != p->host_bd || bl != p->host_bl) {
        for (int i = 0; i < 3; ++i)
            if ((e = cudaStreamSynchronize(p->hs[i])) != cudaSuccess) return cuda_fail(p, e, "cudaStreamSynchronize");
        p->host_chunk = 0;
        p->host_bh = bh;
        p->host_by = by;
        p->host_bd = bd;
        p->host_bl = bl;
    }
    if (p->ws_bytes < need) {
        if (p->ws) {
            for (int i = 0; i < 3; ++i) cudaStreamSynchronize(p->hs[i]);
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_bytes = 0;
        }
        e = cudaMalloc(&p->ws, need);
        if (e != cudaSuccess) return cuda_fail(p, e, "cudaMalloc(host-path workspace)");
        p->ws_bytes = need;
    }
    // order after work already enqueued on the plan's stream
    if ((e = cudaEventRecord(p->ev, p->stream)) != cudaSuccess) return cuda_fail(p, e, "cudaEventRecord");
    for (int i = 0; i < 3; ++i) cudaStreamWaitEvent(p->hs[i], p->ev, 0);
    cudaStream_t s_in = p->hs[0], s_k = p->hs[1], s_out = p->hs[2];

    int chunk = 0;
    for (int s0 = 0; s0 < n_slots; s0 += cs, ++chunk) {
        const int ns = (n_slots - s0) < cs ? (n_slots - s0) : cs;
        const int b = (int)(p->host_chunk++ % NB);  // the ring continues across (asynchronous) calls
        char* base = p->ws + (size_t)b * (bh + by + bd + bl);
        char *dH = base, *dy = base + bh, *dd = base + bh + by, *dl = base + bh + by + bd;
        // buffer b's previous use (this call's chunk - NB, or a previous asynchronous call's chunk) is
        // over: its inputs consumed / its outputs drained (waiting on a never-recorded event is a no-op)
        cudaStreamWaitEvent(s_in, p->e_k[b], 0);
        e = cudaMemcpyAsync(dH, (const char*)H_host + h_slot * s0, h_slot * ns, cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dy, (const char*)y_host + y_slot * s0, y_slot * ns, cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaEventRecord(p->e_in[b], s_in);
        if (e != cudaSuccess) return cuda_fail(p, e, "cudaMemcpyAsync H2D");
        cudaStreamWaitEvent(s_k, p->e_in[b], 0);
        cudaStreamWaitEvent(s_k, p->e_out[b], 0);
        mimo::DetectArgs a = make_args(p, dH, !bfp.iq_width ? dy : bfp_fused ? nullptr : dd, sigma2, n_sc, ns * symph,
                                       dl, nullptr, nullptr);
        a.overlap = 0;
        if (bfp.iq_width && !bfp_fused) {
            if ((e = mimo::launch_bfp_decode(dy, reinterpret_cast<float2*>(dd), n_rx, n_sc, ns * symph, bfp.iq_width,
                                             bfp.scale, s_k)) != cudaSuccess)
                return cuda_fail(p, e, "BFP decode");
            st = launch(p, a, s_k, 1);
            if (st != MIMO_OK) return st;
        } else if (bfp.iq_width) {
            st = ensure_ws(p, 1, mimo::bfp_workspace(a), s_k);
            if (st != MIMO_OK) return st;
            a.ws = p->kws[1];
            if ((e = mimo::launch_bfp(a, dy, bfp.iq_width, bfp.scale, s_k)) != cudaSuccess) return cuda_fail(p, e, "BFP route");
        } else {
            st = launch(p, a, s_k, 1);
            if (st != MIMO_OK) return st;
        }
        if ((e = cudaEventRecord(p->e_k[b], s_k)) != cudaSuccess) return cuda_fail(p, e, "cudaEventRecord");
        cudaStreamWaitEvent(s_out, p->e_k[b], 0);
        e = cudaMemcpyAsync((char*)llr_host + l_slot * s0, dl, l_slot * ns, cudaMemcpyDeviceToHost, s_out);
        if (e == cudaSuccess) e = cudaEventRecord(p->e_out[b], s_out);
        if (e != cudaSuccess) return cuda_fail(p, e, "cudaMemcpyAsync D2H");
    }
    // asynchronous form: mimo_plan_sync_status synchronises the host-path streams. No join into the
    // plan's stream -- the next call orders after that stream's tail, and a join there would
    // serialise consecutive calls (no H2D of call i+1 under the D2H of call i)
    if (!wait) return MIMO_OK;
    for (int i = 0; i < 3; ++i)
        if ((e = cudaStreamSynchronize(p->hs[i])) != cudaSuccess) return cuda_fail(p, e, "cudaStreamSynchronize");
    return MIMO_OK;
}

mimo_status_t mimo_detect_mmse_host(mimo_plan_t p, const void* H_host, const void* y_host, float sigma2, int n_rx,
                                    int n_layers, int n_sc, int n_sym, int qm, void* llr_host) {
    return host_path(p, H_host, y_host, sigma2, n_rx, n_layers, n_sc, n_sym, qm, llr_host, true);
}

mimo_status_t mimo_detect_mmse_host_async(mimo_plan_t p, const void* H_host, const void* y_host, float sigma2,
                                          int n_rx, int n_layers, int n_sc, int n_sym, int qm, void* llr_host) {
    return host_path(p, H_host, y_host, sigma2, n_rx, n_layers, n_sc, n_sym, qm, llr_host, false);
}

mimo_status_t mimo_detect_mmse_bfp_host(mimo_plan_t p, const void* H_host, const void* y_bfp_host, float sigma2,
                                        int n_rx, int n_layers, int n_sc, int n_sym, int qm, int iq_width,
                                        float bfp_scale, void* llr_host) {
    return host_path(p, H_host, y_bfp_host, sigma2, n_rx, n_layers, n_sc, n_sym, qm, llr_host, true,
                     BfpY{iq_width, bfp_scale});
}

mimo_status_t mimo_detect_mmse_bfp_host_async(mimo_plan_t p, const void* H_host, const void* y_bfp_host, float sigma2,
                                              int n_rx, int n_layers, int n_sc, int n_sym, int qm, int iq_width,
                                              float bfp_scale, void* llr_host) {
    return host_path(p, H_host, y_bfp_host, sigma2, n_rx, n_layers, n_sc, n_sym, qm, llr_host, false,
                     BfpY{iq_width, bfp_scale});
}

mimo_status_t mimo_detect_lmmse_lu(mimo_plan_t p, const void* H, const void* y, float sigma2, int n_rx,
                                   int n_layers, int n_sc, int n_sym, int qm, int precision_bits, void* llr_out,
                                   void* xhat_out, float* sinr_out, float* stage_us) {
    if (!p) return arg_fail(nullptr, "null plan");
    if (precision_bits != 32 && precision_bits != 64) return arg_fail(p, "precision_bits must be 32 or 64");
    mimo_status_t st = check_dims(p, sigma2, n_rx, n_layers, n_sc, n_sym, qm);
    if (st != MIMO_OK) return st;
    if (!mimo::lu_route_supported(n_rx)) {
        snprintf(p->err, sizeof(p->err), "LU route: n_rx must be 1, 2, 4, 8 or 16");
        return MIMO_ERR_UNSUPPORTED;
    }
    if (stage_us)
        for (int i = 0; i < MIMO_LU_STAGES; ++i) stage_us[i] = 0.f;
    if ((long long)n_sc * n_sym == 0) return MIMO_OK;
    if (!H || !y) return arg_fail(p, "null H or y");
    if (!llr_out && !xhat_out && !sinr_out) return arg_fail(p, "no output requested");
    if (!aligned(H, 16) || !aligned(y, 16) || !aligned(llr_out, 16) || !aligned(xhat_out, 16) ||
        !aligned(sinr_out, 4))
        return arg_fail(p, "pointer not 16-byte aligned");
    const int dev = p->d.device;
    if (!is_device_ptr(H, dev) || !is_device_ptr(y, dev) || !is_device_ptr(llr_out, dev) ||
        !is_device_ptr(xhat_out, dev) || !is_device_ptr(sinr_out, dev))
        return arg_fail(p, "pointer is not device memory on the plan's device");
    DeviceGuard g(dev);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    mimo::DetectArgs a = make_args(p, H, y, sigma2, n_sc, n_sym, llr_out, xhat_out, sinr_out);
    a.overlap = 0;
    const size_t need = mimo::lu_route_workspace(n_rx, a.n_units, precision_bits);
    cudaError_t e;
    if (p->lu_ws_bytes < need) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (p->stream) cudaStreamIsCapturing(p->stream, &cs);
        if (cs != cudaStreamCaptureStatusNone) return arg_fail(p, "LU workspace must grow while capturing a graph");
        if (p->lu_ws) {
            cudaStreamSynchronize(p->stream);
            cudaFree(p->lu_ws);
            p->lu_ws = nullptr;
            p->lu_ws_bytes = 0;
        }
        if ((e = cudaMalloc(&p->lu_ws, need)) != cudaSuccess) {
            p->lu_ws = nullptr;
            return cuda_fail(p, e, "cudaMalloc(LU workspace)");
        }
        p->lu_ws_bytes = need;
    }
    a.ws = p->lu_ws;
    cudaEvent_t* ev = nullptr;
    if (stage_us) {
        for (int i = 0; i <= MIMO_LU_STAGES; ++i)
            if (!p->lu_ev[i] && (e = cudaEventCreate(&p->lu_ev[i])) != cudaSuccess)
                return cuda_fail(p, e, "cudaEventCreate");
        ev = p->lu_ev;
    }
    if ((e = mimo::launch_lu_route(a, precision_bits, p->stream, ev)) != cudaSuccess)
        return cuda_fail(p, e, "LU route");
    if (stage_us) {
        if ((e = cudaEventSynchronize(ev[MIMO_LU_STAGES])) != cudaSuccess) return cuda_fail(p, e, "LU route sync");
        for (int i = 0; i < MIMO_LU_STAGES; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            stage_us[i] = ms * 1000.f;
        }
    }
    return MIMO_OK;
}

mimo_status_t mimo_detect_irc(mimo_plan_t p, const void* H, const void* y, const void* Rnn, int n_rx, int n_layers,
                              int n_sc, int n_sym, int qm, void* llr_out, void* xhat_out, float* sinr_out) {
    if (!p) return arg_fail(nullptr, "null plan");
    mimo_status_t st = check_dims(p, 1.0f, n_rx, n_layers, n_sc, n_sym, qm);
    if (st != MIMO_OK) return st;
    if (!mimo::irc_supported(n_rx, n_layers)) {
        snprintf(p->err, sizeof(p->err), "IRC route: n_rx must be <= 16");
        return MIMO_ERR_UNSUPPORTED;
    }
    if ((long long)n_sc * n_sym == 0) return MIMO_OK;
    if (!H || !y || !Rnn) return arg_fail(p, "null H, y or Rnn");
    if (!llr_out && !xhat_out && !sinr_out) return arg_fail(p, "no output requested");
    if (!aligned(H, 8) || !aligned(y, 8) || !aligned(Rnn, 8) || !aligned(llr_out, 8) || !aligned(xhat_out, 8) ||
        !aligned(sinr_out, 4))
        return arg_fail(p, "pointer not 8-byte aligned");
    const int dev = p->d.device;
    if (!is_device_ptr(H, dev) || !is_device_ptr(y, dev) || !is_device_ptr(Rnn, dev) ||
        !is_device_ptr(llr_out, dev) || !is_device_ptr(xhat_out, dev) || !is_device_ptr(sinr_out, dev))
        return arg_fail(p, "pointer is not device memory on the plan's device");
    DeviceGuard g(dev);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    mimo::DetectArgs a = make_args(p, H, y, 1.0f, n_sc, n_sym, llr_out, xhat_out, sinr_out);
    a.overlap = 0;
    cudaError_t e = mimo::launch_irc(a, static_cast<const float2*>(Rnn), p->stream);
    if (e != cudaSuccess) return cuda_fail(p, e, "IRC route");
    return MIMO_OK;
}

mimo_status_t mimo_detect_mmse_bfp(mimo_plan_t p, const void* H, const void* y_bfp, float sigma2, int n_rx,
                                   int n_layers, int n_sc, int n_sym, int qm, int iq_width, float bfp_scale,
                                   void* llr_out, void* xhat_out, float* sinr_out) {
    if (!p) return arg_fail(nullptr, "null plan");
    mimo_status_t st = check_dims(p, sigma2, n_rx, n_layers, n_sc, n_sym, qm);
    if (st != MIMO_OK) return st;
    if (iq_width < 8 || iq_width > 16) return arg_fail(p, "iq_width must be in 8..16");
    if (!(bfp_scale > 0.f) || !std::isfinite(bfp_scale)) return arg_fail(p, "bfp_scale must be finite > 0");
    if (n_sc % 12) return arg_fail(p, "BFP y: n_sc must be a multiple of 12 (one block per PRB)");
    const bool fused = mimo::bfp_supported(n_rx, n_layers, p->d.sc_per_h, p->d.sym_per_h);
    if ((long long)n_sc * n_sym == 0) return MIMO_OK;
    if (!H || !y_bfp) return arg_fail(p, "null H or y_bfp");
    if (!llr_out && !xhat_out && !sinr_out) return arg_fail(p, "no output requested");
    if (!aligned(H, 32) || !aligned(y_bfp, 16) || !aligned(llr_out, 16) || !aligned(xhat_out, 16) ||
        !aligned(sinr_out, 4))
        return arg_fail(p, "pointer misaligned (H 32 B, y_bfp 16 B, outputs 16 B)");
    const int dev = p->d.device;
    if (!is_device_ptr(H, dev) || !is_device_ptr(y_bfp, dev) || !is_device_ptr(llr_out, dev) ||
        !is_device_ptr(xhat_out, dev) || !is_device_ptr(sinr_out, dev))
        return arg_fail(p, "pointer is not device memory on the plan's device");
    DeviceGuard g(dev);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    if (!fused) {  // expand into the plan's complex64 y buffer, then the shape's detector
        const size_t need = (size_t)n_sym * n_sc * n_rx * 8;
        if (p->ydec_bytes < need) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (p->stream) cudaStreamIsCapturing(p->stream, &cs);
            if (cs != cudaStreamCaptureStatusNone)
                return arg_fail(p, "BFP y buffer too small while capturing a graph: make one call before capturing");
            cudaError_t e = cudaStreamSynchronize(p->stream);
            if (e != cudaSuccess) return cuda_fail(p, e, "cudaStreamSynchronize");
            cudaFree(p->ydec);
            p->ydec = nullptr;
            p->ydec_bytes = 0;
            if ((e = cudaMalloc(&p->ydec, need)) != cudaSuccess) return cuda_fail(p, e, "cudaMalloc(BFP y buffer)");
            p->ydec_bytes = need;
        }
        cudaError_t e = mimo::launch_bfp_decode(y_bfp, static_cast<float2*>(p->ydec), n_rx, n_sc, n_sym, iq_width,
                                                bfp_scale, p->stream);
        if (e != cudaSuccess) return cuda_fail(p, e, "BFP decode");
        return launch(p, make_args(p, H, p->ydec, sigma2, n_sc, n_sym, llr_out, xhat_out, sinr_out), p->stream);
    }
    mimo::DetectArgs a = make_args(p, H, nullptr, sigma2, n_sc, n_sym, llr_out, xhat_out, sinr_out);
    st = ensure_ws(p, 0, mimo::bfp_workspace(a), p->stream);
    if (st != MIMO_OK) return st;
    a.ws = p->kws[0];
    cudaError_t e = mimo::launch_bfp(a, y_bfp, iq_width, bfp_scale, p->stream);
    if (e != cudaSuccess) return cuda_fail(p, e, "BFP route");
    return MIMO_OK;
}

mimo_status_t mimo_plan_reserve(mimo_plan_t p, int n_sc, int n_sym) {
    if (!p) return arg_fail(nullptr, "null plan");
    if (n_sc < 0 || n_sym < 0 || n_sc % p->d.sc_per_h || n_sym % p->d.sym_per_h)
        return arg_fail(p, "n_sc / n_sym not multiples of sc_per_h / sym_per_h");
    const mimo::KernelEntry* k = p->fast;
    if (!k || !k->workspace) return MIMO_OK;
    DeviceGuard g(p->d.device);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    mimo::DetectArgs a = make_args(p, nullptr, nullptr, 0.f, n_sc, n_sym, nullptr, nullptr, nullptr);
    return ensure_ws(p, 0, k->workspace(a), p->stream);
}

mimo_status_t mimo_plan_sync_status(mimo_plan_t p, long long* n_failed) {
    if (n_failed) *n_failed = 0;
    if (!p) return arg_fail(nullptr, "null plan");
    DeviceGuard g(p->d.device);
    if (g.err != cudaSuccess) return cuda_fail(p, g.err, "cudaSetDevice");
    unsigned long long h = 0;
    cudaError_t e = cudaStreamSynchronize(p->stream);
    for (int i = 0; i < 3 && e == cudaSuccess; ++i)
        if (p->hs[i]) e = cudaStreamSynchronize(p->hs[i]);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, p->d_fail, sizeof(h), cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->d_fail, 0, sizeof(h), p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    if (e != cudaSuccess) return cuda_fail(p, e, "sync_status");
    if (n_failed) *n_failed = (long long)h;
    return h ? MIMO_ERR_NOT_PD : MIMO_OK;
}

mimo_status_t mimo_plan_destroy(mimo_plan_t p) {
    if (!p) return MIMO_OK;
    {
        DeviceGuard g(p->d.device);
        cudaStreamSynchronize(p->stream);
        for (int i = 0; i < 3; ++i)
            if (p->hs[i]) {
                cudaStreamSynchronize(p->hs[i]);
                cudaStreamDestroy(p->hs[i]);
            }
        if (p->ev) cudaEventDestroy(p->ev);
        for (int i = 0; i < mimo_plan_s::kNB; ++i) {
            if (p->e_in[i]) cudaEventDestroy(p->e_in[i]);
            if (p->e_k[i]) cudaEventDestroy(p->e_k[i]);
            if (p->e_out[i]) cudaEventDestroy(p->e_out[i]);
        }
        if (p->ws) cudaFree(p->ws);
        if (p->lu_ws) cudaFree(p->lu_ws);
        if (p->ydec) cudaFree(p->ydec);
        for (int i = 0; i <= MIMO_LU_STAGES; ++i)
            if (p->lu_ev[i]) cudaEventDestroy(p->lu_ev[i]);
        for (int i = 0; i < 3; ++i)
            if (p->kws[i]) cudaFree(p->kws[i]);
        if (p->d_fail) cudaFree(p->d_fail);
    }
    delete p;
    return MIMO_OK;
}

}  // extern "C"
