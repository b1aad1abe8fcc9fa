/*
 * mimo.h -- C ABI of the B200-native per-RE linear-MMSE MIMO detector and
 * max-log soft demapper (hot path of arxiv 2510.07843, "Accelerating vRAN and
 * O-RAN with SIMD", BASELINE.json north_star).
 *
 * The operation (§IV; Fig. 4 caption PAPER.md:93): for every
 * resource element (RE) = (OFDM symbol, subcarrier) of a slot, detect the
 * n_layers transmitted symbols from the n_rx received samples y with the LMMSE
 * filter, "which involves inverting the received signal covariance matrix R".
 * This library computes, per H-unit (one channel H shared by sym_per_h
 * symbols x sc_per_h subcarriers; "one weight matrix per subcarrier per slot",
 * SPEC.md:440):
 *   a2  G = H^H H + sigma2 I                         (Gram form of R; reading R1)
 *   a3  G = L L^H (Cholesky)                         (replaces the paper's LU; reading R2)
 *   a4  A_kk = [G^-1]_kk,  W = G^-1 H^H = L^-H L^-1 H^H   (forward/backward substitution)
 *   a5  mu_k = 1 - sigma2 A_kk,  SINR_k = 1/(sigma2 A_kk) - 1,  W~ = diag(1/mu) W   (readings R3, R4)
 * and per RE:
 *   a6  x~ = W~ y                                    (unbiased LMMSE estimate)
 *   a7  exact max-log LLRs of the 38.211 Gray QAM labels (readings R5, R6):
 *       LLR(b) = SINR_k * (min_{s: b=1} |x~_k - s|^2 - min_{s: b=0} |x~_k - s|^2) * llr_scale,
 *       > 0 means bit 0; quantised to fp32 / fp16 / int8 (reading R10).
 * Everything runs in hand-written sm_100a CUDA kernels; there is no CPU path.
 *
 * LAYOUTS (all row-major, complex = interleaved (re, im) float32 = complex64):
 *   H        [n_sym/sym_per_h][n_sc/sc_per_h][n_rx][n_layers]  complex64 (row = rx antenna)
 *   y        [n_sym][n_sc][n_rx]                               complex64
 *   llr_out  [n_sym][n_sc][n_layers][qam_order]                llr_type; bit j = b_j of 38.211
 *   xhat_out [n_sym][n_sc][n_layers]                           complex64 (unbiased x~; optional)
 *   sinr_out [n_units][n_layers]                               float32   (optional)
 * with n_units = (n_sym/sym_per_h) * (n_sc/sc_per_h), unit u = slot * n_fb + fb.
 *
 * OWNERSHIP: the caller owns every data buffer. A plan owns only its failure
 * counter and (for mimo_detect_mmse_host) a device staging workspace. A plan
 * must outlive all work it enqueued; mimo_plan_destroy synchronises first.
 *
 * ERRORS: no call throws. Argument problems are detected synchronously and
 * return MIMO_ERR_INVALID_ARG without enqueuing anything. Kernel-side numerical
 * failures (a Cholesky pivot p_j <= 16 * 2^-24 * max_i G_ii, or NaN; reading
 * R17) never abort: the unit's outputs are written as erasures (LLR 0, x~ 0,
 * SINR 0) and counted; mimo_plan_sync_status reports them as MIMO_ERR_NOT_PD.
 *
 * THREADING: a plan is not thread-safe; use one plan per (host thread, device).
 * DETERMINISM: outputs are bitwise reproducible for identical inputs and plan
 * (no floating-point atomics; fixed reduction order).
 */
#ifndef MIMO_H
#define MIMO_H

#ifdef __cplusplus
extern "C" {
#endif

#define MIMO_ABI_VERSION 2

typedef struct mimo_plan_s* mimo_plan_t;

typedef enum {
    MIMO_OK = 0,
    MIMO_ERR_INVALID_ARG = 1, /* null / misaligned pointer, bad dims, dims != plan, sigma2 < 0 or NaN */
    MIMO_ERR_UNSUPPORTED = 2, /* shape or modulation with no compiled kernel */
    MIMO_ERR_CUDA = 3,        /* CUDA runtime error; text via mimo_plan_last_error / mimo_last_error */
    MIMO_ERR_NOT_PD = 4,      /* >= 1 unit failed the Cholesky guard since the last sync_status */
    MIMO_ERR_OOM = 5          /* host or device allocation failed */
} mimo_status_t;

typedef enum {
    MIMO_LLR_F32 = 0, /* float32, saturating at +-FLT_MAX */
    MIMO_LLR_F16 = 1, /* IEEE binary16, round-to-nearest-even, saturating at +-65504 */
    MIMO_LLR_I8 = 2   /* int8, rint (half to even), saturating at +-127 (-128 unused) */
} mimo_llr_type_t;

typedef struct {
    int device;      /* CUDA device ordinal the plan is bound to */
    void* stream;    /* cudaStream_t to enqueue on (0 = legacy default stream) */
    int n_rx;        /* receive antennas, 1..64 */
    int n_layers;    /* spatial layers, 1..min(16, n_rx) */
    int qam_order;   /* Qm = bits per symbol in {2,4,6,8} (QPSK..256-QAM), NOT M (reading R7) */
    int sc_per_h;    /* subcarriers sharing one H: >= 1 (1 = per subcarrier, 12 = per PRB) */
    int sym_per_h;   /* OFDM symbols sharing one H: >= 1 (14 = one H per slot) */
    int llr_type;    /* mimo_llr_type_t */
    float llr_scale; /* multiplier applied to natural-log LLRs before quantisation (> 0, finite) */
    int flags;       /* bitwise OR of MIMO_PLAN_* flags (0 = none) */
    /* The descriptor is the library's only configuration (no environment
     * variables). The two fields below default to 0 / NULL. */
    const char* kernel; /* NULL or "" = the default kernel specialisation for the shape; "generic" =
                           the generic CTA-per-unit kernel; otherwise the exact name of another compiled
                           specialisation of the same shape (mimo_plan_kernel_name) -- an unknown name is
                           MIMO_ERR_UNSUPPORTED. Only shape-serving, result-exact kernels are compiled in. */
    long long host_chunk_bytes; /* mimo_detect_mmse_host*: input bytes (H + y) per pipeline chunk of whole
                                   H time blocks; 0 = default (4 MiB synchronous, 16 MiB asynchronous) */
} mimo_plan_desc_t;

/* Plan flags.
 * MIMO_PLAN_OVERLAP_CALLS: launch with programmatic dependent launch, so that
 *   a detect call may start loading H / y and running its per-unit setup while
 *   the previous detect call on the same stream is still writing its outputs
 *   (its own writes wait for the previous call to complete). Precondition: a
 *   call's H and y are not outputs of the immediately preceding detect call on
 *   the same stream. Work enqueued by anything else orders normally. */
#define MIMO_PLAN_OVERLAP_CALLS 1

/* Create a plan: validates the descriptor, selects the kernel specialisation
 * for (n_rx, n_layers, qam_order, sc_per_h, sym_per_h, llr_type), allocates the
 * device failure counter on desc->device. *out_plan is set only on MIMO_OK.
 * Errors: INVALID_ARG (null args, out-of-range fields), UNSUPPORTED, CUDA (no
 * device / context creation failed), OOM. */
mimo_status_t mimo_plan_create(const mimo_plan_desc_t* desc, mimo_plan_t* out_plan);

/* Change the stream later calls enqueue on (e.g. torch's current stream). */
mimo_status_t mimo_plan_set_stream(mimo_plan_t plan, void* stream);

/* Detect all REs (north_star signature, with the plan as first argument).
 * H, y, llr_out: DEVICE pointers on the plan's device, 16-byte aligned, in the
 * layouts above. sigma2: total complex noise variance (CN(0, sigma2) per rx
 * antenna), finite and >= 0; sigma2 = 0 is zero-forcing with SINR = +inf and
 * saturated LLRs (reading R11). n_rx, n_layers, qam_order must equal the
 * plan's; n_sc % sc_per_h == 0 and n_sym % sym_per_h == 0; n_sc, n_sym >= 0
 * (0 REs is a no-op). Asynchronous: validates, enqueues one kernel on the plan's
 * stream and returns. Errors: INVALID_ARG, CUDA (launch error). */
mimo_status_t mimo_detect_mmse(mimo_plan_t plan, const void* H, const void* y, float sigma2,
                               int n_rx, int n_layers, int n_sc, int n_sym, int qam_order,
                               void* llr_out);

/* As mimo_detect_mmse, plus optional debug outputs (either may be NULL):
 * xhat_out complex64 [n_sym][n_sc][n_layers] (unbiased x~), sinr_out float32
 * [n_units][n_layers] (post-equalisation SINR_k, +inf when sigma2 = 0). llr_out
 * may be NULL when only the debug outputs are wanted. */
mimo_status_t mimo_detect_mmse_ex(mimo_plan_t plan, const void* H, const void* y, float sigma2,
                                  int n_rx, int n_layers, int n_sc, int n_sym, int qam_order,
                                  void* llr_out, void* xhat_out, float* sinr_out);

/* Per-slot noise variance (SURVEY.md 8(f) NEXT-3 "per-slot sigma2 arrays"; the
 * paper uses one sigma2 per configuration). Same computation as
 * mimo_detect_mmse_ex with sigma2 replaced, for every H-unit of H time block t
 * (units t * (n_sc / sc_per_h) ... ; t = slot when sym_per_h = 14), by
 * sigma2_v[t]. sigma2_v: DEVICE float32 [n_sym / sym_per_h], 4-byte aligned,
 * owned by the caller, read on the plan's stream. Each entry must be finite
 * and > 0 (no zero-forcing on this path): a bad entry makes that block's units
 * fail the pivot guard -- outputs zeroed and counted, mimo_plan_sync_status ->
 * MIMO_ERR_NOT_PD. Served by the same kernels as mimo_detect_mmse_ex.
 * Errors: as mimo_detect_mmse_ex (sigma2 checks replaced by: null, misaligned
 * or non-device sigma2_v -> INVALID_ARG). */
mimo_status_t mimo_detect_mmse_sv(mimo_plan_t plan, const void* H, const void* y, const float* sigma2_v,
                                  int n_rx, int n_layers, int n_sc, int n_sym, int qam_order,
                                  void* llr_out, void* xhat_out, float* sinr_out);

/* End-to-end form with HOST buffers (same layouts): copies H and y to a
 * plan-owned device workspace, detects, copies the LLRs back, and returns after
 * the stream has drained. Work is split into slot chunks (~4 MiB of input)
 * on a 3-deep device buffer ring over three streams (host->device, kernels,
 * device->host) so both PCIe directions and the kernels overlap; pinned
 * (page-locked) host buffers are required for overlap but not for correctness.
 * Errors: as mimo_detect_mmse, plus OOM. */
mimo_status_t mimo_detect_mmse_host(mimo_plan_t plan, const void* H_host, const void* y_host,
                                    float sigma2, int n_rx, int n_layers, int n_sc, int n_sym,
                                    int qam_order, void* llr_host);

/* Asynchronous form of mimo_detect_mmse_host: the same copies and kernels are
 * enqueued (ordered after the work already on the plan's stream) and the call
 * returns at once; mimo_plan_sync_status and mimo_plan_destroy wait for it. Consecutive calls overlap -- the next call's host->device copies run
 * while the previous call's results drain -- so a stream of TTIs is bound by
 * the busier PCIe direction, not by each call's fill and drain. The host
 * buffers must stay valid and unmodified (inputs) / unread (llr_host) until
 * then. Errors: as mimo_detect_mmse_host (enqueue errors only; execution
 * errors surface at the sync). */
mimo_status_t mimo_detect_mmse_host_async(mimo_plan_t plan, const void* H_host, const void* y_host,
                                          float sigma2, int n_rx, int n_layers, int n_sc, int n_sym,
                                          int qam_order, void* llr_host);

/* Paper-literal route: the LMMSE pipeline exactly as
 * the paper states it -- "LU decomposition, forward/backward substitution, and
 * matrix inversion" (Fig. 4 caption) of "the
 * received signal covariance matrix R" -- run as five UNFUSED
 * stage kernels so that each stage can be timed (the B200 analogue of Fig. 5b,
 * PAPER.md:108-109):
 *   stage 0  R = H H^H + sigma2 I                     (n_rx x n_rx)
 *   stage 1  P R = L U, partial pivoting (largest |a_ik|); a unit fails when a
 *            pivot |u_kk| <= 16 u max|a_ij| (u = unit roundoff of the working
 *            precision) or on NaN -- e.g. sigma2 = 0 with n_rx > n_layers
 *   stage 2  R^-1, column by column: L z = P e_c, U x = z
 *   stage 3  W = H^H R^-1, mu_k = [W H]_kk, SINR_k = mu_k / (1 - mu_k)
 *            (+inf at sigma2 = 0), W~ = W / mu_k (readings R3, R4)
 *   stage 4  x~ = W~ y, exact max-log LLRs, quantise (as mimo_detect_mmse)
 * Stages 0-3 run in precision_bits = 32 ("PS", fp32) or 64 ("PD", fp64)
 * arithmetic; W~ is rounded once to fp32 and stage 4 is
 * fp32. Arguments, layouts and outputs are those of mimo_detect_mmse_ex; the
 * plan's n_rx must be 1, 2, 4, 8 or 16 (else MIMO_ERR_UNSUPPORTED); the plan's
 * sc_per_h / sym_per_h / llr_type / llr_scale apply. The intermediate R, L\U,
 * R^-1 and W~ live in a plan-owned workspace (grown on demand; not during
 * graph capture). Failed units are erasures (LLR 0, x~ 0, SINR 0) and counted
 * (mimo_plan_sync_status -> MIMO_ERR_NOT_PD).
 * stage_us: NULL (asynchronous, like mimo_detect_mmse), or a host array of
 * MIMO_LU_STAGES floats that receives each stage's device time in
 * microseconds (CUDA events on the plan's stream; the call then synchronises
 * that stream before returning).
 * Errors: INVALID_ARG (as mimo_detect_mmse_ex; precision_bits not 32 or 64),
 * UNSUPPORTED, CUDA, OOM. */
#define MIMO_LU_STAGES 5
mimo_status_t mimo_detect_lmmse_lu(mimo_plan_t plan, const void* H, const void* y, float sigma2,
                                   int n_rx, int n_layers, int n_sc, int n_sym, int qam_order,
                                   int precision_bits, void* llr_out, void* xhat_out, float* sinr_out,
                                   float* stage_us);

/* Coloured-noise detection / interference-rejection combining (SURVEY.md §8(f)
 * NEXT-3; reading R24): y = H x + n with n ~ CN(0, R_nn) and a Hermitian
 * positive-definite R_nn per H-unit (e.g. the covariance of known interferers
 * plus noise, or sigma2_u I for a per-unit noise level). Computes the LMMSE filter
 *   W = H^H (H H^H + R_nn)^-1
 * (for R_nn = sigma2 I this is the paper's R of PAPER.md:117 and equals
 * mimo_detect_mmse), by whitening: R_nn = L_R L_R^H, H~ = L_R^-1 H, the white
 * Gram/Cholesky route with sigma2 = 1 on H~, and W = G^-1 H~^H L_R^-1 applied to
 * the un-whitened y. mu_k = 1 - [G^-1]_kk, SINR_k = 1/[G^-1]_kk - 1, x~ = (W y)/mu
 * and the LLRs as in mimo_detect_mmse. Setup in fp64, per-RE apply in fp32.
 *   Rnn: DEVICE complex64 [n_units][n_rx][n_rx], full Hermitian matrix (the lower
 *        triangle is read), 8-byte aligned.
 * Other arguments, layouts and outputs as mimo_detect_mmse_ex; n_rx <= 16 (else
 * MIMO_ERR_UNSUPPORTED). Units whose R_nn or G fails the Cholesky guard (R17) or
 * contain NaN are erasures and counted (MIMO_ERR_NOT_PD from sync_status).
 * Asynchronous. Errors: INVALID_ARG, UNSUPPORTED, CUDA. */
mimo_status_t mimo_detect_irc(mimo_plan_t plan, const void* H, const void* y, const void* Rnn,
                              int n_rx, int n_layers, int n_sc, int n_sym, int qam_order,
                              void* llr_out, void* xhat_out, float* sinr_out);

/* Detection from BLOCK-FLOATING-POINT compressed y (fronthaul format; SURVEY.md
 * §8(f) NEXT-4, reading R25), decompressed inside the detector's y loads so the
 * fp32 y never exists in HBM. One block per (symbol, PRB, antenna):
 *   block_bytes = roundup4(1 + 3 * iq_width); byte 0 = exponent e (bits 0..3);
 *   then the 24 two's-complement iq_width-bit mantissas I0,Q0,...,I11,Q11 of the
 *   PRB's 12 subcarriers, packed MSB-first; value = m * 2^e * bfp_scale.
 *   y_bfp: DEVICE bytes [n_sym][n_sc/12][n_rx][block_bytes], 16-byte aligned.
 * iq_width in 8..16; bfp_scale finite > 0; n_sc a multiple of 12. Everything else as
 * mimo_detect_mmse_ex. For n_rx = 8, n_layers = 4, sc_per_h = 12, sym_per_h = 14 (the C3
 * family) the decode is fused into the apply kernel's y loads; every other shape has the blocks
 * expanded by one kernel into a plan-owned complex64 y buffer (n_sym * n_sc * n_rx * 8 bytes,
 * grown by a call outside graph capture) that the shape's detector then reads. Asynchronous.
 * Errors: INVALID_ARG, CUDA, OOM (workspace / y buffer). */
mimo_status_t mimo_detect_mmse_bfp(mimo_plan_t plan, const void* H, const void* y_bfp, float sigma2,
                                   int n_rx, int n_layers, int n_sc, int n_sym, int qam_order,
                                   int iq_width, float bfp_scale,
                                   void* llr_out, void* xhat_out, float* sinr_out);

/* Host-buffer (end-to-end) forms of mimo_detect_mmse_bfp: H_host complex64 and y_bfp_host BFP
 * bytes [n_sym][n_sc/12][n_rx][block_bytes] in (pinned) host memory, llr_host host memory; the same
 * slot-chunk pipeline as mimo_detect_mmse_host / _host_async (H and the compressed y cross PCIe,
 * are decompressed inside the apply kernel's loads, LLRs come back). This is where the fronthaul
 * format pays: y crosses the host link at 28 B instead of 96 B per (symbol, PRB, antenna) at
 * iq_width 9 (D-MIMO fronthaul). Every shape: the C3 family decodes in its apply
 * loads, the others expand each chunk's blocks into the chunk's complex64 y buffer on the kernel
 * stream. Errors as mimo_detect_mmse_bfp plus those of mimo_detect_mmse_host; the _async form
 * returns after enqueuing (synchronise with mimo_plan_sync_status). */
mimo_status_t mimo_detect_mmse_bfp_host(mimo_plan_t plan, const void* H_host, const void* y_bfp_host, float sigma2,
                                        int n_rx, int n_layers, int n_sc, int n_sym, int qam_order, int iq_width,
                                        float bfp_scale, void* llr_host);
mimo_status_t mimo_detect_mmse_bfp_host_async(mimo_plan_t plan, const void* H_host, const void* y_bfp_host,
                                              float sigma2, int n_rx, int n_layers, int n_sc, int n_sym,
                                              int qam_order, int iq_width, float bfp_scale, void* llr_host);

/* Pre-allocate the plan's kernel workspace for calls of up to n_sc x n_sym
 * (some kernel families keep per-unit W~ in a plan-owned buffer). Calls grow the
 * workspace on demand, but not while the stream is being captured into a CUDA
 * graph: reserve before capturing. Errors: INVALID_ARG, CUDA, OOM. */
mimo_status_t mimo_plan_reserve(mimo_plan_t plan, int n_sc, int n_sym);

/* Synchronise the plan's stream (and the host-buffer path's streams, which
 * mimo_detect_mmse_host_async leaves running), return the number of units flagged by the
 * Cholesky guard since the previous call (and reset the count). Returns
 * MIMO_ERR_NOT_PD if that number is > 0, MIMO_ERR_CUDA on a sticky CUDA
 * error. n_failed_units may be NULL. */
mimo_status_t mimo_plan_sync_status(mimo_plan_t plan, long long* n_failed_units);

/* Synchronise and free the plan. NULL is a no-op returning MIMO_OK. */
mimo_status_t mimo_plan_destroy(mimo_plan_t plan);

/* Name of the kernel specialisation the plan launches (static string). */
const char* mimo_plan_kernel_name(mimo_plan_t plan);

/* Number of kernel launches one mimo_detect_mmse call enqueues. */
int mimo_plan_launches_per_call(mimo_plan_t plan);

/* Text of the last CUDA error seen by this plan ("" if none). */
const char* mimo_plan_last_error(mimo_plan_t plan);

/* Text of the last error seen by mimo_plan_create on this thread ("" if none). */
const char* mimo_last_error(void);

/* Static description of a status code. */
const char* mimo_status_string(mimo_status_t status);

/* MIMO_ABI_VERSION of the loaded library. */
int mimo_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MIMO_H */
