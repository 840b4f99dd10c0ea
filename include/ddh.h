/*
 * ddh.h -- C ABI of the B200-native DDH-MBIR hot path (libddh.so).
 *
 * Dynamic DH-MBIR (Sheikh, Pellizzari, Kisner, Buzzard, Bouman, arXiv
 * 2305.03284) estimates, for every time step n of a stream of single-shot
 * digital-holography (DH) frames y_n, the pupil phase error phi_n and the
 * image reflectance r_n of the model
 *
 *     y_n = A_{phi_n} g_n + w_n,   A_phi = D_a D(e^{j phi}) F_c^{-1},   g_n ~ CN(0, D(r_n))
 *
 * (Eq. 1; Gamma = I and F vs F^{-1} per DESIGN.md
 * readings R3/R5).  Citations "P:<line>" are lines of PAPER.md; "R<k>" are
 * the readings listed in DESIGN.md (where the paper is silent).
 *
 * Conventions shared by every entry point
 *   - Grid: N x N, row-major, index (i = row, j = column), centre (N/2, N/2).
 *     N is one of 64, 128, 256, 512, 1024.
 *   - Frames: complex64 = two little-endian IEEE float32 (re, im), layout
 *     [T][S][N][N] (frame-major, then stream, then row, then column).
 *   - Fields (phi, r): float32 [S][N][N] or [T][S][N][N].
 *   - Unless an argument says "host", pointers are CUDA device pointers on
 *     the ctx's device (e.g. torch tensors' data_ptr()).  The CALLER owns all
 *     input/output buffers and keeps them alive until ddh_sync() returns; the
 *     ctx owns its per-stream state and workspace.
 *   - Execution is asynchronous on the CUDA stream given to ddh_create unless
 *     an entry point says "synchronous".
 *   - Every function returns a ddh_status and never throws.  DDH_E_INVAL
 *     leaves the ctx unchanged.  A CUDA error is sticky (DDH_E_CUDA from then
 *     on; the ctx can only be destroyed).  ddh_last_error() explains the last
 *     failure.
 *   - A degenerate frame (||y - mean(y)|| = 0, Eq. 4 undefined) does not fail
 *     the call: its status byte is 1 and that stream's (r, phi) are left
 *     unchanged; the frame counter still advances.
 */
#ifndef DDH_H_
#define DDH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DDH_OK = 0,
  DDH_E_INVAL = 1,  /* bad argument / unsupported configuration      */
  DDH_E_CUDA = 2,   /* CUDA runtime error (sticky)                    */
  DDH_E_NOMEM = 3,  /* device or host allocation failed               */
  DDH_E_STATE = 4   /* ctx unusable (after a sticky error)            */
} ddh_status;

/* flags */
#define DDH_F_NO_TIPTILT 1u /* skip RemoveTipTilt (Fig. 1) in ddh_step  */
#define DDH_F_UNFUSED 2u    /* force the multi-pass kernels K0-K3b (reference
                               structure, used as a second implementation)      */
#define DDH_F_CLUSTER 4u    /* retired (round 2): the cluster-fused iteration was slower
                               than the streaming one at every config; ddh_create
                               returns DDH_E_INVAL when it is set                   */
#define DDH_F_SERIAL 8u     /* enqueue every kernel on the ctx stream in order (no
                               lanes, no side stream): per-kernel event timing     */
#define DDH_F_GRAPHS 32u    /* latency mode for synchronous per-frame calls: a single-
                               frame ddh_step whose frame/output pointers recur is
                               captured once into a CUDA graph and replayed (fewer
                               host launch gaps); back-to-back calls are faster
                               without it (graph boundaries stop the overlap of
                               consecutive steps)                                 */

#define DDH_F_CALL_GRAPHS 128u /* opt-in host-bound mode for multi-frame ddh_step: whole
                               chunks of 8 frames (DDH_CHUNK) of a call are replayed
                               from CUDA graphs captured once per (state parity,
                               outputs) with stand-in buffers, the call's buffers
                               passed through a device-side descriptor, so the host
                               enqueues 2 operations per chunk instead of ~25 per
                               frame (c3: 105 -> 2 us of host time per frame).  The
                               device runs the replayed graph ~2 % slower than the
                               directly launched streams (c3 126.7 vs 124.0 us per
                               step), so it pays only when the host is the bound.
                               The first chunk of each key is captured (~ms of host
                               time); results are bit-identical either way         */

#define DDH_F_NO_ADAPTIVE_GRAPHS 256u /* By default a multi-frame ddh_step on the streaming
                               path switches to the chunk graphs of DDH_F_CALL_GRAPHS by
                               itself when, at three consecutive frame boundaries (from
                               frame 8 on, more than four chunks left), the device holds
                               no whole frame of backlog: it is waiting for the host.
                               The rest of that call and the ctx's next four long calls
                               then come from graphs (tools/adapt_ab.sh).  This flag
                               keeps direct launches whatever the host does.  Results
                               are bit-identical.                                   */

#define DDH_F_L2_PERSIST 64u /* opt-in (device-wide side effect): raise the device's
                               persisting-L2 carve-out to the ctx's spectrum buffer
                               (<= 48 MiB) and give the ctx's own lane streams an
                               access-policy window over it (c3: +1.3 %); the last
                               such ctx on the device restores the previous limit  */

typedef struct ddh_ctx ddh_ctx; /* opaque */

/* Algorithm and layout parameters.  Fill with ddh_default_params() first. */
typedef struct {
  int32_t n;        /* grid side N: 64, 128, 256, 512 or 1024                         */
  int32_t streams;  /* S independent sensor streams owned by this ctx (>= 1)           */
  int32_t device;   /* CUDA device ordinal                                             */
  float aperture_diam;          /* D_a: circle of diameter D px (0 < D <= N; 0 with
                                   no mask means D = N), pixel centres strictly inside,
                                   centred at (N/2, N/2); < 0 selects aperture_mask      */
  const uint8_t *aperture_mask; /* host [N][N] {0,1}, used when aperture_diam <= 0 and it is
                                   not NULL; every row must be empty or one contiguous run
                                   of ones                                              */
  double noise_var; /* sigma^2 of the reconstruction in normalised-data units (R19), > 0  */
  double lambda;    /* Eq. 3 weight lambda in [0,1], default 0.45                 */
  double alpha;     /* Eq. 3 weight alpha in [0,1], default 0.025                 */
  int32_t n_k;      /* EM iterations per time step N_k >= 1 (Fig. 1)                */
  double r_min;     /* floor on r (replaces r <- 0 of Fig. 1, R14), > 0, default 1e-4      */
  double r_sigma;   /* qGGMRF scale sigma_r; <= 0 disables the r prior (R6/R7), def. 0.5  */
  double r_T;       /* qGGMRF threshold T > 0, default 1                                  */
  double r_q;       /* qGGMRF tail exponent q in [1,2], default 1.2                       */
  double phi_sigma; /* GMRF scale sigma_phi; <= 0 disables the phi prior (R11), def. 0.5 */
  int32_t icd_sweeps;   /* 4-colour ICD sweeps per M-step >= 1, default 1 (R8)             */
  int32_t boot_period;  /* bootstrap reset period P_b >= 1, default 200            */
  double boot_alpha;    /* bootstrap back-projection weight alpha_b > 0, default 1 (R15)   */
  int32_t chunk_streams;/* streams per launch group; 0 = auto (all, up to 8 GiB workspace) */
  uint32_t flags;       /* DDH_F_*                                                        */
  int32_t lanes;        /* streaming path: concurrent sub-groups of a launch group, each on
                           its own CUDA stream forked from / joined to the ctx stream, so
                           the kernels of different sub-groups share the SMs; 1..8, 0 =
                           auto (up to 3 lanes of >= 16 streams that keep >= 2 64-pixel
                           ICD tiles per SM).  Results do not depend on it.               */
} ddh_params;

/* Defaults: N=256, S=1, device 0, D=N, sigma^2=0.1, lambda=0.45, alpha=0.025,
 * N_k=1, r_min=1e-4, sigma_r=0.5, T=1, q=1.2, sigma_phi=0.5, 1 sweep,
 * P_b=200, alpha_b=1, chunk auto, flags 0, lanes auto.  Errors: DDH_E_INVAL if p is NULL. */
ddh_status ddh_default_params(ddh_params *p);

/* Create a ctx for S streams on p->device: validates p, allocates the state
 * r = r_min, phi = 0, frame counter n = 0 (Fig. 1 P:163 with R14), and the
 * workspace.  cuda_stream: a cudaStream_t (NULL = legacy default stream) on
 * which all work of this ctx is enqueued and ordered (the ctx may fork work
 * onto streams of its own and joins them back before returning control to
 * that stream's order).  *out receives the ctx (caller frees it with
 * ddh_destroy).  Synchronous.  No device-wide side effect unless
 * DDH_F_L2_PERSIST is set (see there).
 * Errors: DDH_E_INVAL (params out of range, unsupported N, non-interval mask),
 * DDH_E_NOMEM, DDH_E_CUDA. */
ddh_status ddh_create(const ddh_params *p, void *cuda_stream, ddh_ctx **out);

/* Free a ctx and everything it owns (synchronises its stream first). */
ddh_status ddh_destroy(ddh_ctx *c);

/* Bootstrap on the first frame (R15): every stream is cold-
 * started (r = r_min, phi = 0), y0 is normalised (Eq. 4), then k_b EM
 * iterations run; before iteration k with k mod boot_period == 0 the
 * reflectance is reset to max(boot_alpha |A_phi^H y|^2, r_min).  The frame is
 * consumed (frame counter += 1).  k_b == 0 is a no-op (Fig. 1 cold start).
 * y0: device complex64 [S][N][N], 16-byte aligned.  status: device uint8 [S] or NULL (0 ok,
 * 1 degenerate frame: the stream stays cold).  Errors: DDH_E_INVAL (k_b < 0,
 * NULL y0), DDH_E_CUDA. */
ddh_status ddh_bootstrap(ddh_ctx *c, const void *y0, int32_t k_b, uint8_t *status);

/* The hot path: T time steps of DDH_MBIR (Fig. 1) for all S streams.
 * For each t: y <- Normalize(y_t) (Eq. 4); phi <- RemoveTipTilt(phi) (
 * LS plane incl. piston, R17); r <- max((1-lambda) r + lambda alpha
 * |A_phi^H y|^2, r_min) (Eq. 3); then N_k EM iterations (E-step, qGGMRF r-ICD,
 * GMRF phi-ICD; R1-R12), two 2-D FFTs each (R13); WriteData.
 * y: device complex64 [T][S][N][N], 16-byte aligned (bulk asynchronous copies
 * of whole rows).  phi_out, r_out: device float32 [T][S][N][N], 8-byte
 * aligned, or NULL (the state always advances).  status: device uint8 [T][S]
 * or NULL.  Errors: DDH_E_INVAL (T < 0, NULL y with T > 0, misaligned
 * pointers), DDH_E_CUDA.
 * At N = 64 the frame's N_k iterations may run as one on-chip chain kernel
 * (one CTA per stream, the frame in shared memory) where that measured faster
 * (N_k >= 2, or N_k = 1 with one full wave of resident CTAs); the results
 * agree with the six-kernel path at the parity tolerance. */
ddh_status ddh_step(ddh_ctx *c, const void *y, int32_t T, float *phi_out, float *r_out,
                    uint8_t *status);

/* Same as ddh_step with HOST buffers (the end-to-end path): for each t the
 * frame batch y_t is copied host->device, stepped, and phi/r/status of that
 * step copied device->host.  The copies run on their own CUDA streams with
 * triple-buffered device staging, so for T > 1 the upload of frame t+1 and
 * the download of frame t-1 overlap the step of frame t.  y_host: host
 * complex64 [T][S][N][N] (pinned memory needed for the overlap);
 * phi_out/r_out/status: host [T][S][N][N] / [T][S] or NULL.  Synchronous.
 * Errors as ddh_step, plus DDH_E_NOMEM; on an error the copies already
 * enqueued are waited for before returning. */
ddh_status ddh_step_host(ddh_ctx *c, const void *y_host, int32_t T, float *phi_out,
                         float *r_out, uint8_t *status);

/* Asynchronous form of ddh_step_host: returns once the T frames are enqueued;
 * consecutive calls continue one copy/compute pipeline (no drain between
 * calls).  The caller keeps y_host and the output buffers alive and unread
 * until ddh_sync(c) returns.  Errors as ddh_step_host. */
ddh_status ddh_step_host_async(ddh_ctx *c, const void *y_host, int32_t T, float *phi_out,
                               float *r_out, uint8_t *status);

/* Conventional single-shot DH-MBIR on each of T frame
 * batches independently: cold start, `iters` EM iterations with bootstrap
 * resets every boot_period.  The ctx state is left equal to the last frame's
 * result.  Arguments as ddh_step.  Errors: DDH_E_INVAL (iters < 1). */
ddh_status ddh_static(ddh_ctx *c, const void *y, int32_t T, int32_t iters, float *phi_out,
                      float *r_out, uint8_t *status);

/* Copy the state out / in (checkpoint / resume; SPEC state continuity).
 * r, phi: device float32 [S][N][N] (either may be NULL); frame_index: host
 * int64 (may be NULL).  Errors: DDH_E_CUDA. */
ddh_status ddh_get_state(ddh_ctx *c, float *r, float *phi, int64_t *frame_index);
ddh_status ddh_set_state(ddh_ctx *c, const float *r, const float *phi, int64_t frame_index);

/* Peak Strehl ratio of B phase estimates against truth:
 * S_b = max |F_c^{-1}(a e^{j psi_b})|^2 / max |F_c^{-1}(a)|^2,
 * psi_b = phi_hat_b - phi_true_b minus its LS plane over the aperture (R26).
 * phi_hat, phi_true: device float32 [B][N][N].  strehl_out: HOST double [B].
 * Synchronous.  Errors: DDH_E_INVAL (B < 0, NULL), DDH_E_CUDA. */
ddh_status ddh_strehl(ddh_ctx *c, const float *phi_hat, const float *phi_true, int32_t B,
                      double *strehl_out);

/* Residual phase and residual PSF ("residual phase error"; Fig. 5
 * caption P:320, tip and tilt removed) of B estimates, with their Strehl
 * ratios: psi_b = phi_hat_b - phi_true_b minus its LS plane over the aperture
 * (R26); resid_b = angle(e^{-j psi_b}) in (-pi, pi] on the aperture, 0 off it;
 * psf_b = |F_c^{-1}(a e^{j psi_b})|^2 / max |F_c^{-1}(a)|^2 (centred; its
 * maximum is the peak Strehl ratio).  phi_hat, phi_true: device float32
 * [B][N][N]; resid, psf: device float32 [B][N][N] or NULL; strehl_out: HOST
 * double [B].  Synchronous.  Errors as ddh_strehl. */
ddh_status ddh_residual(ddh_ctx *c, const float *phi_hat, const float *phi_true, int32_t B, float *resid,
                        float *psf, double *strehl_out);

/* Wait for all work enqueued by this ctx (including the downloads of
 * ddh_step_host_async). */
ddh_status ddh_sync(ddh_ctx *c);

/* Human-readable description of the last error of c (or of the last failed
 * ddh_create when c is NULL).  Never NULL; owned by the library. */
const char *ddh_last_error(const ddh_ctx *c);

/* Number of CUDA kernels this ctx has launched so far (instrumentation). */
uint64_t ddh_kernel_launches(const ddh_ctx *c);

/* Frames processed so far (the n of Fig. 1). */
int64_t ddh_frame_index(const ddh_ctx *c);

/* ---- instrumentation: per-kernel device time (CUDA events on the ctx stream) ----
 * Kernel kinds: 0 K0 stats, 1 K1 rows_fwd, 2 K2a cols, 3 K2b r-ICD,
 * 4 K3a rows_inv, 5 K3b phi-ICD, 6 fill, 7 Strehl (multi-pass path);
 * 8 ks_chain (the on-chip multi-iteration chain at N = 64: one launch per
 * launch group and frame, all N_k iterations); 9-10 unused (the retired
 * cluster path); 11 S0 ks_stats, 12 S1 ks_rows_fwd,
 * 13 S2 ks_cols, 14 S3 ks_ricd (for large launches the four colour passes
 * ks_ricd_pass, timed as one), 15 S4 ks_rows_inv, 16 S5 ks_phiicd
 * (streaming path, default).
 * When enabled, every launch of the ctx is bracketed by two events. */
#define DDH_KIND_COUNT 17
ddh_status ddh_profile_enable(ddh_ctx *c, int32_t enable);
/* Synchronises the ctx stream and ADDS the accumulated totals since the last
 * read into ms[k] (milliseconds) and launches[k] (host arrays of
 * DDH_KIND_COUNT), then clears the pending records. */
ddh_status ddh_profile_read(ddh_ctx *c, double *ms, int64_t *launches);
/* Static name of kernel kind k (or "?"). */
const char *ddh_kind_name(int32_t k);

/* ---- stage entry points for parity tests ----
 * With the default (streaming) path these run the streaming kernels' own
 * device code: the register FFT of S1/S2/S4, the E-step epilogue of S2, the
 * S3 and S5 tile kernels.  With DDH_F_UNFUSED they run the multi-pass
 * kernels.  All buffers are device buffers owned by the caller; the calls are
 * asynchronous on the ctx stream.  Errors: DDH_E_INVAL (B < 0, NULL buffer),
 * DDH_E_CUDA. */

/* Centred unitary 2-D DFT F_c (inverse = 0) or F_c^{-1} (inverse = 1) of B
 * fields ("normalized 2D discrete Fourier transform"; R4): in, out
 * complex64 [B][N][N] (may alias). */
ddh_status ddh_test_fft2c(ddh_ctx *c, const void *in, void *out, int32_t B, int32_t inverse);

/* Eq. 3 + E-step of B fields (Eq. 3; P:93-95, 121 E-step, reading
 * R1): u = A^H y-hat complex64 [B][N][N], r_prev float32 [B][N][N];
 * warm != 0: r0 = max((1 - lambda) r_prev + lambda alpha |u|^2, r_min), else
 * r0 = r_prev; w = r0/(r0 + noise_var); mu = w u (complex64), q = |mu|^2 +
 * w noise_var.  Outputs r0, q float32 [B][N][N], mu complex64 [B][N][N]. */
ddh_status ddh_test_estep(ddh_ctx *c, const void *u, const float *r_prev, int32_t B, int32_t warm,
                          float *r0, void *mu, float *q);

/* One r M-step (colour-ordered qGGMRF ICD, icd_sweeps sweeps; R6-R9) of B
 * fields: r_in, q, r_out float32 [B][N][N] (r_out must not alias r_in). */
ddh_status ddh_test_ricd(ddh_ctx *c, const float *r_in, const float *q, int32_t B, float *r_out);

/* One phi M-step (colour-ordered GMRF ICD, icd_sweeps sweeps; R10-R11) of B
 * fields given the phase-correlation terms c, theta: float32 [B][N][N]
 * (phi_out must not alias phi_in). */
ddh_status ddh_test_phiicd(ddh_ctx *c, const float *phi_in, const float *cc, const float *theta,
                           int32_t B, float *phi_out);

/* ---- on-device frame synthesiser (input generation) ----
 * Synthetic DH frame sequences of the BASELINE recipe: blurred
 * uniform reflectance r (R23), FFT-method Kolmogorov screen on a periodic 2N x 2N
 * grid moved by frozen flow (Fourier shift, R22/R24) with piston/tip/tilt removed
 * over the aperture, fresh speckle g = sqrt(r/2)(z1 + j z2) per frame
 * (R21), complex AWGN sigma_n^2 = mean(r)/10^{SNR/10} (R20),
 * y = a e^{j phi} F_c^{-1}(g) + w (Eq. 1).  Philox-4x32-10 counters keyed by
 * (pixel, frame, stream, purpose) and `seed`: deterministic, independent of
 * the batching of frames.  Not the estimator: no part of the DDH-MBIR update. */
typedef struct ddh_synth ddh_synth; /* opaque */

/* n in {64,128,256,512,1024}; aperture: circle of diameter `diam` px strictly inside,
 * centre (n/2, n/2); d_r0: host [streams] turbulence strengths D/r0 (0: no
 * turbulence); velocity: host [streams][2] frozen-flow velocity (rows, cols) in
 * px/frame; sigma_b: reflectance blur (px, > 0); snr_db: per-pixel SNR in dB.
 * Synchronous setup on cuda_stream.  Errors: DDH_E_INVAL, DDH_E_NOMEM, DDH_E_CUDA. */
ddh_status ddh_synth_create(int32_t n, float diam, int32_t streams, const double *d_r0,
                            const double *velocity, double sigma_b, double snr_db, uint64_t seed,
                            void *cuda_stream, ddh_synth **out);

/* Frames t0 .. t0+T-1 of every stream: y device complex64 [T][S][n][n]; phi
 * device float32 [T][S][n][n] (the true, plane-removed phase) or NULL.
 * Asynchronous on the synthesiser's stream.  Errors: DDH_E_INVAL, DDH_E_CUDA. */
ddh_status ddh_synth_frames(ddh_synth *z, int64_t t0, int32_t T, void *y, float *phi);

/* The true reflectance r: device float32 [S][n][n]. */
ddh_status ddh_synth_reflectance(ddh_synth *z, float *r);

/* Free a synthesiser (synchronises its stream first). */
ddh_status ddh_synth_destroy(ddh_synth *z);

#ifdef __cplusplus
}
#endif
#endif /* DDH_H_ */
