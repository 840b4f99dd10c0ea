// ddh_kernels.h -- internal interface between the host library (ddh_api.cpp)
// and the sm_100a kernels (ddh_kernels.cu).  Not part of the public ABI.
//
// Kernel map of one EM iteration:
//   K0  k0_stats     per-stream sums of y (Eq. 4 mean) and of the phase over
//                    the aperture (RemoveTipTilt normal equations)
//   K1  k1_rows_fwd  Normalize-apply (y - mu), plane removal, aperture,
//                    e^{-j phi}, chi, forward row DFT; partial ||y - mu||^2
//   K2a k2a_cols     forward column DFT -> u = A^H y (Eq. 3 back-projection =
//                    first E-step transform, R13); Eq. 3 warm start; E-step;
//                    chi mu -> inverse column DFT
//   K2b k2b_ricd     colour-ordered qGGMRF r-ICD (4 colours, halo 4, periodic)
//   K3a k3a_rows_inv inverse row DFT -> f = F_c^{-1} mu; c = (2/s2) a |y||f|,
//                    theta = arg(y conj f)
//   K3b k3b_phiicd   colour-ordered GMRF phi-ICD (4 colours, halo 4, free edge)
// State pointers passed to kernels are pre-offset to the first stream of the
// launch group ("chunk"); blockIdx.{y|z} is the stream within the chunk.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ddh {

// Base pointers of one multi-frame call replayed from a CUDA graph (ddh_api.cpp
// call graphs): the graph's kernels carry offsets from fixed stand-in bases and
// add these deltas (real base - stand-in base, modulo 2^64) at entry, so one
// captured chunk of frames serves every call whatever its buffers.
struct CallDesc {
  unsigned long long dy, dphi, dr, dst;  // y (and the next frame), phi_out, r_out, status
};
enum : int { kRelY = 1, kRelCopyPhi = 2, kRelCopyR = 4, kRelStatus = 8 };

struct StepArgs {
  int n;        // N
  int sc;       // streams in this launch group
  int nb0;      // K0 blocks per stream
  int nb1;      // K1 / K3a row blocks per stream
  const float2 *y;        // frame batch for this chunk: [sc][N][N]
  const float *phi_sub;   // K0 only: subtract this field (Strehl residual), else null
  float *r_state;         // [sc][N][N]
  const float *phi_in;    // [sc][N][N]
  float2 *cbuf;           // [sc][N][N] spectrum scratch (row DFT out / col IDFT out)
  float *rinit, *q;       // [sc][N][N] E-step outputs (r after Eq. 3, second moment)
  float *cc, *theta;      // [sc][N][N] phase-correlation terms
  double *part0;          // [sc][nb0][5]: sum re y, sum im y, sum phi, sum phi x, sum phi y
  double *part1;          // [sc][nb1]: sum |y - mu|^2
  const int2 *rowspan;    // [N] aperture row intervals [lo, hi)
  const float2 *tw;       // [N] twiddles e^{-2 pi i m / N}
  uint8_t *status;        // [sc] degenerate-frame flags or null (written by K2a)
  int want_y;             // K0: accumulate y sums
  int apply_plane;        // K0: accumulate plane sums; K1/K3b: subtract the plane
  int warm;               // K2a: apply Eq. 3 (or a bootstrap reset)
  float oml, la;          // K2a: r0 = max(oml r + la |u|^2, r_min)
  float s2, r_min;        // noise variance, r floor
  float P;                // N*N
  double minv[9];         // inverse of the aperture plane normal matrix
  double *stats;          // [sc][5] scratch (Strehl)
  int r_prior;            // qGGMRF on
  float r_b0, r_inv_Tsig, r_tmq;  // 1/(2 sig_r^2), 1/(T sig_r), 2 - q
  float r_b6, r_h, r_g, r_k;       // r_b0/6, (2-q)/2, (2-q) log2(1/(T sig_r)), q/2 (qgg_w2)
  int phi_prior;          // GMRF on
  float phi_w;            // 1/sig_phi^2
  int sweeps;             // ICD colour sweeps per M-step (R8)
  // streaming path (ddh_stream.cu)
  const float4 *tw4;      // [N] (w.x, w.y, -w.y, w.x), w = e^{-2 pi i m / N}
  const float *icd_in;    // S3: r before the sweep; S5: phi before the sweep [sc][N][N]
  float *icd_out;         // S3 / S5 output [sc][N][N]
  float *icd_copy;        // optional user copy of the output or null
  float *sstat;           // [sc][8] per-stream scalars of the step (ddh_stream.cu kStatW)
  double *psum_in;        // [sc][3] RemoveTipTilt sums of phi_in, 2^-16 fixed point (integer-valued; S0 adds / S1 reads)
  double *psum_out;       // [sc][3] the same sums of the output phase (S1 zeroes, last S5 adds) or null
  const CallDesc *desc;   // call-graph replay: deltas for the pointers flagged in `rel`, else unused
  int rel;                // kRel* bits: y / ynx, icd_copy (phi_out or r_out), status are stand-in pointers
  const float2 *ynx;      // S4: the next frame of the call [sc][N][N] (its S0 y sums are formed here) or null
  int dbg_fault;          // debug build only (DDH_DEBUG_FAULT): a deliberately failing check, to show the checks run
};

// On-chip multi-iteration chain (ddh_chain.cu, N = 64): one CTA per stream runs
// the whole frame, N_k iterations, in shared memory.
struct ChainArgs {
  StepArgs a;        // y, r_state (updated in place), phi_in, status, priors, plane, Eq. 3 weights
  float *phi_next;   // new phase state [sc][N][N]
  float *phi_copy;   // caller's phi_out or null
  float *r_copy;     // caller's r_out or null
  int iters;         // N_k
};

struct IcdArgs {
  int n;
  const float *in;       // r_in or phi_in [sc][N][N]
  const float *q;        // r-ICD: second moment; phi-ICD: c
  const float *theta;    // phi-ICD only
  float *out;            // [sc][N][N]
  float *copy;           // optional second output (user buffer) or null
  const double *part0;   // plane sums (phi-ICD with apply_plane) or null
  const double *part1;   // ||y - mu||^2 partials for degenerate detection, or null
  int nb0, nb1;
  int apply_plane;
  double minv[9];
  int prior;             // prior enabled
  float r_min;
  float b0;              // r: 1/(2 sig_r^2) ; phi: 1/sig_phi^2
  float inv_Tsig;        // r: 1/(T sig_r)
  float two_minus_q;     // r: 2 - q
};

struct StrehlArgs {
  int n, nb;             // nb: column blocks per field (partial maxima per field)
  const float *phi_hat, *phi_true;  // [B][N][N] (phi_hat null: psi = 0)
  const double *part0;   // plane sums of psi [B][nb0][5]
  int nb0;
  double minv[9];
  const int2 *rowspan;
  const float2 *tw;
  float2 *cbuf;          // [B][N][N]
  float *pmax;           // [B][nb]
  float *resid;          // optional [B][N][N]: wrapped residual phase (phi_true - phi_hat) - plane, 0 off the aperture
  float *psf;            // optional [B][N][N]: residual PSF |F_c^{-1}(a e^{j psi})|^2 / max |F_c^{-1} a|^2
  float inv_den;         // 1 / max |F_c^{-1} a|^2 (psf normalisation)
};

// Returns the first launch error (cudaGetLastError) of the sequence.
cudaError_t init_kernels(int n);
int row_block_rows(int n);    // H rows per K1/K3a CTA
int col_block_cols(int n);    // W columns per K2a CTA
int icd_tile(int n);          // ICD tile side
int k0_blocks(int n);         // K0 blocks per stream

cudaError_t launch_k0(const StepArgs &a, cudaStream_t st);
cudaError_t launch_k1(const StepArgs &a, cudaStream_t st);
cudaError_t launch_k2a(const StepArgs &a, cudaStream_t st);
cudaError_t launch_k3a(const StepArgs &a, cudaStream_t st);
cudaError_t launch_ricd(const IcdArgs &a, int sc, cudaStream_t st);
cudaError_t launch_phiicd(const IcdArgs &a, int sc, cudaStream_t st);
cudaError_t launch_fill(float *p, float v, size_t count, cudaStream_t st);
cudaError_t launch_strehl(const StrehlArgs &a, int B, cudaStream_t st);

// streaming (cluster-free) EM iteration, ddh_stream.cu: S0 stats, S1 rows,
// S2 cols + E-step, S3 r-ICD tiles, S4 inverse rows + c/theta, S5 phi-ICD tiles
cudaError_t init_stream(int n);
int stream_nb0(int n);  // S0 blocks per stream
int stream_nb1(int n);  // S1 row blocks per stream (part1 entries)
cudaError_t launch_s0(const StepArgs &a, cudaStream_t st);
cudaError_t launch_s1(const StepArgs &a, cudaStream_t st);
cudaError_t launch_s2(const StepArgs &a, cudaStream_t st);
cudaError_t launch_s3(const StepArgs &a, cudaStream_t st);
cudaError_t launch_s4(const StepArgs &a, cudaStream_t st);
cudaError_t launch_set_desc(CallDesc *d, const CallDesc &v, cudaStream_t st);
// S4 can form the next frame's S0 y sums (StepArgs::ynx) at this N
bool s4_sums_next(int n);
cudaError_t launch_s5(const StepArgs &a, cudaStream_t st);
int icd_launches(const StepArgs &a, bool r_icd);  // kernels one launch_s3 / launch_s5 enqueues (4: colour passes)

bool chain_fits(int n);  // the on-chip chain holds an N x N frame in one CTA
int chain_ctas_per_sm();  // its resident CTAs per SM
cudaError_t launch_chain(const ChainArgs &c, cudaStream_t st);

// stage entry points of the streaming kernels (ddh_test_*)
cudaError_t launch_test_fft_stream(int n, const float2 *in, float2 *out, int B, int inverse, const float4 *tw4,
                                   cudaStream_t st);
cudaError_t launch_test_estep(const float2 *u, const float *r_prev, float *r0, float2 *mu, float *q, size_t count,
                              int warm, float oml, float la, float r_min, float s2, cudaStream_t st);
cudaError_t launch_test_pack(const float *c, const float *th, float2 *out, size_t count, cudaStream_t st);
cudaError_t launch_test_fft2c(int n, const float2 *in, float2 *out, int B, int inverse, const float2 *tw,
                              cudaStream_t st);

}  // namespace ddh
