// ddh_api.cpp -- host side of libddh.so: the C ABI declared in include/ddh.h.
//
// Owns per-stream state (r, phi ping-pong) and the launch-group workspace,
// validates parameters and sequences the kernels of ddh_kernels.cu:
//   per frame batch t, per launch group (chunk of streams):
//     K0 ; N_k x [ K1 ; K2a ; icd_sweeps x K2b ; K3a ; icd_sweeps x K3b ]
// (Fig. 1; Eq. 3 only in the first iteration; RemoveTipTilt's plane
// is subtracted by K1/K3b of the first iteration).  Everything is enqueued on
// the ctx stream; nothing here computes on the host except the aperture's
// constant tables (row intervals, 3x3 normal-matrix inverse, twiddles).
#include "../../include/ddh.h"
#include "ddh_kernels.h"
#ifndef DDH_DEBUG_BOUNDS
#define DDH_DEBUG_BOUNDS 0
#endif

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using ddh::ChainArgs;
using ddh::IcdArgs;
using ddh::StepArgs;
using ddh::StrehlArgs;
using ddh::CallDesc;
using ddh::kRelY;
using ddh::kRelCopyPhi;
using ddh::kRelCopyR;
using ddh::kRelStatus;

struct ddh_ctx {
  ddh_params p{};
  cudaStream_t st = nullptr;
  int n = 0, S = 0, sc = 0, nb0 = 0, nb1 = 0, strehl_nb = 0;
  size_t P = 0;
  // state
  float *r = nullptr;
  float *phi[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t frame = 0;
  // streaming path: RemoveTipTilt sums of the phase state in 2^-16 fixed point
  // (integer-valued doubles), [2][S][3]; psum[pcur] holds the sums of phi[cur] when psum_valid (written
  // by the last S5 of the previous frame), so S0 reads only y
  double *psum[2] = {nullptr, nullptr};
  int pcur = 0;
  bool psum_valid = false;
  // the S0 y sums of frame t+1 of one call run on the r-ICD side stream of
  // frame t: the frame batch whose sums are already in part0, or null
  const void *y_prefetched = nullptr;
  // launch-group workspace
  float2 *cbuf = nullptr;
  float *rinit = nullptr, *q = nullptr, *cc = nullptr, *theta = nullptr;
  float *rtmp[2] = {nullptr, nullptr}, *ptmp[2] = {nullptr, nullptr};
  double *part0 = nullptr, *part1 = nullptr, *stats = nullptr;
  float *sstat = nullptr;  // streaming path: per-stream scalars of a step [SC][8]
  bool streaming = false;  // cluster-free 6-kernel path (ddh_stream.cu)
  float4 *tw4 = nullptr;
  float *pmax = nullptr;
  // constants
  int2 *rowspan = nullptr;
  float2 *tw = nullptr;
  double minv[9] = {};
  double strehl_den = 1.0;
  // host-buffer path: triple-buffered staging, H2D / compute / D2H on three
  // streams so the copies of frames t+1 and t-1 overlap the step of frame t
#ifndef DDH_HOST_STAGES
#define DDH_HOST_STAGES 3
#endif
  static constexpr int kStages = DDH_HOST_STAGES;  // host pipeline depth (frames in flight)
  float2 *y_stage[kStages] = {};
  float *phi_stage[kStages] = {}, *r_stage[kStages] = {};
  uint8_t *status_stage[kStages] = {};
  cudaStream_t h2d_st = nullptr, d2h_st = nullptr;
  cudaEvent_t h2d_ev[kStages] = {}, comp_ev[kStages] = {}, d2h_ev[kStages] = {};
  bool host_pending = false;  // an asynchronous host-buffer call is in flight
  uint64_t host_t = 0;        // frames through the host pipeline since it was last drained
  // concurrent launch lanes of the streaming path: the streams of a launch
  // group are split over `lanes` CUDA streams so that the kernels of different
  // sub-groups (S1 of one, S3 of another, ...) share the SMs
  int lanes = 1;
  cudaStream_t lane_st[8] = {};
  cudaEvent_t lane_ev[9] = {};
  // streaming path: the r M-step (S3) of a lane runs on a side stream,
  // concurrently with the phi branch (S4, S5) it does not depend on (R12)
  bool split_r = false;
  // on-chip multi-iteration chain (ddh_chain.cu): Step frames of the streaming path at
  // N = 64 run as one CTA per stream holding the frame in shared memory when that
  // is faster than the six kernels (profiles/r02e_chain64.json, use_chain()).
  // DDH_CHAIN: 0 never, 1 always (tests, measurements)
  bool chain = false;
  bool chain_force = false;
  int chain_slots = 0;  // resident chain CTAs on the device (use_chain)
  bool l2_window = false;  // holds the device's persisting-L2 carve-out
  cudaStream_t side_st[8] = {};
  cudaEvent_t side_fork[8] = {}, side_join[8] = {};
  // inside a multi-frame call the join of a lane's r-ICD side stream is
  // deferred to the next S2 (the first kernel that needs it), so S1 of the next
  // frame overlaps the r-ICD; the next frame's S0 y sums run on a stream of
  // their own, forked after S1 (which reads the partials they overwrite)
  bool side_pending[8] = {};
  cudaStream_t ypf_st[8] = {};
  cudaEvent_t ypf_fork[8] = {}, ypf_join[8] = {};
  bool ypf_pending[8] = {};
  // CUDA graphs of single-frame steps (DDH_F_GRAPHS): a key (frame, outputs,
  // phi parity) seen twice within the last kKeyWindow calls is captured once
  // and replayed afterwards (the host then enqueues one graph instead of ~10
  // launches and events, so a synchronous per-frame call is not host-bound)
  struct GraphKey {
    const void *y;
    const void *phi, *r, *st;
    int cur, pcur;
    bool pvalid;
    bool operator==(const GraphKey &o) const {
      return y == o.y && phi == o.phi && r == o.r && st == o.st && cur == o.cur && pcur == o.pcur && pvalid == o.pvalid;
    }
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t launches, last;
  };
  bool graphs = false;
  cudaStream_t cap_st = nullptr;  // capture stream (the ctx stream may be the legacy default stream)
  // Call graphs (DDH_F_CALL_GRAPHS; streaming path, multi-frame ddh_step): chunks of `chunk`
  // frames are captured once per (state parity, outputs) with stand-in
  // buffer pointers and replayed for every later chunk, the call's real
  // buffers passed as deltas through a device-side CallDesc (ddh_kernels.h):
  // the host then enqueues 2 operations per chunk instead of ~25 per frame.
  struct ChunkKey {
    int len, cur, pcur;
    bool pvalid, phi, r, st;
    bool operator==(const ChunkKey &o) const {
      return len == o.len && cur == o.cur && pcur == o.pcur && pvalid == o.pvalid && phi == o.phi && r == o.r &&
             st == o.st;
    }
  };
  struct ChunkEntry {
    ChunkKey key;
    cudaGraphExec_t exec;
    uint64_t launches;
    int cur, pcur;  // state after the chunk (psum_valid is then true)
  };
  bool call_graphs = false;
  // Adaptive call graphs (default; DDH_F_NO_ADAPTIVE_GRAPHS / DDH_ADAPTIVE_GRAPHS=0 turn it off):
  // a long multi-frame call that finds the device waiting for the host (no whole frame of
  // backlog at three consecutive frame boundaries) finishes from chunk graphs.
  // adapt: 0 off, 1 on, 2 test mode (every check counts as starved)
  int adapt = 0, adapt_hot = 0;
  cudaEvent_t adapt_ev[2] = {nullptr, nullptr};  // ends of the last two directly launched frames
  double host_delay_us = 0.0;  // DDH_HOST_DELAY_US (diagnostic)
  uint64_t adapt_switches = 0;
  int chunk = 8;
  bool rel_mode = false;  // capturing a call graph: pointers are stand-ins (StepArgs::rel)
  CallDesc *desc = nullptr;
  std::vector<ChunkEntry> ccache;
  std::vector<GraphEntry> gcache;
  std::vector<GraphKey> gseen;
  uint64_t gclock = 0;
  // instrumentation
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_kind;  // kind of pending record i (events 2i, 2i+1)
  // stage entry points of the streaming path: stand-in per-stream partial sums
  // (no plane, ||y - mu||^2 > 0) for kernels that read them
  double *test_part0 = nullptr, *test_part1 = nullptr;
  float *test_sstat = nullptr;
  // bookkeeping
  uint64_t launches = 0;
  bool sticky = false;
  std::string err;
};

namespace {

std::mutex g_err_mu;
// persisting-L2 carve-out (device-wide): contexts holding one per device, and
// the limit found before the first of them raised it (restored by the last)
std::mutex g_l2_mu;
int g_l2_users[64] = {};
size_t g_l2_prev[64] = {};
std::string g_create_err;

ddh_status fail(ddh_ctx *c, ddh_status s, const std::string &msg) {
  if (c) {
    c->err = msg;
    if (s == DDH_E_CUDA) c->sticky = true;
  } else {
    std::lock_guard<std::mutex> lk(g_err_mu);
    g_create_err = msg;
  }
  return s;
}

#define DDH_CK(c, call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail((c), DDH_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

enum Kind { K_STATS = 0, K_ROWS_FWD, K_COLS, K_RICD, K_ROWS_INV, K_PHIICD, K_FILL, K_STREHL, K_CHAIN, K_KB, K_KC,
            K_S0, K_S1, K_S2, K_S3, K_S4, K_S5 };
const char *kKindNames[DDH_KIND_COUNT] = {"k0_stats", "k1_rows_fwd", "k2a_cols", "k2b_ricd",
                                          "k3a_rows_inv", "k3b_phiicd", "k_fill", "ks_strehl",
                                          "ks_chain", "unused9", "unused10",
                                          "ks_stats", "ks_rows_fwd", "ks_cols", "ks_ricd", "ks_rows_inv", "ks_phiicd"};

// Event pair for a launch of `kind` when profiling (nullptr otherwise).
cudaEvent_t *prof_begin(ddh_ctx *c, int kind, cudaStream_t st) {
  if (!c->profiling) return nullptr;
  const size_t i = c->ev_kind.size();
  while (c->ev_pool.size() < 2 * (i + 1)) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    c->ev_pool.push_back(e);
  }
  c->ev_kind.push_back(kind);
  cudaEventRecord(c->ev_pool[2 * i], st);
  return &c->ev_pool[2 * i + 1];
}

// DDH_SKIP=<mask of S0..S5>: those launches are not issued (diagnostic: marginal cost
// of a kernel inside the concurrent step; results invalid)
static int skip_mask() {
  static const int m = std::getenv("DDH_SKIP") ? std::atoi(std::getenv("DDH_SKIP")) : 0;
  return m;
}
#define DDH_LAUNCH_ON(c, kind, st, call)                \
  do {                                                  \
    cudaEvent_t *end_ = prof_begin((c), (kind), (st));  \
    if ((kind) < K_S0 || !(skip_mask() & (1 << ((kind) - K_S0)))) DDH_CK(c, call); \
    if (end_) cudaEventRecord(*end_, (st));             \
    (c)->launches++;                                    \
  } while (0)
#define DDH_LAUNCH(c, kind, call) DDH_LAUNCH_ON(c, kind, (c)->st, call)

bool valid_n(int n) { return n == 64 || n == 128 || n == 256 || n == 512 || n == 1024; }

ddh_status check_usable(ddh_ctx *c) {
  if (!c) return DDH_E_INVAL;
  if (c->sticky) return DDH_E_STATE;
  return DDH_OK;
}

template <class T>
cudaError_t dalloc(T **p, size_t count) {
  return cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T));
}

StepArgs base_args(ddh_ctx *c, int s0, int sc) {
  StepArgs a{};
  a.n = c->n;
  a.sc = sc;
  a.nb0 = c->nb0;
  a.nb1 = c->nb1;
  a.r_state = c->r + (size_t)s0 * c->P;
  a.cbuf = c->cbuf;
  a.rinit = c->rinit;
  a.q = c->q;
  a.cc = c->cc;
  a.theta = c->theta;
  a.part0 = c->part0;
  a.part1 = c->part1;
  a.rowspan = c->rowspan;
  a.tw = c->tw;
  a.tw4 = c->tw4;
  a.s2 = (float)c->p.noise_var;
  a.r_min = (float)c->p.r_min;
  a.P = (float)c->P;
  std::memcpy(a.minv, c->minv, sizeof(a.minv));
  a.stats = c->stats;
  a.sstat = c->sstat;
  a.r_prior = c->p.r_sigma > 0 ? 1 : 0;
  if (a.r_prior) {
    a.r_b0 = (float)(1.0 / (2.0 * c->p.r_sigma * c->p.r_sigma));
    a.r_inv_Tsig = (float)(1.0 / (c->p.r_T * c->p.r_sigma));
    a.r_tmq = (float)(2.0 - c->p.r_q);
    a.r_b6 = (float)(1.0 / (12.0 * c->p.r_sigma * c->p.r_sigma));
    a.r_h = (float)(0.5 * (2.0 - c->p.r_q));
    a.r_g = (float)((2.0 - c->p.r_q) * std::log2(1.0 / (c->p.r_T * c->p.r_sigma)));
    a.r_k = (float)(0.5 * c->p.r_q);
  }
  a.sweeps = c->p.icd_sweeps;
#if DDH_DEBUG_BOUNDS
  static const int fault = std::getenv("DDH_DEBUG_FAULT") ? std::atoi(std::getenv("DDH_DEBUG_FAULT")) : 0;
  a.dbg_fault = fault;
#endif
  a.phi_prior = c->p.phi_sigma > 0 ? 1 : 0;
  if (a.phi_prior) a.phi_w = (float)(1.0 / (c->p.phi_sigma * c->p.phi_sigma));
  return a;
}

IcdArgs ricd_args(ddh_ctx *c) {
  IcdArgs a{};
  a.n = c->n;
  a.nb0 = c->nb0;
  a.nb1 = c->nb1;
  a.prior = c->p.r_sigma > 0 ? 1 : 0;
  a.r_min = (float)c->p.r_min;
  if (a.prior) {
    a.b0 = (float)(1.0 / (2.0 * c->p.r_sigma * c->p.r_sigma));
    a.inv_Tsig = (float)(1.0 / (c->p.r_T * c->p.r_sigma));
    a.two_minus_q = (float)(2.0 - c->p.r_q);
  }
  return a;
}

IcdArgs phiicd_args(ddh_ctx *c) {
  IcdArgs a{};
  a.n = c->n;
  a.nb0 = c->nb0;
  a.nb1 = c->nb1;
  a.prior = c->p.phi_sigma > 0 ? 1 : 0;
  if (a.prior) a.b0 = (float)(1.0 / (c->p.phi_sigma * c->p.phi_sigma));
  std::memcpy(a.minv, c->minv, sizeof(a.minv));
  return a;
}

// r M-step: icd_sweeps sweeps of K2b from r_in into r_final (+ copy).
ddh_status run_ricd(ddh_ctx *c, const float *r_in, const float *q, float *r_final, float *copy,
                    const double *part1, int sc) {
  IcdArgs a = ricd_args(c);
  a.q = q;
  a.part1 = part1;
  const int sw = c->p.icd_sweeps;
  const float *in = r_in;
  for (int k = 0; k < sw; ++k) {
    const bool last = (k == sw - 1);
    float *out = last ? r_final : c->rtmp[k & 1];
    a.in = in;
    a.out = out;
    a.copy = last ? copy : nullptr;
    DDH_LAUNCH(c, K_RICD, ddh::launch_ricd(a, sc, c->st));
    in = out;
  }
  return DDH_OK;
}

// phi M-step: icd_sweeps sweeps of K3b (plane subtracted in the first sweep).
ddh_status run_phiicd(ddh_ctx *c, const float *phi_in, const float *cc, const float *theta, float *phi_final,
                      float *copy, const double *part0, const double *part1, int apply_plane, int sc) {
  IcdArgs a = phiicd_args(c);
  a.q = cc;
  a.theta = theta;
  a.part0 = part0;
  a.part1 = part1;
  const int sw = c->p.icd_sweeps;
  const float *in = phi_in;
  for (int k = 0; k < sw; ++k) {
    const bool last = (k == sw - 1);
    float *out = last ? phi_final : c->ptmp[k & 1];
    a.in = in;
    a.out = out;
    a.copy = last ? copy : nullptr;
    a.apply_plane = (k == 0) ? apply_plane : 0;
    DDH_LAUNCH(c, K_PHIICD, ddh::launch_phiicd(a, sc, c->st));
    in = out;
  }
  return DDH_OK;
}

enum class Mode { Step, Boot };

// The chain for a Step frame of N_k iterations (measured at 64^2, one B200,
// profiles/r02e_chain64.json, device us per step, chain / six kernels): every
// N_k >= 2 (N_k = 2: 47.4 / 47.9, 71.9 / 94.7, 231.6 / 245.2 at 64 / 296 / 1024
// streams; N_k = 8: 161 / 193, 246 / 381, 814 / 942); N_k = 1 only when the
// launch group is one full wave of resident CTAs (296 streams: 43.1 / 47.5; 64
// streams, 0.2 waves: 28.9 / 27.8; 1024 streams, 3.46 waves: 137.2 / 125.9).
bool use_chain(const ddh_ctx *c, int iters) {
  if (!c->chain) return false;
  if (c->chain_force || iters >= 2) return true;
  return c->sc >= 0.95 * c->chain_slots && c->sc <= c->chain_slots;
}

// One frame batch (all streams) through the loop body.  y: device frames
// [S][N][N] of this time step.  Outputs (may be null) are [S][N][N] / [S].
// Mode::Step: DDH step (Fig. 1).  Mode::Boot: cold start + `iters` iterations
// with resets every boot_period (bootstrap / static DH-MBIR).
// y_next: the next frame batch of the same call (streaming path, Step mode:
// its S0 y sums are computed during this frame, on the r-ICD side stream), or null.
ddh_status run_frame(ddh_ctx *c, const float2 *y, float *phi_out, float *r_out, uint8_t *status, Mode mode,
                     int iters, const float2 *y_next = nullptr) {
  // (one launch group only: the S0 partials are launch-group workspace)
  if (mode != Mode::Step || !c->streaming || c->sc < c->S) y_next = nullptr;
  const size_t P = c->P;
  const int cur0 = c->cur;
  const bool plane = (mode == Mode::Step) && !(c->p.flags & DDH_F_NO_TIPTILT);
  if (mode == Mode::Step && use_chain(c, iters)) {  // the on-chip chain: all N_k iterations
    for (int l = 0; l < 8; ++l) {  // streaming work still pending from a bootstrap
      if (c->side_pending[l]) DDH_CK(c, cudaStreamWaitEvent(c->st, c->side_join[l], 0));
      if (c->ypf_pending[l]) DDH_CK(c, cudaStreamWaitEvent(c->st, c->ypf_join[l], 0));
      c->side_pending[l] = c->ypf_pending[l] = false;
    }
    for (int s0 = 0; s0 < c->S; s0 += c->sc) {
      const int sc = std::min(c->sc, c->S - s0);
      const size_t so = (size_t)s0 * P;
      ChainArgs ca{};
      ca.a = base_args(c, s0, sc);
      ca.a.y = y + so;
      ca.a.phi_in = c->phi[cur0] + so;
      ca.a.apply_plane = plane ? 1 : 0;
      ca.a.warm = 1;
      ca.a.oml = (float)(1.0 - c->p.lambda);
      ca.a.la = (float)(c->p.lambda * c->p.alpha);
      ca.a.status = status ? status + s0 : nullptr;
      ca.phi_next = c->phi[cur0 ^ 1] + so;
      ca.phi_copy = phi_out ? phi_out + so : nullptr;
      ca.r_copy = r_out ? r_out + so : nullptr;
      ca.iters = iters;
      DDH_LAUNCH(c, K_CHAIN, ddh::launch_chain(ca, c->st));
    }
    c->cur = cur0 ^ 1;
    c->y_prefetched = nullptr;
    c->psum_valid = false;  // the streaming path's fixed-point plane sums are not kept
    return DDH_OK;
  }
  for (int s0 = 0; s0 < c->S; s0 += c->sc) {
    const int sc = std::min(c->sc, c->S - s0);
    const size_t so = (size_t)s0 * P;
    int cur = cur0;
    if (mode == Mode::Boot) {  // cold start r = r_min, phi = 0 (Fig. 1, R14)
      DDH_LAUNCH(c, K_FILL, ddh::launch_fill(c->r + so, (float)c->p.r_min, (size_t)sc * P, c->st));
      DDH_CK(c, cudaMemsetAsync(c->phi[cur] + so, 0, (size_t)sc * P * sizeof(float), c->st));
    }
    StepArgs a = base_args(c, s0, sc);
    a.y = y + so;
    a.phi_in = c->phi[cur] + so;
    a.want_y = 1;
    a.apply_plane = plane ? 1 : 0;
    if (c->streaming) {  // S0 ; N_k x [S1 ; S2 ; sweeps x S3 ; S4 ; sweeps x S5]
      const int L = std::min(c->lanes, sc);
      if (L > 1) {
        DDH_CK(c, cudaEventRecord(c->lane_ev[8], c->st));
        for (int l = 0; l < L; ++l) DDH_CK(c, cudaStreamWaitEvent(c->lane_st[l], c->lane_ev[8], 0));
      }
      const int nb0 = ddh::stream_nb0(c->n), nb1 = ddh::stream_nb1(c->n);
      const int sw = c->p.icd_sweeps;
      for (int l = 0; l < L; ++l) {
        const int g0 = (int)((long)sc * l / L), g1 = (int)((long)sc * (l + 1) / L);
        const size_t go = (size_t)(s0 + g0) * P, wo = (size_t)g0 * P;  // state / workspace offsets
        cudaStream_t st = L > 1 ? c->lane_st[l] : c->st;
        StepArgs b = a;
        b.sc = g1 - g0;
        b.nb0 = nb0;
        b.nb1 = nb1;
        b.y = y + go;
        b.r_state = c->r + go;
        b.cbuf = c->cbuf + wo;
        b.rinit = c->rinit + wo;
        b.q = c->q + wo;
        b.cc = c->cc + wo;
        b.theta = c->theta + wo;
        b.part0 = c->part0 + (size_t)g0 * nb0 * 5;
        b.part1 = c->part1 + (size_t)g0 * nb1;
        b.sstat = c->sstat + (size_t)g0 * 8;
        b.desc = c->desc;
        b.rel = c->rel_mode ? kRelY : 0;
        b.want_y = 1;
        b.apply_plane = plane ? 1 : 0;
        b.phi_in = c->phi[cur] + go;
        const bool stepm = mode == Mode::Step;
        b.psum_in = c->psum[c->pcur] + (size_t)(s0 + g0) * 3;
        double *psum_next = stepm ? c->psum[c->pcur ^ 1] + (size_t)(s0 + g0) * 3 : nullptr;
        // S0: the y sums (unless frame t-1 of this call prefetched them) and, when the
        // fixed-point plane sums of phi are not already there, those too
        const bool need_plane = plane && !c->psum_valid;
        const bool y_ready = c->y_prefetched == (const void *)y;
        if (need_plane)
          DDH_CK(c, cudaMemsetAsync(b.psum_in, 0, (size_t)b.sc * 3 * sizeof(double), st));
        if (!y_ready || need_plane) {
          b.want_y = y_ready ? 0 : 1;
          b.apply_plane = need_plane ? 1 : 0;
          DDH_LAUNCH_ON(c, K_S0, st, ddh::launch_s0(b, st));
          b.want_y = 1;
        }
        int cl = cur;
        for (int it = 0; it < iters; ++it) {
          const bool first = (it == 0), last = (it == iters - 1);
          b.phi_in = c->phi[cl] + go;
          b.apply_plane = (plane && first) ? 1 : 0;
          if (mode == Mode::Step) {
            b.warm = first ? 1 : 0;
            b.oml = (float)(1.0 - c->p.lambda);
            b.la = (float)(c->p.lambda * c->p.alpha);
          } else {
            b.warm = (it % c->p.boot_period == 0) ? 1 : 0;
            b.oml = 0.f;
            b.la = (float)c->p.boot_alpha;
          }
          b.status = (first && status) ? status + s0 + g0 : nullptr;
          b.rel = c->rel_mode ? (kRelY | (b.status ? kRelStatus : 0)) : 0;
          b.psum_out = first ? psum_next : nullptr;  // S1 zeroes the next frame's sums
          if (first && c->ypf_pending[l]) {  // this frame's S0 y sums, prefetched during the last frame
            DDH_CK(c, cudaStreamWaitEvent(st, c->ypf_join[l], 0));
            c->ypf_pending[l] = false;
          }
          DDH_LAUNCH_ON(c, K_S1, st, ddh::launch_s1(b, st));
          const bool s4_sums = last && y_next && ddh::s4_sums_next(c->n);
          if (last && y_next && !s4_sums) {  // y sums of the next frame of this call, after S1 read the partials
            StepArgs yb = b;
            yb.y = y_next + go;
            yb.want_y = 1;
            yb.apply_plane = 0;
            cudaStream_t yst = st;
            if (c->split_r) {
              yst = c->ypf_st[l];
              DDH_CK(c, cudaEventRecord(c->ypf_fork[l], st));
              DDH_CK(c, cudaStreamWaitEvent(yst, c->ypf_fork[l], 0));
            }
            DDH_LAUNCH_ON(c, K_S0, yst, ddh::launch_s0(yb, yst));
            if (c->split_r) {
              DDH_CK(c, cudaEventRecord(c->ypf_join[l], yst));
              c->ypf_pending[l] = true;
            }
          }
          if (c->side_pending[l]) {  // S2 overwrites r0, q and reads r: the previous r-ICD must be done
            DDH_CK(c, cudaStreamWaitEvent(st, c->side_join[l], 0));
            c->side_pending[l] = false;
          }
          DDH_LAUNCH_ON(c, K_S2, st, ddh::launch_s2(b, st));
          cudaStream_t rst = st;
          if (c->split_r) {  // fork: S3 after S2, beside S4/S5
            rst = c->side_st[l];
            DDH_CK(c, cudaEventRecord(c->side_fork[l], st));
            DDH_CK(c, cudaStreamWaitEvent(rst, c->side_fork[l], 0));
          }
          for (int k = 0; k < sw; ++k) {  // r M-step sweeps
            b.icd_in = k == 0 ? c->rinit + wo : c->rtmp[(k - 1) & 1] + wo;
            b.icd_out = k == sw - 1 ? c->r + go : c->rtmp[k & 1] + wo;
            b.icd_copy = (k == sw - 1 && last && r_out) ? r_out + go : nullptr;
            if (c->rel_mode) b.rel = (b.rel & ~(kRelCopyPhi | kRelCopyR)) | (b.icd_copy ? kRelCopyR : 0);
            DDH_LAUNCH_ON(c, K_S3, rst, ddh::launch_s3(b, rst));
            c->launches += ddh::icd_launches(b, true) - 1;
          }
          b.ynx = s4_sums ? y_next + go : nullptr;  // S4 forms the next frame's y sums (after S1 read them)
          DDH_LAUNCH_ON(c, K_S4, st, ddh::launch_s4(b, st));
          b.ynx = nullptr;
          const int plane_it = b.apply_plane;
          for (int k = 0; k < sw; ++k) {  // phi M-step sweeps (plane removed in the first)
            b.icd_in = k == 0 ? c->phi[cl] + go : c->ptmp[(k - 1) & 1] + wo;
            b.icd_out = k == sw - 1 ? c->phi[cl ^ 1] + go : c->ptmp[k & 1] + wo;
            b.icd_copy = (k == sw - 1 && last && phi_out) ? phi_out + go : nullptr;
            if (c->rel_mode) b.rel = (b.rel & ~(kRelCopyPhi | kRelCopyR)) | (b.icd_copy ? kRelCopyPhi : 0);
            b.apply_plane = k == 0 ? plane_it : 0;
            b.psum_out = (k == sw - 1 && last) ? psum_next : nullptr;  // sums of the frame's phase
            DDH_LAUNCH_ON(c, K_S5, st, ddh::launch_s5(b, st));
            c->launches += ddh::icd_launches(b, false) - 1;
            b.psum_out = nullptr;
          }
          if (c->split_r) {  // join: the next S2 reads r; S1 overwrites nothing S3 reads
            DDH_CK(c, cudaEventRecord(c->side_join[l], rst));
            if (last && y_next) {
              c->side_pending[l] = true;  // deferred to the next frame's S2
            } else {
              DDH_CK(c, cudaStreamWaitEvent(st, c->side_join[l], 0));
            }
          }
          cl ^= 1;
        }
      }
      if (L > 1) {
        for (int l = 0; l < L; ++l) {
          DDH_CK(c, cudaEventRecord(c->lane_ev[l], c->lane_st[l]));
          DDH_CK(c, cudaStreamWaitEvent(c->st, c->lane_ev[l], 0));
        }
      }
      cur ^= (iters & 1);
      continue;
    }
    DDH_LAUNCH(c, K_STATS, ddh::launch_k0(a, c->st));
    for (int it = 0; it < iters; ++it) {
      const bool first = (it == 0), last = (it == iters - 1);
      a.phi_in = c->phi[cur] + so;
      a.apply_plane = (plane && first) ? 1 : 0;
      if (mode == Mode::Step) {
        a.warm = first ? 1 : 0;
        a.oml = (float)(1.0 - c->p.lambda);
        a.la = (float)(c->p.lambda * c->p.alpha);
      } else {
        a.warm = (it % c->p.boot_period == 0) ? 1 : 0;
        a.oml = 0.f;
        a.la = (float)c->p.boot_alpha;
      }
      a.status = (first && status) ? status + s0 : nullptr;
      DDH_LAUNCH(c, K_ROWS_FWD, ddh::launch_k1(a, c->st));
      DDH_LAUNCH(c, K_COLS, ddh::launch_k2a(a, c->st));
      ddh_status rs = run_ricd(c, c->rinit, c->q, c->r + so, (last && r_out) ? r_out + so : nullptr, c->part1, sc);
      if (rs != DDH_OK) return rs;
      DDH_LAUNCH(c, K_ROWS_INV, ddh::launch_k3a(a, c->st));
      rs = run_phiicd(c, c->phi[cur] + so, c->cc, c->theta, c->phi[cur ^ 1] + so,
                      (last && phi_out) ? phi_out + so : nullptr, c->part0, c->part1, a.apply_plane, sc);
      if (rs != DDH_OK) return rs;
      cur ^= 1;
    }
  }
  c->cur = cur0 ^ (iters & 1);
  c->y_prefetched = y_next;
  if (c->streaming) {
    if (mode == Mode::Step) {
      c->pcur ^= 1;  // the last S5 left the sums of the new phase in psum[pcur ^ 1]
      c->psum_valid = true;
    } else {
      c->psum_valid = false;  // bootstrap / static: no epilogue sums
    }
  }
  return DDH_OK;
}

constexpr size_t kGraphCache = 16, kKeyWindow = 64;

// One DDH step of one frame batch, replayed from a CUDA graph when this exact
// call (same frame and output pointers, same phi parity) recurs.
ddh_status step_frame(ddh_ctx *c, const float2 *y, float *phi_out, float *r_out, uint8_t *status,
                      const float2 *y_next) {
  // Opt-in (DDH_F_GRAPHS) for synchronous per-frame use, where a graph removes
  // the host launch gaps from the frame's latency.  Back-to-back calls are
  // better served by direct launches, whose programmatic dependent launches
  // overlap one step's tail with the next step's head (graph boundaries do not).
  if (!c->graphs || c->profiling) return run_frame(c, y, phi_out, r_out, status, Mode::Step, c->p.n_k, y_next);
  if (c->y_prefetched) return run_frame(c, y, phi_out, r_out, status, Mode::Step, c->p.n_k, y_next);
  if (y_next) return run_frame(c, y, phi_out, r_out, status, Mode::Step, c->p.n_k, y_next);
  const ddh_ctx::GraphKey key{y, phi_out, r_out, status, c->cur, c->pcur, c->psum_valid};
  ++c->gclock;
  for (auto &g : c->gcache) {
    if (g.key == key) {
      g.last = c->gclock;
      DDH_CK(c, cudaGraphLaunch(g.exec, c->st));
      c->launches += g.launches;
      c->cur ^= (c->p.n_k & 1);
      if (c->streaming) c->pcur ^= 1, c->psum_valid = true;
      return DDH_OK;
    }
  }
  const bool seen = std::find(c->gseen.begin(), c->gseen.end(), key) != c->gseen.end();
  if (!seen) {
    c->gseen.push_back(key);
    if (c->gseen.size() > kKeyWindow) c->gseen.erase(c->gseen.begin());
    return run_frame(c, y, phi_out, r_out, status, Mode::Step, c->p.n_k);
  }
  // capture the sequence on a private stream standing in for the ctx stream
  // (lane and side streams join through their events); replays go to the ctx stream
  if (!c->cap_st) DDH_CK(c, cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
  const int cur0 = c->cur, pcur0 = c->pcur;
  const bool pvalid0 = c->psum_valid;
  const uint64_t l0 = c->launches;
  cudaStream_t user_st = c->st;
  DDH_CK(c, cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeThreadLocal));
  c->st = c->cap_st;
  ddh_status s = run_frame(c, y, phi_out, r_out, status, Mode::Step, c->p.n_k);
  c->st = user_st;
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(c->cap_st, &graph);
  c->cur = cur0;
  c->pcur = pcur0;
  c->psum_valid = pvalid0;
  const uint64_t nl = c->launches - l0;
  c->launches = l0;
  if (s != DDH_OK) {
    if (graph) cudaGraphDestroy(graph);
    return s;
  }
  if (ec != cudaSuccess) return fail(c, DDH_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ec));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return fail(c, DDH_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
  if (c->gcache.size() >= kGraphCache) {  // evict the least recently used
    auto lru = std::min_element(c->gcache.begin(), c->gcache.end(),
                                [](const ddh_ctx::GraphEntry &a, const ddh_ctx::GraphEntry &b) { return a.last < b.last; });
    cudaGraphExecDestroy(lru->exec);
    c->gcache.erase(lru);
  }
  c->gcache.push_back({key, exec, nl, c->gclock});
  DDH_CK(c, cudaGraphLaunch(exec, c->st));
  c->launches += nl;
  c->cur ^= (c->p.n_k & 1);
  if (c->streaming) c->pcur ^= 1, c->psum_valid = true;
  return DDH_OK;
}

// Stand-in bases of a captured call graph (never dereferenced: the kernels add
// the CallDesc deltas first).  Far apart, so a chunk's offsets never overlap.
const uintptr_t kFakeY = (uintptr_t)1 << 44, kFakePhi = (uintptr_t)2 << 44, kFakeR = (uintptr_t)3 << 44,
                kFakeSt = (uintptr_t)4 << 44;

// `len` frames of a multi-frame call (streaming path, Step mode) from a
// chunk graph, captured on first use for this (state parity, outputs) key.
// Chunks start and end with no cross-frame work pending (the last frame of a
// chunk prefetches nothing), so a graph depends only on the key.
ddh_status run_chunk(ddh_ctx *c, const float2 *y, float *phi_out, float *r_out, uint8_t *status, int len) {
  const ddh_ctx::ChunkKey key{len, c->cur, c->pcur, c->psum_valid, phi_out != nullptr, r_out != nullptr,
                              status != nullptr};
  const ddh_ctx::ChunkEntry *hit = nullptr;
  for (const auto &e : c->ccache)
    if (e.key == key) hit = &e;
  if (!hit) {
    if (!c->cap_st) DDH_CK(c, cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
    const int cur0 = c->cur, pcur0 = c->pcur;
    const bool pvalid0 = c->psum_valid;
    const uint64_t l0 = c->launches;
    const size_t fs = (size_t)c->S * c->P;
    cudaStream_t user_st = c->st;
    DDH_CK(c, cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeThreadLocal));
    c->st = c->cap_st;
    c->rel_mode = true;
    ddh_status s = DDH_OK;
    for (int k = 0; k < len && s == DDH_OK; ++k) {
      const float2 *yk = reinterpret_cast<const float2 *>(kFakeY) + k * fs;
      s = run_frame(c, yk, phi_out ? reinterpret_cast<float *>(kFakePhi) + k * fs : nullptr,
                    r_out ? reinterpret_cast<float *>(kFakeR) + k * fs : nullptr,
                    status ? reinterpret_cast<uint8_t *>(kFakeSt) + (size_t)k * c->S : nullptr, Mode::Step,
                    c->p.n_k, k + 1 < len ? yk + fs : nullptr);
    }
    c->rel_mode = false;
    c->st = user_st;
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->cap_st, &graph);
    const int cur1 = c->cur, pcur1 = c->pcur;
    c->cur = cur0;
    c->pcur = pcur0;
    c->psum_valid = pvalid0;
    c->y_prefetched = nullptr;
    const uint64_t nl = c->launches - l0;
    c->launches = l0;
    if (s != DDH_OK || ec != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      if (s != DDH_OK) return s;
      return fail(c, DDH_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ec));
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return fail(c, DDH_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
    if (c->ccache.size() >= kGraphCache) {
      cudaGraphExecDestroy(c->ccache.front().exec);
      c->ccache.erase(c->ccache.begin());
    }
    c->ccache.push_back({key, exec, nl, cur1, pcur1});
    hit = &c->ccache.back();
  }
  CallDesc d;
  d.dy = (unsigned long long)((uintptr_t)y - kFakeY);
  d.dphi = (unsigned long long)((uintptr_t)phi_out - kFakePhi);
  d.dr = (unsigned long long)((uintptr_t)r_out - kFakeR);
  d.dst = (unsigned long long)((uintptr_t)status - kFakeSt);
  DDH_CK(c, ddh::launch_set_desc(c->desc, d, c->st));
  DDH_CK(c, cudaGraphLaunch(hit->exec, c->st));
  c->launches += hit->launches + 1;
  c->cur = hit->cur;
  c->pcur = hit->pcur;
  c->psum_valid = true;
  c->y_prefetched = nullptr;
  return DDH_OK;
}

double inv3(const double G[9], double out[9]) {
  const double a = G[0], b = G[1], cc = G[2], d = G[3], e = G[4], f = G[5], g = G[6], h = G[7], i = G[8];
  const double A = e * i - f * h, B = -(d * i - f * g), C = d * h - e * g;
  const double det = a * A + b * B + cc * C;
  if (!(std::fabs(det) > 0)) return 0.0;
  out[0] = A / det;
  out[1] = -(b * i - cc * h) / det;
  out[2] = (b * f - cc * e) / det;
  out[3] = B / det;
  out[4] = (a * i - cc * g) / det;
  out[5] = -(a * f - cc * d) / det;
  out[6] = C / det;
  out[7] = -(a * h - b * g) / det;
  out[8] = (a * e - b * d) / det;
  return det;
}

void free_ctx(ddh_ctx *c) {
  if (!c) return;
  if (c->l2_window) {  // the last context on the device restores the limit it found
    std::lock_guard<std::mutex> lk(g_l2_mu);
    const int d = c->p.device & 63;
    if (--g_l2_users[d] == 0) {
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(c->p.device);
      cudaCtxResetPersistingL2Cache();
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_prev[d]);
      if (prev >= 0) cudaSetDevice(prev);
      cudaGetLastError();
    }
  }
  for (auto &g : c->gcache) cudaGraphExecDestroy(g.exec);
  for (auto &g : c->ccache) cudaGraphExecDestroy(g.exec);
  if (c->desc) cudaFree(c->desc);
  if (c->cap_st) cudaStreamDestroy(c->cap_st);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->adapt_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->lane_ev)
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : c->lane_st)
    if (s) cudaStreamDestroy(s);
  for (int k = 0; k < ddh_ctx::kStages; ++k) {
    if (c->h2d_ev[k]) cudaEventDestroy(c->h2d_ev[k]);
    if (c->comp_ev[k]) cudaEventDestroy(c->comp_ev[k]);
    if (c->d2h_ev[k]) cudaEventDestroy(c->d2h_ev[k]);
  }
  if (c->h2d_st) cudaStreamDestroy(c->h2d_st);
  if (c->d2h_st) cudaStreamDestroy(c->d2h_st);
  for (int l = 0; l < 8; ++l) {
    if (c->side_st[l]) cudaStreamDestroy(c->side_st[l]);
    if (c->side_fork[l]) cudaEventDestroy(c->side_fork[l]);
    if (c->side_join[l]) cudaEventDestroy(c->side_join[l]);
    if (c->ypf_st[l]) cudaStreamDestroy(c->ypf_st[l]);
    if (c->ypf_fork[l]) cudaEventDestroy(c->ypf_fork[l]);
    if (c->ypf_join[l]) cudaEventDestroy(c->ypf_join[l]);
  }
  void *ptrs[] = {c->r, c->phi[0], c->phi[1], c->cbuf, c->cc, c->theta, c->rtmp[0], c->rtmp[1],
                  c->ptmp[0], c->ptmp[1], c->part0, c->part1, c->stats, c->pmax, c->rowspan, c->tw, c->tw4,
                  c->y_stage[0], c->phi_stage[0], c->r_stage[0], c->status_stage[0],
                  c->y_stage[1], c->phi_stage[1], c->r_stage[1], c->status_stage[1],
                  c->y_stage[2], c->phi_stage[2], c->r_stage[2], c->status_stage[2], c->test_part0, c->test_part1, c->sstat, c->test_sstat, c->psum[0], c->psum[1]};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  delete c;
}

}  // namespace

extern "C" {

ddh_status ddh_default_params(ddh_params *p) {
  if (!p) return DDH_E_INVAL;
  std::memset(p, 0, sizeof(*p));
  p->n = 256;
  p->streams = 1;
  p->device = 0;
  p->aperture_diam = 0.f;  // D = N
  p->aperture_mask = nullptr;
  p->noise_var = 0.1;
  p->lambda = 0.45;
  p->alpha = 0.025;
  p->n_k = 1;
  p->r_min = 1e-4;
  p->r_sigma = 0.5;
  p->r_T = 1.0;
  p->r_q = 1.2;
  p->phi_sigma = 0.5;
  p->icd_sweeps = 1;
  p->boot_period = 200;
  p->boot_alpha = 1.0;
  p->chunk_streams = 0;
  p->flags = 0;
  p->lanes = 0;
  return DDH_OK;
}

ddh_status ddh_create(const ddh_params *pp, void *cuda_stream, ddh_ctx **out) {
  if (!pp || !out) return fail(nullptr, DDH_E_INVAL, "ddh_create: NULL argument");
  *out = nullptr;
  const ddh_params &p = *pp;
  if (!valid_n(p.n)) return fail(nullptr, DDH_E_INVAL, "ddh_create: n must be 64, 128, 256, 512 or 1024");
  if (p.streams < 1) return fail(nullptr, DDH_E_INVAL, "ddh_create: streams must be >= 1");
  if (!(p.noise_var > 0)) return fail(nullptr, DDH_E_INVAL, "ddh_create: noise_var must be > 0");
  if (!(p.lambda >= 0 && p.lambda <= 1) || !(p.alpha >= 0 && p.alpha <= 1))
    return fail(nullptr, DDH_E_INVAL, "ddh_create: lambda and alpha must be in [0,1] (P:189)");
  if (p.n_k < 1) return fail(nullptr, DDH_E_INVAL, "ddh_create: n_k must be >= 1");
  if (!(p.r_min > 0)) return fail(nullptr, DDH_E_INVAL, "ddh_create: r_min must be > 0");
  if (p.r_sigma > 0 && (!(p.r_T > 0) || !(p.r_q >= 1 && p.r_q <= 2)))
    return fail(nullptr, DDH_E_INVAL, "ddh_create: qGGMRF needs r_T > 0 and r_q in [1,2]");
  if (p.icd_sweeps < 1) return fail(nullptr, DDH_E_INVAL, "ddh_create: icd_sweeps must be >= 1");
  if (p.boot_period < 1 || !(p.boot_alpha > 0))
    return fail(nullptr, DDH_E_INVAL, "ddh_create: boot_period >= 1 and boot_alpha > 0 required");
  if (p.chunk_streams < 0) return fail(nullptr, DDH_E_INVAL, "ddh_create: chunk_streams must be >= 0");
  if (p.lanes < 0 || p.lanes > 8) return fail(nullptr, DDH_E_INVAL, "ddh_create: lanes must be in [0, 8]");
  if (p.flags & DDH_F_CLUSTER)
    return fail(nullptr, DDH_E_INVAL, "ddh_create: the cluster path (DDH_F_CLUSTER) was retired (slower than the streaming path at every config)");
  const int n = p.n;
  // aperture_diam 0 with no mask: the configs' D = N; a circle wider than the grid is refused
  const float diam = (p.aperture_diam == 0.f && !p.aperture_mask) ? (float)n : p.aperture_diam;
  if (!(diam > 0) && !p.aperture_mask)
    return fail(nullptr, DDH_E_INVAL, "ddh_create: aperture_diam < 0 requires aperture_mask");
  if (diam > (float)n) return fail(nullptr, DDH_E_INVAL, "ddh_create: aperture_diam must be <= n");

  // aperture row intervals and plane normal matrix (RemoveTipTilt)
  std::vector<int2> span(n);
  double G[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  size_t count = 0;
  for (int i = 0; i < n; ++i) {
    int lo = n, hi = n;
    bool seen = false, ended = false;
    for (int j = 0; j < n; ++j) {
      bool in;
      if (diam > 0) {
        const double di = i - n / 2, dj = j - n / 2, rr = 0.5 * (double)diam;
        in = di * di + dj * dj < rr * rr;
      } else {
        in = p.aperture_mask[(size_t)i * n + j] != 0;
      }
      if (in) {
        if (ended) return fail(nullptr, DDH_E_INVAL, "ddh_create: aperture mask rows must be contiguous runs");
        if (!seen) lo = j;
        seen = true;
        hi = j + 1;
        const double x = j - n / 2, y = i - n / 2;
        const double b[3] = {1.0, x, y};
        for (int u = 0; u < 3; ++u)
          for (int v = 0; v < 3; ++v) G[u * 3 + v] += b[u] * b[v];
        ++count;
      } else if (seen) {
        ended = true;
      }
    }
    if (!seen) lo = hi = 0;
    span[i] = make_int2(lo, hi);
  }
  double minv[9];
  if (count < 3 || inv3(G, minv) == 0.0)
    return fail(nullptr, DDH_E_INVAL, "ddh_create: aperture too small for the tip/tilt plane fit");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || p.device < 0 || p.device >= ndev)
    return fail(nullptr, DDH_E_CUDA, "ddh_create: CUDA device not available");
  if (cudaSetDevice(p.device) != cudaSuccess) return fail(nullptr, DDH_E_CUDA, "ddh_create: cudaSetDevice failed");

  ddh_ctx *c = new ddh_ctx();
  c->p = p;
  c->p.aperture_mask = nullptr;  // not retained
  c->p.aperture_diam = diam;
  c->st = (cudaStream_t)cuda_stream;
  c->n = n;
  c->S = p.streams;
  c->P = (size_t)n * n;
  std::memcpy(c->minv, minv, sizeof(minv));
  c->nb0 = ddh::k0_blocks(n);
  c->nb1 = n / ddh::row_block_rows(n);
  c->strehl_nb = n / ddh::col_block_cols(n);
  // launch group: all streams up to an 8 GiB workspace cap (~40-48 B/px per
  // stream); one launch per kernel per step keeps the grids large (c4, 512
  // streams at 512^2 = 5.4 GB in one group: 106.9 -> 109.0 k frames/s
  // against 204-stream groups)
  int sc = p.chunk_streams;
  if (sc <= 0) {
    const double bytes = 48.0 * (double)c->P;
    sc = (int)std::max(1.0, std::floor(8.0 * 1024 * 1024 * 1024 / bytes));
  }
  c->sc = std::min(sc, c->S);
  const size_t S = c->S, P = c->P, SC = c->sc;

  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  A(dalloc(&c->r, S * P));
  A(dalloc(&c->phi[0], S * P));
  A(dalloc(&c->phi[1], S * P));
  // spectrum, r0 and q in one allocation [cbuf | r0 | q] (one persisting-L2 window can cover any of them)
  A(dalloc(&c->cbuf, 2 * SC * P));
  c->rinit = c->cbuf ? reinterpret_cast<float *>(c->cbuf + SC * P) : nullptr;
  c->q = c->rinit ? c->rinit + SC * P : nullptr;
  A(dalloc(&c->cc, SC * P));
  A(dalloc(&c->theta, SC * P));
  A(dalloc(&c->tw4, (size_t)n));
  if (p.icd_sweeps > 1) {
    A(dalloc(&c->rtmp[0], SC * P));
    A(dalloc(&c->rtmp[1], SC * P));
    A(dalloc(&c->ptmp[0], SC * P));
    A(dalloc(&c->ptmp[1], SC * P));
  }
  A(dalloc(&c->part0, SC * std::max(c->nb0, ddh::stream_nb0(n)) * 5));
  A(dalloc(&c->part1, SC * std::max(std::max(c->nb1, 16), ddh::stream_nb1(n))));
  A(dalloc(&c->stats, SC * 5));
  A(dalloc(&c->sstat, SC * 8));
  A(dalloc(&c->psum[0], S * 3));
  A(dalloc(&c->psum[1], S * 3));
  A(dalloc(&c->pmax, SC * c->strehl_nb));
  A(dalloc(&c->rowspan, (size_t)n));
  A(dalloc(&c->tw, (size_t)n));
  if (e != cudaSuccess) {
    free_ctx(c);
    return fail(nullptr, e == cudaErrorMemoryAllocation ? DDH_E_NOMEM : DDH_E_CUDA,
                std::string("ddh_create: allocation failed: ") + cudaGetErrorString(e));
  }
  // twiddles W_N^m = e^{-2 pi i m/N}, FP64 -> FP32
  std::vector<float2> tw(n);
  for (int m = 0; m < n; ++m) {
    const double ang = -2.0 * M_PI * (double)m / (double)n;
    tw[m] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  A(cudaMemcpy(c->tw, tw.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
  {  // packed twiddles (w.x, w.y, -w.y, w.x) of the streaming path
    std::vector<float4> tw4(n);
    for (int m = 0; m < n; ++m) tw4[m] = make_float4(tw[m].x, tw[m].y, -tw[m].y, tw[m].x);
    A(cudaMemcpy(c->tw4, tw4.data(), n * sizeof(float4), cudaMemcpyHostToDevice));
  }
  A(cudaMemcpy(c->rowspan, span.data(), n * sizeof(int2), cudaMemcpyHostToDevice));
  A(ddh::init_kernels(n));
  {
    const char *pe = std::getenv("DDH_PATH");  // diagnostic override: stream | cluster | multipass
    const std::string path = pe ? pe : "";
    if (path == "multipass" || (path.empty() && (p.flags & DDH_F_UNFUSED))) {
      c->streaming = false;
    } else {
      c->streaming = true;
    }
  }
  {
    const char *gr = std::getenv("DDH_GRAPHS");  // diagnostic override
    c->graphs = gr ? std::atoi(gr) != 0 : (p.flags & DDH_F_GRAPHS) != 0;
  }
  if (c->streaming) A(ddh::init_stream(n));
  if (c->streaming) {  // call graphs (DDH_F_CALL_GRAPHS; DDH_CALL_GRAPHS=0/1 overrides; DDH_CHUNK: frames per graph)
    const char *cg = std::getenv("DDH_CALL_GRAPHS");
    const char *ck = std::getenv("DDH_CHUNK");
    c->call_graphs = cg ? std::atoi(cg) != 0 : (p.flags & DDH_F_CALL_GRAPHS) && !(p.flags & DDH_F_SERIAL);
    c->chunk = std::max(2, ck ? std::atoi(ck) : 8);
    if (const char *hd = std::getenv("DDH_HOST_DELAY_US")) c->host_delay_us = std::atof(hd);
    const char *ad = std::getenv("DDH_ADAPTIVE_GRAPHS");  // 0 off, 1 on, 2 test mode
    c->adapt = (p.flags & (DDH_F_SERIAL | DDH_F_GRAPHS)) ? 0
               : ad ? std::atoi(ad)
                    : ((p.flags & DDH_F_NO_ADAPTIVE_GRAPHS) || (cg && std::atoi(cg) == 0)) ? 0 : 1;
    A(cudaMalloc((void **)&c->desc, sizeof(CallDesc)));
    A(cudaMemset(c->desc, 0, sizeof(CallDesc)));
  }
  if (c->streaming) {
    const char *ev = std::getenv("DDH_LANES");  // diagnostic override
    c->lanes = (p.flags & DDH_F_SERIAL) ? 1 : ev ? std::atoi(ev) : p.lanes;
    if (c->lanes <= 0) {  // auto: up to 3 lanes, each keeping the large-launch kernels
      // (ICD tiles of 64 / r-ICD colour passes: >= 2 64-tiles per SM) and >= 16 streams
      // (c3, 64 streams at 256^2: 1 lane 140.8, 2 lanes 126.5, 3 lanes 125.6 us per step)
      int sms = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const long tiles = (long)(n / 64) * (n / 64);
      c->lanes = 1;
      for (int L = 3; L > 1; --L)
        if (c->sc / L >= 16 && tiles * (c->sc / L) >= 2L * sms) {
          c->lanes = L;
          break;
        }
    }
    c->lanes = std::max(1, std::min(8, c->lanes));
    if (c->lanes > 1) {
      {  // diagnostic: DDH_LANE_PRIO = priority of the lane streams (lower = higher priority)
        const char *lp = std::getenv("DDH_LANE_PRIO");
        for (int l = 0; l < c->lanes; ++l) {
          if (lp) A(cudaStreamCreateWithPriority(&c->lane_st[l], cudaStreamNonBlocking, std::atoi(lp)));
          else A(cudaStreamCreateWithFlags(&c->lane_st[l], cudaStreamNonBlocking));
        }
      }
      for (int l = 0; l < 9; ++l) A(cudaEventCreateWithFlags(&c->lane_ev[l], cudaEventDisableTiming));
    }
    const char *sr = std::getenv("DDH_SPLIT_R");  // diagnostic override
    c->split_r = c->streaming && !(p.flags & DDH_F_SERIAL) && (sr ? std::atoi(sr) != 0 : true);
    const char *ch = std::getenv("DDH_CHAIN");
    c->chain = c->streaming && ddh::chain_fits(n) && (ch ? std::atoi(ch) != 0 : true);
    c->chain_force = c->chain && ch && std::atoi(ch) == 1;
    if (c->chain) {
      int sms = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      c->chain_slots = ddh::chain_ctas_per_sm() * sms;
    }

    if (c->split_r) {
      for (int l = 0; l < c->lanes; ++l) {
        {  // diagnostic: DDH_SIDE_PRIO = priority of the r-ICD side streams (lower = higher priority)
          const char *sp = std::getenv("DDH_SIDE_PRIO");
          if (sp) A(cudaStreamCreateWithPriority(&c->side_st[l], cudaStreamNonBlocking, std::atoi(sp)));
          else A(cudaStreamCreateWithFlags(&c->side_st[l], cudaStreamNonBlocking));
        }
        A(cudaEventCreateWithFlags(&c->side_fork[l], cudaEventDisableTiming));
        A(cudaEventCreateWithFlags(&c->side_join[l], cudaEventDisableTiming));
        A(cudaStreamCreateWithFlags(&c->ypf_st[l], cudaStreamNonBlocking));
        A(cudaEventCreateWithFlags(&c->ypf_fork[l], cudaEventDisableTiming));
        A(cudaEventCreateWithFlags(&c->ypf_join[l], cudaEventDisableTiming));
      }
    }
  }
  // Streaming path: the spectrum buffer is written by S1 and read / rewritten
  // by S2, S4 and S5 within a step; a persisting-L2 window over it keeps it
  // resident against the frames and state streaming through (c3: 32 MiB,
  // 449.7 -> 455.5 k frames/s; a larger carve-out than the buffer, or a
  // partial window over a buffer much larger than L2, does not pay).  The
  // carve-out is a device-wide limit; DDH_L2P=0 disables it (diagnostic).
  if (c->streaming && (p.flags & DDH_F_L2_PERSIST)) {
    const char *pl = std::getenv("DDH_L2P");
    const size_t cb = SC * P * sizeof(float2);
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, p.device);
    if ((!pl || std::atoi(pl) != 0) && cb <= ((size_t)48 << 20) && cb <= (size_t)maxp) {
      std::lock_guard<std::mutex> lk(g_l2_mu);
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (g_l2_users[p.device & 63] == 0) g_l2_prev[p.device & 63] = cur;
      // best effort (not available under some sharing modes): failures are ignored
      if (cur >= cb || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, cb) == cudaSuccess) {
        ++g_l2_users[p.device & 63];
        c->l2_window = true;
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.base_ptr = c->cbuf;
        v.accessPolicyWindow.num_bytes = cb;
        v.accessPolicyWindow.hitRatio = 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        // only the library's own streams (lanes, r-ICD side streams); the
        // caller's stream is left as it is
        // the r-ICD side streams' window covers r0 and q (read four times by the colour
        // passes) when the carve-out allows both windows (c3: 509.2 -> 510.3 k frames/s;
        // one window over spectrum, r0 and q on every stream: 509.3 k)
        const char *ps = std::getenv("DDH_L2P_SIDE");  // diagnostic: 0 = the spectrum window everywhere
        cudaStreamAttrValue vs = v;
        const size_t rq = 2 * SC * P * sizeof(float);
        const bool side_rq = (!ps || std::atoi(ps) != 0) && cb + rq <= (size_t)maxp &&
                             cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, cb + rq) == cudaSuccess;
        if (side_rq) {
          vs.accessPolicyWindow.base_ptr = c->rinit;
          vs.accessPolicyWindow.num_bytes = rq;
        }
        for (int l = 0; l < 8; ++l) {
          if (c->lane_st[l]) cudaStreamSetAttribute(c->lane_st[l], cudaStreamAttributeAccessPolicyWindow, &v);
          if (c->side_st[l]) cudaStreamSetAttribute(c->side_st[l], cudaStreamAttributeAccessPolicyWindow, &vs);
        }
      }
      cudaGetLastError();
    }
  }
  // state: n = 0, r = r_min, phi = 0 (Fig. 1; R14)
  A(ddh::launch_fill(c->r, (float)p.r_min, S * P, c->st));
  A(cudaMemsetAsync(c->phi[0], 0, S * P * sizeof(float), c->st));
  A(cudaMemsetAsync(c->phi[1], 0, S * P * sizeof(float), c->st));
  A(cudaMemsetAsync(c->psum[0], 0, S * 3 * sizeof(double), c->st));  // the sums of phi = 0
  c->psum_valid = true;
  A(cudaStreamSynchronize(c->st));
  if (e != cudaSuccess) {
    free_ctx(c);
    return fail(nullptr, DDH_E_CUDA, std::string("ddh_create: ") + cudaGetErrorString(e));
  }
  c->launches = 1;
  // Strehl denominator max |F_c^{-1}(a)|^2 ("back-propagation through a vacuum")
  {
    StrehlArgs s{};
    s.n = n;
    s.nb = c->strehl_nb;
    s.phi_hat = nullptr;
    s.phi_true = nullptr;
    s.part0 = c->part0;
    s.nb0 = c->nb0;
    std::memcpy(s.minv, c->minv, sizeof(s.minv));
    s.rowspan = c->rowspan;
    s.tw = c->tw;
    s.cbuf = c->cbuf;
    s.pmax = c->pmax;
    A(ddh::launch_strehl(s, 1, c->st));
    std::vector<float> pm(c->strehl_nb);
    A(cudaMemcpyAsync(pm.data(), c->pmax, pm.size() * sizeof(float), cudaMemcpyDeviceToHost, c->st));
    A(cudaStreamSynchronize(c->st));
    double m = 0;
    for (float v : pm) m = std::max(m, (double)v);
    c->strehl_den = m;
    c->launches += 2;
  }
  if (e != cudaSuccess) {
    free_ctx(c);
    return fail(nullptr, DDH_E_CUDA, std::string("ddh_create: ") + cudaGetErrorString(e));
  }
  *out = c;
  return DDH_OK;
}

ddh_status ddh_destroy(ddh_ctx *c) {
  if (!c) return DDH_E_INVAL;
  cudaSetDevice(c->p.device);
  if (c->d2h_st) cudaStreamSynchronize(c->d2h_st);
  cudaStreamSynchronize(c->st);
  free_ctx(c);
  return DDH_OK;
}

ddh_status ddh_bootstrap(ddh_ctx *c, const void *y0, int32_t k_b, uint8_t *status) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (k_b < 0 || (!y0 && k_b > 0)) return fail(c, DDH_E_INVAL, "ddh_bootstrap: bad arguments");
  if ((uintptr_t)y0 & 15) return fail(c, DDH_E_INVAL, "ddh_bootstrap: y0 must be 16-byte aligned");
  if (k_b == 0) return DDH_OK;
  DDH_CK(c, cudaSetDevice(c->p.device));
  s = run_frame(c, (const float2 *)y0, nullptr, nullptr, status, Mode::Boot, k_b);
  if (s != DDH_OK) return s;
  c->frame += 1;
  return DDH_OK;
}

ddh_status ddh_step(ddh_ctx *c, const void *y, int32_t T, float *phi_out, float *r_out, uint8_t *status) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (T < 0 || (!y && T > 0)) return fail(c, DDH_E_INVAL, "ddh_step: bad arguments");
  if (((uintptr_t)y & 15) || ((uintptr_t)phi_out & 7) || ((uintptr_t)r_out & 7))
    return fail(c, DDH_E_INVAL, "ddh_step: y must be 16-byte aligned, phi_out / r_out 8-byte aligned");
  DDH_CK(c, cudaSetDevice(c->p.device));
  const size_t fs = (size_t)c->S * c->P;
  int t = 0;
  // whole chunks from call graphs (one launch group, no profiling; frames still in
  // flight from the host pipeline are ordered by the ctx stream)
  if (c->call_graphs && c->streaming && !use_chain(c, c->p.n_k) && !c->profiling && c->sc == c->S &&
      !c->y_prefetched) {
    for (; t + c->chunk <= T; t += c->chunk) {
      s = run_chunk(c, (const float2 *)y + t * fs, phi_out ? phi_out + t * fs : nullptr,
                    r_out ? r_out + t * fs : nullptr, status ? status + (size_t)t * c->S : nullptr, c->chunk);
      if (s != DDH_OK) return s;
      c->frame += c->chunk;
    }
  }
  // Adaptive call graphs: directly launched frames need ~105 us of host time each at c3, a
  // little less than the device needs, so a slow host makes a long call enqueue-bound (c3,
  // 300 frames, the enqueue thread sharing its core: 552 k -> 330-350 k frames/s; from graphs
  // 541 k either way, profiles/r02i_graphs_ab.txt).  When the device is found waiting for the
  // host (below), the rest of the call runs from chunk graphs (~2 % slower on the device, ~2 us of
  // host time per frame).  Only with at least four chunks left (a capture costs ~ms once).
  const bool can_adapt = c->adapt > 0 && c->streaming && !c->call_graphs && !use_chain(c, c->p.n_k) &&
                         !c->profiling && c->sc == c->S;
  // a ctx that switched keeps its next four long calls on graphs from their first frame
  // (a busy host cannot be observed from a graph call), then probes again
  bool graph_mode = can_adapt && c->adapt_hot > 0 && T > 4 * c->chunk;
  if (graph_mode) --c->adapt_hot;
  // The observable: when the host has enqueued frame t-1 and is about to enqueue frame t, is
  // frame t-2 already complete?  A device-bound pipeline keeps at least one whole frame of
  // backlog (the host runs ahead: at c3 by 11 us more per frame), a host-bound one executes
  // kernels as they arrive.  (The ctx stream itself is never found drained at a frame boundary:
  // the kernels enqueued last are still running.)  Checked from frame 8 on (the host's lead has
  // built up by then); three consecutive observations switch.
  const bool probing = can_adapt && !graph_mode && T > 4 * c->chunk + 8;
  int consec = 0;
  if (probing && !c->adapt_ev[0]) {
    DDH_CK(c, cudaEventCreateWithFlags(&c->adapt_ev[0], cudaEventDisableTiming));
    DDH_CK(c, cudaEventCreateWithFlags(&c->adapt_ev[1], cudaEventDisableTiming));
  }
  while (t < T) {
    if (graph_mode && !c->y_prefetched && t + c->chunk <= T) {
      s = run_chunk(c, (const float2 *)y + t * fs, phi_out ? phi_out + t * fs : nullptr,
                    r_out ? r_out + t * fs : nullptr, status ? status + (size_t)t * c->S : nullptr, c->chunk);
      if (s != DDH_OK) return s;
      c->frame += c->chunk;
      t += c->chunk;
      continue;
    }
    if (probing && !graph_mode && t >= 8 && T - t > 4 * c->chunk) {
      const cudaError_t q = c->adapt == 2 ? cudaSuccess : cudaEventQuery(c->adapt_ev[t & 1]);  // end of frame t-2
      if (q == cudaSuccess) {
        if (++consec >= 3) graph_mode = true, ++c->adapt_switches, c->adapt_hot = 4;
      } else if (q == cudaErrorNotReady) {
        consec = 0;
      } else {
        DDH_CK(c, q);
      }
    }
    if (c->host_delay_us > 0) {  // diagnostic (DDH_HOST_DELAY_US): a uniformly slower host, per directly launched frame
      const auto t0 = std::chrono::steady_clock::now();
      while (std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() < c->host_delay_us) {
      }
    }
    // the frame before the first chunk prefetches nothing (chunks start with no cross-frame work pending)
    const bool pf = t + 1 < T && !(graph_mode && t + 1 + c->chunk <= T);
    s = step_frame(c, (const float2 *)y + t * fs, phi_out ? phi_out + t * fs : nullptr,
                   r_out ? r_out + t * fs : nullptr, status ? status + (size_t)t * c->S : nullptr,
                   pf ? (const float2 *)y + (t + 1) * fs : nullptr);
    if (s != DDH_OK) return s;
    if (probing && !graph_mode) DDH_CK(c, cudaEventRecord(c->adapt_ev[t & 1], c->st));  // end of frame t
    c->frame += 1;
    ++t;
  }
  return DDH_OK;
}

ddh_status ddh_static(ddh_ctx *c, const void *y, int32_t T, int32_t iters, float *phi_out, float *r_out,
                      uint8_t *status) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (T < 0 || iters < 1 || (!y && T > 0)) return fail(c, DDH_E_INVAL, "ddh_static: bad arguments");
  if (((uintptr_t)y & 15) || ((uintptr_t)phi_out & 7) || ((uintptr_t)r_out & 7))
    return fail(c, DDH_E_INVAL, "ddh_static: y must be 16-byte aligned, phi_out / r_out 8-byte aligned");
  DDH_CK(c, cudaSetDevice(c->p.device));
  const size_t fs = (size_t)c->S * c->P;
  for (int t = 0; t < T; ++t) {
    s = run_frame(c, (const float2 *)y + t * fs, phi_out ? phi_out + t * fs : nullptr,
                  r_out ? r_out + t * fs : nullptr, status ? status + (size_t)t * c->S : nullptr, Mode::Boot,
                  iters);
    if (s != DDH_OK) return s;
    c->frame += 1;
  }
  return DDH_OK;
}

namespace {
// Host-buffer path: frame t of the pipeline uses stage k = t mod 3.  H2D(t)
// waits for the step of t-3 (reader of y_stage[k]); the step of t waits for
// H2D(t) and for D2H(t-3) (reader of the output stages); D2H(t) waits for the
// step of t.  `host_t` continues across asynchronous calls, so consecutive
// calls keep the copy pipeline full; a synchronous call (or ddh_sync) drains it.
ddh_status step_host_impl(ddh_ctx *c, const void *y_host, int32_t T, float *phi_out, float *r_out,
                          uint8_t *status, bool sync) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (T < 0 || (!y_host && T > 0)) return fail(c, DDH_E_INVAL, "ddh_step_host: bad arguments");
  DDH_CK(c, cudaSetDevice(c->p.device));
  const size_t fs = (size_t)c->S * c->P;
  if (!c->y_stage[0]) {
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < ddh_ctx::kStages && e == cudaSuccess; ++k) {
      e = dalloc(&c->y_stage[k], fs);
      if (e == cudaSuccess) e = dalloc(&c->phi_stage[k], fs);
      if (e == cudaSuccess) e = dalloc(&c->r_stage[k], fs);
      if (e == cudaSuccess) e = dalloc(&c->status_stage[k], (size_t)c->S);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->h2d_ev[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->comp_ev[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->d2h_ev[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->h2d_st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->d2h_st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(c, DDH_E_NOMEM, "ddh_step_host: staging allocation failed");
  }
  // on any error after copies were enqueued: wait for them (best effort) so that
  // no copy into or out of the caller's host buffers is in flight on return
  auto drain = [c](ddh_status st) {
    cudaStreamSynchronize(c->h2d_st);
    cudaStreamSynchronize(c->d2h_st);
    cudaGetLastError();
    c->host_pending = false;
    return st;
  };
#define DDH_HCK(call)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return drain(fail(c, DDH_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)));   \
  } while (0)
  if (!c->host_pending) {  // order after prior work on the ctx stream (fresh pipeline)
    for (int k = 0; k < ddh_ctx::kStages; ++k) {
      DDH_HCK(cudaEventRecord(c->comp_ev[k], c->st));
      DDH_HCK(cudaEventRecord(c->d2h_ev[k], c->st));
    }
    c->host_t = 0;
  }
  c->host_pending = true;
  for (int t = 0; t < T; ++t) {
    const int k = (int)((c->host_t++) % ddh_ctx::kStages);
    DDH_HCK(cudaStreamWaitEvent(c->h2d_st, c->comp_ev[k], 0));
    DDH_HCK(cudaMemcpyAsync(c->y_stage[k], (const float2 *)y_host + t * fs, fs * sizeof(float2),
                            cudaMemcpyHostToDevice, c->h2d_st));
    DDH_HCK(cudaEventRecord(c->h2d_ev[k], c->h2d_st));
    DDH_HCK(cudaStreamWaitEvent(c->st, c->h2d_ev[k], 0));
    DDH_HCK(cudaStreamWaitEvent(c->st, c->d2h_ev[k], 0));
    s = run_frame(c, c->y_stage[k], phi_out ? c->phi_stage[k] : nullptr, r_out ? c->r_stage[k] : nullptr,
                  status ? c->status_stage[k] : nullptr, Mode::Step, c->p.n_k);
    if (s != DDH_OK) return drain(s);
    c->frame += 1;
    DDH_HCK(cudaEventRecord(c->comp_ev[k], c->st));
    DDH_HCK(cudaStreamWaitEvent(c->d2h_st, c->comp_ev[k], 0));
    if (phi_out)
      DDH_HCK(cudaMemcpyAsync(phi_out + t * fs, c->phi_stage[k], fs * sizeof(float), cudaMemcpyDeviceToHost, c->d2h_st));
    if (r_out)
      DDH_HCK(cudaMemcpyAsync(r_out + t * fs, c->r_stage[k], fs * sizeof(float), cudaMemcpyDeviceToHost, c->d2h_st));
    if (status)
      DDH_HCK(cudaMemcpyAsync(status + (size_t)t * c->S, c->status_stage[k], c->S, cudaMemcpyDeviceToHost, c->d2h_st));
    DDH_HCK(cudaEventRecord(c->d2h_ev[k], c->d2h_st));
  }
#undef DDH_HCK
  if (sync) {
    c->host_pending = false;
    DDH_CK(c, cudaStreamSynchronize(c->d2h_st));
    DDH_CK(c, cudaStreamSynchronize(c->st));
  }
  return DDH_OK;
}
}  // namespace

ddh_status ddh_step_host(ddh_ctx *c, const void *y_host, int32_t T, float *phi_out, float *r_out,
                         uint8_t *status) {
  return step_host_impl(c, y_host, T, phi_out, r_out, status, true);
}

ddh_status ddh_step_host_async(ddh_ctx *c, const void *y_host, int32_t T, float *phi_out, float *r_out,
                               uint8_t *status) {
  return step_host_impl(c, y_host, T, phi_out, r_out, status, false);
}

ddh_status ddh_get_state(ddh_ctx *c, float *r, float *phi, int64_t *frame_index) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  DDH_CK(c, cudaSetDevice(c->p.device));
  const size_t bytes = (size_t)c->S * c->P * sizeof(float);
  if (r) DDH_CK(c, cudaMemcpyAsync(r, c->r, bytes, cudaMemcpyDeviceToDevice, c->st));
  if (phi) DDH_CK(c, cudaMemcpyAsync(phi, c->phi[c->cur], bytes, cudaMemcpyDeviceToDevice, c->st));
  if (frame_index) *frame_index = c->frame;
  return DDH_OK;
}

ddh_status ddh_set_state(ddh_ctx *c, const float *r, const float *phi, int64_t frame_index) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  DDH_CK(c, cudaSetDevice(c->p.device));
  const size_t bytes = (size_t)c->S * c->P * sizeof(float);
  if (r) DDH_CK(c, cudaMemcpyAsync(c->r, r, bytes, cudaMemcpyDeviceToDevice, c->st));
  if (phi) {
    DDH_CK(c, cudaMemcpyAsync(c->phi[c->cur], phi, bytes, cudaMemcpyDeviceToDevice, c->st));
    c->psum_valid = false;  // the next S0 recomputes the RemoveTipTilt sums
  }
  c->frame = frame_index;
  return DDH_OK;
}

namespace {
ddh_status strehl_impl(ddh_ctx *c, const float *phi_hat, const float *phi_true, int32_t B, double *out, float *resid,
                       float *psf);
}

ddh_status ddh_strehl(ddh_ctx *c, const float *phi_hat, const float *phi_true, int32_t B, double *out) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (B < 0 || (B > 0 && (!phi_hat || !phi_true || !out))) return fail(c, DDH_E_INVAL, "ddh_strehl: bad arguments");
  return strehl_impl(c, phi_hat, phi_true, B, out, nullptr, nullptr);
}

ddh_status ddh_residual(ddh_ctx *c, const float *phi_hat, const float *phi_true, int32_t B, float *resid,
                        float *psf, double *strehl_out) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (B < 0 || (B > 0 && (!phi_hat || !phi_true || !strehl_out)))
    return fail(c, DDH_E_INVAL, "ddh_residual: bad arguments");
  return strehl_impl(c, phi_hat, phi_true, B, strehl_out, resid, psf);
}

namespace {
ddh_status strehl_impl(ddh_ctx *c, const float *phi_hat, const float *phi_true, int32_t B, double *out, float *resid,
                       float *psf) {
  ddh_status s = DDH_OK;
  DDH_CK(c, cudaSetDevice(c->p.device));
  std::vector<float> pm((size_t)c->sc * c->strehl_nb);
  for (int b0 = 0; b0 < B; b0 += c->sc) {
    const int bn = std::min(c->sc, B - b0);
    const size_t off = (size_t)b0 * c->P;
    StepArgs a = base_args(c, 0, bn);
    a.want_y = 0;
    a.apply_plane = 1;
    a.phi_in = phi_hat + off;
    a.phi_sub = phi_true + off;
    DDH_LAUNCH(c, K_STATS, ddh::launch_k0(a, c->st));
    StrehlArgs sa{};
    sa.n = c->n;
    sa.nb = c->strehl_nb;
    sa.phi_hat = phi_hat + off;
    sa.phi_true = phi_true + off;
    sa.part0 = c->part0;
    sa.nb0 = c->nb0;
    std::memcpy(sa.minv, c->minv, sizeof(sa.minv));
    sa.rowspan = c->rowspan;
    sa.tw = c->tw;
    sa.cbuf = c->cbuf;
    sa.pmax = c->pmax;
    sa.resid = resid ? resid + off : nullptr;
    sa.psf = psf ? psf + off : nullptr;
    sa.inv_den = (float)(1.0 / c->strehl_den);
    DDH_CK(c, ddh::launch_strehl(sa, bn, c->st));
    c->launches += 2;
    DDH_CK(c, cudaMemcpyAsync(pm.data(), c->pmax, (size_t)bn * c->strehl_nb * sizeof(float),
                              cudaMemcpyDeviceToHost, c->st));
    DDH_CK(c, cudaStreamSynchronize(c->st));
    for (int b = 0; b < bn; ++b) {
      double m = 0;
      for (int k = 0; k < c->strehl_nb; ++k) m = std::max(m, (double)pm[(size_t)b * c->strehl_nb + k]);
      out[b0 + b] = m / c->strehl_den;
    }
  }
  (void)s;
  return DDH_OK;
}
}  // namespace

ddh_status ddh_sync(ddh_ctx *c) {
  if (!c) return DDH_E_INVAL;
  DDH_CK(c, cudaSetDevice(c->p.device));
  if (c->d2h_st) {  // the host-buffer pipeline's downloads (ddh_step_host_async)
    c->host_pending = false;
    DDH_CK(c, cudaStreamSynchronize(c->d2h_st));
  }
  DDH_CK(c, cudaStreamSynchronize(c->st));
  return c->sticky ? DDH_E_STATE : DDH_OK;
}

const char *ddh_last_error(const ddh_ctx *c) {
  if (c) return c->err.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_create_err.c_str();
}

uint64_t ddh_kernel_launches(const ddh_ctx *c) { return c ? c->launches : 0; }

ddh_status ddh_profile_enable(ddh_ctx *c, int32_t enable) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  c->profiling = enable != 0;
  return DDH_OK;
}

ddh_status ddh_profile_read(ddh_ctx *c, double *ms, int64_t *launches) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (!ms || !launches) return fail(c, DDH_E_INVAL, "ddh_profile_read: NULL output");
  DDH_CK(c, cudaSetDevice(c->p.device));
  DDH_CK(c, cudaStreamSynchronize(c->st));
  for (size_t i = 0; i < c->ev_kind.size(); ++i) {
    float t = 0.f;
    DDH_CK(c, cudaEventElapsedTime(&t, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
    ms[c->ev_kind[i]] += t;
    launches[c->ev_kind[i]] += 1;
  }
  c->ev_kind.clear();
  return DDH_OK;
}

const char *ddh_kind_name(int32_t k) { return (k >= 0 && k < DDH_KIND_COUNT) ? kKindNames[k] : "?"; }

int64_t ddh_frame_index(const ddh_ctx *c) { return c ? c->frame : -1; }

ddh_status ddh_test_fft2c(ddh_ctx *c, const void *in, void *out, int32_t B, int32_t inverse) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (B < 0 || (B > 0 && (!in || !out))) return fail(c, DDH_E_INVAL, "ddh_test_fft2c: bad arguments");
  if (B == 0) return DDH_OK;
  DDH_CK(c, cudaSetDevice(c->p.device));
  if (c->streaming)  // the register FFT of S1 / S2 / S4 (ks_test_rows + ks_test_cols)
    DDH_CK(c, ddh::launch_test_fft_stream(c->n, (const float2 *)in, (float2 *)out, B, inverse, c->tw4, c->st));
  else
    DDH_CK(c, ddh::launch_test_fft2c(c->n, (const float2 *)in, (float2 *)out, B, inverse, c->tw, c->st));
  c->launches += 2;
  return DDH_OK;
}

namespace {
ddh_status ensure_test_parts(ddh_ctx *c) {
  if (c->test_part0) return DDH_OK;
  const size_t n0 = (size_t)c->sc * std::max(c->nb0, ddh::stream_nb0(c->n)) * 5;
  const size_t n1 = (size_t)c->sc * std::max(std::max(c->nb1, 16), ddh::stream_nb1(c->n));
  DDH_CK(c, dalloc(&c->test_part0, n0));
  DDH_CK(c, dalloc(&c->test_part1, n1));
  DDH_CK(c, dalloc(&c->test_sstat, (size_t)c->sc * 8));
  DDH_CK(c, cudaMemset(c->test_sstat, 0, (size_t)c->sc * 8 * sizeof(float)));  // no plane, not degenerate
  std::vector<double> ones(n1, 1.0);
  DDH_CK(c, cudaMemset(c->test_part0, 0, n0 * sizeof(double)));
  DDH_CK(c, cudaMemcpy(c->test_part1, ones.data(), n1 * sizeof(double), cudaMemcpyHostToDevice));
  return DDH_OK;
}

// StepArgs for a streaming ICD stage entry point over streams [b0, b0 + bn) of caller buffers
StepArgs test_icd_args(ddh_ctx *c, int bn) {
  StepArgs a = base_args(c, 0, bn);
  a.nb0 = ddh::stream_nb0(c->n);
  a.nb1 = ddh::stream_nb1(c->n);
  a.part0 = c->test_part0;
  a.part1 = c->test_part1;
  a.sstat = c->test_sstat;
  a.apply_plane = 0;
  return a;
}
}  // namespace

ddh_status ddh_test_ricd(ddh_ctx *c, const float *r_in, const float *q, int32_t B, float *r_out) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (B < 0 || (B > 0 && (!r_in || !q || !r_out))) return fail(c, DDH_E_INVAL, "ddh_test_ricd: bad arguments");
  if (B == 0) return DDH_OK;
  DDH_CK(c, cudaSetDevice(c->p.device));
  if (!c->streaming) {
    if (c->p.icd_sweeps > 1 && B > c->sc) return fail(c, DDH_E_INVAL, "ddh_test_ricd: B > chunk with sweeps > 1");
    return run_ricd(c, r_in, q, r_out, nullptr, nullptr, B);
  }
  if ((s = ensure_test_parts(c)) != DDH_OK) return s;
  const int sw = c->p.icd_sweeps;
  for (int b0 = 0; b0 < B; b0 += c->sc) {  // S3, icd_sweeps sweeps, per launch group
    const int bn = std::min(c->sc, B - b0);
    const size_t off = (size_t)b0 * c->P;
    StepArgs a = test_icd_args(c, bn);
    a.q = const_cast<float *>(q) + off;
    for (int k = 0; k < sw; ++k) {
      a.icd_in = k == 0 ? r_in + off : c->rtmp[(k - 1) & 1];
      a.icd_out = k == sw - 1 ? r_out + off : c->rtmp[k & 1];
      a.icd_copy = nullptr;
      DDH_LAUNCH(c, K_S3, ddh::launch_s3(a, c->st));
      c->launches += ddh::icd_launches(a, true) - 1;
    }
  }
  return DDH_OK;
}

ddh_status ddh_test_phiicd(ddh_ctx *c, const float *phi_in, const float *cc, const float *theta, int32_t B,
                           float *phi_out) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (B < 0 || (B > 0 && (!phi_in || !cc || !theta || !phi_out)))
    return fail(c, DDH_E_INVAL, "ddh_test_phiicd: bad arguments");
  if (B == 0) return DDH_OK;
  DDH_CK(c, cudaSetDevice(c->p.device));
  if (!c->streaming) {
    if (c->p.icd_sweeps > 1 && B > c->sc) return fail(c, DDH_E_INVAL, "ddh_test_phiicd: B > chunk with sweeps > 1");
    return run_phiicd(c, phi_in, cc, theta, phi_out, nullptr, nullptr, nullptr, 0, B);
  }
  if ((s = ensure_test_parts(c)) != DDH_OK) return s;
  const int sw = c->p.icd_sweeps;
  for (int b0 = 0; b0 < B; b0 += c->sc) {  // (c, theta) pairs as S4 leaves them, then S5 sweeps
    const int bn = std::min(c->sc, B - b0);
    const size_t off = (size_t)b0 * c->P;
    DDH_CK(c, ddh::launch_test_pack(cc + off, theta + off, c->cbuf, (size_t)bn * c->P, c->st));
    c->launches++;
    StepArgs a = test_icd_args(c, bn);
    for (int k = 0; k < sw; ++k) {
      a.icd_in = k == 0 ? phi_in + off : c->ptmp[(k - 1) & 1];
      a.icd_out = k == sw - 1 ? phi_out + off : c->ptmp[k & 1];
      a.icd_copy = nullptr;
      DDH_LAUNCH(c, K_S5, ddh::launch_s5(a, c->st));
      c->launches += ddh::icd_launches(a, false) - 1;
    }
  }
  return DDH_OK;
}

ddh_status ddh_test_estep(ddh_ctx *c, const void *u, const float *r_prev, int32_t B, int32_t warm, float *r0,
                          void *mu, float *q) {
  ddh_status s = check_usable(c);
  if (s != DDH_OK) return s;
  if (B < 0 || (B > 0 && (!u || !r_prev || !r0 || !mu || !q))) return fail(c, DDH_E_INVAL, "ddh_test_estep: bad arguments");
  if (B == 0) return DDH_OK;
  DDH_CK(c, cudaSetDevice(c->p.device));
  DDH_CK(c, ddh::launch_test_estep((const float2 *)u, r_prev, r0, (float2 *)mu, q, (size_t)B * c->P, warm,
                                   (float)(1.0 - c->p.lambda), (float)(c->p.lambda * c->p.alpha),
                                   (float)c->p.r_min, (float)c->p.noise_var, c->st));
  c->launches++;
  return DDH_OK;
}

}  // extern "C"
