// ddh_chain.cu -- the on-chip multi-iteration chain for
// N = 64: one CTA per stream holds the whole frame (y, the complex work
// array, r, q / c, theta, phi: 97 KB of shared memory, two CTAs per SM; y is re-read from L2) and runs Fig. 1's
// loop body for the frame -- Normalize (Eq. 4), RemoveTipTilt,
// then N_k x [FFT1 = back-projection (Eq. 3 on the first), E-step, qGGMRF
// r-ICD, FFT2 + phase correlation, GMRF phi-ICD] -- reading y, r and phi from
// HBM once and writing r and phi once, whatever N_k is.  Each extra EM
// iteration costs shared-memory passes only (the streaming path's six
// kernels move ~112 B/px through HBM / L2 per iteration).
//
// The arithmetic is the other paths': the multi-pass path's Stockham FFT and
// elementwise stages (ddh_kernels.cu K1-K3a), the streaming path's packed
// qGGMRF weights, E-step reciprocal, reduced sincos and polynomial atan2
// (ddh_common.cuh), r_update / phi_update; reductions in FP64 in a fixed order.
// Parity with the oracle in tests/test_gpu_parity.py (test_chain_*).
#include "ddh_common.cuh"
#include "ddh_fft.cuh"
#include "ddh_kernels.h"

namespace ddh {
namespace {

constexpr int kCN = 64, kCP = kCN * kCN, kCPitch = kCN + 1, kCThreads = 512;
// phi with a zero border (pitch N + 2): the free-boundary neighbours read 0 without a test
constexpr int kPP = kCN + 2;
__device__ __forceinline__ int pidx(int i, int j) { return (i + 1) * kPP + j + 1; }

#ifndef DDH_CHAIN_MINB
#define DDH_CHAIN_MINB 2
#endif
// y stays in global memory (L2-resident after the first read; 32 KB more shared
// memory per CTA would leave one CTA per SM instead of two)
struct ChainSmem {
  float2 X[kCN * kCPitch];  // complex work array (row pitch N + 1)
  float rs[kCP];            // r (in place through Eq. 3 and the r-ICD)
  float qs[kCP];            // q (E-step), then c (phase correlation)
  float ts[kCP];            // theta
  float ps[kPP * kPP];      // phi (plane removed), zero border
  float2 tw[kCN];
  int2 span[kCN];
  double red[32 * 5];
  double scal[8];
};

// One qGGMRF r update of pixel (i, j) (R6-R9, periodic 8-neighbourhood) in
// place: the streaming path's packed-pair weights (qgg_w2) and the shared root
// finder r_update
__device__ __forceinline__ void chain_rupd(float *rs, const float *qs, int i, int j, const StepArgs &A) {
  const int im = ((i - 1) & (kCN - 1)) * kCN, i0 = i * kCN, ip = ((i + 1) & (kCN - 1)) * kCN;
  const int jm = (j - 1) & (kCN - 1), jp = (j + 1) & (kCN - 1);
  DDH_DBG(i >= 0 && i < kCN && j >= 0 && j < kCN);
  const float ri = rs[i0 + j];
  const float2 nA = make_float2(rs[im + j], rs[ip + j]), nB = make_float2(rs[i0 + jm], rs[i0 + jp]);
  const float2 dA = make_float2(rs[im + jm], rs[im + jp]), dB = make_float2(rs[ip + jm], rs[ip + jp]);
  const float2 wA = qgg_w2(ri, nA, A.r_h, A.r_g, A.r_k), wB = qgg_w2(ri, nB, A.r_h, A.r_g, A.r_k);
  const float2 wC = qgg_w2(ri, dA, A.r_h, A.r_g, A.r_k), wD = qgg_w2(ri, dB, A.r_h, A.r_g, A.r_k);
  const float2 bs = p_fma(p_add(wC, wD), bc2(0.5f), p_add(wA, wB));
  const float2 ss = p_fma(p_fma(wC, dA, p_mul(wD, dB)), bc2(0.5f), p_fma(wA, nA, p_mul(wB, nB)));
  rs[i0 + j] = r_update(ri, qs[i0 + j], A.r_b6 * (bs.x + bs.y), A.r_b6 * (ss.x + ss.y), A.r_min);
}

// One GMRF phi update of pixel (i, j) (R10-R11) in place, free boundary: the
// neighbours outside the frame read the zero border and are dropped from sum b
// (the streaming path's edge expression), so no lane of a warp diverges
__device__ __forceinline__ void chain_phiupd(float *ps, const float *cs, const float *ts, int i, int j,
                                             const StepArgs &A) {
  const int g = i * kCN + j, gp = pidx(i, j);
  DDH_DBG(i >= 0 && i < kCN && j >= 0 && j < kCN);
  float nb = 0.f, sb = 0.f;
  if (A.phi_prior) {
    const float n4 = (ps[gp - kPP] + ps[gp + kPP]) + (ps[gp - 1] + ps[gp + 1]);
    const float nd = (ps[gp - kPP - 1] + ps[gp - kPP + 1]) + (ps[gp + kPP - 1] + ps[gp + kPP + 1]);
    nb = fmaf(nd, 1.f / 12.f, n4 * (1.f / 6.f));
    const bool tp = i == 0, bt = i == kCN - 1, lf = j == 0, rt = j == kCN - 1;
    sb = 1.f - (1.f / 6.f) * (float)(tp + bt + lf + rt) -
         (1.f / 12.f) * (float)((tp | lf) + (tp | rt) + (bt | lf) + (bt | rt));
  }
  ps[gp] = phi_update(ps[gp], cs[g], ts[g], nb, sb, A.phi_w, A.phi_prior != 0);
}

__global__ void __launch_bounds__(kCThreads, DDH_CHAIN_MINB) ks_chain(ChainArgs C) {
  const StepArgs &A = C.a;
  extern __shared__ __align__(16) unsigned char chain_sm[];
  ChainSmem &M = *reinterpret_cast<ChainSmem *>(chain_sm);
  const int tid = threadIdx.x, s = blockIdx.x;
  const size_t off = (size_t)s * kCP;
  if (tid < kCN) {
    M.tw[tid] = A.tw[tid];
    M.span[tid] = A.rowspan[tid];
  }
  for (int k = tid; k < 4 * (kCN + 1); k += kCThreads) {  // the zero border of phi
    const int e = k / (kCN + 1), t = k % (kCN + 1);
    const int idx = e == 0 ? t : e == 1 ? (kCN + 1) * kPP + t + 1 : e == 2 ? (t + 1) * kPP : t * kPP + kCN + 1;
    M.ps[idx] = 0.f;
  }
  __syncthreads();
  auto ap = [&](int i, int j) { return j >= M.span[i].x && j < M.span[i].y; };
  // ---- load the frame and the state; sums for Normalize (Eq. 4) and RemoveTipTilt
  double v[5] = {0, 0, 0, 0, 0};
  for (int idx = tid; idx < kCP; idx += kCThreads) {
    const int i = idx / kCN, j = idx & (kCN - 1);
    const float2 y = A.y[off + idx];
    v[0] += (double)y.x;
    v[1] += (double)y.y;
    const float ph = A.phi_in[off + idx];
    M.ps[pidx(i, j)] = ph;
    M.rs[idx] = A.r_state[off + idx];
    if (A.apply_plane && ap(i, j)) {
      v[2] += (double)ph;
      v[3] += (double)ph * (double)(j - kCN / 2);
      v[4] += (double)ph * (double)(i - kCN / 2);
    }
  }
  block_sum<5>(v, M.red);
  if (tid == 0) {
    M.scal[0] = v[0] / kCP;
    M.scal[1] = v[1] / kCP;
    double c[3] = {0, 0, 0};
    if (A.apply_plane) plane_from_sums(v, A.minv, c);
    M.scal[2] = c[0];
    M.scal[3] = c[1];
    M.scal[4] = c[2];
  }
  __syncthreads();
  const float mur = (float)M.scal[0], mui = (float)M.scal[1];
  const float c0 = (float)M.scal[2], c1 = (float)M.scal[3], c2 = (float)M.scal[4];
  double a1[1] = {0.0};
  for (int idx = tid; idx < kCP; idx += kCThreads) {
    const float2 y = A.y[off + idx];
    const float dr = y.x - mur, di = y.y - mui;
    a1[0] += (double)dr * dr + (double)di * di;
  }
  block_sum<1>(a1, M.red);
  if (tid == 0) M.scal[5] = a1[0];
  __syncthreads();
  const double d2 = M.scal[5];
  const bool degenerate = !(d2 > 0.0);
  if (A.status && tid == 0) A.status[s] = degenerate ? 1 : 0;
  if (degenerate) {  // state unchanged (no tip/tilt removal either)
    for (int idx = tid; idx < kCP; idx += kCThreads) {
      const float p = M.ps[pidx(idx / kCN, idx & (kCN - 1))], r = M.rs[idx];
      C.phi_next[off + idx] = p;
      if (C.phi_copy) C.phi_copy[off + idx] = p;
      if (C.r_copy) C.r_copy[off + idx] = r;
    }
    return;
  }
  const float kappa = (float)sqrt((double)kCP / d2);  // Eq. 4: sqrt(p) / ||y - mu||
  const float scale = kappa / (float)kCN;             // unitary F_c = chi F chi / N
  if (A.apply_plane) {
    for (int idx = tid; idx < kCP; idx += kCThreads) {
      const int i = idx / kCN, j = idx & (kCN - 1);
      M.ps[pidx(i, j)] -= (c0 + c1 * (float)(j - kCN / 2) + c2 * (float)(i - kCN / 2));
    }
  }
  const int fb = tid % kCN, ft = tid / kCN;  // FFT: vector fb, lane ft (8 threads per 64-point vector)
  const float inv_n = 1.f / (float)kCN, two_s2 = 2.f / A.s2;
  for (int it = 0; it < C.iters; ++it) {
    __syncthreads();
    // ---- FFT1: z = chi a e^{-j phi'} (y - mu), forward rows then columns (K1, K2a)
    for (int idx = tid; idx < kCP; idx += kCThreads) {
      const int i = idx / kCN, j = idx & (kCN - 1);
      float2 z = make_float2(0.f, 0.f);
      if (ap(i, j)) {
        const float2 y = __ldg(A.y + off + idx);
        const float dr = y.x - mur, di = y.y - mui;
        float sn, cs;
        sincos_red(M.ps[pidx(i, j)], sn, cs);
        z = make_float2(dr * cs + di * sn, di * cs - dr * sn);
        if ((i + j) & 1) z = make_float2(-z.x, -z.y);
      }
      M.X[i * kCPitch + j] = z;
    }
    __syncthreads();
    block_fft<kCN, -1>(M.X + fb * kCPitch, true, ft, 1, M.tw);
    block_fft<kCN, -1>(M.X + fb, true, ft, kCPitch, M.tw);
    // ---- u = A^H y-hat; Eq. 3 warm start on the first iteration; E-step (R1)
    const bool warm = A.warm && it == 0;
    for (int idx = tid; idx < kCP; idx += kCThreads) {
      const int ki = idx / kCN, kj = idx & (kCN - 1);
      const float sg = ((ki + kj) & 1) ? -scale : scale;
      const float2 X = M.X[ki * kCPitch + kj];
      const float2 u = make_float2(X.x * sg, X.y * sg);
      const float rp = M.rs[idx];
      float r0 = rp;
      if (warm) r0 = fmaxf(fmaf(A.oml, rp, A.la * (u.x * u.x + u.y * u.y)), A.r_min);  // Eq. 3
      const float w = r0 * rcp_approx(r0 + A.s2);
      const float2 mu = make_float2(w * u.x, w * u.y);
      M.rs[idx] = r0;
      M.qs[idx] = fmaf(mu.x, mu.x, fmaf(mu.y, mu.y, w * A.s2));
      const float cs = ((ki + kj) & 1) ? -1.f : 1.f;
      M.X[ki * kCPitch + kj] = make_float2(cs * mu.x, cs * mu.y);
    }
    __syncthreads();
    // ---- r M-step: colour-ordered qGGMRF ICD in place (R6-R9), periodic
    if (A.r_prior) {
      for (int sw = 0; sw < A.sweeps; ++sw) {
        for (int c = 0; c < 4; ++c) {
          const int ci = c >> 1, cj = c & 1;
          for (int p = tid; p < kCP / 4; p += kCThreads) {
            const int i = 2 * (p / (kCN / 2)) + ci, j = 2 * (p % (kCN / 2)) + cj;
            DDH_DBG((i & 1) == ci && (j & 1) == cj);
            chain_rupd(M.rs, M.qs, i, j, A);
          }
          __syncthreads();
        }
      }
    } else {
      for (int idx = tid; idx < kCP; idx += kCThreads) M.rs[idx] = fmaxf(M.qs[idx], A.r_min);
    }
    // ---- FFT2: f = F_c^{-1} mu (inverse columns then rows: K2a, K3a)
    block_fft<kCN, +1>(M.X + fb, true, ft, kCPitch, M.tw);
    block_fft<kCN, +1>(M.X + fb * kCPitch, true, ft, 1, M.tw);
    // ---- phase correlation: c = (2/s2) a |y-hat| |f|, theta = arg(y-hat conj f)
    for (int idx = tid; idx < kCP; idx += kCThreads) {
      const int i = idx / kCN, j = idx & (kCN - 1);
      float c = 0.f, th = 0.f;
      if (ap(i, j)) {
        const float sg = ((i + j) & 1) ? -inv_n : inv_n;
        const float2 X = M.X[i * kCPitch + j];
        const float2 f = make_float2(X.x * sg, X.y * sg);
        const float2 y = __ldg(A.y + off + idx);
        const float2 yh = make_float2(kappa * (y.x - mur), kappa * (y.y - mui));
        const float2 z = make_float2(yh.x * f.x + yh.y * f.y, yh.y * f.x - yh.x * f.y);
        c = two_s2 * sqrt_approx(fmaf(z.x, z.x, z.y * z.y) + 1e-37f);
        th = atan2_fast(z.y, z.x);
      }
      M.qs[idx] = c;
      M.ts[idx] = th;
    }
    __syncthreads();
    // ---- phi M-step: colour-ordered GMRF ICD in place (R10-R11), free boundary
    for (int sw = 0; sw < A.sweeps; ++sw) {
      for (int c = 0; c < 4; ++c) {
        const int ci = c >> 1, cj = c & 1;
        for (int p = tid; p < kCP / 4; p += kCThreads) {
          const int i = 2 * (p / (kCN / 2)) + ci, j = 2 * (p % (kCN / 2)) + cj;
          DDH_DBG((i & 1) == ci && (j & 1) == cj);
          chain_phiupd(M.ps, M.qs, M.ts, i, j, A);
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  // ---- WriteData: the new state (and the caller's copies)
  for (int idx = tid; idx < kCP; idx += kCThreads) {
    const float p = M.ps[pidx(idx / kCN, idx & (kCN - 1))], r = M.rs[idx];
    C.phi_next[off + idx] = p;
    A.r_state[off + idx] = r;
    if (C.phi_copy) C.phi_copy[off + idx] = p;
    if (C.r_copy) C.r_copy[off + idx] = r;
  }
}

}  // namespace

bool chain_fits(int n) { return n == kCN; }

// resident chain CTAs per SM on the current device (occupancy calculator; cached)
int chain_ctas_per_sm() {
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 1;
  if (!cache[dev]) {
    int nb = 0;
    if (cudaFuncSetAttribute(ks_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ChainSmem)) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, ks_chain, kCThreads, sizeof(ChainSmem)) != cudaSuccess)
      nb = 1;
    cache[dev] = nb > 0 ? nb : 1;
  }
  return cache[dev];
}

cudaError_t launch_chain(const ChainArgs &c, cudaStream_t st) {
  if (c.a.n != kCN) return cudaErrorInvalidValue;
  static bool init[64] = {};  // the shared-memory opt-in is per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!init[dev]) {
    e = cudaFuncSetAttribute(ks_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ChainSmem));
    if (e != cudaSuccess) return e;
    init[dev] = true;
  }
  ks_chain<<<c.a.sc, kCThreads, sizeof(ChainSmem), st>>>(c);
  return cudaGetLastError();
}

}  // namespace ddh
