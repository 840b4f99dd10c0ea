// ddh_kernels.cu -- sm_100a kernels of the DDH-MBIR hot path (one EM
// iteration = K1 -> K2a -> K2b -> K3a -> K3b, preceded by K0 once per frame).
// See ddh_kernels.h for the kernel map and DESIGN.md for the roofline of each.
//
// Paper references: P:<line> = PAPER.md line; R<k> = DESIGN.md reading.
//   Normalize (Eq. 4), RemoveTipTilt, Eq. 3
//   (P:183-187), A_phi^H, EM (R1-R12).
#include "ddh_kernels.h"
#include "ddh_common.cuh"
#include "ddh_fft.cuh"

#include <math.h>

namespace ddh {

// ---------------------------------------------------------------- geometry

template <int N> struct RowCfg { static constexpr int H = (N <= 512) ? 16 : 8; };
template <int N> struct ColCfg { static constexpr int W = (N <= 512) ? 16 : 8; };
constexpr int kIcdTile = 64;       // ICD tile side (owned); halo 4 on each side
constexpr int kIcdHalo = 4;        // = 4 colour phases x 1 sweep (R8)
constexpr int kIcdRegion = kIcdTile + 2 * kIcdHalo;
constexpr int kIcdThreads = 256;
constexpr int kK0Threads = 256;

int row_block_rows(int n) { return n <= 512 ? 16 : 8; }
int col_block_cols(int n) { return n <= 512 ? 16 : 8; }
int icd_tile(int n) { return kIcdTile < n ? kIcdTile : n; }
int k0_blocks(int n) {
  int b = (n * n) / 4096;
  return b < 1 ? 1 : b;
}

// ------------------------------------------------------------- reductions

// Warp 0 only: per-stream totals of the K0 partials -> out[0..4]
// (sum re y, sum im y, sum phi, sum phi x, sum phi y) in fixed order.
__device__ __forceinline__ void reduce_part0(const double *__restrict__ part0, int nb0, int s, double *out) {
  const int lane = threadIdx.x & 31;
  double v[5] = {0, 0, 0, 0, 0};
  for (int b = lane; b < nb0; b += 32) {
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] += part0[((size_t)s * nb0 + b) * 5 + k];
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    v[k] = warp_sum(v[k]);
    if (lane == 0) out[k] = v[k];
  }
}

// Warp 0 only: ||y - mu||^2 of stream s from the K1 partials.
__device__ __forceinline__ double reduce_part1(const double *__restrict__ part1, int nb1, int s) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int b = lane; b < nb1; b += 32) v += part1[(size_t)s * nb1 + b];
  return warp_sum(v);
}

// ---------------------------------------------------------------- K0: sums

// Per-stream sums for Normalize (Eq. 4: mean of y over all N^2 entries, R16)
// and for the RemoveTipTilt least-squares plane over the aperture.
// grid (nb0, sc), block 256.  FP64 accumulation, fixed reduction order.
__global__ void __launch_bounds__(kK0Threads) k0_stats(StepArgs A) {
  __shared__ double sh[32 * 5];
  const int s = blockIdx.y;
  const int n = A.n;
  const int P = n * n;
  const int per = P / A.nb0;
  const int base = blockIdx.x * per;
  const int lg = 31 - __clz(n);
  const size_t off = (size_t)s * P;
  double v[5] = {0, 0, 0, 0, 0};
  for (int idx = base + threadIdx.x; idx < base + per; idx += kK0Threads) {
    if (A.want_y) {
      const float2 y = A.y[off + idx];
      v[0] += (double)y.x;
      v[1] += (double)y.y;
    }
    if (A.apply_plane) {
      const int i = idx >> lg, j = idx & (n - 1);
      if (in_ap(A.rowspan, i, j)) {
        double f = (double)A.phi_in[off + idx];
        if (A.phi_sub) f -= (double)A.phi_sub[off + idx];
        v[2] += f;
        v[3] += f * (double)(j - n / 2);
        v[4] += f * (double)(i - n / 2);
      }
    }
  }
  block_sum<5>(v, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) A.part0[((size_t)s * A.nb0 + blockIdx.x) * 5 + k] = v[k];
  }
}

// ------------------------------------------------------- K1: forward rows

// z = chi a e^{-j phi'} (y - mu) for H pupil rows, forward row DFT -> cbuf.
// Also the partial sums of |y - mu|^2 (Eq. 4 denominator, all N^2 entries).
// grid (N/H, sc), block H*N/E.
template <int N>
__global__ void __launch_bounds__(RowCfg<N>::H *(N / FftPlan<N>::E)) k1_rows_fwd(StepArgs A) {
  constexpr int H = RowCfg<N>::H, E = FftPlan<N>::E, NT = H * (N / E), PITCH = N + 1;
  constexpr int P = N * N;
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + H * PITCH;
  __shared__ double st[8];
  __shared__ double red[32];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * H;
  const size_t off = (size_t)s * P;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = A.tw[k];
  if (threadIdx.x < 32) {
    double sums[5];
    reduce_part0(A.part0, A.nb0, s, sums);
    if (threadIdx.x == 0) {
      st[0] = sums[0] / P;
      st[1] = sums[1] / P;
      double c[3] = {0, 0, 0};
      if (A.apply_plane) plane_from_sums(sums, A.minv, c);
      st[2] = c[0];
      st[3] = c[1];
      st[4] = c[2];
    }
  }
  __syncthreads();
  const float mur = (float)st[0], mui = (float)st[1];
  const float c0 = (float)st[2], c1 = (float)st[3], c2 = (float)st[4];
  double acc = 0.0;
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    const size_t g = off + (size_t)i * N + j;
    const float2 y = A.y[g];
    const float dr = y.x - mur, di = y.y - mui;
    acc += (double)dr * dr + (double)di * di;
    float2 z = make_float2(0.f, 0.f);
    if (in_ap(A.rowspan, i, j)) {
      const float ph = A.phi_in[g] - (c0 + c1 * (float)(j - N / 2) + c2 * (float)(i - N / 2));
      float sn, cs;
      sincosf(ph, &sn, &cs);
      z = make_float2(dr * cs + di * sn, di * cs - dr * sn);  // (y - mu) e^{-j phi'}
      if ((i + j) & 1) z = make_float2(-z.x, -z.y);
    }
    tile[r * PITCH + j] = z;
  }
  double a1[1] = {acc};
  block_sum<1>(a1, red);
  if (threadIdx.x == 0) A.part1[(size_t)s * A.nb1 + blockIdx.x] = a1[0];
  const int b = threadIdx.x % H, t = threadIdx.x / H;
  block_fft<N, -1>(tile + b * PITCH, true, t, 1, tw);
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1);
    A.cbuf[off + (size_t)(i0 + r) * N + j] = tile[r * PITCH + j];
  }
}

// ------------------------------------------------- K2a: forward columns + E

// Column DFT -> u = A^H y-hat (back-projection; first E-step transform,
// R13), Eq. 3 warm start, E-step (R1), then chi mu -> inverse column DFT.
// grid (N/W, sc), block W*N/E.
template <int N>
__global__ void __launch_bounds__(ColCfg<N>::W *(N / FftPlan<N>::E)) k2a_cols(StepArgs A) {
  constexpr int W = ColCfg<N>::W, E = FftPlan<N>::E, NT = W * (N / E);
  constexpr int P = N * N;
  extern __shared__ float2 sm[];
  float2 *tile = sm;  // [N][W]
  float2 *tw = sm + N * W;
  __shared__ double st[2];
  const int s = blockIdx.y;
  const int c0 = blockIdx.x * W;
  const size_t off = (size_t)s * P;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = A.tw[k];
  if (threadIdx.x < 32) {
    const double d2 = reduce_part1(A.part1, A.nb1, s);
    if (threadIdx.x == 0) st[0] = d2;
  }
  for (int idx = threadIdx.x; idx < N * W; idx += NT) {
    const int i = idx / W, c = idx % W;
    tile[idx] = A.cbuf[off + (size_t)i * N + c0 + c];
  }
  __syncthreads();
  const double d2 = st[0];
  const bool degenerate = !(d2 > 0.0);
  if (A.status && blockIdx.x == 0 && threadIdx.x == 0) A.status[s] = degenerate ? 1 : 0;
  const float kappa = degenerate ? 0.f : (float)sqrt((double)P / d2);  // Eq. 4: sqrt(p)/||y - mu||
  const float scale = kappa / (float)N;                                 // unitary F_c = chi F chi / N
  const int b = threadIdx.x % W, t = threadIdx.x / W;
  block_fft<N, -1>(tile + b, true, t, W, tw);
  const bool warm = A.warm && !degenerate;
  for (int idx = threadIdx.x; idx < N * W; idx += NT) {
    const int ki = idx / W, kj = c0 + idx % W;
    const float sg = ((ki + kj) & 1) ? -scale : scale;
    const float2 X = tile[idx];
    const float2 u = make_float2(X.x * sg, X.y * sg);
    const size_t g = off + (size_t)ki * N + kj;
    const float rp = A.r_state[g];
    float r0 = rp;
    if (warm) r0 = fmaxf(fmaf(A.oml, rp, A.la * (u.x * u.x + u.y * u.y)), A.r_min);  // Eq. 3
    const float w = r0 / (r0 + A.s2);                                                 // E-step (R1)
    const float2 mu = make_float2(w * u.x, w * u.y);
    A.rinit[g] = r0;
    A.q[g] = fmaf(mu.x, mu.x, fmaf(mu.y, mu.y, w * A.s2));
    const float cs = ((ki + kj) & 1) ? -1.f : 1.f;
    tile[idx] = make_float2(cs * mu.x, cs * mu.y);
  }
  __syncthreads();
  block_fft<N, +1>(tile + b, true, t, W, tw);
  for (int idx = threadIdx.x; idx < N * W; idx += NT) {
    const int i = idx / W, c = idx % W;
    A.cbuf[off + (size_t)i * N + c0 + c] = tile[idx];
  }
}

// --------------------------------------------------- K3a: inverse rows + c

// Inverse row DFT -> f = F_c^{-1} mu; phase-correlation terms of the phi
// M-step: c = (2/s2) a |y-hat| |f|, theta = arg(y-hat conj f).
// grid (N/H, sc), block H*N/E.
template <int N>
__global__ void __launch_bounds__(RowCfg<N>::H *(N / FftPlan<N>::E)) k3a_rows_inv(StepArgs A) {
  constexpr int H = RowCfg<N>::H, E = FftPlan<N>::E, NT = H * (N / E), PITCH = N + 1;
  constexpr int P = N * N;
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + H * PITCH;
  __shared__ double st[4];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * H;
  const size_t off = (size_t)s * P;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = A.tw[k];
  if (threadIdx.x < 32) {
    double sums[5];
    reduce_part0(A.part0, A.nb0, s, sums);
    const double d2 = reduce_part1(A.part1, A.nb1, s);
    if (threadIdx.x == 0) {
      st[0] = sums[0] / P;
      st[1] = sums[1] / P;
      st[2] = d2;
    }
  }
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1);
    tile[r * PITCH + j] = A.cbuf[off + (size_t)(i0 + r) * N + j];
  }
  __syncthreads();
  const float mur = (float)st[0], mui = (float)st[1];
  const double d2 = st[2];
  const float kappa = d2 > 0.0 ? (float)sqrt((double)P / d2) : 0.f;
  const int b = threadIdx.x % H, t = threadIdx.x / H;
  block_fft<N, +1>(tile + b * PITCH, true, t, 1, tw);
  const float inv_n = 1.f / (float)N;
  const float two_s2 = 2.f / A.s2;
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    const size_t g = off + (size_t)i * N + j;
    float c = 0.f, th = 0.f;
    if (in_ap(A.rowspan, i, j)) {
      const float sg = ((i + j) & 1) ? -inv_n : inv_n;
      const float2 X = tile[r * PITCH + j];
      const float2 f = make_float2(X.x * sg, X.y * sg);
      const float2 y = A.y[g];
      const float2 yh = make_float2(kappa * (y.x - mur), kappa * (y.y - mui));
      const float2 z = make_float2(yh.x * f.x + yh.y * f.y, yh.y * f.x - yh.x * f.y);  // yh conj(f)
      c = two_s2 * hypotf(z.x, z.y);
      th = atan2f(z.y, z.x);
    }
    A.cc[g] = c;
    A.theta[g] = th;
  }
}

// ------------------------------------------------------------ r-ICD (K2b)

// grid (N/tile, N/tile, sc), block 256.  One 4-colour sweep (R8) over a tile
// with a halo of 4 (periodic): after colour phase k the values at distance >= k
// from the region edge equal those of the global colour-ordered sweep.
__global__ void __launch_bounds__(kIcdThreads) k2b_ricd(IcdArgs A) {
  constexpr int RW = kIcdRegion;
  __shared__ float rs[RW * RW];
  __shared__ float qs[RW * RW];
  __shared__ double st[1];
  const int n = A.n;
  const int TT = n < kIcdTile ? n : kIcdTile;  // n >= 64 in practice -> 64
  const int s = blockIdx.z;
  const int i0 = blockIdx.y * TT, j0 = blockIdx.x * TT;
  const size_t off = (size_t)s * n * n;
  const int R = TT + 2 * kIcdHalo;
  bool degenerate = false;
  if (A.part1) {
    if (threadIdx.x < 32) {
      const double d2 = reduce_part1(A.part1, A.nb1, s);
      if (threadIdx.x == 0) st[0] = d2;
    }
    __syncthreads();
    degenerate = !(st[0] > 0.0);
  }
  for (int idx = threadIdx.x; idx < R * R; idx += kIcdThreads) {
    const int li = idx / R, lj = idx % R;
    const int gi = (i0 - kIcdHalo + li + n) & (n - 1), gj = (j0 - kIcdHalo + lj + n) & (n - 1);
    rs[li * RW + lj] = A.in[off + (size_t)gi * n + gj];
    qs[li * RW + lj] = A.q[off + (size_t)gi * n + gj];
  }
  __syncthreads();
  if (A.prior && !degenerate) {
    const float rmin = A.r_min;
    const float b0 = A.b0;
    const int half = R / 2;
    for (int c = 0; c < 4; ++c) {
      const int ci = c >> 1, cj = c & 1;  // colours (0,0),(0,1),(1,0),(1,1)
      const int lo = c + 1, hi = R - (c + 1);
      for (int p = threadIdx.x; p < half * half; p += kIcdThreads) {
        const int li = 2 * (p / half) + ci, lj = 2 * (p % half) + cj;
        if (li < lo || li >= hi || lj < lo || lj >= hi) continue;
        const float ri = rs[li * RW + lj];
        float B = 0.f, S = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int di = nb_di(k), dj = nb_dj(k);
          const float bw = nb_w(k);
          const float rj = rs[(li + di) * RW + lj + dj];
          const float bt = bw * b0 * qgg_w(ri - rj, A.inv_Tsig, A.two_minus_q);
          B += bt;
          S = fmaf(bt, rj, S);
        }
        rs[li * RW + lj] = r_update(ri, qs[li * RW + lj], B, S, rmin);
      }
      __syncthreads();
    }
  }
  for (int idx = threadIdx.x; idx < TT * TT; idx += kIcdThreads) {
    const int oi = idx / TT, oj = idx % TT;
    const int li = oi + kIcdHalo, lj = oj + kIcdHalo;
    float v = rs[li * RW + lj];
    if (!A.prior && !degenerate) v = fmaxf(qs[li * RW + lj], A.r_min);  // prior off: max(q, r_min)
    const size_t g = off + (size_t)(i0 + oi) * n + (j0 + oj);
    A.out[g] = v;
    if (A.copy) A.copy[g] = v;
  }
}

// ---------------------------------------------------------- phi-ICD (K3b)

// grid (N/tile, N/tile, sc), block 256, dynamic smem 3 R^2 floats.  One
// 4-colour sweep of the GMRF phi update (R10-R11), free boundary.  The symmetric
// bound of -c cos(.) at x0 = wrap(phi - theta) gives
// phi <- (c s th~ + w sum b phi_j) / (c s + w sum b), s = sin x0 / x0.
__global__ void __launch_bounds__(kIcdThreads) k3b_phiicd(IcdArgs A) {
  extern __shared__ float smf[];
  constexpr int RW = kIcdRegion;
  float *ps = smf;
  float *cs = smf + RW * RW;
  float *ts = smf + 2 * RW * RW;
  __shared__ double st[8];
  const int n = A.n;
  const int TT = n < kIcdTile ? n : kIcdTile;
  const int s = blockIdx.z;
  const int i0 = blockIdx.y * TT, j0 = blockIdx.x * TT;
  const size_t off = (size_t)s * n * n;
  const int R = TT + 2 * kIcdHalo;
  if (threadIdx.x < 32) {
    double c[3] = {0, 0, 0};
    if (A.apply_plane) {
      double sums[5];
      reduce_part0(A.part0, A.nb0, s, sums);
      if (threadIdx.x == 0) plane_from_sums(sums, A.minv, c);
    }
    double d2 = 1.0;
    if (A.part1) d2 = reduce_part1(A.part1, A.nb1, s);
    if (threadIdx.x == 0) {
      st[0] = c[0];
      st[1] = c[1];
      st[2] = c[2];
      st[3] = d2;
    }
  }
  __syncthreads();
  const bool degenerate = !(st[3] > 0.0);
  const float c0 = (float)st[0], c1 = (float)st[1], c2 = (float)st[2];
  if (degenerate) {  // state unchanged (no tip/tilt removal either)
    for (int idx = threadIdx.x; idx < TT * TT; idx += kIcdThreads) {
      const size_t g = off + (size_t)(i0 + idx / TT) * n + (j0 + idx % TT);
      const float v = A.in[g];
      A.out[g] = v;
      if (A.copy) A.copy[g] = v;
    }
    return;
  }
  for (int idx = threadIdx.x; idx < R * R; idx += kIcdThreads) {
    const int li = idx / R, lj = idx % R;
    const int gi = i0 - kIcdHalo + li, gj = j0 - kIcdHalo + lj;
    float ph = 0.f, cv = 0.f, tv = 0.f;
    if (gi >= 0 && gi < n && gj >= 0 && gj < n) {
      const size_t g = off + (size_t)gi * n + gj;
      ph = A.in[g] - (c0 + c1 * (float)(gj - n / 2) + c2 * (float)(gi - n / 2));
      cv = A.q[g];
      tv = A.theta[g];
    }
    ps[li * RW + lj] = ph;
    cs[li * RW + lj] = cv;
    ts[li * RW + lj] = tv;
  }
  __syncthreads();
  const float w = A.b0;
  const int half = R / 2;
  for (int c = 0; c < 4; ++c) {
    const int ci = c >> 1, cj = c & 1;
    const int lo = c + 1, hi = R - (c + 1);
    for (int p = threadIdx.x; p < half * half; p += kIcdThreads) {
      const int li = 2 * (p / half) + ci, lj = 2 * (p % half) + cj;
      if (li < lo || li >= hi || lj < lo || lj >= hi) continue;
      const int gi = i0 - kIcdHalo + li, gj = j0 - kIcdHalo + lj;
      if (gi < 0 || gi >= n || gj < 0 || gj >= n) continue;
      float nb = 0.f, sb = 0.f;
      if (A.prior) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int di = nb_di(k), dj = nb_dj(k);
          const int ni = gi + di, nj = gj + dj;
          if (ni >= 0 && ni < n && nj >= 0 && nj < n) {
            nb = fmaf(nb_w(k), ps[(li + di) * RW + lj + dj], nb);
            sb += nb_w(k);
          }
        }
      }
      const float outv = phi_update(ps[li * RW + lj], cs[li * RW + lj], ts[li * RW + lj], nb, sb, w, A.prior != 0);
      ps[li * RW + lj] = outv;
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < TT * TT; idx += kIcdThreads) {
    const int oi = idx / TT, oj = idx % TT;
    const float v = ps[(oi + kIcdHalo) * RW + oj + kIcdHalo];
    const size_t g = off + (size_t)(i0 + oi) * n + (j0 + oj);
    A.out[g] = v;
    if (A.copy) A.copy[g] = v;
  }
}

// ------------------------------------------------------------------ utils

__global__ void k_fill(float *p, float v, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------ Strehl (Ks)

// Rows: psi' = (phi_hat - phi_true) - plane; z = chi a e^{j psi'}; inverse row DFT.
template <int N>
__global__ void __launch_bounds__(RowCfg<N>::H *(N / FftPlan<N>::E)) ks1_rows(StrehlArgs A) {
  constexpr int H = RowCfg<N>::H, E = FftPlan<N>::E, NT = H * (N / E), PITCH = N + 1;
  constexpr int P = N * N;
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + H * PITCH;
  __shared__ double st[4];
  const int s = blockIdx.y;
  const int i0 = blockIdx.x * H;
  const size_t off = (size_t)s * P;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = A.tw[k];
  if (threadIdx.x < 32) {
    double c[3] = {0, 0, 0};
    if (A.phi_hat) {
      double sums[5];
      reduce_part0(A.part0, A.nb0, s, sums);
      if (threadIdx.x == 0) plane_from_sums(sums, A.minv, c);
    }
    if (threadIdx.x == 0) {
      st[0] = c[0];
      st[1] = c[1];
      st[2] = c[2];
    }
  }
  __syncthreads();
  const float c0 = (float)st[0], c1 = (float)st[1], c2 = (float)st[2];
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    float2 z = make_float2(0.f, 0.f);
    if (in_ap(A.rowspan, i, j)) {
      float psi = 0.f;
      if (A.phi_hat) {
        const size_t g = off + (size_t)i * N + j;
        psi = (A.phi_hat[g] - A.phi_true[g]) - (c0 + c1 * (float)(j - N / 2) + c2 * (float)(i - N / 2));
      }
      float sn, cs;
      sincosf(psi, &sn, &cs);
      z = ((i + j) & 1) ? make_float2(-cs, -sn) : make_float2(cs, sn);
      // residual phase angle(e^{j(phi - phi_hat)}) with tip/tilt removed: -psi wrapped
      if (A.resid) A.resid[off + (size_t)i * N + j] = atan2f(-sn, cs);
    } else if (A.resid) {
      A.resid[off + (size_t)i * N + j] = 0.f;
    }
    tile[r * PITCH + j] = z;
  }
  __syncthreads();
  const int b = threadIdx.x % H, t = threadIdx.x / H;
  block_fft<N, +1>(tile + b * PITCH, true, t, 1, tw);
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1);
    A.cbuf[off + (size_t)(i0 + r) * N + j] = tile[r * PITCH + j];
  }
}

// Columns: inverse column DFT, |.|^2 / N^2, per-CTA maximum.
template <int N>
__global__ void __launch_bounds__(ColCfg<N>::W *(N / FftPlan<N>::E)) ks2_cols(StrehlArgs A) {
  constexpr int W = ColCfg<N>::W, E = FftPlan<N>::E, NT = W * (N / E);
  constexpr int P = N * N;
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + N * W;
  __shared__ float red[32];
  const int s = blockIdx.y;
  const int c0 = blockIdx.x * W;
  const size_t off = (size_t)s * P;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = A.tw[k];
  for (int idx = threadIdx.x; idx < N * W; idx += NT) {
    const int i = idx / W, c = idx % W;
    tile[idx] = A.cbuf[off + (size_t)i * N + c0 + c];
  }
  __syncthreads();
  const int b = threadIdx.x % W, t = threadIdx.x / W;
  block_fft<N, +1>(tile + b, true, t, W, tw);
  float m = 0.f;
  for (int idx = threadIdx.x; idx < N * W; idx += NT) {
    const float2 X = tile[idx];
    const float I = X.x * X.x + X.y * X.y;
    m = fmaxf(m, I);
    if (A.psf) A.psf[off + (size_t)(idx / W) * N + c0 + idx % W] = I / ((float)N * (float)N) * A.inv_den;
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (NT + 31) / 32 ? red[threadIdx.x] : 0.f;
    v = warp_max(v);
    if (threadIdx.x == 0) A.pmax[(size_t)s * A.nb + blockIdx.x] = v / ((float)N * (float)N);
  }
}

// ------------------------------------------------------- test: F_c, F_c^-1

template <int N, int DIR>
__global__ void __launch_bounds__(RowCfg<N>::H *(N / FftPlan<N>::E))
    kt_rows(const float2 *in, float2 *out, const float2 *tw_g) {
  constexpr int H = RowCfg<N>::H, E = FftPlan<N>::E, NT = H * (N / E), PITCH = N + 1;
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + H * PITCH;
  const size_t off = (size_t)blockIdx.y * N * N;
  const int i0 = blockIdx.x * H;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = tw_g[k];
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    float2 z = in[off + (size_t)i * N + j];
    if ((i + j) & 1) z = make_float2(-z.x, -z.y);
    tile[r * PITCH + j] = z;
  }
  __syncthreads();
  block_fft<N, DIR>(tile + (threadIdx.x % H) * PITCH, true, threadIdx.x / H, 1, tw);
  for (int idx = threadIdx.x; idx < H * N; idx += NT) {
    const int r = idx / N, j = idx & (N - 1);
    out[off + (size_t)(i0 + r) * N + j] = tile[r * PITCH + j];
  }
}

template <int N, int DIR>
__global__ void __launch_bounds__(ColCfg<N>::W *(N / FftPlan<N>::E)) kt_cols(float2 *io, const float2 *tw_g) {
  constexpr int W = ColCfg<N>::W, E = FftPlan<N>::E, NT = W * (N / E);
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + N * W;
  const size_t off = (size_t)blockIdx.y * N * N;
  const int c0 = blockIdx.x * W;
  for (int k = threadIdx.x; k < N; k += NT) tw[k] = tw_g[k];
  for (int idx = threadIdx.x; idx < N * W; idx += NT)
    tile[idx] = io[off + (size_t)(idx / W) * N + c0 + idx % W];
  __syncthreads();
  block_fft<N, DIR>(tile + threadIdx.x % W, true, threadIdx.x / W, W, tw);
  const float inv_n = 1.f / (float)N;
  for (int idx = threadIdx.x; idx < N * W; idx += NT) {
    const int i = idx / W, j = c0 + idx % W;
    const float sg = ((i + j) & 1) ? -inv_n : inv_n;
    const float2 X = tile[idx];
    io[off + (size_t)i * N + j] = make_float2(X.x * sg, X.y * sg);
  }
}

// ------------------------------------------------------------- launchers

template <int N> constexpr int row_threads() { return RowCfg<N>::H * (N / FftPlan<N>::E); }
template <int N> constexpr int col_threads() { return ColCfg<N>::W * (N / FftPlan<N>::E); }
template <int N> constexpr size_t row_smem() { return (size_t)(RowCfg<N>::H * (N + 1) + N) * sizeof(float2); }
template <int N> constexpr size_t col_smem() { return (size_t)(N * ColCfg<N>::W + N) * sizeof(float2); }
constexpr size_t phi_smem() { return (size_t)3 * kIcdRegion * kIcdRegion * sizeof(float); }

template <int N>
static cudaError_t init_n() {
  cudaFuncSetAttribute(k1_rows_fwd<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<N>());
  cudaFuncSetAttribute(k3a_rows_inv<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<N>());
  cudaFuncSetAttribute(ks1_rows<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<N>());
  cudaFuncSetAttribute(kt_rows<N, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<N>());
  cudaFuncSetAttribute(kt_rows<N, +1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<N>());
  cudaFuncSetAttribute(k2a_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_smem<N>());
  cudaFuncSetAttribute(ks2_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_smem<N>());
  cudaFuncSetAttribute(kt_cols<N, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_smem<N>());
  cudaFuncSetAttribute(kt_cols<N, +1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_smem<N>());
  return cudaGetLastError();
}

cudaError_t init_kernels(int n) {
  cudaFuncSetAttribute(k3b_phiicd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)phi_smem());
  switch (n) {
    case 64: return init_n<64>();
    case 128: return init_n<128>();
    case 256: return init_n<256>();
    case 512: return init_n<512>();
    case 1024: return init_n<1024>();
  }
  return cudaErrorInvalidValue;
}

#define DDH_DISPATCH(n, CALL)          \
  switch (n) {                         \
    case 64: { constexpr int N = 64; CALL; } break;     \
    case 128: { constexpr int N = 128; CALL; } break;   \
    case 256: { constexpr int N = 256; CALL; } break;   \
    case 512: { constexpr int N = 512; CALL; } break;   \
    case 1024: { constexpr int N = 1024; CALL; } break; \
    default: return cudaErrorInvalidValue;              \
  }

cudaError_t launch_k0(const StepArgs &a, cudaStream_t st) {
  k0_stats<<<dim3(a.nb0, a.sc), kK0Threads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_k1(const StepArgs &a, cudaStream_t st) {
  DDH_DISPATCH(a.n, (k1_rows_fwd<N><<<dim3(N / RowCfg<N>::H, a.sc), row_threads<N>(), row_smem<N>(), st>>>(a)));
  return cudaGetLastError();
}

cudaError_t launch_k2a(const StepArgs &a, cudaStream_t st) {
  DDH_DISPATCH(a.n, (k2a_cols<N><<<dim3(N / ColCfg<N>::W, a.sc), col_threads<N>(), col_smem<N>(), st>>>(a)));
  return cudaGetLastError();
}

cudaError_t launch_k3a(const StepArgs &a, cudaStream_t st) {
  DDH_DISPATCH(a.n, (k3a_rows_inv<N><<<dim3(N / RowCfg<N>::H, a.sc), row_threads<N>(), row_smem<N>(), st>>>(a)));
  return cudaGetLastError();
}

cudaError_t launch_ricd(const IcdArgs &a, int sc, cudaStream_t st) {
  const int tt = icd_tile(a.n);
  k2b_ricd<<<dim3(a.n / tt, a.n / tt, sc), kIcdThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_phiicd(const IcdArgs &a, int sc, cudaStream_t st) {
  const int tt = icd_tile(a.n);
  k3b_phiicd<<<dim3(a.n / tt, a.n / tt, sc), kIcdThreads, phi_smem(), st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fill(float *p, float v, size_t count, cudaStream_t st) {
  const int blocks = (int)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
  k_fill<<<blocks, 256, 0, st>>>(p, v, count);
  return cudaGetLastError();
}

cudaError_t launch_strehl(const StrehlArgs &a, int B, cudaStream_t st) {
  DDH_DISPATCH(a.n, ({
                 ks1_rows<N><<<dim3(N / RowCfg<N>::H, B), row_threads<N>(), row_smem<N>(), st>>>(a);
                 ks2_cols<N><<<dim3(N / ColCfg<N>::W, B), col_threads<N>(), col_smem<N>(), st>>>(a);
               }));
  return cudaGetLastError();
}

cudaError_t launch_test_fft2c(int n, const float2 *in, float2 *out, int B, int inverse, const float2 *tw,
                              cudaStream_t st) {
  DDH_DISPATCH(n, ({
                 if (inverse) {
                   kt_rows<N, +1><<<dim3(N / RowCfg<N>::H, B), row_threads<N>(), row_smem<N>(), st>>>(in, out, tw);
                   kt_cols<N, +1><<<dim3(N / ColCfg<N>::W, B), col_threads<N>(), col_smem<N>(), st>>>(out, tw);
                 } else {
                   kt_rows<N, -1><<<dim3(N / RowCfg<N>::H, B), row_threads<N>(), row_smem<N>(), st>>>(in, out, tw);
                   kt_cols<N, -1><<<dim3(N / ColCfg<N>::W, B), col_threads<N>(), col_smem<N>(), st>>>(out, tw);
                 }
               }));
  return cudaGetLastError();
}

}  // namespace ddh
