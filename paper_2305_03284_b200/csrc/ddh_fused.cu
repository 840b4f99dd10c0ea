// ddh_fused.cu -- cluster-fused EM iteration for N <= 512 (sm_100a).
//
// One thread-block cluster per stream covers the whole N x N frame: KA and KC
// split it into row slabs (H rows per CTA), KB into column slabs (W columns
// per CTA).  Everything that needs a view wider than one slab goes through
// distributed shared memory (DSMEM) inside the cluster instead of HBM:
//   KA  kf_rows_fwd  y and phi rows -> per-stream sums (Eq. 4 mean, RemoveTipTilt
//                    plane) reduced across the cluster over
//                    DSMEM; z = chi a e^{-j phi'} (y - mu); forward row DFT
//   KB  kf_cols      column DFT -> u = A^H y-hat (R13); Eq. 3; E-step (R1);
//                    inverse column DFT of chi mu; qGGMRF r-ICD (R6-R9) over
//                    the slab, exchanging the boundary columns with the
//                    neighbouring CTAs over DSMEM before each colour phase
//   KC  kf_rows_inv  inverse row DFT -> f; c, theta (registers); GMRF phi-ICD
//                    (R10-R11) with boundary rows exchanged over DSMEM
// HBM traffic per pixel and EM iteration: KA 20 B, KB 24 B, KC 24 B (68 B),
// against 112 B and 3 more launches for the unfused pass design.
//
// Race-freedom of the halo exchange: before colour phase c every CTA passes a
// cluster barrier (all phase c-1 writes visible), copies the neighbour's
// boundary column/row into its halo, then updates its colour-c pixels.  A
// neighbour may modify the copied column during phase c only if that column
// has the parity of colour c, in which case the adjacent own column has the
// other parity and is not updated in phase c, so the possibly stale halo values
// are not used before the next phase re-copies them.
#include "ddh_common.cuh"
#include "ddh_fft.cuh"
#include "ddh_kernels.h"

#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

// Phase timestamps (instrumentation build only: -DDDH_PHASE_TIMING): thread 0
// of rank-0 CTAs of streams 0..3 prints clock64() deltas at phase boundaries.
#ifdef DDH_PHASE_TIMING
#define DDH_T0() long long t_ph[12]; int n_ph = 0; if (threadIdx.x == 0) t_ph[n_ph++] = clock64();
#define DDH_TS() do { if (threadIdx.x == 0 && n_ph < 12) t_ph[n_ph++] = clock64(); } while (0)
#define DDH_TPRINT(tag) do { if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y < 4) { long long d_[11]; \
    for (int k_ = 0; k_ < 11; ++k_) d_[k_] = (k_ + 1 < n_ph) ? t_ph[k_ + 1] - t_ph[k_] : 0; \
    printf("%s %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n", tag, d_[0], d_[1], d_[2], d_[3], d_[4], \
           d_[5], d_[6], d_[7], d_[8], d_[9], d_[10]); } } while (0)
#define DDH_SYNC_T(stmt) do { long long a_ = clock64(); stmt; if (threadIdx.x == 0) t_sync += clock64() - a_; } while (0)
#define DDH_SYNC_DECL long long t_sync = 0;
#define DDH_SYNC_PRINT(tag) do { if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y < 4) printf("%s %lld\n", tag, t_sync); } while (0)
#else
#define DDH_SYNC_T(stmt) stmt
#define DDH_SYNC_DECL
#define DDH_SYNC_PRINT(tag)
#define DDH_T0()
#define DDH_TS()
#define DDH_TPRINT(tag)
#endif

namespace ddh {

template <int N> struct FusedCfg {
  static constexpr int CS = (N <= 128) ? 8 : 16;  // CTAs per stream (cluster size)
  static constexpr int H = N / CS;                // rows per CTA (KA, KC)
  static constexpr int W = N / CS;                // columns per CTA (KB)
  static constexpr int E = FftPlan<N>::E;
  static constexpr int NT = H * (N / E);          // threads per CTA (all three kernels)
  static constexpr int EPT = H * N / NT;          // pixels per thread (= E)
  static constexpr int RP = W + 2;                // pitch of the r-ICD slab (1-column halos)
  static constexpr int MINB = NT >= 1024 ? 1 : (NT >= 256 ? 4 : 8);  // CTAs/SM for __launch_bounds__
};

// L2 prefetch of [p, p + bytes) by the threads of a CTA (one request per 128 B line)
__device__ __forceinline__ void prefetch_l2(const void *p, size_t bytes, int tid, int nt) {
  const char *c = reinterpret_cast<const char *>(p);
  for (size_t o = (size_t)tid * 128; o < bytes; o += (size_t)nt * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
}

bool fused_supported(int n) { return n == 64 || n == 128 || n == 256 || n == 512; }
int fused_cluster(int n) { return n <= 128 ? 8 : 16; }

template <int N> __host__ __device__ constexpr size_t ka_smem() { return (size_t)(FusedCfg<N>::H * (N + 1) + N) * sizeof(float2); }
template <int N> __host__ __device__ constexpr size_t kb_smem() {
  using C = FusedCfg<N>;
  return (size_t)N * C::W * sizeof(float2) + (size_t)(N + 2) * C::RP * sizeof(float) + (size_t)N * sizeof(float2);
}
template <int N> __host__ __device__ constexpr size_t kc_smem() {
  using C = FusedCfg<N>;
  return (size_t)C::H * (N + 1) * sizeof(float2) + (size_t)(C::H + 2) * (N + 8) * sizeof(float) + (size_t)N * sizeof(float2);
}

// ------------------------------------------------------------------- KA

template <int N>
__device__ __forceinline__ void phase_a(const StepArgs &A, const int s) {
  using C = FusedCfg<N>;
  constexpr int H = C::H, NT = C::NT, CS = C::CS, EPT = C::EPT, PITCH = N + 1, P = N * N;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ float2 sm[];
  float2 *tile = sm;
  float2 *tw = sm + H * PITCH;
  __shared__ double red[32 * 5];
  __shared__ double part[5];
  __shared__ double tot[5];
  const int tid = threadIdx.x;
  const int i0 = rank * H;
  DDH_T0();
  const size_t off = (size_t)s * P;
  __syncthreads();  // previous phase's shared-memory reads are done
  for (int k = tid; k < N; k += NT) tw[k] = A.tw[k];
  float ph[EPT];
  double v[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    const size_t g = off + (size_t)i * N + j;
    const float2 y = A.y[g];
    tile[r * PITCH + j] = y;
    const float f = A.phi_in[g];
    ph[k] = f;
    v[0] += (double)y.x;
    v[1] += (double)y.y;
    if (A.apply_plane && in_ap(A.rowspan, i, j)) {
      v[2] += (double)f;
      v[3] += (double)f * (double)(j - N / 2);
      v[4] += (double)f * (double)(i - N / 2);
    }
  }
  DDH_TS();  // 1: loaded + local sums
  block_sum<5>(v, red);
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) part[k] = v[k];
  }
  cl.sync();  // all partials of the stream written
  if (tid < 5) {
    double acc = 0.0;
    for (int r = 0; r < CS; ++r) acc += cl.map_shared_rank(part, r)[tid];  // fixed rank order
    tot[tid] = acc;
  }
  cl.barrier_arrive();  // remote reads of `part` done (waited on before exit)
  __syncthreads();
  DDH_TS();  // 2: cluster reduction
  double c[3] = {0, 0, 0};
  if (A.apply_plane) plane_from_sums(tot, A.minv, c);
  const double mu_r = tot[0] / P, mu_i = tot[1] / P;
  if (rank == 0 && tid == 0) {
    double *st = A.stats + (size_t)s * 5;
    st[0] = mu_r;
    st[1] = mu_i;
    st[2] = c[0];
    st[3] = c[1];
    st[4] = c[2];
  }
  const float mur = (float)mu_r, mui = (float)mu_i;
  const float c0 = (float)c[0], c1 = (float)c[1], c2 = (float)c[2];
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    const float2 y = tile[r * PITCH + j];
    const float dr = y.x - mur, di = y.y - mui;
    acc += (double)dr * dr + (double)di * di;
    float2 z = make_float2(0.f, 0.f);
    if (in_ap(A.rowspan, i, j)) {
      const float p = ph[k] - (c0 + c1 * (float)(j - N / 2) + c2 * (float)(i - N / 2));
      float sn, cs;
      __sincosf(fmaf(-6.283185307179586f, rintf(p * 0.15915494309189535f), p), &sn, &cs);  // |arg| <= pi
      z = make_float2(dr * cs + di * sn, di * cs - dr * sn);  // (y - mu) e^{-j phi'}
      if ((i + j) & 1) z = make_float2(-z.x, -z.y);
    }
    tile[r * PITCH + j] = z;
  }
  double a1[1] = {acc};
  block_sum<1>(a1, red);  // also orders the tile writes before the FFT
  if (tid == 0) A.part1[(size_t)s * CS + rank] = a1[0];
  DDH_TS();  // 3: z, |y - mu|^2
  block_fft<N, -1>(tile + (tid % H) * PITCH, true, tid / H, 1, tw);
  DDH_TS();  // 4: row DFT
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int r = idx / N, j = idx & (N - 1);
    A.cbuf[off + (size_t)(i0 + r) * N + j] = tile[r * PITCH + j];
  }
  DDH_TS();  // 5: stored
  cl.barrier_wait();
  DDH_TS();  // 6: exit barrier
  DDH_TPRINT("KA");
}

template <int N>
__global__ void __launch_bounds__(FusedCfg<N>::NT, FusedCfg<N>::MINB) kf_rows_fwd(StepArgs A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  phase_a<N>(A, blockIdx.y);
}

// ------------------------------------------------------------------- KB

// Column slab of W columns x N rows.  Order: column DFT -> Eq. 3 + E-step
// (r0 -> rS, q -> registers, chi mu -> tile) -> r-ICD over rS (each thread
// updates exactly the pixels whose q it holds) -> write r -> inverse column
// DFT of the tile -> write the spectrum slab.
template <int N>
__device__ __forceinline__ void phase_b(const StepArgs &A, const int s, const int s_next) {
  using C = FusedCfg<N>;
  constexpr int W = C::W, NT = C::NT, CS = C::CS, EPT = C::EPT, RP = C::RP, P = N * N;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ float2 sm[];
  float2 *tile = sm;                                       // [N][W]
  // rS: [N+2][RP]; data row i at padded row i+1, columns 1..W; column 0 / W+1 and
  // rows 0 / N+1 are halos (neighbour CTAs' columns, periodic row wrap)
  float *rS = reinterpret_cast<float *>(sm + N * W);
  float2 *tw = reinterpret_cast<float2 *>(rS + (N + 2) * RP);
  __shared__ double st[1];
  const int tid = threadIdx.x;
  const int c0 = rank * W;
  __syncthreads();  // previous phase's shared-memory reads are done
  for (int k = tid; k < N; k += NT) tw[k] = A.tw[k];
  {
    const int sn = s_next;  // next stream of this cluster: pull its inputs into L2 now
    if (sn < A.sc) {
      for (int i = tid; i < N; i += NT) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(A.cbuf + (size_t)sn * P + (size_t)i * N + c0));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(A.r_state + (size_t)sn * P + (size_t)i * N + c0));
      }
    }
  }
  const size_t off = (size_t)s * P;
  DDH_T0();
  if (tid == 0) {
    double d2 = 0.0;
    for (int r = 0; r < CS; ++r) d2 += A.part1[(size_t)s * CS + r];
    st[0] = d2;
  }
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    tile[idx] = A.cbuf[off + (size_t)(idx / W) * N + c0 + idx % W];
  }
  // r_prev slab -> rS (asynchronous copy; consumed after the forward column DFT)
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int i = idx / W, c = idx % W;
    const unsigned dst = (unsigned)__cvta_generic_to_shared(rS + (i + 1) * RP + c + 1);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(A.r_state + off + (size_t)i * N + c0 + c));
  }
  asm volatile("cp.async.commit_group;");
  __syncthreads();
  DDH_TS();  // 1: loaded
  const double d2 = st[0];
  const bool degenerate = !(d2 > 0.0);
  if (A.status && rank == 0 && tid == 0) A.status[s] = degenerate ? 1 : 0;
  const float kappa = degenerate ? 0.f : (float)sqrt((double)P / d2);  // Eq. 4
  const float scale = kappa / (float)N;                                 // F_c = chi F chi / N
  block_fft<N, -1>(tile + tid % W, true, tid / W, W, tw);
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
  DDH_TS();  // 2: forward column DFT
  const bool warm = A.warm && !degenerate;
  float qreg[EPT];
  // Eq. 3 + E-step over 2x2 pixel blocks (one pixel of each colour per block)
#pragma unroll
  for (int k = 0; k < EPT / 4; ++k) {
    const int b = tid + k * NT;
    const int br = b / (W / 2), bc = b % (W / 2);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int ki = 2 * br + (q4 >> 1), lc = 2 * bc + (q4 & 1), kj = c0 + lc;
      const float sg = ((ki + kj) & 1) ? -scale : scale;
      const float2 X = tile[ki * W + lc];
      const float2 u = make_float2(X.x * sg, X.y * sg);
      const float rp = rS[(ki + 1) * RP + lc + 1];  // prefetched r_prev
      float r0 = rp;
      if (warm) r0 = fmaxf(fmaf(A.oml, rp, A.la * (u.x * u.x + u.y * u.y)), A.r_min);
      const float w = r0 * rcp_approx(r0 + A.s2);
      const float2 mu = make_float2(w * u.x, w * u.y);
      qreg[k * 4 + q4] = fmaf(mu.x, mu.x, fmaf(mu.y, mu.y, w * A.s2));
      rS[(ki + 1) * RP + lc + 1] = r0;
      const float cs = ((ki + kj) & 1) ? -1.f : 1.f;
      tile[ki * W + lc] = make_float2(cs * mu.x, cs * mu.y);
    }
  }
  DDH_TS();  // 3: Eq. 3 + E-step
  const bool icd = A.r_prior && !degenerate;  // uniform over the cluster (one stream)
  DDH_SYNC_DECL
  if (icd) {
    float *left = cl.map_shared_rank(rS, (rank + CS - 1) % CS);
    float *right = cl.map_shared_rank(rS, (rank + 1) % CS);
#pragma unroll 1
    for (int sw = 0; sw < A.sweeps; ++sw) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        DDH_SYNC_T(cl.sync());
        // halos: neighbour columns for all padded rows (rows 0 / N+1 take the
        // neighbours' data rows N / 1) and the periodic row wrap of own columns
        for (int i = tid; i < N + 2; i += NT) {
          const int src = i == 0 ? N : (i == N + 1 ? 1 : i);
          rS[i * RP] = left[src * RP + W];
          rS[i * RP + W + 1] = right[src * RP + 1];
        }
        for (int w = tid; w < W; w += NT) {
          rS[w + 1] = rS[N * RP + w + 1];
          rS[(N + 1) * RP + w + 1] = rS[RP + w + 1];
        }
        DDH_SYNC_T(__syncthreads());
        const int ci = c >> 1, cj = c & 1;
        // pixels of one colour never neighbour each other: gather B, S of all
        // of this thread's colour-c pixels first (independent chains the
        // scheduler can interleave), then update, then store
        float Bv[EPT / 4], Sv[EPT / 4], Rv[EPT / 4];
#pragma unroll
        for (int k = 0; k < EPT / 4; ++k) {
          const int b = tid + k * NT;
          const int br = b / (W / 2), bc = b % (W / 2);
          const int ki = 2 * br + ci + 1, lj = 2 * bc + cj + 1;  // padded coordinates
          const float ri = rS[ki * RP + lj];
          // neighbour pairs (nearest: up/down, left/right; diagonal: upper, lower)
          const float2 nA = make_float2(rS[(ki - 1) * RP + lj], rS[(ki + 1) * RP + lj]);
          const float2 nB = make_float2(rS[ki * RP + lj - 1], rS[ki * RP + lj + 1]);
          const float2 dA = make_float2(rS[(ki - 1) * RP + lj - 1], rS[(ki - 1) * RP + lj + 1]);
          const float2 dB = make_float2(rS[(ki + 1) * RP + lj - 1], rS[(ki + 1) * RP + lj + 1]);
          const float2 wA = qgg_w2(ri, nA, A.r_h, A.r_g, A.r_k), wB = qgg_w2(ri, nB, A.r_h, A.r_g, A.r_k);
          const float2 wC = qgg_w2(ri, dA, A.r_h, A.r_g, A.r_k), wD = qgg_w2(ri, dB, A.r_h, A.r_g, A.r_k);
          // b = 1/6 (nearest), 1/12 (diagonal), times 1/(2 sig_r^2) = r_b0:
          // B = (r_b0/6) (sum_4 w + sum_d w / 2), S likewise with w r_j
          const float2 bs = p_fma(p_add(wC, wD), bc2(0.5f), p_add(wA, wB));
          const float2 ss = p_fma(p_fma(wC, dA, p_mul(wD, dB)), bc2(0.5f), p_fma(wA, nA, p_mul(wB, nB)));
          Bv[k] = A.r_b6 * (bs.x + bs.y);
          Sv[k] = A.r_b6 * (ss.x + ss.y);
          Rv[k] = ri;
        }
#pragma unroll
        for (int k = 0; k < EPT / 4; ++k) Rv[k] = r_update(Rv[k], qreg[k * 4 + c], Bv[k], Sv[k], A.r_min);
#pragma unroll
        for (int k = 0; k < EPT / 4; ++k) {
          const int b = tid + k * NT;
          const int br = b / (W / 2), bc = b % (W / 2);
          rS[(2 * br + ci + 1) * RP + 2 * bc + cj + 1] = Rv[k];
        }
      }
    }
    cl.barrier_arrive();  // last remote read of a neighbour's slab done (wait before exit)
  } else if (!degenerate) {  // prior off: r = max(q, r_min)
#pragma unroll
    for (int k = 0; k < EPT / 4; ++k) {
      const int b = tid + k * NT;
      const int br = b / (W / 2), bc = b % (W / 2);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        rS[(2 * br + (q4 >> 1) + 1) * RP + 2 * bc + (q4 & 1) + 1] = fmaxf(qreg[k * 4 + q4], A.r_min);
    }
  }
  __syncthreads();
  DDH_TS();  // 4: r-ICD
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int i = idx / W, c = idx % W;
    const float v = rS[(i + 1) * RP + c + 1];
    const size_t g = off + (size_t)i * N + c0 + c;
    A.r_state[g] = v;
    if (A.r_copy) A.r_copy[g] = v;
  }
  DDH_TS();  // 5: r written
  block_fft<N, +1>(tile + tid % W, true, tid / W, W, tw);
  DDH_TS();  // 6: inverse column DFT
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    A.cbuf[off + (size_t)(idx / W) * N + c0 + idx % W] = tile[idx];
  }
  DDH_TS();  // 7: spectrum stored
  if (icd) cl.barrier_wait();  // neighbours may still read our slab until they arrive
  DDH_TS();  // 8: final cluster barrier
  DDH_TPRINT("KB");
  DDH_SYNC_PRINT("KBsync");
}

template <int N>
__global__ void __launch_bounds__(FusedCfg<N>::NT, FusedCfg<N>::MINB) kf_cols(StepArgs A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int s = blockIdx.y; s < A.sc; s += gridDim.y)  // persistent: one stream per iteration
    phase_b<N>(A, s, s + gridDim.y);
}

// ------------------------------------------------------------------- KC

template <int N>
__device__ __forceinline__ void phase_c(const StepArgs &A, const int s) {
  using C = FusedCfg<N>;
  constexpr int H = C::H, NT = C::NT, CS = C::CS, EPT = C::EPT, PITCH = N + 1, P = N * N;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ float2 sm[];
  float2 *tile = sm;                                                       // [H][N+1]
  // phS: [H+2][PP], data row r at row r+1, column j at j+4; zero borders make
  // missing neighbours of the free boundary contribute nothing
  constexpr int PP = N + 8;
  float *phS = reinterpret_cast<float *>(sm + H * PITCH);
  float2 *tw = reinterpret_cast<float2 *>(phS + (H + 2) * PP);
  __shared__ double st[6];
  const int tid = threadIdx.x;
  __syncthreads();  // previous phase's shared-memory reads are done
  const int i0 = rank * H;
  DDH_T0();
  const size_t off = (size_t)s * P;
  for (int k = tid; k < N; k += NT) tw[k] = A.tw[k];
  for (int k = tid; k < (H + 2) * 8; k += NT) {  // pad columns
    const int r = k >> 3, c = k & 7;
    phS[r * PP + (c < 4 ? c : N + c)] = 0.f;
  }
  for (int k = tid; k < N; k += NT) {  // halo rows (overwritten where a neighbour CTA exists)
    phS[4 + k] = 0.f;
    phS[(H + 1) * PP + 4 + k] = 0.f;
  }
  if (tid == 0) {
    double d2 = 0.0;
    for (int r = 0; r < CS; ++r) d2 += A.part1[(size_t)s * CS + r];
    const double *sv = A.stats + (size_t)s * 5;
    st[0] = sv[0];
    st[1] = sv[1];
    st[2] = sv[2];
    st[3] = sv[3];
    st[4] = sv[4];
    st[5] = d2;
  }
  // y rows -> L2 now (read in the epilogue); phi rows -> phS asynchronously
  prefetch_l2(A.y + off + (size_t)i0 * N, (size_t)H * N * sizeof(float2), tid, NT);
#pragma unroll
  for (int k = 0; k < EPT / 4; ++k) {
    const int idx = (tid + k * NT) * 4;  // 16-byte chunks of the H x N phi slab
    const unsigned dst = (unsigned)__cvta_generic_to_shared(phS + (idx / N + 1) * PP + 4 + (idx & (N - 1)));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(A.phi_in + off + (size_t)i0 * N + idx));
  }
  asm volatile("cp.async.commit_group;");
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int r = idx / N, j = idx & (N - 1);
    tile[r * PITCH + j] = A.cbuf[off + (size_t)(i0 + r) * N + j];
  }
  __syncthreads();
  const float mur = (float)st[0], mui = (float)st[1];
  const float c0 = (float)st[2], c1 = (float)st[3], c2 = (float)st[4];
  const double d2 = st[5];
  const bool degenerate = !(d2 > 0.0);
  const float kappa = degenerate ? 0.f : (float)sqrt((double)P / d2);
  DDH_TS();  // 1: loaded
  block_fft<N, +1>(tile + (tid % H) * PITCH, true, tid / H, 1, tw);
  DDH_TS();  // 2: inverse row DFT
  // phase-correlation terms for this thread's pixels (2x2 blocks), kept in registers
  float creg[EPT], treg[EPT];
  const float inv_n = 1.f / (float)N, two_s2 = 2.f / A.s2;
#pragma unroll
  for (int k = 0; k < EPT / 4; ++k) {
    const int b = tid + k * NT;
    const int br = b / (N / 2), bc = b % (N / 2);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int r = 2 * br + (q4 >> 1), j = 2 * bc + (q4 & 1), i = i0 + r;
      float c = 0.f, th = 0.f;
      if (in_ap(A.rowspan, i, j)) {
        const float sg = ((i + j) & 1) ? -inv_n : inv_n;
        const float2 X = tile[r * PITCH + j];
        const float2 f = make_float2(X.x * sg, X.y * sg);
        const float2 y = A.y[off + (size_t)i * N + j];
        const float2 yh = make_float2(kappa * (y.x - mur), kappa * (y.y - mui));
        const float2 z = make_float2(yh.x * f.x + yh.y * f.y, yh.y * f.x - yh.x * f.y);  // yh conj(f)
        c = two_s2 * sqrtf(fmaf(z.x, z.x, z.y * z.y));
        th = atan2f(z.y, z.x);
      }
      creg[k * 4 + q4] = c;
      treg[k * 4 + q4] = th;
    }
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
  DDH_TS();  // 3: c, theta
  if (degenerate) {  // state unchanged (no tip/tilt removal either)
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int idx = tid + k * NT;
      const size_t g = off + (size_t)(i0 + idx / N) * N + (idx & (N - 1));
      const float v = A.phi_in[g];
      A.phi_out[g] = v;
      if (A.phi_copy) A.phi_copy[g] = v;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int r = idx / N, j = idx & (N - 1), i = i0 + r;
    phS[(r + 1) * PP + 4 + j] -= c0 + c1 * (float)(j - N / 2) + c2 * (float)(i - N / 2);  // phi' = phi - plane
  }
  __syncthreads();
  DDH_TS();  // 4: phi loaded
  const bool prior = A.phi_prior != 0;
  const float w = A.phi_w;
  DDH_SYNC_DECL
  if (prior) {
    const float *up = rank > 0 ? cl.map_shared_rank(phS, rank - 1) : nullptr;
    const float *dn = rank < CS - 1 ? cl.map_shared_rank(phS, rank + 1) : nullptr;
#pragma unroll 1
    for (int cc = 0; cc < 4 * A.sweeps; ++cc) {
      const int c = cc & 3;
      // Row parity changes only every two phases: the halo row above (global
      // row i0-1, odd) is read in phases 0/1 and modified by its owner only in
      // phases 2/3; the halo row below (i0+H, even) is read in phases 2/3 and
      // modified only in phases 0/1.  So one cluster barrier + copy before
      // phase 0 (row above) and one before phase 2 (row below) per sweep.
      if (c == 0 || c == 2) {
        DDH_SYNC_T(cl.sync());
        for (int j = tid; j < N; j += NT) {
          if (c == 0 && up) phS[4 + j] = up[H * PP + 4 + j];
          if (c == 2 && dn) phS[(H + 1) * PP + 4 + j] = dn[PP + 4 + j];
        }
      }
      DDH_SYNC_T(__syncthreads());
      const int ci = c >> 1, cj = c & 1;
#pragma unroll
      for (int k = 0; k < EPT / 4; ++k) {
        const int b = tid + k * NT;
        const int br = b / (N / 2), bc = b % (N / 2);
        const int r = 2 * br + ci, j = 2 * bc + cj, i = i0 + r, li = r + 1, lj = j + 4;
        float n4 = 0.f, nd = 0.f;  // zero borders: no bounds checks
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const float v = phS[(li + nb_di(m)) * PP + lj + nb_dj(m)];
          if (m < 4) n4 += v; else nd += v;
        }
        const float nb = fmaf(nd, 1.f / 12.f, n4 * (1.f / 6.f));
        // sum of b over the existing neighbours (1 inside the grid)
        const bool tp = i == 0, bt = i == N - 1, lf = j == 0, rt = j == N - 1;
        const float sb = 1.f - (1.f / 6.f) * (float)(tp + bt + lf + rt) -
                         (1.f / 12.f) * (float)((tp | lf) + (tp | rt) + (bt | lf) + (bt | rt));
        const float cv = c == 0 ? creg[k * 4] : c == 1 ? creg[k * 4 + 1] : c == 2 ? creg[k * 4 + 2] : creg[k * 4 + 3];
        const float tv = c == 0 ? treg[k * 4] : c == 1 ? treg[k * 4 + 1] : c == 2 ? treg[k * 4 + 2] : treg[k * 4 + 3];
        phS[li * PP + lj] = phi_update(phS[li * PP + lj], cv, tv, nb, sb, w, true);
      }
    }
    cl.barrier_arrive();  // last remote read done (wait before exit)
    __syncthreads();
  } else {
#pragma unroll
    for (int k = 0; k < EPT / 4; ++k) {
      const int b = tid + k * NT;
      const int br = b / (N / 2), bc = b % (N / 2);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int li = 2 * br + (q4 >> 1) + 1, lj = 2 * bc + (q4 & 1) + 4;
        phS[li * PP + lj] = phi_update(phS[li * PP + lj], creg[k * 4 + q4], treg[k * 4 + q4], 0.f, 0.f, 0.f, false);
      }
    }
    __syncthreads();
  }
  DDH_TS();  // 5: phi-ICD
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int idx = tid + k * NT;
    const int r = idx / N, j = idx & (N - 1);
    const size_t g = off + (size_t)(i0 + r) * N + j;
    const float v = phS[(r + 1) * PP + 4 + j];
    A.phi_out[g] = v;
    if (A.phi_copy) A.phi_copy[g] = v;
  }
  DDH_TS();  // 6: phi stored
  if (prior) cl.barrier_wait();  // neighbours may still read our boundary rows until they arrive
  DDH_TS();  // 7: exit barrier
  DDH_TPRINT("KC");
  DDH_SYNC_PRINT("KCsync");
}

template <int N>
__global__ void __launch_bounds__(FusedCfg<N>::NT, FusedCfg<N>::MINB) kf_rows_inv(StepArgs A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  phase_c<N>(A, blockIdx.y);
}

// ------------------------------------------------------------- launchers

template <typename... KArgs, typename... Args>
static cudaError_t launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, int cs,
                                  cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol in the phases)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int N>
static void init_grids();

template <int N>
static cudaError_t init_fused_n() {
  cudaFuncSetAttribute(kf_rows_fwd<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ka_smem<N>());
  cudaFuncSetAttribute(kf_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kb_smem<N>());
  cudaFuncSetAttribute(kf_rows_inv<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kc_smem<N>());
  if (FusedCfg<N>::CS > 8) {
    cudaFuncSetAttribute(kf_rows_fwd<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kf_cols<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kf_rows_inv<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  init_grids<N>();
  return cudaGetLastError();
}

#define DDH_FDISPATCH(n, CALL)                          \
  switch (n) {                                          \
    case 64: { constexpr int N = 64; CALL; } break;     \
    case 128: { constexpr int N = 128; CALL; } break;   \
    case 256: { constexpr int N = 256; CALL; } break;   \
    case 512: { constexpr int N = 512; CALL; } break;   \
    default: return cudaErrorInvalidValue;              \
  }

cudaError_t init_fused(int n) { DDH_FDISPATCH(n, return init_fused_n<N>()); }

// Persistent grids: as many clusters as can be co-resident (queried once per
// kernel with cudaOccupancyMaxActiveClusters), each looping over streams.
static int g_max_clusters[3][11];  // [kernel][log2 N]

template <typename... KArgs>
static int max_clusters(void (*kernel)(KArgs...), int cs, int nt, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1024);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void *)kernel, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1 << 20;  // unknown: one cluster per stream
  }
  return n;
}

template <int N>
static void init_grids() {
  using C = FusedCfg<N>;
  const int l = 31 - __builtin_clz(N);
  // measured at 256^2 x 64 streams: the persistent grid helps KB (94 vs 99 us)
  // and hurts KA/KC (52 vs 44, 82 vs 70 us), which keep one cluster per stream
  g_max_clusters[0][l] = 1 << 20;
  g_max_clusters[1][l] = max_clusters(kf_cols<N>, C::CS, C::NT, kb_smem<N>());
  g_max_clusters[2][l] = 1 << 20;
}

static inline int grid_y(int which, int n, int sc) {
  const int m = g_max_clusters[which][31 - __builtin_clz(n)];
  return m > 0 && m < sc ? m : sc;
}

cudaError_t launch_ka(const StepArgs &a, cudaStream_t st) {
  DDH_FDISPATCH(a.n, return launch_cluster(kf_rows_fwd<N>, dim3(FusedCfg<N>::CS, grid_y(0, N, a.sc)),
                                           dim3(FusedCfg<N>::NT), ka_smem<N>(), FusedCfg<N>::CS, st, a));
}
cudaError_t launch_kb(const StepArgs &a, cudaStream_t st) {
  DDH_FDISPATCH(a.n, return launch_cluster(kf_cols<N>, dim3(FusedCfg<N>::CS, grid_y(1, N, a.sc)),
                                           dim3(FusedCfg<N>::NT), kb_smem<N>(), FusedCfg<N>::CS, st, a));
}
cudaError_t launch_kc(const StepArgs &a, cudaStream_t st) {
  DDH_FDISPATCH(a.n, return launch_cluster(kf_rows_inv<N>, dim3(FusedCfg<N>::CS, grid_y(2, N, a.sc)),
                                           dim3(FusedCfg<N>::NT), kc_smem<N>(), FusedCfg<N>::CS, st, a));
}

}  // namespace ddh
