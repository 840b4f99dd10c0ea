// ddh_stream.cu -- the streaming (cluster-free) EM iteration, sm_100a.
//
// One EM iteration of S independent streams (Fig. 1) as six
// kernels with no inter-CTA dependency inside a launch, so every launch
// packs the SMs freely (no thread-block-cluster co-scheduling, no wave
// quantisation at the cluster granularity) and the launches of different
// stream sub-groups ("lanes", ddh_api.cpp) overlap on the GPU:
//
//   S0 ks_stats     per stream: sum y (Eq. 4 mean) and the
//                   RemoveTipTilt normal-equation sums of phi
//   S1 ks_rows_fwd_p  z = chi a e^{-j phi'} (y - mu); forward row DFT;
//                   partial ||y - mu||^2; persistent, rows streamed in by
//                   bulk asynchronous copies (ks_rows_fwd: one-shot form)
//   S2 ks_cols      column DFT -> u = A^H y-hat (R13); Eq. 3; E-step (R1)
//                   -> r0, q to HBM; FFT of conj(chi mu) (the inverse column
//                   DFT by conjugation); ks_cols_p (staged) for small launches
//   S3 ks_ricd      qGGMRF r-ICD on 64x64 (32x32, 16x16 for small launches)
//                   tiles with a 4-pixel periodic halo (one colour sweep,
//                   R6-R9), recomputing the halo ring
//   S4 ks_rows_inv  row DFT of the conjugated spectrum -> f = F_c^{-1} mu;
//                   c = (2/s2)|y-hat||f|, theta = arg(y-hat conj f), written
//                   as (c, theta) pairs in place over the spectrum rows
//   S5 ks_phiicd    GMRF phi-ICD on 64x64 tiles, 4-pixel halo, free edge
//                   (R10-R11)
//
// FFTs are register-resident (ddh_fft_reg.cuh: one shared-memory exchange at
// N <= 256), all arithmetic on complex pairs uses packed FP32x2 instructions.
// The ICD kernels store the tile colour-separated (four (i mod 2, j mod 2)
// sub-grids), so a colour phase reads and writes consecutive words.
#include <algorithm>
#include <cstdlib>

#include "ddh_common.cuh"
#include "ddh_fft_reg.cuh"
#include "ddh_kernels.h"

// Programmatic dependent launch (sm_90+): every streaming kernel is launched
// with programmatic stream serialisation.  It lets its successor launch at
// once (launch_dependents) and waits for its predecessor's completion and
// memory (griddepcontrol.wait) only after the prologue that touches constant
// tables and the user's read-only frames, so launch latency and the
// predecessor's tail overlap the prologue.  No kernel reads or writes any
// buffer a predecessor produces or consumes before the wait.
#define DDH_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#define DDH_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
// DDH_PDL_NOTRIG (build knob, bits S0 1, S1 2, S2 4 (only launches with more items than
// CTAs: with the bit applied to single-item launches too the single-stream latency rose
// from 25.5 to 31.5 us p50, profiles/r02h_bench.json vs r02g_bench.json), S4 8, r-ICD 16,
// phi-ICD 32, the large-launch S2 form `ks_cols` 64):
// kernels whose bit is set issue no early launch_dependents, so their
// dependent launches only as their CTAs exit (no dependent CTAs resident
// and waiting beside them while other lanes' kernels need the slots).
// Default: S2 only (its dependent S4 resident and waiting during the whole
// persistent S2 cost the c3 step 1 %: 546.1-546.2 k -> 551.8-552.1 k frames/s,
// profiles/r02h_pdl_ab.txt; every other kernel measured best with the early
// trigger, e.g. S4 without it 546 -> 539 k)
#ifndef DDH_PDL_NOTRIG
#define DDH_PDL_NOTRIG 4
#endif
// DDH_PDL_LATE (bits S1 2, S2 4 of the persistent forms): launch_dependents
// when a CTA starts its last item (with the bit also set in DDH_PDL_NOTRIG)
#ifndef DDH_PDL_LATE
#define DDH_PDL_LATE 0
#endif
#define DDH_PDL_TRIGGER_K(bit)                  \
  do {                                          \
    if (!(DDH_PDL_NOTRIG & (bit))) DDH_PDL_TRIGGER(); \
  } while (0)

namespace ddh {

namespace {

// Per-stream scalars of a step, written once by the kernel that first has
// them (S1: mu, plane; S2: kappa, degenerate flag) and read by the later
// kernels instead of re-reducing the partial sums in every CTA.
//   [0] Re mu  [1] Im mu  [2..4] plane c0, c1, c2  [5] kappa  [6] degenerate (0 / 1)
constexpr int kStatW = 8;

// Call-graph replay (CallDesc): the stand-in pointers of a captured chunk
// become this call's buffers at their point of use (the kernels never modify
// their argument struct: a written kernel parameter is copied to local memory).
template <typename T>
__device__ __forceinline__ T *add_delta(T *p, unsigned long long d) {
  return reinterpret_cast<T *>(reinterpret_cast<unsigned long long>(p) + d);
}
__device__ __forceinline__ const float2 *call_y(const StepArgs &A, const float2 *p) {
  return (A.rel & kRelY) ? add_delta(p, A.desc->dy) : p;
}
__device__ __forceinline__ float *call_copy(const StepArgs &A) {
  if (A.rel & kRelCopyPhi) return add_delta(A.icd_copy, A.desc->dphi);
  if (A.rel & kRelCopyR) return add_delta(A.icd_copy, A.desc->dr);
  return A.icd_copy;
}
__device__ __forceinline__ uint8_t *call_status(const StepArgs &A) {
  return (A.rel & kRelStatus) ? add_delta(A.status, A.desc->dst) : A.status;
}

constexpr int kSThreads = 256;
#ifndef DDH_S5_LOAD_UNROLL
#define DDH_S5_LOAD_UNROLL 4  // S5 tile-load loop unroll (build knob)
#endif
constexpr int kS5LoadUnroll = DDH_S5_LOAD_UNROLL;
// 128-thread row CTAs (S1, S4) and S0 blocks: c3 124.0 -> 120.4 us per step, c4 +1.8 %,
// c2 -0.5 %, c5 -1.8 % against 256 (the S4-fused next-frame sums need S0's thread count)
#ifndef DDH_ROW_THREADS
#define DDH_ROW_THREADS 128
#endif
#ifndef DDH_COL_THREADS
#define DDH_COL_THREADS 256
#endif
#ifndef DDH_COL_MINW
#define DDH_COL_MINW 16
#endif
constexpr int kRowThreads = DDH_ROW_THREADS, kColThreads = DDH_COL_THREADS;
#ifndef DDH_S0_THREADS
#define DDH_S0_THREADS DDH_ROW_THREADS
#endif
constexpr int kS0Threads = DDH_S0_THREADS;  // S0 (and S4's fused next-frame sums): threads per block

template <int N> struct SCfg {
  static constexpr int E = RPlan<N>::E;
  static constexpr int TPV = N / E;                                  // threads per vector
  static constexpr int H = (kRowThreads / TPV) < 1 ? 1 : kRowThreads / TPV;  // rows per row CTA
  static constexpr int NTR = H * TPV;                                // threads per row CTA
  static constexpr int W = (kColThreads / TPV) < DDH_COL_MINW ? DDH_COL_MINW : kColThreads / TPV;  // cols per col CTA
  static constexpr int NTC = W * TPV;                                // threads per col CTA
  static constexpr int RPITCH = N + N / 16;                          // padded row pitch
};

// sincos_red, atan2_fast: ddh_common.cuh (shared with the on-chip chain)

__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Per warp (no barrier): per-stream totals of the S0 partials, fixed order,
// identical in every warp and lane -> out[0..4]
__device__ __forceinline__ void sum_part0(const double *__restrict__ part0, int nb0, int s, double *out) {
  const int lane = threadIdx.x & 31;
  double v[5] = {0, 0, 0, 0, 0};
  for (int b = lane; b < nb0; b += 32) {
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] += part0[((size_t)s * nb0 + b) * 5 + k];
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) out[k] = warp_sum(v[k]);  // xor tree: every lane holds the totals
}
// RemoveTipTilt normal-equation sums (R17) in 2^-16 fixed point: every
// phase value is rounded to an integer multiple of 2^-16 (FP32 rint of f 2^16)
// and the sums of those integers (and of their integer x / y moments) are
// accumulated in FP64, where they are exact while below 2^53 (|phi| < 256 rad
// at N = 1024, < 16384 rad at 256^2).  So any partition and order of the
// pixels (S0 over row blocks, S5's epilogue over ICD tiles, double atomics)
// gives the same bits.  Quantisation 1.5e-5 rad per pixel, random: the plane
// coefficients move by ~1e-9 rad per pixel.
constexpr float kFix = 65536.f;  // 2^16
__device__ __forceinline__ float fixq(float f) { return rintf(f * kFix); }
// Block sum of (s0, sx, sy) (exact: integer-valued doubles) and one atomic add each into out[0..2]
__device__ __forceinline__ void plane_sums_add(double s0, double sx, double sy, double *red, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  s0 = warp_sum(s0);
  sx = warp_sum(sx);
  sy = warp_sum(sy);
  if (lane == 0) red[warp * 3] = s0, red[warp * 3 + 1] = sx, red[warp * 3 + 2] = sy;
  __syncthreads();
  if (warp == 0) {
    double v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = warp_sum(lane < nw ? red[lane * 3 + k] : 0.0);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (v[k] != 0.0) atomicAdd(out + k, v[k]);
  }
}
// plane coefficients from the fixed-point sums
__device__ __forceinline__ void plane_from_fix(const double *__restrict__ ps, const double *minv, double *c) {
  const double sums[5] = {0.0, 0.0, ps[0] / kFix, ps[1] / kFix, ps[2] / kFix};
  plane_from_sums(sums, minv, c);
}

__device__ __forceinline__ double sum_part1(const double *__restrict__ part1, int nb1, int s) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int b = lane; b < nb1; b += 32) v += part1[(size_t)s * nb1 + b];
  return warp_sum(v);
}

template <int N>
__device__ __forceinline__ void load_tw(float4 *tw, const float4 *__restrict__ g, int tid, int nt) {
  for (int k = tid; k < N; k += nt) tw[k] = g[k];
}
// the same table by 16-byte cp.async (one commit group; the caller waits for it
// before the barrier that precedes the first FFT): no register round trip, so
// the table's L2 latency overlaps the kernel's other loads
template <int N>
__device__ __forceinline__ void load_tw_async(float4 *tw, const float4 *__restrict__ g, int tid, int nt) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(tw);
  for (int k = tid; k < N; k += nt) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * k), "l"(g + k));
  asm volatile("cp.async.commit_group;");
}

}  // namespace

// ------------------------------------------------------------------ S0

// grid (nb0, sc), block kS0Threads: block b sums pixels [b P/nb0, (b+1) P/nb0) of
// stream s in chunks of 8 consecutive pixels (16-byte loads); nb0 depends on
// N only (2048-pixel blocks, at most 64), so the partials and everything
// downstream are independent of the launch grouping, and a single stream's
// S0 is 32 short CTAs (c2 step 32.9 -> 30.9 us; 8192-pixel blocks, the former
// layout, is 0.5 % faster at 64 streams).  y: each chunk is summed as a
// balanced FP32 tree (exact for a constant frame, so the degenerate test
// ||y - mu|| = 0 of R31 stays exact) and accumulated in FP64; phi plane sums:
// FP32 per-thread partials; FP64 block sums.
__global__ void __launch_bounds__(kS0Threads) ks_stats(StepArgs A) {
  __shared__ double red[32 * 3];
  const int n = A.n, lg = 31 - __clz(n);
  const size_t P = (size_t)n * n;
  const int s = blockIdx.y;
  const size_t per = P / A.nb0;
  const size_t base = blockIdx.x * per;
  const size_t off = (size_t)s * P;
  double l0 = 0.0, lx = 0.0, ly = 0.0;
  double yr = 0.0, yi = 0.0;
  DDH_PDL_TRIGGER_K(1);
  DDH_PDL_WAIT();
  const float2 *Y = A.want_y ? call_y(A, A.y) : nullptr;
  for (size_t p0 = base + (size_t)threadIdx.x * 8; p0 < base + per; p0 += (size_t)kS0Threads * 8) {
    if (A.want_y) {
      const float4 *y4 = reinterpret_cast<const float4 *>(Y + off + p0);
      float4 a[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] = __ldg(y4 + k);  // kept in L2 for S1
      yr += (double)(((a[0].x + a[0].z) + (a[1].x + a[1].z)) + ((a[2].x + a[2].z) + (a[3].x + a[3].z)));
      yi += (double)(((a[0].y + a[0].w) + (a[1].y + a[1].w)) + ((a[2].y + a[2].w) + (a[3].y + a[3].w)));
    }
    if (A.apply_plane) {
      const int i = (int)(p0 >> lg), j0 = (int)(p0 & (n - 1));
      const int2 sp = __ldg(A.rowspan + i);
      if (j0 + 8 > sp.x && j0 < sp.y) {
        const float4 *f4 = reinterpret_cast<const float4 *>(A.phi_in + off + p0);
        const float4 f0 = __ldg(f4), f1 = __ldg(f4 + 1);
        const float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
        double s0 = 0.0, sx = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = j0 + k;
          const double q = (j >= sp.x && j < sp.y) ? (double)fixq(f[k]) : 0.0;
          s0 += q;
          sx = fma(q, (double)(j - n / 2), sx);
        }
        l0 += s0;
        lx += sx;
        ly = fma(s0, (double)(i - n / 2), ly);
      }
    }
  }
  if (A.want_y) {
    double d[2] = {yr, yi};
    block_sum<2>(d, red);
    if (threadIdx.x == 0) {
      A.part0[((size_t)s * A.nb0 + blockIdx.x) * 5 + 0] = d[0];
      A.part0[((size_t)s * A.nb0 + blockIdx.x) * 5 + 1] = d[1];
    }
  }
  if (A.apply_plane) plane_sums_add(l0, lx, ly, red, A.psum_in + (size_t)s * 3);
}

// ------------------------------------------------------------------ S1

template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTR, 1024 / SCfg<N>::NTR) ks_rows_fwd(StepArgs A) {
  using C = SCfg<N>;
  constexpr int E = C::E, TPV = C::TPV, H = C::H, NT = C::NTR, P = N * N;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;                                             // [N]
  float2 *buf = reinterpret_cast<float2 *>(smem4 + N);            // [H][RPITCH]
  __shared__ double red[32];
  const int tid = threadIdx.x, s = blockIdx.y;
  const int t = tid % TPV, b = tid / TPV;
  const int i = blockIdx.x * H + b;
  const size_t off = (size_t)s * P;
  const size_t row = off + (size_t)i * N;
  // issue the loads first (y: 8 B, phi: 4 B per pixel, comb t + TPV e); the
  // frames are read-only user input, so they may be read before the wait
  DDH_PDL_TRIGGER_K(2);
  const float2 *Y = call_y(A, A.y);
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = Y[row + t + TPV * e];
  load_tw<N>(tw, A.tw4, tid, NT);
  DDH_PDL_WAIT();
  if (t == 0) {  // phi row -> L2 (read after the stats)
    for (int k = 0; k < N * 4; k += 128) prefetch_l2(reinterpret_cast<const char *>(A.phi_in + row) + k);
  }
  double sums[5], cpl[3] = {0, 0, 0};
  sum_part0(A.part0, A.nb0, s, sums);
  if (A.apply_plane) plane_from_fix(A.psum_in + (size_t)s * 3, A.minv, cpl);
  const float mur = (float)(sums[0] / P), mui = (float)(sums[1] / P);
  const float c0 = (float)cpl[0], c1 = (float)cpl[1], c2 = (float)cpl[2];
  if (blockIdx.x == 0 && tid == 0) {  // per-stream scalars for S4 / S5
    float *st = A.sstat + (size_t)s * kStatW;
    st[0] = mur;
    st[1] = mui;
    if (A.apply_plane) st[2] = c0, st[3] = c1, st[4] = c2;
    if (A.psum_out) A.psum_out[(size_t)s * 3] = A.psum_out[(size_t)s * 3 + 1] = A.psum_out[(size_t)s * 3 + 2] = 0.0;
  }
  const int2 sp = __ldg(A.rowspan + i);
  const float pyi = fmaf(c2, (float)(i - N / 2), c0);
  float acc = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = t + TPV * e;
    const float2 d = p_sub(v[e], make_float2(mur, mui));
    acc = fmaf(d.x, d.x, fmaf(d.y, d.y, acc));
    float2 z = make_float2(0.f, 0.f);
    if (j >= sp.x && j < sp.y) {
      float sn, cs;
      sincos_red(A.phi_in[row + j] - fmaf(c1, (float)(j - N / 2), pyi), sn, cs);
      // (y - mu) e^{-j phi'} = d (cs - i sn), times chi = (-1)^(i+j)
      const float sg = ((i + j) & 1) ? -1.f : 1.f;
      z = p_fma(bc2(d.x * sg), make_float2(cs, -sn), p_mul(bc2(d.y * sg), make_float2(sn, cs)));
    }
    v[e] = z;
  }
#ifndef DDH_RF_NORED
  double a1[1] = {(double)acc};
  block_sum<1>(a1, red);  // also: every thread is past its smem use before the FFT
  if (tid == 0) A.part1[(size_t)s * A.nb1 + blockIdx.x] = a1[0];
#else
  if (acc == 12345.f) A.part1[0] = 1.0;
#endif
#ifndef DDH_RF_NOFFT
  fft_reg<N>(v, t, buf + b * C::RPITCH, [](int p) { return rpad(p); }, tw);
#endif
#pragma unroll
  for (int e = 0; e < E; ++e) A.cbuf[row + t + TPV * out_comb<N>(e)] = v[e];
}

// S1, persistent form: grid = 2 CTAs per SM; each CTA walks its row blocks
// (item = (row block, stream)) through a two-stage shared-memory ring filled
// by bulk asynchronous copies (cp.async.bulk, completion on an mbarrier): the
// H contiguous y rows (H N 8 B) and phi rows (H N 4 B) of item k+2 stream in
// while item k is transformed.  The stage of the item being transformed also
// serves as its FFT exchange buffer.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(m)),
      "r"(parity)
      : "memory");
}

template <int N> struct S1P {
  using C = SCfg<N>;
  static constexpr int YB = C::H * N * 8, FB = C::H * N * 4;   // bytes per stage: y rows, phi rows
  static constexpr int STAGE = YB + FB;
  static_assert(C::H * C::RPITCH * 8 <= STAGE, "FFT exchange fits in a stage");
  static constexpr size_t SMEM = N * sizeof(float4) + 2 * (size_t)STAGE;
};

template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTR, 512 / SCfg<N>::NTR) ks_rows_fwd_p(StepArgs A) {
  using C = SCfg<N>;
  using Q = S1P<N>;
  constexpr int E = C::E, TPV = C::TPV, H = C::H, NT = C::NTR, P = N * N, NR = N / H;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;                                           // [N]
  char *stage0 = reinterpret_cast<char *>(smem4 + N);           // 2 x [y rows | phi rows]
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t mb[2];
  // per-item stream scalars, staged one item ahead by 8-byte cp.async: the S0
  // partials (sum y re, im of nb0 blocks) and the fixed-point plane sums
  __shared__ double scal[2][2 * 64 + 3];
  const int tid = threadIdx.x, G = gridDim.x, total = NR * A.sc;
  const int nsc = 2 * A.nb0 + (A.apply_plane ? 3 : 0);
  auto issue_scal = [&](int item, int slot) {
    const int s = item / NR;
    const unsigned dst = smem_u32(&scal[slot][0]);
    for (int idx = tid; idx < nsc; idx += NT) {
      const double *src = idx < 2 * A.nb0 ? A.part0 + ((size_t)s * A.nb0 + (idx >> 1)) * 5 + (idx & 1)
                                          : A.psum_in + (size_t)s * 3 + (idx - 2 * A.nb0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8 * idx), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int t = tid % TPV, b = tid / TPV;
  auto issue = [&](int item, int st, bool y_part, bool phi_part) {  // thread 0
    const int bx = item % NR, s = item / NR;
    char *dst = stage0 + st * Q::STAGE;
    const size_t row0 = (size_t)s * P + (size_t)bx * H * N;
    if (y_part) {
      mbar_expect_tx(&mb[st], Q::YB + Q::FB);
      bulk_g2s(dst, call_y(A, A.y) + row0, Q::YB, &mb[st]);
    }
    if (phi_part) bulk_g2s(dst + Q::YB, A.phi_in + row0, Q::FB, &mb[st]);
  };
  if (tid == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  DDH_PDL_TRIGGER_K(2);
  // y is read-only user input: its copies may start before the wait; phi after
  if (tid == 0) {
    if (blockIdx.x < total) issue(blockIdx.x, 0, true, false);
    if (blockIdx.x + G < total) issue(blockIdx.x + G, 1, true, false);
  }
  load_tw_async<N>(tw, A.tw4, tid, NT);  // completed by the wait_group 0 below
  DDH_PDL_WAIT();
  if (tid == 0) {
    if (blockIdx.x < total) issue(blockIdx.x, 0, false, true);
    if (blockIdx.x + G < total) issue(blockIdx.x + G, 1, false, true);
  }
  if ((int)blockIdx.x < total) issue_scal(blockIdx.x, 0);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();  // twiddles, first item's scalars
  int k = 0;
  for (int item = blockIdx.x; item < total; item += G, ++k) {
#if DDH_PDL_LATE & 2
    if (item + G >= total) DDH_PDL_TRIGGER();  // the dependent launches as the last items start
#endif
    const int st = k & 1, bx = item % NR, s = item / NR;
    const int i = bx * H + b;
    const size_t row = (size_t)s * P + (size_t)i * N;
    char *stg = stage0 + st * Q::STAGE;
    const float2 *ys = reinterpret_cast<const float2 *>(stg) + b * N;
    const float *fs = reinterpret_cast<const float *>(stg + Q::YB) + b * N;
    const int2 sp = __ldg(A.rowspan + i);  // issued first: consumed after the mbarrier wait
    if (item + G < total) issue_scal(item + G, st ^ 1);  // the next item's scalars, in flight during this one
    double sums[5] = {0, 0, 0, 0, 0}, cpl[3] = {0, 0, 0};
    {  // stream totals from the staged partials (same order as sum_part0: lane b, b + 32, ...; xor tree)
      const int lane = tid & 31;
      double v0 = 0.0, v1 = 0.0;
      for (int bb = lane; bb < A.nb0; bb += 32) v0 += scal[st][2 * bb], v1 += scal[st][2 * bb + 1];
      sums[0] = warp_sum(v0);
      sums[1] = warp_sum(v1);
      if (A.apply_plane) plane_from_fix(&scal[st][2 * A.nb0], A.minv, cpl);
    }
    const float mur = (float)(sums[0] / P), mui = (float)(sums[1] / P);
    const float c0 = (float)cpl[0], c1 = (float)cpl[1], c2 = (float)cpl[2];
    if (bx == 0 && tid == 0) {  // per-stream scalars for S4 / S5
      float *ss = A.sstat + (size_t)s * kStatW;
      ss[0] = mur;
      ss[1] = mui;
      if (A.apply_plane) ss[2] = c0, ss[3] = c1, ss[4] = c2;
      if (A.psum_out) A.psum_out[(size_t)s * 3] = A.psum_out[(size_t)s * 3 + 1] = A.psum_out[(size_t)s * 3 + 2] = 0.0;
    }
    const float pyi = fmaf(c2, (float)(i - N / 2), c0);
    mbar_wait(&mb[st], (k >> 1) & 1);
    float2 v[E];
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int j = t + TPV * e;
      const float2 d = p_sub(ys[j], make_float2(mur, mui));
      acc = fmaf(d.x, d.x, fmaf(d.y, d.y, acc));
      float2 z = make_float2(0.f, 0.f);
      if (j >= sp.x && j < sp.y) {
        float sn, cs;
        sincos_red(fs[j] - fmaf(c1, (float)(j - N / 2), pyi), sn, cs);
        const float sg = ((i + j) & 1) ? -1.f : 1.f;
        z = p_fma(bc2(d.x * sg), make_float2(cs, -sn), p_mul(bc2(d.y * sg), make_float2(sn, cs)));
      }
      v[e] = z;
    }
    double a1[1] = {(double)acc};
    block_sum<1>(a1, red);  // also: every thread is past its reads of the stage
    if (tid == 0) A.part1[(size_t)s * A.nb1 + bx] = a1[0];
    fft_reg<N>(v, t, reinterpret_cast<float2 *>(stg) + b * C::RPITCH, [](int p) { return rpad(p); }, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) A.cbuf[row + t + TPV * out_comb<N>(e)] = v[e];
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // the next item's scalars
    __syncthreads();  // the stage (FFT exchange) is free; the next item's scalars are visible
    if (tid == 0 && item + 2 * G < total) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(item + 2 * G, st, true, true);
    }
  }
}

// ------------------------------------------------------------------ S2

// Eq. 3 + E-step of one pixel (R1, R14): from u = A^H y-hat and
// r_prev, r0 = max(oml r_prev + la |u|^2, r_min) when `warm` (else r_prev),
// w = r0/(r0 + s2), mu = w u, q = |mu|^2 + w s2.  Shared by both S2 forms and
// the stage entry point ddh_test_estep.
__device__ __forceinline__ float2 estep_px(float2 u, float r_prev, bool warm, float oml, float la, float r_min,
                                           float s2, float &r0, float &q) {
  r0 = r_prev;
  if (warm) r0 = fmaxf(fmaf(oml, r0, la * fmaf(u.x, u.x, u.y * u.y)), r_min);  // Eq. 3
  const float w = r0 * rcp_approx(r0 + s2);                                   // E-step (R1)
  const float2 mu = p_mul(u, bc2(w));
  q = fmaf(mu.x, mu.x, fmaf(mu.y, mu.y, w * s2));
  return mu;
}

template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTC, 1024 / SCfg<N>::NTC) ks_cols(StepArgs A) {
  using C = SCfg<N>;
  constexpr int E = C::E, TPV = C::TPV, W = C::W, NT = C::NTC, P = N * N;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;                                   // [N]
  float2 *buf = reinterpret_cast<float2 *>(smem4 + N);  // [N][W]
  const int tid = threadIdx.x, s = blockIdx.y;
  const int b = tid % W, t = tid / W;
  const int col = blockIdx.x * W + b;
  const size_t off = (size_t)s * P;
  DDH_PDL_TRIGGER_K(64);  // the small-launch form keeps the early trigger (bit 64, not S2's 4): latency path
  load_tw_async<N>(tw, A.tw4, tid, NT);
  DDH_PDL_WAIT();
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = A.cbuf[off + (size_t)(t + TPV * e) * N + col];
  if (b == 0) {  // r_prev of this column slab -> L2 (read in the E-step)
#pragma unroll
    for (int e = 0; e < E; ++e) prefetch_l2(A.r_state + off + (size_t)(t + TPV * e) * N + blockIdx.x * W);
  }
  const double d2 = sum_part1(A.part1, A.nb1, s);
  const bool degenerate = !(d2 > 0.0);
  const float kappa = degenerate ? 0.f : (float)sqrt((double)P / d2);  // Eq. 4
  if (blockIdx.x == 0 && tid == 0) {
    if (A.status) call_status(A)[s] = degenerate ? 1 : 0;
    A.sstat[(size_t)s * kStatW + 5] = kappa;
    A.sstat[(size_t)s * kStatW + 6] = degenerate ? 1.f : 0.f;
  }
  const float scale = kappa / (float)N;                                 // F_c = chi F chi / N
  asm volatile("cp.async.wait_group 0;" ::: "memory");  // twiddles (visible after the FFT's first barrier)
  fft_reg<N>(v, t, buf + b, [](int p) { return p * W; }, tw);
  const bool warm = A.warm && !degenerate;
  float2 w2[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int ki = t + TPV * out_comb<N>(e);
    const size_t g = off + (size_t)ki * N + col;
    const float sg = ((ki + col) & 1) ? -scale : scale;
    const float2 u = p_mul(v[e], bc2(sg));
    float r0, q;
    const float2 mu = estep_px(u, A.r_state[g], warm, A.oml, A.la, A.r_min, A.s2, r0, q);
    A.rinit[g] = r0;
    A.q[g] = q;
    // conj(chi mu) into input position out_comb(e) of the next FFT
    const float cs = ((ki + col) & 1) ? -1.f : 1.f;
    w2[out_comb<N>(e)] = make_float2(cs * mu.x, -cs * mu.y);
  }
  __syncthreads();  // exchange buffer free
  fft_reg<N>(w2, t, buf + b, [](int p) { return p * W; }, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) A.cbuf[off + (size_t)(t + TPV * out_comb<N>(e)) * N + col] = w2[e];
}

// S2, persistent form (N <= 256): 2 CTAs per SM walk their column slabs
// (item = (W-column block, stream)) through a two-stage ring filled with
// 16-byte cp.async copies: the spectrum slab [N][W] (also the stage's FFT
// exchange buffer) and the r_prev slab [N][W] of item k+2 stream in while
// item k is transformed.
template <int N> struct S2P {
  using C = SCfg<N>;
  static constexpr int CB = N * C::W * 8, RB = N * C::W * 4, STAGE = CB + RB;
  static constexpr size_t SMEM = N * sizeof(float4) + 2 * (size_t)STAGE;
};

template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTC, 512 / SCfg<N>::NTC) ks_cols_p(StepArgs A) {
  using C = SCfg<N>;
  using Q = S2P<N>;
  constexpr int E = C::E, TPV = C::TPV, W = C::W, NT = C::NTC, P = N * N, NC = N / W;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;
  char *stage0 = reinterpret_cast<char *>(smem4 + N);
  const int tid = threadIdx.x, G = gridDim.x, total = NC * A.sc;
  const int b = tid % W, t = tid / W;
  auto issue = [&](int item, int st) {  // all threads: 16-byte chunks of the two slabs
    const int bx = item % NC, s = item / NC;
    const size_t base = (size_t)s * P + (size_t)bx * W;
    const unsigned dc = smem_u32(stage0 + st * Q::STAGE), dr = dc + Q::CB;
    for (int c = tid; c < N * W / 2; c += NT) {  // spectrum: W/2 chunks (2 complex) per row
      const int row = c / (W / 2), part = c % (W / 2);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dc + 16 * c),
                   "l"(A.cbuf + base + (size_t)row * N + 2 * part));
    }
    for (int c = tid; c < N * W / 4; c += NT) {  // r_prev: W/4 chunks per row
      const int row = c / (W / 4), part = c % (W / 4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dr + 16 * c),
                   "l"(A.r_state + base + (size_t)row * N + 4 * part));
    }
  };
  // a launch of one item per CTA (single-stream latency mode) keeps the early trigger: S2's
  // NOTRIG bit is about the dependent sitting beside a *persistent* S2 (c2 p50 31.5 -> 25.5 us)
  if (total <= G) DDH_PDL_TRIGGER();
  else DDH_PDL_TRIGGER_K(4);
  load_tw_async<N>(tw, A.tw4, tid, NT);  // the oldest group: complete at the first wait_group 1
  DDH_PDL_WAIT();
  double p1n = 0.0;  // the first item's partial (nb1 <= 32: one per lane, before the slab copies), then one item ahead
  if (A.nb1 <= 32 && (int)blockIdx.x < total && (tid & 31) < A.nb1)
    p1n = __ldg(A.part1 + (size_t)(blockIdx.x / NC) * A.nb1 + (tid & 31));
  if ((int)blockIdx.x < total) issue(blockIdx.x, 0);
  asm volatile("cp.async.commit_group;");
  if ((int)blockIdx.x + G < total) issue(blockIdx.x + G, 1);
  asm volatile("cp.async.commit_group;");
  int k = 0;
  for (int item = blockIdx.x; item < total; item += G, ++k) {
#if DDH_PDL_LATE & 4
    if (item + G >= total) DDH_PDL_TRIGGER();  // the dependent launches as the last items start
#endif
    const int st = k & 1, bx = item % NC, s = item / NC;
    const int col = bx * W + b;
    const size_t off = (size_t)s * P;
    float2 *slab = reinterpret_cast<float2 *>(stage0 + st * Q::STAGE);  // [N][W]
    const float *rsl = reinterpret_cast<const float *>(stage0 + st * Q::STAGE + Q::CB);
    // the stream's ||y - mu||^2 partials (one per lane at nb1 <= 32, loaded one item ahead:
    // issued at the item start their L2 latency was 28-32 % of the kernel's stall samples,
    // the compiler hoisting the reduction up to the load)
    double p1 = p1n;
    if (A.nb1 <= 32) {
      const int lane = tid & 31;
      p1n = (item + G < total && lane < A.nb1) ? __ldg(A.part1 + (size_t)((item + G) / NC) * A.nb1 + lane) : 0.0;
    } else {
      p1 = 0.0;
      for (int bb = tid & 31; bb < A.nb1; bb += 32) p1 += A.part1[(size_t)s * A.nb1 + bb];
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // item k's group (one newer may be pending)
    __syncthreads();  // every thread's chunks (and the twiddles) visible
    float2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = slab[(t + TPV * e) * W + b];
    __syncthreads();  // the slab becomes the exchange buffer
    fft_reg<N>(v, t, slab + b, [](int p) { return p * W; }, tw);
    const double d2 = warp_sum(p1);
    const bool degenerate = !(d2 > 0.0);
    const float kappa = degenerate ? 0.f : (float)sqrt((double)P / d2);  // Eq. 4
    if (bx == 0 && tid == 0) {
      if (A.status) call_status(A)[s] = degenerate ? 1 : 0;
      A.sstat[(size_t)s * kStatW + 5] = kappa;
      A.sstat[(size_t)s * kStatW + 6] = degenerate ? 1.f : 0.f;
    }
    const float scale = kappa / (float)N;  // F_c = chi F chi / N
    const bool warm = A.warm && !degenerate;
    float2 w2[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int ki = t + TPV * out_comb<N>(e);
      const size_t g = off + (size_t)ki * N + col;
      const float sg = ((ki + col) & 1) ? -scale : scale;
      const float2 u = p_mul(v[e], bc2(sg));
      float r0, q;
      const float2 mu = estep_px(u, rsl[ki * W + b], warm, A.oml, A.la, A.r_min, A.s2, r0, q);
      A.rinit[g] = r0;
      A.q[g] = q;
      const float cs = ((ki + col) & 1) ? -1.f : 1.f;
      w2[out_comb<N>(e)] = make_float2(cs * mu.x, -cs * mu.y);
    }
    __syncthreads();  // exchange buffer free
    fft_reg<N>(w2, t, slab + b, [](int p) { return p * W; }, tw);
#pragma unroll
    for (int e = 0; e < E; ++e) A.cbuf[off + (size_t)(t + TPV * out_comb<N>(e)) * N + col] = w2[e];
    __syncthreads();  // stage st free
    if (item + 2 * G < total) issue(item + 2 * G, st);
    asm volatile("cp.async.commit_group;");
  }
}

// ------------------------------------------------------------------ S4

template <int N>
__device__ __forceinline__ void rows_inv_body(const StepArgs &A, const int bx, const int s) {
  using C = SCfg<N>;
  constexpr int E = C::E, TPV = C::TPV, H = C::H, NT = C::NTR, P = N * N;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;
  float2 *buf = reinterpret_cast<float2 *>(smem4 + N);
  float2 *ys = buf + H * C::RPITCH;  // [H][N]: y rows staged by cp.async (read in the epilogue)
  const int tid = threadIdx.x;
  const int t = tid % TPV, b = tid / TPV;
  const int i = bx * H + b;
  const size_t row = (size_t)s * P + (size_t)i * N;
  DDH_PDL_TRIGGER_K(8);
  const int2 sp = __ldg(A.rowspan + i);  // constant: loaded before the wait, used in the epilogue
  load_tw_async<N>(tw, A.tw4, tid, NT);  // commit group 1 of 2
  {  // y is read-only user input: staged before the wait (commit group 2 of 2)
    const char *src = reinterpret_cast<const char *>(call_y(A, A.y) + (size_t)s * P + (size_t)bx * H * N);
    const unsigned dst = (unsigned)__cvta_generic_to_shared(ys);
    for (int k = tid * 16; k < H * N * 8; k += NT * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + k), "l"(src + k));
    asm volatile("cp.async.commit_group;");
  }
  DDH_PDL_WAIT();
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = A.cbuf[row + t + TPV * e];
  const float *stt = A.sstat + (size_t)s * kStatW;  // from S1 (mu) and S2 (kappa)
  const float mur = stt[0], mui = stt[1], kappa = stt[5];
  asm volatile("cp.async.wait_group 1;" ::: "memory");  // the twiddle group (y may still be in flight)
  __syncthreads();  // twiddles
  fft_reg<N>(v, t, buf + b * C::RPITCH, [](int p) { return rpad(p); }, tw);
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();  // y rows staged
  // v = G = conj(F) with F = inverse row DFT; f = chi F / N, so
  // z = y-hat conj(f) = y-hat chi G / N
  const float kn = kappa / (float)N, two_s2 = 2.f / A.s2;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = t + TPV * out_comb<N>(e);
    float c = 0.f, th = 0.f;
    if (j >= sp.x && j < sp.y) {
      const float sg = ((i + j) & 1) ? -kn : kn;
      const float2 yh = p_mul(p_sub(ys[b * N + j], make_float2(mur, mui)), bc2(sg));
      const float2 g = v[e];
      const float2 z = p_fma(bc2(yh.x), g, p_mul(bc2(yh.y), make_float2(-g.y, g.x)));  // yh * g
      c = two_s2 * sqrt_approx(fmaf(z.x, z.x, z.y * z.y) + 1e-37f);
      th = atan2_fast(z.y, z.x);
    }
    A.cbuf[row + j] = make_float2(c, th);  // in place: this CTA read its spectrum rows before the FFT
  }
  if constexpr (NT == kS0Threads) {  // S0's thread mapping (s4_sums_next checks it on the host)
  if (A.ynx) {  // the next frame's S0 y sums over this CTA's rows (after S1 of this frame read part0)
    __shared__ double red[32 * 2];
    const int per = P / A.nb0, nbk = H * N / per;  // S0 blocks in this CTA (s4_sums_next: integral)
    const float2 *YN = call_y(A, A.ynx);
    for (int kb = 0; kb < nbk; ++kb) {
      const size_t base = (size_t)bx * H * N + (size_t)kb * per;
      double yr = 0.0, yi = 0.0;
      // ks_stats' partition and order: thread t sums the 8-pixel chunks base + 8 t + 8 kS0Threads k
      // (balanced FP32 tree per chunk, FP64 accumulation), then the same block tree
      for (size_t p0 = base + (size_t)tid * 8; p0 < base + per; p0 += (size_t)kS0Threads * 8) {
        const float4 *y4 = reinterpret_cast<const float4 *>(YN + (size_t)s * P + p0);
        float4 a[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = __ldg(y4 + k);
        yr += (double)(((a[0].x + a[0].z) + (a[1].x + a[1].z)) + ((a[2].x + a[2].z) + (a[3].x + a[3].z)));
        yi += (double)(((a[0].y + a[0].w) + (a[1].y + a[1].w)) + ((a[2].y + a[2].w) + (a[3].y + a[3].w)));
      }
      double d[2] = {yr, yi};
      block_sum<2>(d, red);
      if (tid == 0) {
        A.part0[((size_t)s * A.nb0 + base / per) * 5 + 0] = d[0];
        A.part0[((size_t)s * A.nb0 + base / per) * 5 + 1] = d[1];
      }
    }
  }
  }
}

template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTR, 1024 / SCfg<N>::NTR) ks_rows_inv(StepArgs A) {
  rows_inv_body<N>(A, blockIdx.x, blockIdx.y);
}

// ------------------------------------------------------------ ICD tiles

namespace {
constexpr int kHalo = 4;  // = 4 colour phases x 1 sweep (R8)
// Tile geometry: TILE x TILE core, region TILE + 2 kHalo, stored colour-separated:
// sub-grid c = 2 (i&1) + (j&1), element (i>>1, j>>1).  64 for throughput, 32 when
// a launch has too few 64-tiles to fill the SMs (single-stream latency).
template <int TILE> struct Icd {
  static constexpr int kReg = TILE + 2 * kHalo, kSub = kReg / 2, kSubP = kSub + 1;
  static constexpr int kIcdGrid = 4 * kSub * kSubP;  // floats per colour-separated tile
  static __device__ __forceinline__ int sidx(int c, int a, int b) { return (c * kSub + a) * kSubP + b; }
  // debug build: index inside the tile, in colour sub-grid `col` (or any other than `not_col`)
  static __device__ __forceinline__ void chk(int idx, int col, int not_col) {
    DDH_DBG(idx >= 0 && idx < kIcdGrid);
    DDH_DBG(idx % kSubP < kSub);                 // never the padding column
    DDH_DBG(col < 0 || idx / (kSub * kSubP) == col);
    DDH_DBG(not_col < 0 || idx / (kSub * kSubP) != not_col);
  }
  // neighbour (di, dj) of a pixel of colour (ci, cj) at sub coords (a, b):
  // colour ((ci+di)&1, (cj+dj)&1), sub coords (a + floor((ci+di)/2), b + floor((cj+dj)/2))
  template <int CI, int CJ, int DI, int DJ>
  static __device__ __forceinline__ int nidx(int a, int b) {
    constexpr int ti = CI + DI, tj = CJ + DJ;
    constexpr int pi = ti & 1, pj = tj & 1;
    constexpr int oa = (ti - pi) / 2, ob = (tj - pj) / 2;
    return sidx(2 * pi + pj, a + oa, b + ob);
  }
};
// sub-coordinate range of colour parity p updated in a phase covering local
// rows [lo, hi): smallest a with 2a+p >= lo, first a with 2a+p >= hi
__host__ __device__ constexpr int sub_lo(int lo, int p) { return (lo - p + 1) / 2; }
}  // namespace

// r M-step: one 4-colour sweep of the qGGMRF ICD (R6-R9) for the 64x64 tile
// (blockIdx.x, blockIdx.y) of stream blockIdx.z, from A.icd_in (r after Eq. 3,
// or the previous sweep) into A.icd_out (+ A.icd_copy).  The tile is loaded
// colour-separated with a 4-pixel periodic halo; colour phase c updates the
// pixels of colour c in the region shrunk by c+1 on each side, so after the 4
// phases the 64x64 core equals the global colour-ordered sweep.  q is read
// from global (L2) at the pixel's update and only r is staged (21 KB smem),
// within 32 registers.  The 64x64 tile runs 320 threads (6 CTAs, 60 warps
// per SM): its colour phases (1225, 1156, 1089, 1024 pixels) take 4 passes
// each, against 5/5/5/4 at 256 threads.
template <int N, int TILE, int NTH = kSThreads>
__global__ void __launch_bounds__(NTH, 2048 / NTH) ks_ricd(StepArgs A) {
  using G = Icd<TILE>;
  constexpr int T = N < TILE ? N : TILE, P = N * N;
  extern __shared__ float icd_sm[];
  float *rs = icd_sm;
  const int tid = threadIdx.x, s = blockIdx.z;
  const int i0 = blockIdx.y * T, j0 = blockIdx.x * T;
  const size_t off = (size_t)s * P;
  const float *__restrict__ rin = A.icd_in + off;
  const float *__restrict__ qin = A.q + off;
  DDH_PDL_TRIGGER_K(16);
  DDH_PDL_WAIT();
  {  // thread = one pair column pj of the region, rows r0, r0 + RP, ...
    constexpr int RP = NTH / G::kSub;
    const int pj = tid % G::kSub, r0 = tid / G::kSub;
    if (r0 < RP) {
      const float *src = rin + ((j0 - kHalo + 2 * pj) & (N - 1));
#pragma unroll 4
      for (int li = r0; li < G::kReg; li += RP) {
        const float2 v = *reinterpret_cast<const float2 *>(src + (size_t)((i0 - kHalo + li) & (N - 1)) * N);
        DDH_DBG(li < G::kReg && pj < G::kSub && 2 * pj + 1 < G::kReg);
        G::chk(G::sidx(2 * (li & 1), li >> 1, pj) + G::kSub * G::kSubP, 2 * (li & 1) + 1, -1);
        float *d = rs + G::sidx(2 * (li & 1), li >> 1, pj);
        d[0] = v.x;                     // colour (li & 1, 0)
        d[G::kSub * G::kSubP] = v.y;    // colour (li & 1, 1)
      }
    }
  }
  const bool degenerate = A.sstat[(size_t)s * kStatW + 6] != 0.f;
  __syncthreads();
  if (A.r_prior && !degenerate) {
    const float h = A.r_h, g = A.r_g, kq = A.r_k, b6 = A.r_b6, rmin = A.r_min;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ci = c >> 1, cj = c & 1;
      const int alo = sub_lo(c + 1, ci), ahi = sub_lo(G::kReg - c - 1, ci);
      const int blo = sub_lo(c + 1, cj), bhi = sub_lo(G::kReg - c - 1, cj);
      const int nbb = bhi - blo, cnt = (ahi - alo) * nbb;
#pragma unroll 1
      for (int p = tid; p < cnt; p += NTH) {
        const int a = alo + p / nbb, bb = blo + p % nbb;
        float ri, n0, n1, n2, n3, d0, d1, d2v, d3;
#define DDH_NB(CI, CJ)                                                                       \
  ri = rs[G::sidx(2 * CI + CJ, a, bb)];                                                          \
  n0 = rs[G::template nidx<CI, CJ, -1, 0>(a, bb)]; n1 = rs[G::template nidx<CI, CJ, 1, 0>(a, bb)];                    \
  n2 = rs[G::template nidx<CI, CJ, 0, -1>(a, bb)]; n3 = rs[G::template nidx<CI, CJ, 0, 1>(a, bb)];                    \
  d0 = rs[G::template nidx<CI, CJ, -1, -1>(a, bb)]; d1 = rs[G::template nidx<CI, CJ, -1, 1>(a, bb)];                  \
  d2v = rs[G::template nidx<CI, CJ, 1, -1>(a, bb)]; d3 = rs[G::template nidx<CI, CJ, 1, 1>(a, bb)];
        if (c == 0) { DDH_NB(0, 0) } else if (c == 1) { DDH_NB(0, 1) } else if (c == 2) { DDH_NB(1, 0) } else { DDH_NB(1, 1) }
#undef DDH_NB
#if DDH_DEBUG_BOUNDS
        {  // own pixel in sub-grid c; the 8 neighbours in the other sub-grids (no read of a pixel this phase writes)
          G::chk(G::sidx(c, a, bb), c, -1);
          if (A.dbg_fault) G::chk(G::sidx(c, a, bb), -1, c);  // injected: "own pixel not of colour c" fails
          const int ci_ = c >> 1, cj_ = c & 1;
          for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj) {
              if (!di && !dj) continue;
              const int ti = ci_ + di, tj = cj_ + dj, pi = ti & 1, pj2 = tj & 1;
              G::chk(G::sidx(2 * pi + pj2, a + (ti - pi) / 2, bb + (tj - pj2) / 2), -1, c);
            }
        }
#endif
        const int gi = (i0 - kHalo + 2 * a + ci) & (N - 1), gj = (j0 - kHalo + 2 * bb + cj) & (N - 1);
        DDH_DBG(gi >= 0 && gi < N && gj >= 0 && gj < N);
        const float q = __ldg(qin + (size_t)gi * N + gj);
        const float2 nA = make_float2(n0, n1), nB = make_float2(n2, n3);
        const float2 dA = make_float2(d0, d1), dB = make_float2(d2v, d3);
        const float2 wA = qgg_w2(ri, nA, h, g, kq), wB = qgg_w2(ri, nB, h, g, kq);
        const float2 wC = qgg_w2(ri, dA, h, g, kq), wD = qgg_w2(ri, dB, h, g, kq);
        const float2 bs = p_fma(p_add(wC, wD), bc2(0.5f), p_add(wA, wB));
        const float2 ss = p_fma(p_fma(wC, dA, p_mul(wD, dB)), bc2(0.5f), p_fma(wA, nA, p_mul(wB, nB)));
        rs[G::sidx(c, a, bb)] = r_update(ri, q, b6 * (bs.x + bs.y), b6 * (ss.x + ss.y), rmin);
      }
      __syncthreads();
    }
  }
  constexpr int PR = T / 2;  // pixel pairs per tile row
  // one column pair per thread when the thread count allows it (constant address steps)
  constexpr int STEP = NTH % PR == 0 ? NTH : 1;
  const int pj0 = tid % PR, oi0 = tid / PR;
  float *const copy = call_copy(A);
  for (int idx = NTH % PR == 0 ? oi0 * PR + pj0 : tid; idx < T * PR; idx += (NTH % PR == 0 ? STEP : NTH)) {
    const int oi = idx / PR, pj = idx - oi * PR;
    const int li = oi + kHalo;
    const size_t gidx = off + (size_t)(i0 + oi) * N + (j0 + 2 * pj);
    DDH_DBG(i0 + oi < N && j0 + 2 * pj + 1 < N && gidx + 1 < (size_t)A.sc * P);
    G::chk(G::sidx(2 * (li & 1) + 1, li >> 1, pj + kHalo / 2), 2 * (li & 1) + 1, -1);
    float2 v = make_float2(rs[G::sidx(2 * (li & 1), li >> 1, pj + kHalo / 2)], rs[G::sidx(2 * (li & 1) + 1, li >> 1, pj + kHalo / 2)]);
    if (!A.r_prior && !degenerate) {
      const float2 qv = *reinterpret_cast<const float2 *>(A.q + gidx);
      v = make_float2(fmaxf(qv.x, A.r_min), fmaxf(qv.y, A.r_min));
    }
    *reinterpret_cast<float2 *>(A.icd_out + gidx) = v;
    if (copy) *reinterpret_cast<float2 *>(copy + gidx) = v;
  }
}

// Fixed-column thread map of the ICD tiles: thread t owns sub-column
// bcol = t mod kSub and the sub-rows arow0 + R k (arow0 = t / kSub), the same
// slots in every colour phase, so all shared-memory addresses of a phase are
// one per-thread base plus compile-time offsets and the per-pixel operands
// from global memory (q, or the (c, theta) pairs) of a whole phase are issued
// before its first update.  NTH = R kSub threads, KP passes per phase (the
// last one partial): 64-tiles 8 x 36 = 288 threads (7 CTAs per SM), 32-tiles
// 10 x 20 = 200, 16-tiles 12 x 12 = 144.

template <int TILE> struct IcdMap;
template <> struct IcdMap<64> { static constexpr int R = 8; };
template <> struct IcdMap<32> { static constexpr int R = 10; };
template <> struct IcdMap<16> { static constexpr int R = 12; };
template <int TILE> struct IcdT {
  using G = Icd<TILE>;
  static constexpr int R = IcdMap<TILE>::R, NTH = R * G::kSub, KP = (G::kSub + R - 1) / R;
  static constexpr int MINB = 2048 / NTH < 8 ? 2048 / NTH : 8;
};

// One colour phase C of the phi-ICD over this thread's slots (free edge: in
// EDGE tiles, slots outside the frame are absent and the frame-boundary
// pixels drop their missing neighbours from sum b).
template <int N, int TILE, int C, bool EDGE>
__device__ __forceinline__ void phiicd_phase(float *ps, const float2 *cts, int b0, int arow0, int bcol,
                                             int I0, int J0, float w, bool prior) {
  using G = Icd<TILE>;
  using M = IcdT<TILE>;
  constexpr int R = M::R, KP = M::KP, CI = C >> 1, CJ = C & 1;
  constexpr int alo = sub_lo(C + 1, CI), ahi = sub_lo(G::kReg - C - 1, CI);
  constexpr int blo = sub_lo(C + 1, CJ), bhi = sub_lo(G::kReg - C - 1, CJ);
  const int gj = J0 + CJ;
  if (bcol < blo || bcol >= bhi || (EDGE && (unsigned)gj >= (unsigned)N)) return;
  // the thread's slots k of this phase form one range [kb, ke): rows a = arow0 + R k
  // inside [alo, ahi) and, in EDGE tiles, frame rows gi = I0 + CI + 2 R k inside [0, N)
  auto cdiv = [](int x, int d) { return x >= 0 ? (x + d - 1) / d : -((-x) / d); };  // ceil(x / d), d > 0
  int kb = max(0, cdiv(alo - arow0, R)), ke = min(KP, cdiv(ahi - arow0, R));
  if (EDGE) {
    kb = max(kb, cdiv(-(I0 + CI), 2 * R));
    ke = min(ke, cdiv(N - (I0 + CI), 2 * R));
  }
  const bool lr_edge = EDGE && (gj == 0 || gj == N - 1);  // this thread's column is a frame edge
  float2 cn = kb < ke ? ldg_last2(cts + (size_t)(I0 + CI + 2 * R * kb) * N + gj) : make_float2(0.f, 0.f);
#pragma unroll 1
  for (int k = kb; k < ke; ++k) {
    const int a = arow0 + R * k, gi = I0 + 2 * R * k + CI;
    const float2 ctk = cn;
    if (k + 1 < ke) cn = ldg_last2(cts + (size_t)(gi + 2 * R) * N + gj);
    DDH_DBG(a >= alo && a < ahi && (!EDGE || (unsigned)gi < (unsigned)N));
    (void)a;
    const int o = b0 + R * k * G::kSubP;
#if DDH_DEBUG_BOUNDS
    DDH_DBG(o == G::sidx(0, a, bcol));
    G::chk(o + G::sidx(C, 0, 0), C, -1);
    G::chk(o + G::template nidx<CI, CJ, -1, 0>(0, 0), -1, C); G::chk(o + G::template nidx<CI, CJ, 1, 0>(0, 0), -1, C);
    G::chk(o + G::template nidx<CI, CJ, 0, -1>(0, 0), -1, C); G::chk(o + G::template nidx<CI, CJ, 0, 1>(0, 0), -1, C);
    G::chk(o + G::template nidx<CI, CJ, -1, -1>(0, 0), -1, C); G::chk(o + G::template nidx<CI, CJ, -1, 1>(0, 0), -1, C);
    G::chk(o + G::template nidx<CI, CJ, 1, -1>(0, 0), -1, C); G::chk(o + G::template nidx<CI, CJ, 1, 1>(0, 0), -1, C);
    DDH_DBG(!EDGE || ((unsigned)gi < (unsigned)N && (unsigned)gj < (unsigned)N));
#endif
    const float pi_ = ps[o + G::sidx(C, 0, 0)];
    const float n4 = (ps[o + G::template nidx<CI, CJ, -1, 0>(0, 0)] + ps[o + G::template nidx<CI, CJ, 1, 0>(0, 0)]) +
                     (ps[o + G::template nidx<CI, CJ, 0, -1>(0, 0)] + ps[o + G::template nidx<CI, CJ, 0, 1>(0, 0)]);
    const float nd = (ps[o + G::template nidx<CI, CJ, -1, -1>(0, 0)] + ps[o + G::template nidx<CI, CJ, -1, 1>(0, 0)]) +
                     (ps[o + G::template nidx<CI, CJ, 1, -1>(0, 0)] + ps[o + G::template nidx<CI, CJ, 1, 1>(0, 0)]);
    const float nb = fmaf(nd, 1.f / 12.f, n4 * (1.f / 6.f));
    float sb = 1.f;  // sum of b over the existing neighbours (the expression is exactly 1 inside)
    if (EDGE && (lr_edge || gi == 0 || gi == N - 1)) {
      const bool tp = gi == 0, bt = gi == N - 1, lf = gj == 0, rt = gj == N - 1;
      sb = 1.f - (1.f / 6.f) * (float)(tp + bt + lf + rt) -
           (1.f / 12.f) * (float)((tp | lf) + (tp | rt) + (bt | lf) + (bt | rt));
    }
    ps[o + G::sidx(C, 0, 0)] = phi_update(pi_, ctk.x, ctk.y, nb, sb, w, prior);
  }
}

template <int N, int TILE, bool EDGE>
__device__ __forceinline__ void phiicd_sweep(float *ps, const float2 *cts, int tid, int i0, int j0, float w, bool prior) {
  using G = Icd<TILE>;
  const int bcol = tid % G::kSub, arow0 = tid / G::kSub;
  const int b0 = arow0 * G::kSubP + bcol;
  const int I0 = i0 - kHalo + 2 * arow0, J0 = j0 - kHalo + 2 * bcol;
  phiicd_phase<N, TILE, 0, EDGE>(ps, cts, b0, arow0, bcol, I0, J0, w, prior);
  __syncthreads();
  phiicd_phase<N, TILE, 1, EDGE>(ps, cts, b0, arow0, bcol, I0, J0, w, prior);
  __syncthreads();
  phiicd_phase<N, TILE, 2, EDGE>(ps, cts, b0, arow0, bcol, I0, J0, w, prior);
  __syncthreads();
  phiicd_phase<N, TILE, 3, EDGE>(ps, cts, b0, arow0, bcol, I0, J0, w, prior);
  __syncthreads();
}

// phi M-step: one 4-colour sweep of the GMRF ICD (R10-R11) on a TILE x TILE
// tile with a 4-pixel halo; free boundary: neighbours outside the frame are
// absent (value 0 in the tile, excluded from sum b).  The first sweep of a
// time step subtracts the RemoveTipTilt plane (S1's per-stream scalars) on load.
template <int N, int TILE>
__global__ void __launch_bounds__(IcdT<TILE>::NTH, IcdT<TILE>::MINB) ks_phiicd(StepArgs A) {
  using G = Icd<TILE>;
  constexpr int NTH = IcdT<TILE>::NTH, T = N < TILE ? N : TILE, P = N * N;
  extern __shared__ float icd_sm[];
  float *ps = icd_sm;
  const int tid = threadIdx.x, s = blockIdx.z;
  const int i0 = blockIdx.y * T, j0 = blockIdx.x * T;
  const size_t off = (size_t)s * P;
  const float *__restrict__ pin = A.icd_in + off;
  DDH_PDL_TRIGGER_K(32);
  DDH_PDL_WAIT();

  const float *st = A.sstat + (size_t)s * kStatW;
  const bool degenerate = st[6] != 0.f;
  const bool plane = A.apply_plane && !degenerate;
  const float c0 = plane ? st[2] : 0.f, c1 = plane ? st[3] : 0.f, c2 = plane ? st[4] : 0.f;
  {  // thread = one pair column pj of the region, rows r0, r0 + RP, ...
    constexpr int RP = NTH / G::kSub;
    const int pj = tid % G::kSub, r0 = tid / G::kSub;
    if (r0 < RP) {
      const int gj = j0 - kHalo + 2 * pj;
      const bool jin = gj >= 0 && gj < N;  // pairs are both inside or both outside
      const float px = fmaf(c1, (float)(gj - N / 2), c0);
      const float *src = pin + gj;
#pragma unroll kS5LoadUnroll
      for (int li = r0; li < G::kReg; li += RP) {
        const int gi = i0 - kHalo + li;
        float2 v = make_float2(0.f, 0.f);
        if (jin && gi >= 0 && gi < N) {
          const float2 f = *reinterpret_cast<const float2 *>(src + (size_t)gi * N);
          const float pl = fmaf(c2, (float)(gi - N / 2), px);
          v = make_float2(f.x - pl, f.y - (pl + c1));
        }
        float *d = ps + G::sidx(2 * (li & 1), li >> 1, pj);
        d[0] = v.x;
        d[G::kSub * G::kSubP] = v.y;
      }
    }
  }
  const float2 *cts = A.cbuf + off;  // (c, theta) pairs from S4
  __syncthreads();
  if (!degenerate) {
    const bool prior = A.phi_prior != 0;
    const float w = A.phi_w;
    if (i0 == 0 || j0 == 0 || i0 + T == N || j0 + T == N)  // tile touches the frame edge
      phiicd_sweep<N, TILE, true>(ps, cts, tid, i0, j0, w, prior);
    else
      phiicd_sweep<N, TILE, false>(ps, cts, tid, i0, j0, w, prior);
  }
  // output (and the RemoveTipTilt sums of the output phase for the next frame's S1)
  float *const copy = call_copy(A);
  constexpr int PR = T / 2;  // pixel pairs per tile row
  double e0 = 0.0, ex = 0.0, ey = 0.0;
  if constexpr (NTH % PR == 0) {
    // every thread keeps one column pair: addresses advance by constants, the
    // x moments come from the two column sums at the end
    constexpr int RS = NTH / PR;  // tile rows per pass
    const int pj = tid % PR, oi0 = tid / PR;
    const int gj = j0 + 2 * pj;
    const float *psrc = ps + G::sidx(0, 0, pj + kHalo / 2);
    size_t g = off + (size_t)(i0 + oi0) * N + gj;
    double c0 = 0.0, c1 = 0.0;
#pragma unroll 2
    for (int oi = oi0; oi < T; oi += RS, g += (size_t)RS * N) {
      const int li = oi + kHalo;
      const float *q = psrc + (2 * (li & 1) * G::kSub + (li >> 1)) * G::kSubP;
      const float2 v = degenerate ? *reinterpret_cast<const float2 *>(pin + (g - off)) : make_float2(q[0], q[G::kSub * G::kSubP]);
      *reinterpret_cast<float2 *>(A.icd_out + g) = v;
      if (copy) *reinterpret_cast<float2 *>(copy + g) = v;
      if (A.psum_out) {
        const int gi = i0 + oi;
        const int2 sp = __ldg(A.rowspan + gi);
        const double q0 = (gj >= sp.x && gj < sp.y) ? (double)fixq(v.x) : 0.0;
        const double q1 = (gj + 1 >= sp.x && gj + 1 < sp.y) ? (double)fixq(v.y) : 0.0;
        c0 += q0;
        c1 += q1;
        ey = fma(q0 + q1, (double)(gi - N / 2), ey);
      }
    }
    e0 = c0 + c1;
    ex = fma(c0, (double)(gj - N / 2), c1 * (double)(gj + 1 - N / 2));
  } else {
    for (int idx = tid; idx < T * PR; idx += NTH) {
      const int oi = idx / PR, pj = idx - oi * PR;
      const int li = oi + kHalo;
      const size_t g = off + (size_t)(i0 + oi) * N + (j0 + 2 * pj);
      const float2 v = degenerate ? *reinterpret_cast<const float2 *>(pin + (g - off))
                                  : make_float2(ps[G::sidx(2 * (li & 1), li >> 1, pj + kHalo / 2)],
                                                ps[G::sidx(2 * (li & 1) + 1, li >> 1, pj + kHalo / 2)]);
      *reinterpret_cast<float2 *>(A.icd_out + g) = v;
      if (copy) *reinterpret_cast<float2 *>(copy + g) = v;
      if (A.psum_out) {
        const int gi = i0 + oi, gj = j0 + 2 * pj;
        const int2 sp = __ldg(A.rowspan + gi);
        const double q0 = (gj >= sp.x && gj < sp.y) ? (double)fixq(v.x) : 0.0;
        const double q1 = (gj + 1 >= sp.x && gj + 1 < sp.y) ? (double)fixq(v.y) : 0.0;
        e0 += q0 + q1;
        ex = fma(q0, (double)(gj - N / 2), fma(q1, (double)(gj + 1 - N / 2), ex));
        ey = fma(q0 + q1, (double)(gi - N / 2), ey);
      }
    }
  }
  if (A.psum_out) {
    __shared__ double redd[32 * 3];
    plane_sums_add(e0, ex, ey, redd, A.psum_out + (size_t)s * 3);
  }
}

// ----------------------------------------- r-ICD as global colour passes
// Large launches: the colour-ordered sweep (R8) as four kernels, one per
// colour class (i mod 2, j mod 2) in the order (0,0),(0,1),(1,0),(1,1), one
// thread per pixel of the class.  A neighbour of a lower colour is read from
// the sweep's output (already updated by an earlier pass), of a higher colour
// from its input; pixels of one class never neighbour each other, so a pass
// has no intra-kernel dependency: no tile, no halo, no barrier, and the whole
// GPU is one pool of independent updates.  The per-pixel arithmetic is the
// tile kernels' (same expressions, same order), so the results are the same
// bits as the halo-tile kernels (tests/test_gpu_parity.py kernel variants).

// neighbour (DI, DJ) of a colour-C pixel (i, j), periodic boundary (r-ICD)
template <typename T>
__device__ __forceinline__ T *opaque_ptr(T *p) {
  asm("mov.b64 %0, %0;" : "+l"(p));
  return p;
}

// One qGGMRF r update (R6-R9) from the pixel's value ri, its q and its 8
// neighbours as (n(-1,0), n(1,0)), (n(0,-1), n(0,1)), (d(-1,-1), d(-1,1)),
// (d(1,-1), d(1,1)): the expressions and their order of the tile kernels, so
// every r-ICD kernel produces the same bits.
__device__ __forceinline__ float ricd_px(const StepArgs &A, float ri, float q, float2 nA, float2 nB, float2 dA,
                                         float2 dB) {
  const float h = A.r_h, gg = A.r_g, kq = A.r_k;
  const float2 wA = qgg_w2(ri, nA, h, gg, kq), wB = qgg_w2(ri, nB, h, gg, kq);
  const float2 wC = qgg_w2(ri, dA, h, gg, kq), wD = qgg_w2(ri, dB, h, gg, kq);
  const float2 bs = p_fma(p_add(wC, wD), bc2(0.5f), p_add(wA, wB));
  const float2 ss = p_fma(p_fma(wC, dA, p_mul(wD, dB)), bc2(0.5f), p_fma(wA, nA, p_mul(wB, nB)));
  return r_update(ri, q, A.r_b6 * (bs.x + bs.y), A.r_b6 * (ss.x + ss.y), A.r_min);
}

// Indices are 32-bit within the stream (N^2 <= 2^20): one row offset per
// neighbour row and one wrapped column per neighbour column, so each load is
// one 32-bit add and one wide multiply-add onto the stream base.
template <int N, int C, int DI, int DJ>
__device__ __forceinline__ float rnb(const float *__restrict__ in, const float *out, const int (&ro)[3],
                                     const int (&co)[3]) {
  constexpr int CI = C >> 1, CJ = C & 1, NC = 2 * ((CI + DI) & 1) + ((CJ + DJ) & 1);
  const float *src = NC < C ? out : in;  // lower colours were written by earlier passes (read-only now)
  return __ldg(src + (unsigned)(ro[DI + 1] + co[DJ + 1]));
}

template <int N, int C>
__device__ __forceinline__ void ricd_pass_px(const StepArgs &A, int s, int p) {
  constexpr int CI = C >> 1, CJ = C & 1, H = N / 2, P = N * N;
  const int i = 2 * (p / H) + CI, j = 2 * (p % H) + CJ;
  const size_t off = (size_t)s * P;
  const unsigned g = (unsigned)(i * N + j);
  // stream bases made opaque, so every neighbour address is one wide
  // multiply-add of its 32-bit index (not a 64-bit add chain per load)
  const float *__restrict__ in = opaque_ptr(A.icd_in + off);
  float *out = opaque_ptr(A.icd_out + off);
  // the degenerate flag is loaded beside the pixel's operands, not before them
  const float dflag = A.sstat[(size_t)s * kStatW + 6];
  DDH_DBG(i < N && j < N);
  float v;
  if (!A.r_prior) {
    v = dflag != 0.f ? in[g] : fmaxf(__ldg(A.q + off + g), A.r_min);
  } else {
    // q is issued with the neighbour loads (volatile: left to itself the
    // compiler sinks it behind the weights, exposing its latency in r_update)
    const float q = ldg_last(A.q + off + g);
    const float ri = __ldg(in + g);  // written only by this thread, after this read
    // periodic neighbour rows / columns (only one side of a colour class can wrap)
    const int ro[3] = {CI == 0 ? ((i - 1) & (N - 1)) * N : (i - 1) * N, i * N,
                       CI == 1 ? ((i + 1) & (N - 1)) * N : (i + 1) * N};
    const int co[3] = {CJ == 0 ? (j - 1) & (N - 1) : j - 1, j, CJ == 1 ? (j + 1) & (N - 1) : j + 1};
    const float2 nA = make_float2(rnb<N, C, -1, 0>(in, out, ro, co), rnb<N, C, 1, 0>(in, out, ro, co));
    const float2 nB = make_float2(rnb<N, C, 0, -1>(in, out, ro, co), rnb<N, C, 0, 1>(in, out, ro, co));
    const float2 dA = make_float2(rnb<N, C, -1, -1>(in, out, ro, co), rnb<N, C, -1, 1>(in, out, ro, co));
    const float2 dB = make_float2(rnb<N, C, 1, -1>(in, out, ro, co), rnb<N, C, 1, 1>(in, out, ro, co));
    // a degenerate frame keeps r (its root is computed and discarded, so no
    // load waits for the flag)
    const float x = ricd_px(A, ri, q, nA, nB, dA, dB);
    v = dflag != 0.f ? ri : x;
  }
  out[g] = v;
  if (A.icd_copy) call_copy(A)[off + g] = v;
}

// one thread per pixel of the class; grid (N^2/4 / 256, streams).  (A
// grid-stride form sized to the resident CTA slots measured slower in the
// concurrent step: 134.9 vs 128.5 us at c3.)
#ifndef DDH_RICD_MINB
#define DDH_RICD_MINB 8
#endif
template <int N, int C>
__global__ void __launch_bounds__(256, DDH_RICD_MINB) ks_ricd_pass(StepArgs A) {
  DDH_PDL_TRIGGER_K(16);
  DDH_PDL_WAIT();
  ricd_pass_px<N, C>(A, blockIdx.y, blockIdx.x * 256 + threadIdx.x);
}

// ----------------------------------- r-ICD as two row-parity launches
// The four colour passes folded in pairs: launch RP = 0 updates colours 0 and
// 1 (rows i even), launch RP = 1 colours 2 and 3 (rows i odd).  A thread owns
// the pixel pair (i, 2p), (i, 2p+1) and a CTA whole rows, so the pair's
// colour-(RP,1) pixel finds the new colour-(RP,0) values of (i, 2p) and
// (i, 2p+2) -- including the periodic wrap of the row -- in shared memory
// after one barrier.  Each thread loads one float2 from each of rows i-1, i,
// i+1 and of q (the columns 2p-1 and 2p+2 come from the neighbouring pairs
// through shared memory): 4 vector loads per pixel pair instead of 20 scalar
// loads, and two launches per sweep instead of four.  Rows i +- 1 are of the
// other parity: not yet updated for RP = 0 (read from the sweep's input),
// already updated for RP = 1 (read from its output).  Same arithmetic
// (ricd_px) and colour order as the passes and the tiles, so the same bits.
#ifndef DDH_ROWS_NT
#define DDH_ROWS_NT 128
#endif
#ifndef DDH_ROWS_MINB
#define DDH_ROWS_MINB 1
#endif
template <int N> struct RowsCfg {
  static constexpr int H = N / 2, NT = H > DDH_ROWS_NT ? H : DDH_ROWS_NT, RPC = NT / H;  // pairs per row, threads, rows per CTA
  static constexpr int MINB = DDH_ROWS_MINB * DDH_ROWS_NT / NT > 0 ? DDH_ROWS_MINB * DDH_ROWS_NT / NT : 1;
};
template <int N, int RP>
__global__ void __launch_bounds__(RowsCfg<N>::NT, RowsCfg<N>::MINB) ks_ricd_rows(StepArgs A) {
  using RC = RowsCfg<N>;
  constexpr int H = RC::H, NT = RC::NT, RPC = RC::RPC, P = N * N;
  __shared__ float2 sh[3][NT];  // rows i-1, i, i+1 of every pair of the CTA (input values)
  __shared__ float c0n[NT];     // new colour-(RP,0) values
  const int tid = threadIdx.x, s = blockIdx.y;
  const int lr = tid / H, p = tid - lr * H;
  const int i = 2 * (blockIdx.x * RPC + lr) + RP;
  const size_t off = (size_t)s * P;
  const float *__restrict__ in = opaque_ptr(A.icd_in + off);
  const float *__restrict__ nbs = RP == 0 ? in : opaque_ptr(A.icd_out + off);  // rows i +- 1
  const unsigned gm = (unsigned)(((i - 1) & (N - 1)) * N + 2 * p), g0 = (unsigned)(i * N + 2 * p),
                 gp = (unsigned)(((i + 1) & (N - 1)) * N + 2 * p);
  DDH_DBG(i < N && 2 * p + 1 < N && lr < RPC);
  DDH_PDL_TRIGGER_K(16);
  DDH_PDL_WAIT();
  const float dflag = A.sstat[(size_t)s * kStatW + 6];
  const float2 M = __ldg(reinterpret_cast<const float2 *>(in + g0));
  float2 v;
  if (!A.r_prior) {
    const float2 Q = __ldg(reinterpret_cast<const float2 *>(A.q + off + g0));
    v = dflag != 0.f ? M : make_float2(fmaxf(Q.x, A.r_min), fmaxf(Q.y, A.r_min));
  } else {
    const float2 U = __ldg(reinterpret_cast<const float2 *>(nbs + gm));
    const float2 D = __ldg(reinterpret_cast<const float2 *>(nbs + gp));
    const float2 Q = __ldg(reinterpret_cast<const float2 *>(A.q + off + g0));
    const int base = lr * H, pl = base + ((p - 1) & (H - 1)), pr = base + ((p + 1) & (H - 1));
    sh[0][tid] = U;
    sh[1][tid] = M;
    sh[2][tid] = D;
    __syncthreads();
    const float Ul = sh[0][pl].y, Ml = sh[1][pl].y, Dl = sh[2][pl].y;  // column 2p-1
    const float Ur = sh[0][pr].x, Dr = sh[2][pr].x;                    // column 2p+2
    // colour (RP,0) at (i, 2p): every in-row neighbour is of colour (RP,1), not yet updated
    const float x0 = ricd_px(A, M.x, Q.x, make_float2(U.x, D.x), make_float2(Ml, M.y), make_float2(Ul, U.y),
                             make_float2(Dl, D.y));
    const float v0 = dflag != 0.f ? M.x : x0;
    c0n[tid] = v0;
    __syncthreads();
    const float v0r = c0n[pr];  // new value at (i, 2p+2)
    // colour (RP,1) at (i, 2p+1): in-row neighbours (i, 2p), (i, 2p+2) updated just now
    const float x1 = ricd_px(A, M.y, Q.y, make_float2(U.y, D.y), make_float2(v0, v0r), make_float2(U.x, Ur),
                             make_float2(D.x, Dr));
    v = make_float2(v0, dflag != 0.f ? M.y : x1);
  }
  *reinterpret_cast<float2 *>(A.icd_out + off + g0) = v;
  if (A.icd_copy) *reinterpret_cast<float2 *>(call_copy(A) + off + g0) = v;
}

// ------------------------------------------------- stage entry points
// (ddh_test_*: the streaming kernels' own device code on caller buffers)

// Row pass of F_c on B fields: out row = FFT_row(chi . [conj] in row), the
// register FFT and comb layout of S1 / S4.
template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTR) ks_test_rows(const float2 *in, float2 *out, int inverse,
                                                             const float4 *tw4) {
  using C = SCfg<N>;
  constexpr int E = C::E, TPV = C::TPV, H = C::H, NT = C::NTR, P = N * N;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;
  float2 *buf = reinterpret_cast<float2 *>(smem4 + N);
  const int tid = threadIdx.x, s = blockIdx.y;
  const int t = tid % TPV, b = tid / TPV;
  const int i = blockIdx.x * H + b;
  const size_t row = (size_t)s * P + (size_t)i * N;
  load_tw<N>(tw, tw4, tid, NT);
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = t + TPV * e;
    float2 x = in[row + j];
    if (inverse) x.y = -x.y;
    const float sg = ((i + j) & 1) ? -1.f : 1.f;
    v[e] = p_mul(x, bc2(sg));
  }
  __syncthreads();
  fft_reg<N>(v, t, buf + b * C::RPITCH, [](int p) { return rpad(p); }, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) out[row + t + TPV * out_comb<N>(e)] = v[e];
}

// Column pass of F_c: out column = chi/N . FFT_col(in column) [conj], the
// register FFT and comb layout of S2.
template <int N>
__global__ void __launch_bounds__(SCfg<N>::NTC) ks_test_cols(const float2 *in, float2 *out, int inverse,
                                                             const float4 *tw4) {
  using C = SCfg<N>;
  constexpr int E = C::E, TPV = C::TPV, W = C::W, NT = C::NTC, P = N * N;
  extern __shared__ float4 smem4[];
  float4 *tw = smem4;
  float2 *buf = reinterpret_cast<float2 *>(smem4 + N);
  const int tid = threadIdx.x, s = blockIdx.y;
  const int b = tid % W, t = tid / W;
  const int col = blockIdx.x * W + b;
  const size_t off = (size_t)s * P;
  load_tw<N>(tw, tw4, tid, NT);
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = in[off + (size_t)(t + TPV * e) * N + col];
  __syncthreads();
  fft_reg<N>(v, t, buf + b, [](int p) { return p * W; }, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int ki = t + TPV * out_comb<N>(e);
    const float sg = ((ki + col) & 1) ? -1.f / N : 1.f / N;
    float2 x = p_mul(v[e], bc2(sg));
    if (inverse) x.y = -x.y;
    out[off + (size_t)ki * N + col] = x;
  }
}

// Eq. 3 + E-step of S2 (estep_px) on B fields: u complex64, r_prev -> r0, mu, q
__global__ void ks_test_estep(const float2 *u, const float *r_prev, float *r0, float2 *mu, float *q, size_t count,
                              int warm, float oml, float la, float r_min, float s2) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < count; k += (size_t)gridDim.x * blockDim.x) {
    float rr, qq;
    mu[k] = estep_px(u[k], r_prev[k], warm != 0, oml, la, r_min, s2, rr, qq);
    r0[k] = rr;
    q[k] = qq;
  }
}

// (c, theta) pairs in S4's output layout, for the S5 stage entry point
__global__ void ks_test_pack(const float *c, const float *th, float2 *out, size_t count) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < count; k += (size_t)gridDim.x * blockDim.x)
    out[k] = make_float2(c[k], th[k]);
}

// ------------------------------------------------------------- launchers

#define DDH_SDISPATCH(n, CALL)                          \
  switch (n) {                                          \
    case 64: { constexpr int N = 64; CALL; } break;     \
    case 128: { constexpr int N = 128; CALL; } break;   \
    case 256: { constexpr int N = 256; CALL; } break;   \
    case 512: { constexpr int N = 512; CALL; } break;   \
    case 1024: { constexpr int N = 1024; CALL; } break; \
    default: return cudaErrorInvalidValue;              \
  }

// SM count of the current device (queried once per device)
static int device_sms() {
  static int cache[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  if (!cache[d & 63]) cudaDeviceGetAttribute(&cache[d & 63], cudaDevAttrMultiProcessorCount, d);
  return cache[d & 63] > 0 ? cache[d & 63] : 1;
}
template <int N> static size_t srow_smem() { return N * sizeof(float4) + (size_t)SCfg<N>::H * SCfg<N>::RPITCH * sizeof(float2); }
template <int N> static size_t srowi_smem() { return srow_smem<N>() + (size_t)SCfg<N>::H * N * sizeof(float2); }
template <int N> static size_t scol_smem() { return N * sizeof(float4) + (size_t)N * SCfg<N>::W * sizeof(float2); }

template <int N>
static cudaError_t init_stream_n() {
  cudaFuncSetAttribute(ks_rows_fwd<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)srow_smem<N>());
  cudaFuncSetAttribute(ks_rows_fwd_p<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S1P<N>::SMEM);
  cudaFuncSetAttribute(ks_rows_inv<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)srowi_smem<N>());
  cudaFuncSetAttribute(ks_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scol_smem<N>());
  if constexpr (N <= 256) cudaFuncSetAttribute(ks_cols_p<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S2P<N>::SMEM);
  cudaFuncSetAttribute(ks_phiicd<N, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(Icd<64>::kIcdGrid * sizeof(float)));
  cudaFuncSetAttribute(ks_ricd<N, 64, 320>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(Icd<64>::kIcdGrid * sizeof(float)));
  cudaFuncSetAttribute(ks_phiicd<N, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(Icd<32>::kIcdGrid * sizeof(float)));
  cudaFuncSetAttribute(ks_phiicd<N, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(Icd<16>::kIcdGrid * sizeof(float)));
  cudaFuncSetAttribute(ks_ricd<N, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(Icd<32>::kIcdGrid * sizeof(float)));
  cudaFuncSetAttribute(ks_test_rows<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)srow_smem<N>());
  cudaFuncSetAttribute(ks_test_cols<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scol_smem<N>());
  return cudaGetLastError();
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

cudaError_t init_stream(int n) { DDH_SDISPATCH(n, return init_stream_n<N>()); }
int stream_nb1(int n) { DDH_SDISPATCH(n, return N / SCfg<N>::H); }
// S0 pixel blocks per stream: 2048-pixel blocks (8-pixel chunks, kS0Threads
// per pass), at most 64 (the partials every later stage adds per warp)
int stream_nb0(int n) { return n * n / 2048 < 64 ? (n * n / 2048 < 1 ? 1 : n * n / 2048) : 64; }

cudaError_t launch_s0(const StepArgs &a, cudaStream_t st) {
  return launch_pdl(ks_stats, dim3(a.nb0, a.sc), dim3(kS0Threads), 0, st, a);
}
cudaError_t launch_s1(const StepArgs &a, cudaStream_t st) {
  static const int persist = getenv("DDH_S1P") ? atoi(getenv("DDH_S1P")) : 1;
  const int sms = device_sms();
  if (persist) {
    DDH_SDISPATCH(a.n, ({
                    const int total = N / SCfg<N>::H * a.sc;
#ifdef DDH_S1P_PER_SM
                    constexpr int per_sm = DDH_S1P_PER_SM;
#else
                    constexpr int per_sm = 512 / SCfg<N>::NTR;  // resident CTAs per SM (smem, registers)
#endif
                    const int grid = total < per_sm * sms ? total : per_sm * sms;
                    return launch_pdl(ks_rows_fwd_p<N>, dim3(grid), dim3(SCfg<N>::NTR), S1P<N>::SMEM, st, a);
                  }));
  }
  DDH_SDISPATCH(a.n, return launch_pdl(ks_rows_fwd<N>, dim3(N / SCfg<N>::H, a.sc), dim3(SCfg<N>::NTR), srow_smem<N>(), st, a));
}
// staged form for launches of at most two slabs per SM (few streams: c2 step
// 28.8 -> 25.3 us); at 64 streams the plain kernel is as fast
template <int N>
static cudaError_t launch_s2_n(const StepArgs &a, cudaStream_t st, int staged, int sms) {
  if constexpr (N <= 256) {
    const int total = N / SCfg<N>::W * a.sc;
#ifdef DDH_S2P_PER_SM
    constexpr int per_sm = DDH_S2P_PER_SM;
#else
    constexpr int per_sm = 512 / SCfg<N>::NTC;  // resident CTAs per SM (smem, registers)
#endif
    if (staged == 2 || (staged && total <= 2 * sms))  // 2: persistent staged form for every launch (diagnostic)
      return launch_pdl(ks_cols_p<N>, dim3(total < per_sm * sms ? total : per_sm * sms), dim3(SCfg<N>::NTC), S2P<N>::SMEM, st, a);
  }
  return launch_pdl(ks_cols<N>, dim3(N / SCfg<N>::W, a.sc), dim3(SCfg<N>::NTC), scol_smem<N>(), st, a);
}
cudaError_t launch_s2(const StepArgs &a, cudaStream_t st) {
  // the persistent staged form for every launch at N <= 256 (c3: 509.7 -> 513.3 k
  // frames/s; round 1, before the r-ICD passes freed the shared memory, it was neutral
  // there); DDH_S2P=1: only small launches, 0: never (diagnostic)
  static const int staged = getenv("DDH_S2P") ? atoi(getenv("DDH_S2P")) : 2;
  DDH_SDISPATCH(a.n, return launch_s2_n<N>(a, st, staged, device_sms()));
}
template <int N>
static bool s4_sums_fit() {  // a row CTA holds whole S0 blocks, with S0's thread count
  const int per = N * N / stream_nb0(N);
  return SCfg<N>::NTR == kS0Threads && (SCfg<N>::H * N) % per == 0;
}
__global__ void ks_set_desc(CallDesc *d, CallDesc v) { *d = v; }
cudaError_t launch_set_desc(CallDesc *d, const CallDesc &v, cudaStream_t st) {
  ks_set_desc<<<1, 1, 0, st>>>(d, v);
  return cudaGetLastError();
}
bool s4_sums_next(int n) {
  static const int on = getenv("DDH_S4_SUMS") ? atoi(getenv("DDH_S4_SUMS")) : 1;  // 0: S0 on its own stream (diagnostic)
  if (!on) return false;
  switch (n) {
    case 64: return s4_sums_fit<64>();
    case 128: return s4_sums_fit<128>();
    case 256: return s4_sums_fit<256>();
    case 512: return s4_sums_fit<512>();
    case 1024: return s4_sums_fit<1024>();
  }
  return false;
}
cudaError_t launch_s4(const StepArgs &a, cudaStream_t st) {
  DDH_SDISPATCH(a.n, return launch_pdl(ks_rows_inv<N>, dim3(N / SCfg<N>::H, a.sc), dim3(SCfg<N>::NTR), srowi_smem<N>(), st, a));
}
// ICD tile size: 64 (throughput) unless a launch would have fewer 64-tiles
// than two per SM, then 32 (4x the tiles: shorter per-CTA chains, lower
// single-stream latency, +20 % halo recomputation)
template <int N>
static bool small_tiles(int sc) {
  static const int on = getenv("DDH_SMALL_TILES") ? atoi(getenv("DDH_SMALL_TILES")) : 1;  // diagnostic
  return on && N >= 64 && (N / 64) * (N / 64) * sc < 2 * device_sms();
}
// 16x16 tiles when even 32-tiles would leave most SMs idle (one stream at
// N <= 256: 256 CTAs with one pass per colour phase; c2 step 26.3 -> 24.7 us
// despite 2.25x halo work)
template <int N>
static bool tiny_tiles(int sc) {
  static const int on = getenv("DDH_T16") ? atoi(getenv("DDH_T16")) : 1;
  return on && (N / 32) * (N / 32) * sc < device_sms();
}
template <int N, int TILE>
static cudaError_t launch_icd(void (*k)(StepArgs), const StepArgs &a, cudaStream_t st, size_t smem) {
  constexpr int T = N < TILE ? N : TILE;
  return launch_pdl(k, dim3(N / T, N / T, a.sc), dim3(IcdT<TILE>::NTH), smem, st, a);
}
// the global colour passes for the r-ICD launches that would use the 64-tiles
// (DDH_RICD_PASSES=0: the tiles; diagnostic).  The phi-ICD stays on tiles: its
// cheap update is bound by operand traffic, and the passes' per-neighbour
// global loads (no shared tile) measured 44.4 vs 33.3 us at c3.
template <int N>
static bool use_passes(int sc, bool r) {
  static const int on = getenv("DDH_RICD_PASSES") ? atoi(getenv("DDH_RICD_PASSES")) : 1;
  if (on == 2) return r;  // diagnostic: passes at every size
  return r && on && !small_tiles<N>(sc) && !tiny_tiles<N>(sc);
}
// The two row-parity launches (ks_ricd_rows) for every r-ICD launch at
// N >= 512 (measured, one B200: c4 116.0 -> 119.5 k frames/s against the
// passes, c5 15.2 -> 15.6 k against the 32-tiles), not at N <= 256: c3's three
// concurrent lanes 120.3 -> 123.9 us per step (the barrier-free passes fill the
// gaps between the other lanes' kernels better), c2 23.7 -> 26.7 us against
// the 16-tiles.  DDH_RICD_ROWS (diagnostic): 0 never, 2 wherever the passes
// would run, 3 at every size.
template <int N>
static bool use_rows(int sc) {
  static const int on = getenv("DDH_RICD_ROWS") ? atoi(getenv("DDH_RICD_ROWS")) : 1;
  if (on == 0) return false;
  if (on == 3) return true;
  if (on == 2) return use_passes<N>(sc, true);
  return N >= 512;
}
int icd_launches(const StepArgs &a, bool r) {
  DDH_SDISPATCH(a.n, return r && use_rows<N>(a.sc) ? 2 : use_passes<N>(a.sc, r) ? 4 : 1);
  return 1;
}
template <int N>
static cudaError_t launch_rows(const StepArgs &a, cudaStream_t st) {
  using RC = RowsCfg<N>;
  const dim3 grid((N / 2) / RC::RPC, a.sc);
  cudaError_t e = launch_pdl(ks_ricd_rows<N, 0>, grid, dim3(RC::NT), 0, st, a);
  if (e == cudaSuccess) e = launch_pdl(ks_ricd_rows<N, 1>, grid, dim3(RC::NT), 0, st, a);
  return e;
}
template <int N>
static cudaError_t launch_passes(const StepArgs &a, cudaStream_t st, void (*k0)(StepArgs), void (*k1)(StepArgs),
                                 void (*k2)(StepArgs), void (*k3)(StepArgs)) {
  const dim3 grid((N / 2) * (N / 2) / 256, a.sc);
  cudaError_t e = launch_pdl(k0, grid, dim3(256), 0, st, a);
  if (e == cudaSuccess) e = launch_pdl(k1, grid, dim3(256), 0, st, a);
  if (e == cudaSuccess) e = launch_pdl(k2, grid, dim3(256), 0, st, a);
  if (e == cudaSuccess) e = launch_pdl(k3, grid, dim3(256), 0, st, a);
  return e;
}

cudaError_t launch_s3(const StepArgs &a, cudaStream_t st) {
  DDH_SDISPATCH(a.n, ({
                  if (use_rows<N>(a.sc)) return launch_rows<N>(a, st);
                  if (use_passes<N>(a.sc, true))
                    return launch_passes<N>(a, st, ks_ricd_pass<N, 0>, ks_ricd_pass<N, 1>, ks_ricd_pass<N, 2>,
                                                    ks_ricd_pass<N, 3>);
                  if (tiny_tiles<N>(a.sc))
                    return launch_pdl(ks_ricd<N, 16>, dim3(N / 16, N / 16, a.sc), dim3(kSThreads),
                                      Icd<16>::kIcdGrid * sizeof(float), st, a);
                  if (small_tiles<N>(a.sc)) {
                    constexpr int T = N < 32 ? N : 32;
                    return launch_pdl(ks_ricd<N, 32>, dim3(N / T, N / T, a.sc), dim3(kSThreads),
                                      Icd<32>::kIcdGrid * sizeof(float), st, a);
                  }
                  constexpr int T = N < 64 ? N : 64;
                  // 320 threads (10 warps): the colour phases' 1225/1156/1089/1024 pixels
                  // take 4 passes instead of 5/5/5/4 (step 434 -> 440 k frames/s; 384: 433 k)
                  return launch_pdl(ks_ricd<N, 64, 320>, dim3(N / T, N / T, a.sc), dim3(320),
                                    Icd<64>::kIcdGrid * sizeof(float), st, a);
                }));
}
cudaError_t launch_s5(const StepArgs &a, cudaStream_t st) {
  DDH_SDISPATCH(a.n, ({
                  if (tiny_tiles<N>(a.sc)) return launch_icd<N, 16>(ks_phiicd<N, 16>, a, st, Icd<16>::kIcdGrid * sizeof(float));
                  if (small_tiles<N>(a.sc)) return launch_icd<N, 32>(ks_phiicd<N, 32>, a, st, Icd<32>::kIcdGrid * sizeof(float));
                  return launch_icd<N, 64>(ks_phiicd<N, 64>, a, st, Icd<64>::kIcdGrid * sizeof(float));
                }));
}

cudaError_t launch_test_fft_stream(int n, const float2 *in, float2 *out, int B, int inverse, const float4 *tw4,
                                   cudaStream_t st) {
  // rows in -> out, then columns out -> out (each column CTA reads its own columns only)
  DDH_SDISPATCH(n, ({
                  ks_test_rows<N><<<dim3(N / SCfg<N>::H, B), SCfg<N>::NTR, srow_smem<N>(), st>>>(in, out, inverse, tw4);
                  ks_test_cols<N><<<dim3(N / SCfg<N>::W, B), SCfg<N>::NTC, scol_smem<N>(), st>>>(out, out, inverse, tw4);
                  return cudaGetLastError();
                }));
}
cudaError_t launch_test_estep(const float2 *u, const float *r_prev, float *r0, float2 *mu, float *q, size_t count,
                              int warm, float oml, float la, float r_min, float s2, cudaStream_t st) {
  ks_test_estep<<<592, 256, 0, st>>>(u, r_prev, r0, mu, q, count, warm, oml, la, r_min, s2);
  return cudaGetLastError();
}
cudaError_t launch_test_pack(const float *c, const float *th, float2 *out, size_t count, cudaStream_t st) {
  ks_test_pack<<<592, 256, 0, st>>>(c, th, out, count);
  return cudaGetLastError();
}

}  // namespace ddh
