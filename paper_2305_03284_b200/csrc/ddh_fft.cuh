// ddh_fft.cuh -- batched in-shared-memory complex FFTs for sm_100a.
//
// The two 2-D FFTs of every EM iteration ("dominated by the application
// of two FFTs") are split into a row pass and a column pass; each pass runs a
// batch of length-N vectors that a CTA holds in shared memory.  Within a
// vector we use the mixed-radix Stockham autosort formulation (natural order
// in, natural order out, no bit reversal), with radix-8/16 butterflies held in
// registers and the inter-pass exchange through shared memory:
//
//   pass with radix R, sub-transform size Ns (1, R0, R0 R1, ...):
//     for butterfly j in [0, N/R):  k = j mod Ns
//       v[r] = x[j + r N/R] * W_{Ns R}^{r k}          (r = 0..R-1)
//       v    = DFT_R(v)
//       x[(j / Ns) Ns R + k + m Ns] = v[m]             (m = 0..R-1)
//
// Every thread holds E elements (E/R butterflies) of one vector in registers
// across a pass: load all -> __syncthreads -> compute -> store all ->
// __syncthreads, so the pass runs in place.  Thread -> (vector b, lane t)
// mapping is b = tid % nvec (fast), t = tid / nvec, which makes column
// passes (vectors adjacent in memory) and padded row passes (vector pitch
// N+1) bank-conflict free for the loads.
//
// DIR = -1: forward DFT  X_k = sum x_n e^{-2 pi i nk/N};  DIR = +1: inverse
// (unnormalised).  Twiddles W_N^m = e^{-2 pi i m/N} come from a table computed
// in FP64 on the host and stored as FP32 (tw[m], m in [0,N)).
#pragma once
#include <cuda_runtime.h>

#include "ddh_f32x2.cuh"

namespace ddh {

// complex add / subtract / multiply on packed FP32 pairs (FADD2 / FMUL2 /
// FFMA2): every lane rounds as the scalar expression would, so the results are
// the bits of (a.x + b.x, a.y + b.y) and (fma(a.x, b.x, -a.y b.y),
// fma(a.x, b.y, a.y b.x)); only the instruction count drops
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return p_add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return p_sub(a, b); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return p_fma(bc2(a.x), b, p_mul(make_float2(-a.y, a.y), make_float2(b.y, b.x)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// multiply by e^{DIR i pi/2} = DIR * i
template <int DIR>
__device__ __forceinline__ float2 mul_i(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}

// cos / sin of 2 pi m / 16, m = 0..7 (exact decimal expansions to float precision)
#define DDH_C1 0.92387953251128674f
#define DDH_C2 0.70710678118654752f
#define DDH_C3 0.38268343236508977f

template <int DIR>
__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int DIR>
__device__ __forceinline__ void dft4(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
  float2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  float2 t2 = cadd(x1, x3), t3 = mul_i<DIR>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

// W_8^m with sign DIR applied to the sine: e^{DIR 2 pi i m / 8}
template <int DIR>
__device__ __forceinline__ float2 w8(int m) {
  const float s = DIR < 0 ? -1.f : 1.f;
  switch (m & 7) {
    case 0: return make_float2(1.f, 0.f);
    case 1: return make_float2(DDH_C2, s * DDH_C2);
    case 2: return make_float2(0.f, s);
    default: return make_float2(-DDH_C2, s * DDH_C2);
  }
}

template <int DIR>
__device__ __forceinline__ void dft8(float2 *v) {
  // radix-2 DIT over two length-4 DFTs (even / odd samples)
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<DIR>(e0, e1, e2, e3);
  dft4<DIR>(o0, o1, o2, o3);
  o1 = cmul(o1, w8<DIR>(1));
  o2 = mul_i<DIR>(o2);
  o3 = cmul(o3, w8<DIR>(3));
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

template <int DIR>
__device__ __forceinline__ void dft16(float2 *v) {
  float2 e[8], o[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { e[k] = v[2 * k]; o[k] = v[2 * k + 1]; }
  dft8<DIR>(e);
  dft8<DIR>(o);
  const float s = DIR < 0 ? -1.f : 1.f;
  // o[m] *= W16^m  = (cos 2pi m/16, DIR sin 2pi m/16)
  o[1] = cmul(o[1], make_float2(DDH_C1, s * DDH_C3));
  o[2] = cmul(o[2], make_float2(DDH_C2, s * DDH_C2));
  o[3] = cmul(o[3], make_float2(DDH_C3, s * DDH_C1));
  o[4] = mul_i<DIR>(o[4]);
  o[5] = cmul(o[5], make_float2(-DDH_C3, s * DDH_C1));
  o[6] = cmul(o[6], make_float2(-DDH_C2, s * DDH_C2));
  o[7] = cmul(o[7], make_float2(-DDH_C1, s * DDH_C3));
#pragma unroll
  for (int k = 0; k < 8; ++k) { v[k] = cadd(e[k], o[k]); v[k + 8] = csub(e[k], o[k]); }
}

template <int R, int DIR>
__device__ __forceinline__ void dft(float2 *v) {
  if constexpr (R == 2) dft2<DIR>(v[0], v[1]);
  else if constexpr (R == 4) dft4<DIR>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<DIR>(v);
  else if constexpr (R == 16) dft16<DIR>(v);
  else static_assert(R == 2 || R == 4 || R == 8 || R == 16, "unsupported radix");
}

// Radix plan per N: E elements per thread, radices R0 R1 R2 (R2 = 1: unused).
template <int N> struct FftPlan;
template <> struct FftPlan<64>   { static constexpr int E = 8,  R0 = 8,  R1 = 8,  R2 = 1; };
template <> struct FftPlan<128>  { static constexpr int E = 16, R0 = 16, R1 = 8,  R2 = 1; };
template <> struct FftPlan<256>  { static constexpr int E = 16, R0 = 16, R1 = 16, R2 = 1; };
template <> struct FftPlan<512>  { static constexpr int E = 16, R0 = 16, R1 = 16, R2 = 2; };
template <> struct FftPlan<1024> { static constexpr int E = 16, R0 = 16, R1 = 16, R2 = 4; };

// One Stockham pass over a batch held in shared memory.  Element e of the
// vector of this thread lives at buf[e * estride] (buf already offset by the
// vector base).  All threads of the CTA must call it (it synchronises).
template <int N, int R, int E, int DIR>
__device__ __forceinline__ void stockham_pass(float2 *buf, bool active, int t, int estride, int Ns,
                                              const float2 *__restrict__ tw) {
  constexpr int NB = E / R;   // butterflies per thread
  constexpr int TPV = N / E;  // threads per vector
  float2 v[NB][R];
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int j = t + q * TPV;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = buf[(j + r * (N / R)) * estride];
    }
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int j = t + q * TPV;
      const int k = j & (Ns - 1);
      if (Ns > 1) {
        const int step = k * (N / (Ns * R));  // W_{Ns R}^{r k} = W_N^{r k N/(Ns R)}
#pragma unroll
        for (int r = 1; r < R; ++r) {
          float2 w = tw[r * step];
          if (DIR > 0) w.y = -w.y;
          v[q][r] = cmul(v[q][r], w);
        }
      }
      dft<R, DIR>(v[q]);
      const int idxD = (j - k) * R + k;  // (j / Ns) * Ns * R + k
#pragma unroll
      for (int m = 0; m < R; ++m) buf[(idxD + m * Ns) * estride] = v[q][m];
    }
  }
  __syncthreads();
}

// Full length-N FFT of the vectors of a CTA.  `buf` points at element 0 of
// this thread's vector; t in [0, N/E) is the lane within the vector.
template <int N, int DIR>
__device__ __forceinline__ void block_fft(float2 *buf, bool active, int t, int estride,
                                          const float2 *__restrict__ tw) {
  using P = FftPlan<N>;
  stockham_pass<N, P::R0, P::E, DIR>(buf, active, t, estride, 1, tw);
  stockham_pass<N, P::R1, P::E, DIR>(buf, active, t, estride, P::R0, tw);
  if constexpr (P::R2 > 1) stockham_pass<N, P::R2, P::E, DIR>(buf, active, t, estride, P::R0 * P::R1, tw);
}

}  // namespace ddh
