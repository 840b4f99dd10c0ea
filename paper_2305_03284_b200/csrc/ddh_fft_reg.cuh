// ddh_fft_reg.cuh -- register-resident forward FFT of length N for the
// streaming kernels (ddh_stream.cu), sm_100a.
//
// Every thread holds E elements of one length-N vector in registers; the
// TPV = N/E threads of a vector run a Stockham (natural order in and out)
// mixed-radix transform whose first pass reads the registers directly and
// whose last pass leaves the result in registers, so a 2-pass length (64,
// 128, 256) crosses shared memory exactly once and a 3-pass length (512,
// 1024) twice.  Element positions owned by lane t of a vector:
//
//     input  register e  <->  x[t + TPV e]                    (e = 0..E-1)
//     output register e  <->  X[t + TPV (q + NB m)],  e = q RL + m
//
// (RL = radix of the last pass, NB = E/RL), i.e. both are the comb
// t + TPV s, so global loads/stores with lanes on consecutive t coalesce.
// Butterflies use packed FP32 pairs (ddh_f32x2.cuh); twiddles come from a
// shared-memory table tw[m] = (w.x, w.y, -w.y, w.x), w = e^{-2 pi i m/N}.
// Only the forward transform exists: the inverse is conj(FFT(conj x)), and
// the callers fold both conjugations into their elementwise stages.
#pragma once
#include "ddh_f32x2.cuh"

namespace ddh {

template <int N> struct RPlan;
template <> struct RPlan<64>   { static constexpr int E = 8,  NP = 2, R0 = 8,  R1 = 8,  R2 = 1; };
template <> struct RPlan<128>  { static constexpr int E = 16, NP = 2, R0 = 16, R1 = 8,  R2 = 1; };
template <> struct RPlan<256>  { static constexpr int E = 16, NP = 2, R0 = 16, R1 = 16, R2 = 1; };
template <> struct RPlan<512>  { static constexpr int E = 16, NP = 3, R0 = 16, R1 = 16, R2 = 2; };
template <> struct RPlan<1024> { static constexpr int E = 16, NP = 3, R0 = 16, R1 = 16, R2 = 4; };
// (2048: the on-device synthesiser's 2N x 2N screen grid at N = 1024 only)
template <> struct RPlan<2048> { static constexpr int E = 16, NP = 3, R0 = 16, R1 = 16, R2 = 8; };

// ---- forward DFT butterflies on packed pairs -------------------------------

#define DDH_RC1 0.92387953251128674f  // cos(pi/8)
#define DDH_RC2 0.70710678118654752f  // cos(pi/4)
#define DDH_RC3 0.38268343236508977f  // cos(3pi/8)

__device__ __forceinline__ void rdft2(float2 &a, float2 &b) {
  const float2 t = a;
  a = p_add(t, b);
  b = p_sub(t, b);
}
__device__ __forceinline__ void rdft4(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
  const float2 t0 = p_add(x0, x2), t1 = p_sub(x0, x2);
  const float2 t2 = p_add(x1, x3), d = p_sub(x1, x3);
  x0 = p_add(t0, t2);
  x2 = p_sub(t0, t2);
  x1 = pc_add_mi(t1, d);  // t1 - i d
  x3 = pc_sub_mi(t1, d);  // t1 + i d
}
// W8^1 x = (1 - i) x / sqrt2 ;  W8^3 x = (-1 - i) x / sqrt2
__device__ __forceinline__ float2 w8_1(float2 x) { return p_mul(pc_add_mi(x, x), bc2(DDH_RC2)); }
__device__ __forceinline__ float2 w8_3(float2 x) {
  return p_mul(p_fma(swp(x), make_float2(1.f, -1.f), make_float2(-x.x, -x.y)), bc2(DDH_RC2));
}
__device__ __forceinline__ float2 mul_mi(float2 x) { return p_mul(swp(x), make_float2(1.f, -1.f)); }

// 8-point: n = 2 n1 + n2 -> two DFT4 over n1, twiddle W8^(n2 k1), DFT2 over n2
__device__ __forceinline__ void rdft8(float2 *v) {
  float2 a0 = v[0], a1 = v[2], a2 = v[4], a3 = v[6];
  float2 b0 = v[1], b1 = v[3], b2 = v[5], b3 = v[7];
  rdft4(a0, a1, a2, a3);
  rdft4(b0, b1, b2, b3);
  b1 = w8_1(b1);
  b2 = mul_mi(b2);
  b3 = w8_3(b3);
  v[0] = p_add(a0, b0); v[4] = p_sub(a0, b0);
  v[1] = p_add(a1, b1); v[5] = p_sub(a1, b1);
  v[2] = p_add(a2, b2); v[6] = p_sub(a2, b2);
  v[3] = p_add(a3, b3); v[7] = p_sub(a3, b3);
}

// 16-point: n = 4 n1 + n2 -> DFT4 over n1 (4x), twiddle W16^(n2 k1), DFT4 over n2
__device__ __forceinline__ void rdft16(float2 *v) {
  float2 a[4][4];  // a[n2][k1]
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    a[n2][0] = v[n2];
    a[n2][1] = v[n2 + 4];
    a[n2][2] = v[n2 + 8];
    a[n2][3] = v[n2 + 12];
    rdft4(a[n2][0], a[n2][1], a[n2][2], a[n2][3]);
  }
  // W16^m = (cos, -sin)(2 pi m / 16)
  a[1][1] = pc_mul_c(a[1][1], DDH_RC1, -DDH_RC3);
  a[1][2] = w8_1(a[1][2]);
  a[1][3] = pc_mul_c(a[1][3], DDH_RC3, -DDH_RC1);
  a[2][1] = w8_1(a[2][1]);
  a[2][2] = mul_mi(a[2][2]);
  a[2][3] = w8_3(a[2][3]);
  a[3][1] = pc_mul_c(a[3][1], DDH_RC3, -DDH_RC1);
  a[3][2] = w8_3(a[3][2]);
  a[3][3] = pc_mul_c(a[3][3], -DDH_RC1, DDH_RC3);  // W16^9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    float2 x0 = a[0][k1], x1 = a[1][k1], x2 = a[2][k1], x3 = a[3][k1];
    rdft4(x0, x1, x2, x3);
    v[k1] = x0;
    v[k1 + 4] = x1;
    v[k1 + 8] = x2;
    v[k1 + 12] = x3;
  }
}

template <int R>
__device__ __forceinline__ void rdft(float2 *v) {
  if constexpr (R == 2) rdft2(v[0], v[1]);
  else if constexpr (R == 4) rdft4(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) rdft8(v);
  else if constexpr (R == 16) rdft16(v);
  else static_assert(R == 2, "radix");
}

// ---- passes -----------------------------------------------------------------

// Compute one pass (radix R, sub-transform size Ns) on the registers: NB = E/R
// butterflies, butterfly q holds v[q R .. q R + R - 1] = inputs x[j + r N/R]
// with j = t + q TPV.
template <int N, int R, int Ns>
__device__ __forceinline__ void rpass(float2 (&v)[RPlan<N>::E], int t, const float4 *__restrict__ tw) {
  constexpr int E = RPlan<N>::E, NB = E / R, TPV = N / E;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    if constexpr (Ns > 1) {
      const int j = t + q * TPV;
      const int k = j & (Ns - 1);
      const int step = k * (N / (Ns * R));  // W_{Ns R}^{r k} = W_N^{r k N/(Ns R)}
#pragma unroll
      for (int r = 1; r < R; ++r) v[q * R + r] = pc_mul_t(v[q * R + r], tw[r * step]);
    }
    rdft<R>(&v[q * R]);
  }
}

// Store the outputs of a pass (radix R, sub-size Ns) and load the inputs of
// the next pass (radix R2): out index idxD + m Ns with idxD = (j - k) R + k.
// buf[POS(p)] is element p of this thread's vector.
template <int N, int R, int Ns, int R2, class Pos>
__device__ __forceinline__ void rexchange(float2 (&v)[RPlan<N>::E], int t, float2 *buf, Pos pos) {
  constexpr int E = RPlan<N>::E, NB = E / R, TPV = N / E, NB2 = E / R2;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int j = t + q * TPV;
    const int k = j & (Ns - 1);
    const int d = (j - k) * R + k;
#pragma unroll
    for (int m = 0; m < R; ++m) buf[pos(d + m * Ns)] = v[q * R + m];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NB2; ++q) {
    const int j = t + q * TPV;
#pragma unroll
    for (int r = 0; r < R2; ++r) v[q * R2 + r] = buf[pos(j + r * (N / R2))];
  }
}

// Full forward FFT.  The caller must make sure buf is not in use by other
// threads on entry (__syncthreads) and must __syncthreads before reusing it.
template <int N, class Pos>
__device__ __forceinline__ void fft_reg(float2 (&v)[RPlan<N>::E], int t, float2 *buf, Pos pos,
                                        const float4 *__restrict__ tw) {
  using P = RPlan<N>;
  rpass<N, P::R0, 1>(v, t, tw);
  rexchange<N, P::R0, 1, P::R1>(v, t, buf, pos);
  rpass<N, P::R1, P::R0>(v, t, tw);
  if constexpr (P::NP == 3) {
    __syncthreads();  // everyone has read the first exchange
    rexchange<N, P::R1, P::R0, P::R2>(v, t, buf, pos);
    rpass<N, P::R2, P::R0 * P::R1>(v, t, tw);
  }
}

// Comb index of output register e: X[t + TPV out_comb(e)]
template <int N>
__host__ __device__ constexpr int out_comb(int e) {
  using P = RPlan<N>;
  constexpr int RL = P::NP == 3 ? P::R2 : P::R1;
  constexpr int NB = P::E / RL;
  return (e / RL) + NB * (e % RL);
}

// Padded row layout: one float2 of padding per 16 (bank-conflict-free comb
// stores/loads of the exchange); row pitch N + N/16.
__host__ __device__ constexpr int rpad(int p) { return p + (p >> 4); }

}  // namespace ddh
