// ddh_common.cuh -- device helpers shared by the unfused (ddh_kernels.cu) and
// the cluster-fused (ddh_fused.cu) kernels: deterministic reductions, the
// aperture test, the qGGMRF surrogate weight, the per-pixel r and phi
// M-step updates (readings R6-R11 of DESIGN.md).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "ddh_f32x2.cuh"

// Bounds-checked debug build (the sanitizer substitute; compute-sanitizer is
// not available on the GPU pool): -DDDH_DEBUG_BOUNDS=1 turns DDH_DBG checks of
// shared-memory tile indices, colour-phase ownership and global indices into
// device traps with a message.  Compiled out otherwise.
#ifndef DDH_DEBUG_BOUNDS
#define DDH_DEBUG_BOUNDS 0
#endif
#if DDH_DEBUG_BOUNDS
#include <cstdio>
#define DDH_DBG(cond)                                                                                   \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("DDH_DEBUG_BOUNDS %s:%d block (%d,%d,%d) thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
             blockIdx.y, blockIdx.z, threadIdx.x, #cond);                                               \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define DDH_DBG(cond) \
  do {                \
  } while (0)
#endif

namespace ddh {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum of K doubles (fixed shuffle tree + fixed warp order).
// Result valid in thread 0.  sh: >= 32*K doubles of shared memory.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double *sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh[warp * K + k] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = lane < nw ? sh[lane * K + k] : 0.0;
      v[k] = warp_sum(x);
    }
  }
  __syncthreads();
}

// Plane coefficients c = Minv h of the RemoveTipTilt normal equations (R17);
// sums[2..4] = (sum phi, sum phi x, sum phi y) over the aperture.
__device__ __forceinline__ void plane_from_sums(const double *sums, const double *minv, double *c) {
  const double h0 = sums[2], h1 = sums[3], h2 = sums[4];
  c[0] = minv[0] * h0 + minv[1] * h1 + minv[2] * h2;
  c[1] = minv[3] * h0 + minv[4] * h1 + minv[5] * h2;
  c[2] = minv[6] * h0 + minv[7] * h1 + minv[8] * h2;
}

__device__ __forceinline__ bool in_ap(const int2 *__restrict__ rs, int i, int j) {
  const int2 s = __ldg(rs + i);
  return j >= s.x && j < s.y;
}

// 8-neighbour stencil: offsets and weights b (1/6 nearest, 1/12 diagonal; R7)
__device__ __forceinline__ int nb_di(int k) { return (k < 4) ? ((k == 0) ? -1 : (k == 1) ? 1 : 0) : ((k < 6) ? -1 : 1); }
__device__ __forceinline__ int nb_dj(int k) { return (k < 4) ? ((k == 2) ? -1 : (k == 3) ? 1 : 0) : ((k & 1) ? 1 : -1); }
__device__ __forceinline__ float nb_w(int k) { return (k < 4) ? (1.f / 6.f) : (1.f / 12.f); }

// qGGMRF surrogate weight rho'(D)/(2D) in units of 1/(2 sig^2) (R6):
// (1/(1+t)) (1 - (2-q) t / (2(1+t))),  t = |D/(T sig)|^(2-q).
// t via MUFU lg2/ex2 (the 1e-30 floor makes t = 0 at D = 0 and t = 1 at
// q = 2 without a branch); 1/(1+t) via MUFU rcp.  Relative error ~1e-6.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 1/x by one MUFU.RCP (relative error ~1 ulp; inputs here are normal numbers)
__host__ __device__ __forceinline__ float rcp_approx(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return 1.f / x;
#endif
}
// 1/u for u >= 1 on the FMA pipe (no MUFU): magic-constant seed (rel. error
// < 12.5 %) + 3 Newton steps (< 1e-7).  The r-ICD is MUFU-throughput bound
// (3 MUFU per neighbour at 16/clk/SM), so one MUFU per neighbour moves here.
__device__ __forceinline__ float rcp_fma(float u) {
  float y = __int_as_float(0x7EF311C3 - __float_as_int(u));
  y = y * fmaf(-u, y, 2.f);
  y = y * fmaf(-u, y, 2.f);
  y = y * fmaf(-u, y, 2.f);
  return y;
}

__device__ __forceinline__ float qgg_w(float d, float inv_Tsig, float tmq) {
  // (1/(1+t)) (1 - (2-q) t/(2(1+t))) = k/u + (1-k)/u^2,  u = 1+t, k = q/2 = 1 - tmq/2:
  // 3 MUFU (lg2, ex2, rcp) + 6 FMA-pipe instructions
  const float a = fmaf(fabsf(d), inv_Tsig, 1e-30f);
  const float t = ex2_approx(tmq * lg2_approx(a));
  const float r = rcp_approx(1.f + t);
  const float k = 1.f - 0.5f * tmq;
  return fmaf(1.f - k, r, k) * r;
}

// The same weight for a pair of neighbours (rj.x, rj.y) of pixel ri on packed
// FP32 pairs (streaming and cluster paths): t = (|d| / (T sig))^(2-q) =
// 2^(h lg2(d^2 + tiny) + g) with h = (2-q)/2, g = (2-q) lg2(1/(T sig)); the
// 1e-37 floor keeps lg2 finite at d = 0 (t ~ 2^-49 there, and t = 1 exactly at
// q = 2).  3 MUFU per neighbour (lg2, ex2, rcp: 64 ops/clk/SM on this part,
// tools/micro/mufu_rate.cu) and 5 packed FP32 instructions per pair; the
// kernels around it are issue-bound, so the reciprocal stays on MUFU.
// Returns (w(d.x), w(d.y)).
__device__ __forceinline__ float2 qgg_w2(float ri, float2 rj, float h, float g, float k) {
  const float2 d = p_sub(bc2(ri), rj);
  const float2 a = p_fma(d, d, bc2(1e-37f));
  const float2 e = p_fma(make_float2(lg2_approx(a.x), lg2_approx(a.y)), bc2(h), bc2(g));
  const float2 u = p_add(make_float2(ex2_approx(e.x), ex2_approx(e.y)), bc2(1.f));
  const float2 y = make_float2(rcp_approx(u.x), rcp_approx(u.y));
  return p_mul(p_fma(y, bc2(1.f - k), bc2(k)), y);  // (k + (1-k)/u) / u
}

__device__ __forceinline__ void sincos_red(float p, float &sn, float &cs) {
  // |argument| <= pi after one rint reduction, then MUFU sin/cos
  __sincosf(fmaf(-6.283185307179586f, rintf(p * 0.15915494309189535f), p), &sn, &cs);
}

// atan2(y, x) for the phase-correlation angle: octant reduction + odd
// minimax polynomial (degree 13) of atan on [0, 1]; |error| < 5e-7 rad
// (FP32, measured against FP64 atan).  atan2(0, 0) = 0 (c = 0 there, so
// theta is irrelevant).
__device__ __forceinline__ float atan2_fast(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mx > 0.f ? mn * rcp_approx(mx) : 0.f;
  const float s = a * a;
  float p = 0.00681176f;
  p = fmaf(p, s, -0.03360414f);
  p = fmaf(p, s, 0.07962359f);
  p = fmaf(p, s, -0.1323334f);
  p = fmaf(p, s, 0.19807816f);
  p = fmaf(p, s, -0.3331737f);
  p = fmaf(p, s, 0.9999961f);
  float r = p * a;
  if (ay > ax) r = 1.5707963267948966f - r;
  if (x < 0.f) r = 3.141592653589793f - r;
  return copysignf(r, y);
}

// Last read of a buffer in a step (DDH_EVICT_HINTS build knob): a streaming
// load (ld.global.cs, evict-first) lets the lanes' other data stay in L2
// (profiles/r02d_warm_traffic.json); otherwise the read-only path
#ifndef DDH_EVICT_HINTS
#define DDH_EVICT_HINTS 0
#endif
__device__ __forceinline__ float ldg_last(const float *a) {
  float v;
#if DDH_EVICT_HINTS
  v = __ldcs(a);
#else
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(a));
#endif
  return v;
}
__device__ __forceinline__ float2 ldg_last2(const float2 *a) {
#if DDH_EVICT_HINTS
  return __ldcs(a);
#else
  return __ldg(a);
#endif
}

// ---- r M-step, one pixel (R9) -------------------------------------------
// Minimiser over x >= r_min of f(x) = log x + q/x + B x^2 - 2 S x (B > 0).
// f'(x) = g(x)/x^2 with g(x) = 2B x^3 - 2S x^2 + x - q, g(0) = -q < 0; g is
// concave left of its inflection xi = S/(3B) and convex right of it.
//  * If g has two positive stationary points x1 < xi < x2 (S > 0 and
//    4S^2 > 6B): a small root exists iff g(x1) > 0 and lies in (0, x1)
//    (concave, increasing: monotone Newton from 0, whose first iterate is q);
//    a large root exists iff g(x2) < 0 and lies in (x2, U], U = max(S/B, q)
//    with g(U) >= 0 (convex, increasing: monotone Newton from U).  Both
//    present: three roots, the middle one a local maximum of f.
//  * Otherwise g increases on (0, inf): one root, left of xi iff g(xi) > 0.
// The small and large roots are the local minima of f; with both present the
// lower f wins (FP32 difference).  Candidates are clamped to r_min.  No
// transcendental root formula and no FP64 on this path.
__host__ __device__ __forceinline__ float g_of(float x, float B2, float S2, float q) {
  return fmaf(fmaf(fmaf(B2, x, -S2), x, 1.f), x, -q);
}
__host__ __device__ __forceinline__ float dg_of(float x, float B6, float S4) { return fmaf(fmaf(B6, x, -S4), x, 1.f); }

// sqrt(x) for x > 0 normal by one MUFU.RSQ (only classifies the root set)
__host__ __device__ __forceinline__ float sqrt_approx(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return x * y;
#else
  return sqrtf(x);
#endif
}

#define DDH_FDIV(a, b) ((a) * rcp_approx(b))

// Monotone Newton on g: three unrolled steps (enough for ~95% of pixels on the
// BASELINE workloads, measured with tests/tools/check_r_update.py) then a guarded
// loop for the stragglers.
__host__ __device__ __forceinline__ float newton_root(float x, float B2, float S2, float B6, float S4, float q) {
  float dx = 0.f;
#pragma unroll
  for (int it = 0; it < 3; ++it) {
#if defined(DDH_ITER_HOOK) && !defined(__CUDA_ARCH__)
    DDH_ITER_HOOK;
#endif
    const float d = dg_of(x, B6, S4);
    dx = d > 0.f ? DDH_FDIV(g_of(x, B2, S2, q), d) : 0.f;
    x -= dx;
  }
  if (fabsf(dx) <= 2e-7f * fabsf(x)) return x;
#pragma unroll 1
  for (int it = 0; it < 13; ++it) {
#if defined(DDH_ITER_HOOK) && !defined(__CUDA_ARCH__)
    DDH_ITER_HOOK;
#endif
    const float d = dg_of(x, B6, S4);
    if (!(d > 0.f)) break;
    const float dx = DDH_FDIV(g_of(x, B2, S2, q), d);
    x -= dx;
    if (fabsf(dx) <= 2e-7f * fabsf(x)) break;
  }
  return x;
}

// Halley's method on g (cubic convergence; g'' = 12 B x - 4 S), from the same
// start points as the monotone Newton runs: two unrolled steps, then a guarded
// loop.  Checked against the oracle's exact minimiser on 6e5 random cases and
// the c3 ICD inputs (tests/tools/check_r_update.py: same roots, max relative error
// 1e-6); 3.6 instead of 4.9 iterations for the slowest lane of a warp.
__host__ __device__ __forceinline__ float halley_root(float x, float B2, float S2, float B6, float S4, float q) {
  float dx = 0.f, D = 1.f, H = 0.f;
  const float B12 = 2.f * B6;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
#if defined(DDH_ITER_HOOK) && !defined(__CUDA_ARCH__)
    DDH_ITER_HOOK;
#endif
    const float G = g_of(x, B2, S2, q);
    D = dg_of(x, B6, S4);
    H = fmaf(B12, x, -S4);
    const float den = fmaf(2.f * D, D, -G * H);
    dx = (D > 0.f && den > 0.f) ? DDH_FDIV(2.f * G * D, den) : 0.f;
    x -= dx;
  }
#ifndef DDH_HALLEY_STRICT
  // Stop after two steps when Halley's asymptotic error bound says the second
  // step already converged: e3 ~ C dx^3 with C = g''^2/(4 g'^2) - g'''/(6 g')
  // (g''' = 12 B) at the second step's start point, required below 2e-8 |x|,
  // and only inside the region where the bound holds (|dx g''| <= g'/10).
  // Multiplied through by 4 g'^2 (g' > 0): no division.  Saves the third,
  // verifying step in ~3 of 4 warps on the c3 ICD inputs (tests/tools/r_iter_study.py).
  {
    const float adx = fabsf(dx), c4 = fabsf(fmaf(H, H, -4.f * B2 * D));  // |g''^2 - 8 B g'|
    if (D > 0.f && adx * fabsf(H) <= 0.1f * D && c4 * (adx * adx * adx) <= 8e-8f * fabsf(x) * (D * D)) return x;
  }
#endif
  if (fabsf(dx) <= 2e-7f * fabsf(x)) return x;
#pragma unroll 1
  for (int it = 0; it < 14; ++it) {
#if defined(DDH_ITER_HOOK) && !defined(__CUDA_ARCH__)
    DDH_ITER_HOOK;
#endif
    const float G = g_of(x, B2, S2, q), D = dg_of(x, B6, S4), H = fmaf(B12, x, -S4);
    const float den = fmaf(2.f * D, D, -G * H);
    if (!(D > 0.f) || !(den > 0.f)) break;
    const float d = DDH_FDIV(2.f * G * D, den);
    x -= d;
    if (fabsf(d) <= 2e-7f * fabsf(x)) break;
  }
  return x;
}

// Three roots (both local minima present): the lower surrogate value wins.
static __host__ __device__ __noinline__ float r_pick_two(float rc, float q, float B, float S, float r_min, float xs,
                                                  float B2, float S2, float B6, float S4) {
  const float xl = newton_root(fmaxf(S / B, q), B2, S2, B6, S4, q);
  const float a = fmaxf(xs, r_min), b = fmaxf(xl, r_min);
  // f(b) - f(a)
  const float df = logf(b / a) + q * (a - b) / (a * b) + (b - a) * (B * (a + b) - 2.f * S);
  const float tol = 1e-6f * (1.f + fabsf(logf(a)) + q / a);
  if (fabsf(df) <= tol) return fabsf(a - rc) <= fabsf(b - rc) ? a : b;
  return df < 0.f ? b : a;
}

__host__ __device__ __forceinline__ float r_update(float rc, float q, float B, float S, float r_min) {
  const float B2 = 2.f * B, S2 = 2.f * S, B6 = 6.f * B, S4 = 4.f * S;
  const float disc = 4.f * S * S - 6.f * B;
  const float iB = rcp_approx(B);
  // (approximate x1, x2, xi only classify; near a boundary the two minima are
  // within rounding of each other's surrogate value, so either choice is exact)
  bool has_small, has_large;
  if (S > 0.f && disc > 0.f) {
    const float x2 = (2.f * S + sqrt_approx(disc)) * iB * (1.f / 6.f);
    const float x1 = iB * (1.f / 6.f) * rcp_approx(x2);  // x1 x2 = 1/(6B)
    has_small = g_of(x1, B2, S2, q) > 0.f;
    has_large = g_of(x2, B2, S2, q) < 0.f;
  } else {
    const float xi = S * iB * (1.f / 3.f);
    has_small = xi > 0.f && g_of(xi, B2, S2, q) > 0.f;
    has_large = !has_small;
  }
  // one root search per lane: the small root if it exists (start q), else the
  // large root (start max(S/B, q)); the second minimum only when both exist
  // (rare; separate non-inlined path, monotone Newton)
  const float x = halley_root(has_small ? q : fmaxf(S * iB, q), B2, S2, B6, S4, q);
  if (has_small && has_large) return r_pick_two(rc, q, B, S, r_min, x, B2, S2, B6, S4);
  return fmaxf(x, r_min);
}

// ---- phi M-step, one pixel (R10-R11) --------------------------------------
__device__ __forceinline__ float wrap_pi(float x) {  // (-pi, pi]
  const float twopi = 6.283185307179586f;
  float y = fmaf(-twopi, rintf(x * 0.15915494309189535f), x);
  if (y <= -3.14159265358979f) y += twopi;
  if (y > 3.14159265358979f) y -= twopi;
  return y;
}

// phi <- (c s th~ + w sum b phi_j)/(c s + w sum b), s = sin(x0)/x0, th~ = phi - x0,
// x0 = wrap(phi - theta) (symmetric bound of -c cos(.) at x0).  Prior off:
// phi <- th~ where c > 0 (exact argmax).
__device__ __forceinline__ float phi_update(float phi, float c, float th, float nb, float sb, float w, bool prior) {
  const float x0 = wrap_pi(phi - th);
  const float tt = phi - x0;
  if (!prior) return c > 0.f ? tt : phi;
  const float x2 = x0 * x0;
  const float s = fabsf(x0) < 1e-3f ? fmaf(x2, fmaf(x2, 1.f / 120.f, -1.f / 6.f), 1.f) : __sinf(x0) * rcp_approx(x0);
  const float num = fmaf(c * s, tt, w * nb);
  const float den = fmaf(c, s, w * sb);
  return den != 0.f ? num * rcp_approx(den) : phi;
}

}  // namespace ddh
