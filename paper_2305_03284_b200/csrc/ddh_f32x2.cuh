// ddh_f32x2.cuh -- packed FP32 pair arithmetic for sm_100a.
//
// Blackwell executes add/sub/mul/fma on a pair of FP32 values held in a
// 64-bit register pair as ONE instruction (SASS FADD2 / FMUL2 / FFMA2), with
// per-operand broadcast and swap selectors (a scalar operand is replicated
// into both lanes for free).  Every value is rounded exactly as the scalar
// instruction would round it; only the instruction count halves.  ptxas does
// not form these from scalar code, so the hot loops (FFT butterflies, the
// qGGMRF weights of the r-ICD) call them explicitly.
#pragma once
#include <cuda_runtime.h>

namespace ddh {

__device__ __forceinline__ float2 p_add(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, r; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; add.rn.f32x2 r, a, b; mov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 p_sub(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, r; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; sub.rn.f32x2 r, a, b; mov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 p_mul(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, r; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; mul.rn.f32x2 r, a, b; mov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// a * b + c, one rounding per lane
__device__ __forceinline__ float2 p_fma(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 a, b, c, r; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; mov.b64 c, {%6, %7};"
      " fma.rn.f32x2 r, a, b, c; mov.b64 {%0, %1}, r;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 swp(float2 a) { return make_float2(a.y, a.x); }

// complex helpers on packed pairs
// a * w for a twiddle stored as (w.x, w.y, -w.y, w.x): a.x (w.x, w.y) + a.y (-w.y, w.x)
__device__ __forceinline__ float2 pc_mul_t(float2 a, float4 w) {
  return p_fma(bc2(a.y), make_float2(w.z, w.w), p_mul(bc2(a.x), make_float2(w.x, w.y)));
}
// a * (c + i s) for constants c, s
__device__ __forceinline__ float2 pc_mul_c(float2 a, float c, float s) {
  return p_fma(bc2(a.y), make_float2(-s, c), p_mul(bc2(a.x), make_float2(c, s)));
}
// t + (-i) d  and  t - (-i) d   (-i d = (d.y, -d.x))
__device__ __forceinline__ float2 pc_add_mi(float2 t, float2 d) { return p_fma(swp(d), make_float2(1.f, -1.f), t); }
__device__ __forceinline__ float2 pc_sub_mi(float2 t, float2 d) { return p_fma(swp(d), make_float2(-1.f, 1.f), t); }

}  // namespace ddh
