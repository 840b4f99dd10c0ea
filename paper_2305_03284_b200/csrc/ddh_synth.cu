// ddh_synth.cu -- on-device frame synthesiser, sm_100a.
//
// Generates synthetic DH frame sequences of the BASELINE recipe on the GPU
// (the same laws as synth/sim.py, with its own generator):
//   r      iid U[0,1], periodic Gaussian blur (sigma_b, truncated at 4 sigma,
//          weights summing to 1), min-max rescale to [0,1], clamp >= r_min (R23)
//   phi    FFT-method Kolmogorov screen on a periodic 2N x 2N grid,
//          c_k = (z1 + j z2) sqrt(Phi(f_k) / M^2), Phi = 0.023 r0^{-5/3} |f|^{-11/3},
//          DC = 0 (R22); frame t = Re IDFT(c e^{-2 pi i f.(t v)}) cropped to
//          N x N (frozen flow by Fourier shift, R24), piston/tip/tilt removed
//          over the aperture
//   g      sqrt(r/2)(z1 + j z2), fresh every frame (R21)
//   w      complex AWGN, sigma_n^2 = mean(r) / 10^{SNR/10} (R20)
//   y      a e^{j phi} F_c^{-1}(g) + w, complex64 (Eq. 1)
// Random numbers: Philox-4x32-10, counter (pixel, frame, stream, purpose),
// key = seed; Box-Muller in FP32.  Input generation only: none of the
// estimator's arithmetic.  Supported N: 64 .. 1024 (screen grid 2N <= 2048).
#include "../../include/ddh.h"
#include "ddh_common.cuh"
#include "ddh_fft_reg.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace ddh {
namespace {

enum { kPScene = 0, kPScreen = 1, kPSpeckle = 2, kPNoise = 3 };

// Philox-4x32-10 (Salmon et al. 2011): counter-based, no state
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__device__ __forceinline__ float u01(uint32_t x) { return ((float)x + 0.5f) * 2.3283064365386963e-10f; }
// two independent standard complex normals (z1 + j z2 with z ~ N(0,1) each part)
__device__ __forceinline__ void normals4(uint32_t idx, uint32_t frame, uint32_t stream, uint32_t purpose, uint2 key,
                                         float2 &a, float2 &b) {
  const uint4 r = philox(make_uint4(idx, frame, stream, purpose), key);
  const float m0 = sqrtf(-2.f * __logf(u01(r.x))), m1 = sqrtf(-2.f * __logf(u01(r.z)));
  float s0, c0, s1, c1;
  __sincosf(6.283185307179586f * u01(r.y), &s0, &c0);
  __sincosf(6.283185307179586f * u01(r.w), &s1, &c1);
  a = make_float2(m0 * c0, m0 * s0);
  b = make_float2(m1 * c1, m1 * s1);
}

constexpr int kT = 256;

// ---- batched plain FFT passes (forward; inverse = conj FFT conj) ----------
template <int M> struct ZCfg {
  static constexpr int E = RPlan<M>::E, TPV = M / E;
  static constexpr int H = (kT / TPV) < 1 ? 1 : kT / TPV;
  static constexpr int NTR = H * TPV;
  static constexpr int W0 = (kT / TPV) < 16 ? 16 : kT / TPV;
  static constexpr int W = W0 * TPV > 1024 ? 1024 / TPV : W0;  // <= 1024 threads per column CTA
  static constexpr int NTC = W * TPV;
};

// MODE 0: in-place inverse DFT of rows (unnormalised); MODE 1: rows of the
// shifted screen spectrum c e^{-2 pi i f.s} (inverse DFT); MODE 2: rows of
// chi g with g generated here (speckle, inverse DFT)
struct ZArgs {
  float2 *buf;            // [S][M][M] work plane
  const float2 *coef;     // MODE 1: [S][M][M] screen coefficients
  const double *shift;    // MODE 1: [S][2] (row, col) offsets of this frame
  const float *r;         // MODE 2: [S][N][N] reflectance
  uint2 key;
  uint32_t frame;
};

template <int M, int MODE>
__global__ void __launch_bounds__(ZCfg<M>::NTR) kz_rows(ZArgs Z) {
  using C = ZCfg<M>;
  constexpr int E = C::E, TPV = C::TPV, H = C::H;
  extern __shared__ float4 zsm[];
  float4 *tw = zsm;
  float2 *xb = reinterpret_cast<float2 *>(zsm + M);
  const int tid = threadIdx.x, s = blockIdx.y;
  const int t = tid % TPV, b = tid / TPV, i = blockIdx.x * H + b;
  for (int k = tid; k < M; k += C::NTR) {
    float sn, cs;
    sincospif(-2.f * (float)k / (float)M, &sn, &cs);
    tw[k] = make_float4(cs, sn, -sn, cs);
  }
  float2 *row = Z.buf + ((size_t)s * M + i) * M;
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = t + TPV * e;
    float2 x;
    if (MODE == 1) {
      const float2 c = Z.coef[((size_t)s * M + i) * M + j];
      const float fi = (float)(i < M / 2 ? i : i - M) / (float)M, fj = (float)(j < M / 2 ? j : j - M) / (float)M;
      // e^{-2 pi i f.s}, phase reduced in double (large shifts)
      const double ph = -2.0 * ((double)fi * Z.shift[2 * s] + (double)fj * Z.shift[2 * s + 1]);
      float sn, cs;
      sincospif((float)(ph - 2.0 * rint(0.5 * ph)), &sn, &cs);
      x = make_float2(c.x * cs - c.y * sn, c.x * sn + c.y * cs);
    } else if (MODE == 2) {
      float2 z0, z1;
      normals4((uint32_t)(i * M + j), Z.frame, (uint32_t)s, kPSpeckle, Z.key, z0, z1);
      const float amp = sqrtf(0.5f * Z.r[((size_t)s * M + i) * M + j]) * (((i + j) & 1) ? -1.f : 1.f);
      x = make_float2(amp * z0.x, amp * z0.y);
    } else {
      x = row[j];
    }
    v[e] = make_float2(x.x, -x.y);  // conj: inverse DFT by a forward FFT
  }
  __syncthreads();
  fft_reg<M>(v, t, xb + b * (M + M / 16), [](int p) { return rpad(p); }, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) row[t + TPV * out_comb<M>(e)] = make_float2(v[e].x, -v[e].y);
}

template <int M>
__global__ void __launch_bounds__(ZCfg<M>::NTC) kz_cols(ZArgs Z) {  // in-place inverse DFT of columns
  using C = ZCfg<M>;
  constexpr int E = C::E, TPV = C::TPV, W = C::W;
  extern __shared__ float4 zsm[];
  float4 *tw = zsm;
  float2 *xb = reinterpret_cast<float2 *>(zsm + M);
  const int tid = threadIdx.x, s = blockIdx.y;
  const int b = tid % W, t = tid / W, col = blockIdx.x * W + b;
  for (int k = tid; k < M; k += C::NTC) {
    float sn, cs;
    sincospif(-2.f * (float)k / (float)M, &sn, &cs);
    tw[k] = make_float4(cs, sn, -sn, cs);
  }
  float2 *pl = Z.buf + (size_t)s * M * M;
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const float2 x = pl[(size_t)(t + TPV * e) * M + col];
    v[e] = make_float2(x.x, -x.y);
  }
  __syncthreads();
  fft_reg<M>(v, t, xb + b, [](int p) { return p * W; }, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const float2 x = v[e];
    pl[(size_t)(t + TPV * out_comb<M>(e)) * M + col] = make_float2(x.x, -x.y);
  }
}

// ---- scene, screen coefficients, sums, assembly ---------------------------

__global__ void kz_uniform(float *r, int n, uint2 key, int S) {  // r = U[0,1]
  const size_t P = (size_t)n * n;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < S * P; g += (size_t)gridDim.x * blockDim.x) {
    const uint4 x = philox(make_uint4((uint32_t)(g % P), 0u, (uint32_t)(g / P), kPScene), key);
    r[g] = u01(x.x);
  }
}

// periodic separable Gaussian blur, one direction (dir 0: along rows, 1: along columns)
__global__ void kz_blur(const float *in, float *out, int n, int S, const float *kern, int rad, int dir) {
  const size_t P = (size_t)n * n;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < S * P; g += (size_t)gridDim.x * blockDim.x) {
    const size_t s = g / P;
    const int i = (int)((g % P) / n), j = (int)(g % n);
    float acc = 0.f;
    for (int k = -rad; k <= rad; ++k) {
      const int ii = dir ? (i + k + n) % n : i, jj = dir ? j : (j + k + n) % n;
      acc = fmaf(kern[k + rad], in[s * P + (size_t)ii * n + jj], acc);
    }
    out[g] = acc;
  }
}

// per-stream min / max / sum of a field (one block per stream, fixed order)
__global__ void kz_minmax(const float *r, int n, double *out3) {
  __shared__ float smin[kT], smax[kT];
  __shared__ double ssum[kT];
  const size_t P = (size_t)n * n;
  const float *x = r + blockIdx.x * P;
  float mn = 3.4e38f, mx = -3.4e38f;
  double sm = 0.0;
  for (size_t k = threadIdx.x; k < P; k += kT) {
    mn = fminf(mn, x[k]);
    mx = fmaxf(mx, x[k]);
    sm += x[k];
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  ssum[threadIdx.x] = sm;
  __syncthreads();
  for (int o = kT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      smin[threadIdx.x] = fminf(smin[threadIdx.x], smin[threadIdx.x + o]);
      smax[threadIdx.x] = fmaxf(smax[threadIdx.x], smax[threadIdx.x + o]);
      ssum[threadIdx.x] += ssum[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out3[3 * blockIdx.x] = smin[0];
    out3[3 * blockIdx.x + 1] = smax[0];
    out3[3 * blockIdx.x + 2] = ssum[0];
  }
}

__global__ void kz_rescale(float *r, int n, int S, const double *mm, float r_min) {
  const size_t P = (size_t)n * n;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < S * P; g += (size_t)gridDim.x * blockDim.x) {
    const double *m = mm + 3 * (g / P);
    const float v = (float)((r[g] - m[0]) / (m[1] - m[0]));
    r[g] = fmaxf(v, r_min);
  }
}

// screen coefficients c_k = (z1 + j z2) sqrt(Phi(f_k) / M^2) on the M x M grid
__global__ void kz_screen_coef(float2 *coef, int M, int S, const double *r0px, uint2 key) {
  const size_t MM = (size_t)M * M;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < S * MM; g += (size_t)gridDim.x * blockDim.x) {
    const size_t s = g / MM;
    const int i = (int)((g % MM) / M), j = (int)(g % M);
    const double fi = (double)(i < M / 2 ? i : i - M) / M, fj = (double)(j < M / 2 ? j : j - M) / M;
    const double f2 = fi * fi + fj * fj;
    float2 z0, z1;
    normals4((uint32_t)(g % MM), 0u, (uint32_t)s, kPScreen, key, z0, z1);
    float a = 0.f;
    if (f2 > 0.0 && r0px[s] > 0.0)
      a = (float)sqrt(0.023 * pow(r0px[s], -5.0 / 3.0) * pow(f2, -11.0 / 6.0) / ((double)M * M));
    coef[g] = make_float2(a * z0.x, a * z0.y);
  }
}

// plane sums of Re(screen)[0:N, 0:N] over the aperture: (sum phi, phi x, phi y);
// grid (n / 8 row groups, S): FP32 per-thread partials of one row, FP64 block
// sums, then a fixed-order reduction of the row groups (kz_plane_reduce)
__global__ void kz_plane_sums(const float2 *scr, int n, int M, const int2 *span, double *part) {
  __shared__ double red[32 * 5];
  const int s = blockIdx.y, i0 = blockIdx.x * 8;
  double v[3] = {0, 0, 0};
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + r;
    const int2 sp = span[i];
    float a0 = 0.f, a1 = 0.f;
    for (int j = sp.x + threadIdx.x; j < sp.y; j += kT) {
      const float f = scr[((size_t)s * M + i) * M + j].x;
      a0 += f;
      a1 = fmaf(f, (float)(j - n / 2), a1);
    }
    v[0] += a0;
    v[1] += a1;
    v[2] += (double)a0 * (i - n / 2);
  }
  block_sum<3>(v, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) part[((size_t)s * gridDim.x + blockIdx.x) * 3 + k] = v[k];
}
__global__ void kz_plane_reduce(const double *part, int groups, double *sums, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  double v[3] = {0, 0, 0};
  for (int g = 0; g < groups; ++g)
    for (int k = 0; k < 3; ++k) v[k] += part[((size_t)s * groups + g) * 3 + k];
  for (int k = 0; k < 3; ++k) sums[3 * s + k] = v[k];
}

struct AsmArgs {
  const float2 *scr;   // [S][M][M] screen (real part)
  const float2 *spk;   // [S][N][N] IDFT(chi g) (unnormalised)
  const double *sums;  // [S][3]
  const double *sig2;  // [S] noise variance
  const int2 *span;
  double minv[9];
  float2 *y;           // [S][N][N]
  float *phi;          // [S][N][N] or null
  int n, M, S;
  uint2 key;
  uint32_t frame;
};

__global__ void kz_assemble(AsmArgs A) {
  const int n = A.n;
  const size_t P = (size_t)n * n;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < A.S * P; g += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(g / P), i = (int)((g % P) / n), j = (int)(g % n);
    const double *h = A.sums + 3 * s;
    const double c0 = A.minv[0] * h[0] + A.minv[1] * h[1] + A.minv[2] * h[2];
    const double c1 = A.minv[3] * h[0] + A.minv[4] * h[1] + A.minv[5] * h[2];
    const double c2 = A.minv[6] * h[0] + A.minv[7] * h[1] + A.minv[8] * h[2];
    const float ph = A.scr[((size_t)s * A.M + i) * A.M + j].x - (float)(c0 + c1 * (j - n / 2) + c2 * (i - n / 2));
    const float2 x = A.spk[g];
    const float sc = (((i + j) & 1) ? -1.f : 1.f) / (float)n;  // F_c^{-1} = chi F^{-1} chi / N
    const float2 f = make_float2(sc * x.x, sc * x.y);
    float2 w0, w1;
    normals4((uint32_t)(g % P), A.frame, (uint32_t)s, kPNoise, A.key, w0, w1);
    const float sn_ = (float)sqrt(0.5 * A.sig2[s]);
    float2 out = make_float2(sn_ * w0.x, sn_ * w0.y);
    const int2 sp = A.span[i];
    if (j >= sp.x && j < sp.y) {
      float sp_, cp_;
      sincosf(ph, &sp_, &cp_);
      out.x += cp_ * f.x - sp_ * f.y;
      out.y += sp_ * f.x + cp_ * f.y;
    }
    A.y[g] = out;
    if (A.phi) A.phi[g] = ph;
  }
}

#define DDH_ZDISPATCH(m, CALL)                          \
  switch (m) {                                          \
    case 64: { constexpr int M = 64; CALL; } break;     \
    case 128: { constexpr int M = 128; CALL; } break;   \
    case 256: { constexpr int M = 256; CALL; } break;   \
    case 512: { constexpr int M = 512; CALL; } break;   \
    case 1024: { constexpr int M = 1024; CALL; } break; \
    case 2048: { constexpr int M = 2048; CALL; } break; \
    default: return cudaErrorInvalidValue;              \
  }

template <int M> size_t zrow_smem() { return M * sizeof(float4) + (size_t)ZCfg<M>::H * (M + M / 16) * sizeof(float2); }
template <int M> size_t zcol_smem() { return M * sizeof(float4) + (size_t)M * ZCfg<M>::W * sizeof(float2); }

template <int M>
cudaError_t zinit() {
  cudaFuncSetAttribute(kz_rows<M, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zrow_smem<M>());
  cudaFuncSetAttribute(kz_rows<M, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zrow_smem<M>());
  cudaFuncSetAttribute(kz_rows<M, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zrow_smem<M>());
  cudaFuncSetAttribute(kz_cols<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zcol_smem<M>());
  return cudaGetLastError();
}

cudaError_t z_rows(int M, int mode, const ZArgs &z, int S, cudaStream_t st) {
  DDH_ZDISPATCH(M, ({
                  const dim3 g(M / ZCfg<M>::H, S);
                  if (mode == 1) kz_rows<M, 1><<<g, ZCfg<M>::NTR, zrow_smem<M>(), st>>>(z);
                  else if (mode == 2) kz_rows<M, 2><<<g, ZCfg<M>::NTR, zrow_smem<M>(), st>>>(z);
                  else kz_rows<M, 0><<<g, ZCfg<M>::NTR, zrow_smem<M>(), st>>>(z);
                }));
  return cudaGetLastError();
}
cudaError_t z_cols(int M, const ZArgs &z, int S, cudaStream_t st) {
  DDH_ZDISPATCH(M, (kz_cols<M><<<dim3(M / ZCfg<M>::W, S), ZCfg<M>::NTC, zcol_smem<M>(), st>>>(z)));
  return cudaGetLastError();
}
cudaError_t z_init(int M) { DDH_ZDISPATCH(M, return zinit<M>()); return cudaErrorInvalidValue; }

}  // namespace
}  // namespace ddh

using ddh::ZArgs;

struct ddh_synth {
  int n = 0, M = 0, S = 0;
  cudaStream_t st = nullptr;
  uint2 key{};
  float *r = nullptr, *tmp = nullptr;
  float2 *coef = nullptr, *scr = nullptr, *spk = nullptr;
  double *shift = nullptr, *r0px = nullptr, *mm = nullptr, *sums = nullptr, *sig2 = nullptr, *psum = nullptr;
  int2 *span = nullptr;
  double minv[9] = {};
  std::vector<double> vel;  // [S][2]
  std::string err;
};

namespace {
void synth_free(ddh_synth *z) {
  if (!z) return;
  void *p[] = {z->r, z->tmp, z->coef, z->scr, z->spk, z->shift, z->r0px, z->mm, z->sums, z->sig2, z->span, z->psum};
  for (void *q : p)
    if (q) cudaFree(q);
  delete z;
}
double inv3x3(const double G[9], double out[9]) {
  const double a = G[0], b = G[1], c = G[2], d = G[3], e = G[4], f = G[5], g = G[6], h = G[7], i = G[8];
  const double A = e * i - f * h, B = -(d * i - f * g), C = d * h - e * g, det = a * A + b * B + c * C;
  if (!(std::fabs(det) > 0)) return 0.0;
  const double o[9] = {A, -(b * i - c * h), b * f - c * e, B, a * i - c * g, -(a * f - c * d), C, -(a * h - b * g),
                       a * e - b * d};
  for (int k = 0; k < 9; ++k) out[k] = o[k] / det;
  return det;
}
}  // namespace

extern "C" {

ddh_status ddh_synth_create(int32_t n, float diam, int32_t streams, const double *d_r0, const double *velocity,
                            double sigma_b, double snr_db, uint64_t seed, void *cuda_stream, ddh_synth **out) {
  if (!out || !d_r0 || !velocity) return DDH_E_INVAL;
  *out = nullptr;
  if (!(n == 64 || n == 128 || n == 256 || n == 512 || n == 1024) || streams < 1 || !(diam > 0) || !(sigma_b > 0))
    return DDH_E_INVAL;
  ddh_synth *z = new ddh_synth();
  z->n = n;
  z->M = 2 * n;
  z->S = streams;
  z->st = (cudaStream_t)cuda_stream;
  z->key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  z->vel.assign(velocity, velocity + 2 * streams);
  const size_t P = (size_t)n * n, MM = (size_t)z->M * z->M, S = streams;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  A(cudaMalloc(&z->r, S * P * 4));
  A(cudaMalloc(&z->tmp, S * P * 4));
  A(cudaMalloc(&z->coef, S * MM * 8));
  A(cudaMalloc(&z->scr, S * MM * 8));
  A(cudaMalloc(&z->spk, S * P * 8));
  A(cudaMalloc(&z->shift, S * 2 * 8));
  A(cudaMalloc(&z->r0px, S * 8));
  A(cudaMalloc(&z->mm, S * 3 * 8));
  A(cudaMalloc(&z->sums, S * 3 * 8));
  A(cudaMalloc(&z->psum, S * (n / 8) * 3 * 8));
  A(cudaMalloc(&z->sig2, S * 8));
  A(cudaMalloc(&z->span, n * sizeof(int2)));
  if (e != cudaSuccess) {
    synth_free(z);
    return DDH_E_NOMEM;
  }
  // aperture (strictly inside the circle of diameter diam, centre (n/2, n/2)) and plane normal matrix
  std::vector<int2> span(n);
  double G[9] = {};
  for (int i = 0; i < n; ++i) {
    int lo = n, hi = 0;
    for (int j = 0; j < n; ++j) {
      const double di = i - n / 2, dj = j - n / 2, rr = 0.5 * diam;
      if (di * di + dj * dj < rr * rr) {
        lo = std::min(lo, j);
        hi = j + 1;
        const double b3[3] = {1.0, (double)dj, (double)di};
        for (int u = 0; u < 3; ++u)
          for (int v = 0; v < 3; ++v) G[u * 3 + v] += b3[u] * b3[v];
      }
    }
    span[i] = lo < hi ? make_int2(lo, hi) : make_int2(0, 0);
  }
  if (inv3x3(G, z->minv) == 0.0) {
    synth_free(z);
    return DDH_E_INVAL;
  }
  std::vector<double> r0(S);
  for (size_t s = 0; s < S; ++s) r0[s] = d_r0[s] > 0 ? diam / d_r0[s] : 0.0;
  A(cudaMemcpy(z->span, span.data(), n * sizeof(int2), cudaMemcpyHostToDevice));
  A(cudaMemcpy(z->r0px, r0.data(), S * 8, cudaMemcpyHostToDevice));
  // scene: U[0,1] -> blur rows -> blur columns -> min-max rescale, clamp
  const int rad = (int)std::ceil(4.0 * sigma_b);
  std::vector<float> kern(2 * rad + 1);
  double ks = 0;
  for (int k = -rad; k <= rad; ++k) ks += (kern[k + rad] = (float)std::exp(-0.5 * k * k / (sigma_b * sigma_b)));
  for (float &v : kern) v = (float)(v / ks);
  float *dk = nullptr;
  A(cudaMalloc(&dk, kern.size() * 4));
  A(cudaMemcpy(dk, kern.data(), kern.size() * 4, cudaMemcpyHostToDevice));
  ddh::kz_uniform<<<1024, 256, 0, z->st>>>(z->r, n, z->key, streams);
  ddh::kz_blur<<<1024, 256, 0, z->st>>>(z->r, z->tmp, n, streams, dk, rad, 0);
  ddh::kz_blur<<<1024, 256, 0, z->st>>>(z->tmp, z->r, n, streams, dk, rad, 1);
  ddh::kz_minmax<<<streams, ddh::kT, 0, z->st>>>(z->r, n, z->mm);
  ddh::kz_rescale<<<1024, 256, 0, z->st>>>(z->r, n, streams, z->mm, 1e-4f);
  ddh::kz_minmax<<<streams, ddh::kT, 0, z->st>>>(z->r, n, z->mm);  // mean(r) for the noise level
  ddh::kz_screen_coef<<<1024, 256, 0, z->st>>>(z->coef, z->M, streams, z->r0px, z->key);
  A(ddh::z_init(z->M));
  A(ddh::z_init(n));
  A(cudaGetLastError());
  A(cudaStreamSynchronize(z->st));
  std::vector<double> mm(3 * S), sig2(S);
  A(cudaMemcpy(mm.data(), z->mm, S * 3 * 8, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < S; ++s) sig2[s] = mm[3 * s + 2] / (double)P / std::pow(10.0, snr_db / 10.0);
  A(cudaMemcpy(z->sig2, sig2.data(), S * 8, cudaMemcpyHostToDevice));
  cudaFree(dk);
  if (e != cudaSuccess) {
    synth_free(z);
    return DDH_E_CUDA;
  }
  *out = z;
  return DDH_OK;
}

ddh_status ddh_synth_frames(ddh_synth *z, int64_t t0, int32_t T, void *y, float *phi) {
  if (!z || T < 0 || (T > 0 && !y)) return DDH_E_INVAL;
  const size_t P = (size_t)z->n * z->n;
  std::vector<double> sh(2 * z->S);
  for (int t = 0; t < T; ++t) {
    const int64_t f = t0 + t;
    for (int s = 0; s < z->S; ++s) {
      sh[2 * s] = (double)f * z->vel[2 * s];
      sh[2 * s + 1] = (double)f * z->vel[2 * s + 1];
    }
    if (cudaMemcpyAsync(z->shift, sh.data(), sh.size() * 8, cudaMemcpyHostToDevice, z->st) != cudaSuccess)
      return DDH_E_CUDA;
    ZArgs a{};
    a.key = z->key;
    a.frame = (uint32_t)f;
    // screen: rows of c e^{-2 pi i f.s} (inverse DFT), then columns
    a.buf = z->scr;
    a.coef = z->coef;
    a.shift = z->shift;
    if (ddh::z_rows(z->M, 1, a, z->S, z->st) != cudaSuccess) return DDH_E_CUDA;
    if (ddh::z_cols(z->M, a, z->S, z->st) != cudaSuccess) return DDH_E_CUDA;
    ddh::kz_plane_sums<<<dim3(z->n / 8, z->S), ddh::kT, 0, z->st>>>(z->scr, z->n, z->M, z->span, z->psum);
    ddh::kz_plane_reduce<<<(z->S + 127) / 128, 128, 0, z->st>>>(z->psum, z->n / 8, z->sums, z->S);
    // speckle: rows of chi g (inverse DFT), then columns
    a.buf = z->spk;
    a.r = z->r;
    if (ddh::z_rows(z->n, 2, a, z->S, z->st) != cudaSuccess) return DDH_E_CUDA;
    if (ddh::z_cols(z->n, a, z->S, z->st) != cudaSuccess) return DDH_E_CUDA;
    ddh::AsmArgs as{};
    as.scr = z->scr;
    as.spk = z->spk;
    as.sums = z->sums;
    as.sig2 = z->sig2;
    as.span = z->span;
    std::memcpy(as.minv, z->minv, sizeof(as.minv));
    as.y = reinterpret_cast<float2 *>(y) + (size_t)t * z->S * P;
    as.phi = phi ? phi + (size_t)t * z->S * P : nullptr;
    as.n = z->n;
    as.M = z->M;
    as.S = z->S;
    as.key = z->key;
    as.frame = (uint32_t)f;
    ddh::kz_assemble<<<2048, 256, 0, z->st>>>(as);
    if (cudaGetLastError() != cudaSuccess) return DDH_E_CUDA;
  }
  return DDH_OK;
}

ddh_status ddh_synth_reflectance(ddh_synth *z, float *r) {
  if (!z || !r) return DDH_E_INVAL;
  if (cudaMemcpyAsync(r, z->r, (size_t)z->S * z->n * z->n * 4, cudaMemcpyDeviceToDevice, z->st) != cudaSuccess)
    return DDH_E_CUDA;
  return DDH_OK;
}

ddh_status ddh_synth_destroy(ddh_synth *z) {
  if (!z) return DDH_E_INVAL;
  cudaStreamSynchronize(z->st);
  synth_free(z);
  return DDH_OK;
}

}  // extern "C"
