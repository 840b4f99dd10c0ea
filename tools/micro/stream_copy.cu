// Calibration: the memory pattern of ks_rows_fwd alone (read y 8 B + phi 4 B,
// write 8 B per pixel, 64 streams of 256^2), as a plain kernel, to separate
// the HBM-bound part of the row kernels from their compute.
#include <cstdio>
__global__ void __launch_bounds__(256) kcopy(const float2 *__restrict__ y, const float *__restrict__ phi, float2 *__restrict__ out) {
  const int t = threadIdx.x % 16, b = threadIdx.x / 16;
  const size_t row = ((size_t)blockIdx.y * 256 + blockIdx.x * 16 + b) * 256;
  float2 v[16];
  float p[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = y[row + t + 16 * e];
#pragma unroll
  for (int e = 0; e < 16; ++e) p[e] = phi[row + t + 16 * e];
#pragma unroll
  for (int e = 0; e < 16; ++e) out[row + t + 16 * e] = make_float2(v[e].x * p[e], v[e].y + p[e]);
}
__global__ void __launch_bounds__(256) kcopy_y(const float2 *__restrict__ y, float2 *__restrict__ out) {
  const int t = threadIdx.x % 16, b = threadIdx.x / 16;
  const size_t row = ((size_t)blockIdx.y * 256 + blockIdx.x * 16 + b) * 256;
  float2 v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = y[row + t + 16 * e];
#pragma unroll
  for (int e = 0; e < 16; ++e) out[row + t + 16 * e] = v[e];
}
int main() {
  const size_t P = 256 * 256, S = 64;
  float2 *y, *out; float *phi, *flush;
  cudaMalloc(&y, S * P * 8 * 4); cudaMalloc(&out, S * P * 8); cudaMalloc(&phi, S * P * 4 * 4); cudaMalloc(&flush, 256 << 20);
  cudaMemset(y, 0, S * P * 8 * 4); cudaMemset(phi, 0, S * P * 4 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    float tot = 0; int n = 0;
    for (int r = 0; r < 20; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);  // evict L2
      const int k = r % 4;
      cudaEventRecord(a);
      if (mode == 0) kcopy<<<dim3(16, S), 256>>>(y + k * S * P, phi + k * S * P, out);
      else kcopy_y<<<dim3(16, S), 256>>>(y + k * S * P, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 4) { tot += ms; ++n; }
    }
    const double bytes = mode == 0 ? S * P * 20.0 : S * P * 16.0;
    printf("%s: %.1f us, %.0f GB/s\n", mode == 0 ? "y+phi -> out (20 B/px)" : "y -> out (16 B/px)", tot / n * 1000, bytes / (tot / n * 1e-3) / 1e9);
  }
  return 0;
}
