// Back-to-back launch cost of near-empty kernels (1 block / 1024 blocks,
// small vs 320-byte parameter block) on one stream.
#include <cstdio>
struct Big { char b[320]; };
__global__ void kempty(int *p) { if (threadIdx.x == 1023) p[0] = 1; }
__global__ void kbig(Big a, int *p) { if (threadIdx.x == 1023) p[0] = a.b[7]; }
__global__ void kload(const float4 *x, int *p) {  // 1 load per thread, then exit
  float4 v = x[blockIdx.x * blockDim.x + threadIdx.x];
  if (v.x == 123.f) p[0] = 1;
}
int main() {
  int *p; cudaMalloc(&p, 4); float4 *x; cudaMalloc(&x, 1024 * 256 * 16); cudaMemset(x, 0, 1024 * 256 * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  Big big{};
  for (int mode = 0; mode < 5; ++mode) {
    const int grid = (mode == 0) ? 1 : 1024;
    for (int w = 0; w < 10; ++w) kempty<<<grid, 256>>>(p);
    cudaEventRecord(a);
    for (int r = 0; r < 1000; ++r) {
      if (mode <= 1) kempty<<<grid, 256>>>(p);
      else if (mode == 2) kbig<<<grid, 256>>>(big, p);
      else if (mode == 3) kload<<<grid, 256>>>(x, p);
      else { kload<<<grid, 256>>>(x, p); }
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const char *names[] = {"empty 1 block", "empty 1024x256", "320-B params 1024x256", "1 load/thread 1024x256", "same again"};
    printf("%-26s %6.2f us per launch\n", names[mode], ms);
  }
  return 0;
}
