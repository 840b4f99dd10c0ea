// MUFU throughput on this GPU: independent lg2 / ex2 / rcp / sin chains,
// ops per clock per SM (clock64 over the kernel, all SMs busy).
#include <cstdio>
template <int OP>
__global__ void kmufu(float *out, int iters, long long *cyc) {
  float a0 = threadIdx.x * 1e-3f + 1.1f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#define OP1(x) if (OP == 0) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(x)); \
               else if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x)); \
               else if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x)); \
               else asm volatile("sin.approx.ftz.f32 %0, %0;" : "+f"(x));
    OP1(a0) OP1(a1) OP1(a2) OP1(a3) OP1(a4) OP1(a5) OP1(a6) OP1(a7)
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 4096;
  float *out; long long *cyc; cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  const char *names[] = {"lg2", "ex2", "rcp", "sin"};
  for (int op = 0; op < 4; ++op) {
    for (int w = 0; w < 2; ++w) {
      if (op == 0) kmufu<0><<<blocks, threads>>>(out, iters, cyc);
      if (op == 1) kmufu<1><<<blocks, threads>>>(out, iters, cyc);
      if (op == 2) kmufu<2><<<blocks, threads>>>(out, iters, cyc);
      if (op == 3) kmufu<3><<<blocks, threads>>>(out, iters, cyc);
    }
    cudaDeviceSynchronize();
    long long c[1]; cudaMemcpy(c, cyc, 8, cudaMemcpyDeviceToHost);
    // per SM: 4 blocks x 512 threads x iters x 8 ops over c cycles (blocks co-resident)
    printf("%s: %.1f ops/clk/SM\n", names[op], 4.0 * threads * iters * 8 / (double)c[0]);
  }
  return 0;
}
