// Host cost of kernel launches while the device is busy (each kernel spins
// ~10 us, so the queue holds pending work): plain launches vs launches with
// programmatic stream serialisation, 1 and 3 streams, 336-byte arguments.
#include <chrono>
#include <cstdio>
struct Big { char b[336]; long long spin; };
__global__ void kspin(Big a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  long long t0 = clock64();
  while (clock64() - t0 < a.spin) {}
}
static double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  cudaStream_t s[3];
  for (auto &x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  Big a = {};
  a.spin = 20000;  // ~10 us
  const int R = 120;
  for (int rep = 0; rep < 3; ++rep) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      for (int ns = 1; ns <= 3; ns += 2) {
        for (int grid : {148, 296, 1024}) {
          cudaDeviceSynchronize();
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256);
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at; cfg.numAttrs = pdl;
          double t0 = now();
          for (int i = 0; i < R; ++i) { cfg.stream = s[i % ns]; cudaLaunchKernelEx(&cfg, kspin, a); }
          double t1 = now();
          cudaDeviceSynchronize();
          double t2 = now();
          if (rep == 2) printf("pdl %d streams %d grid %4d: host %.2f us/launch (device %.1f us/launch)\n", pdl, ns, grid, (t1 - t0) / R, (t2 - t0) / R);
        }
      }
    }
  }
  return 0;
}
