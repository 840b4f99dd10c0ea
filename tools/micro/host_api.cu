// Host cost of the enqueue operations a streaming step issues (per call, us):
// kernel launch with a 336-byte argument struct (<<<>>> and cudaLaunchKernelEx
// with programmatic stream serialisation), cudaEventRecord, cudaStreamWaitEvent.
#include <chrono>
#include <cstdio>
struct Big { char b[336]; };
__global__ void kempty(Big a) { if (a.b[0] == 123 && threadIdx.x == 9999) a.b[1] = 0; }
static double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  cudaStream_t s[4];
  for (auto &x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t ev[64];
  for (auto &e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  Big a = {};
  const int R = 2000;
  for (int rep = 0; rep < 3; ++rep) {
    cudaDeviceSynchronize();
    double t0 = now();
    for (int i = 0; i < R; ++i) kempty<<<296, 256, 0, s[i & 3]>>>(a);
    double t1 = now();
    cudaDeviceSynchronize();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(296); cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    double t2 = now();
    for (int i = 0; i < R; ++i) { cfg.stream = s[i & 3]; cudaLaunchKernelEx(&cfg, kempty, a); }
    double t3 = now();
    cudaDeviceSynchronize();
    double t4 = now();
    for (int i = 0; i < R; ++i) cudaEventRecord(ev[i & 63], s[i & 3]);
    double t5 = now();
    for (int i = 0; i < R; ++i) cudaStreamWaitEvent(s[(i + 1) & 3], ev[i & 63], 0);
    double t6 = now();
    cudaDeviceSynchronize();
    printf("launch<<<>>> %.2f us, launchEx+PDL %.2f us, eventRecord %.2f us, streamWaitEvent %.2f us\n",
           (t1 - t0) / R, (t3 - t2) / R, (t5 - t4) / R, (t6 - t5) / R);
  }
  return 0;
}
