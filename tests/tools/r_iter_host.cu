// Host harness for tests/tools/r_iter_study.py: ddh::r_update (device helper compiled
// as host code) on (r, q, B, S) columns, counting root iterations per pixel and
// the per-warp maximum (32 consecutive pixels of a colour class).
#include <cstdio>
#include <vector>
static int g_it = 0;
#define DDH_ITER_HOOK (++g_it)
#include "../../paper_2305_03284_b200/csrc/ddh_common.cuh"
int main(int argc, char **argv) {
  FILE *f = fopen(argv[1], "rb");
  int m; fread(&m, 4, 1, f);
  std::vector<float> v(4 * (size_t)m); fread(v.data(), 4, v.size(), f); fclose(f);
  FILE *o = fopen(argv[2], "wb");
  long tot = 0, warp = 0; int wmax = 0;
  std::vector<float> out(m); std::vector<int> its(m);
  for (int i = 0; i < m; ++i) {
    g_it = 0;
    out[i] = ddh::r_update(v[i], v[m + i], v[2 * m + i], v[3 * m + i], 1e-4f);
    its[i] = g_it; tot += g_it; wmax = g_it > wmax ? g_it : wmax;
    if ((i & 31) == 31) { warp += wmax; wmax = 0; }
  }
  fwrite(out.data(), 4, m, o); fwrite(its.data(), 4, m, o); fclose(o);
  printf("mean iters %.3f  mean warp-max %.3f\n", (double)tot / m, (double)warp / (m / 32));
}
