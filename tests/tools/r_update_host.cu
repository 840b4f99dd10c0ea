// Host harness: evaluates ddh::r_update (the device helper compiled as host
// code) on (r, q, B, S) rows read from stdin; used to debug against the oracle.
#include <cstdio>
#include "../../paper_2305_03284_b200/csrc/ddh_common.cuh"
int main() {
  float r, q, B, S, rmin;
  while (scanf("%f %f %f %f %f", &r, &q, &B, &S, &rmin) == 5) printf("%.9g\n", ddh::r_update(r, q, B, S, rmin));
  return 0;
}
