// Prints EvalTC's shared-memory geometry (tc_geom, eval_tc.cuh) for every odd
// L in [3, SK_TC_MAX_L]: the host side of tests/test_tc_layout.py checks that
// tools/tc_emulate.py's Geom is the same layout.
//   nvcc -std=c++17 -arch=sm_100a -I paper_2210_15962_b200/csrc -o /tmp/tc_geom_dump tools/tc_geom_dump.cu
#include <cstdio>

#include "eval_tc.cuh"

int main() {
  for (int L = 3; L <= sk::kTcMaxL; L += 2) {
    const sk::TcGeom g = sk::tc_geom(L);
    std::printf("%d %d %d %d %u %u %u %u %u %u\n", L, g.NT, g.TOFF, g.MT, g.q_off, g.ge_off, g.go_off, g.t_off,
                g.s2_off, g.bytes);
  }
  return 0;
}
