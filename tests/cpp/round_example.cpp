// C++ host driver over the plain C ABI (no Python, no torch): what a
// reference maintainer's co2_round loop (proj/src/outer_algorithms.cpp:
// 110-211, driven by Simulation::step :451-453) looks like on the B200 path.
// Two simulated CO2 workers on one GPU (LOCAL engine), C1-style fp32 buffers,
// tau synthetic inner steps per round with the InnerTrace snapshots, then
// co2_round.  Checks the reference's round contract: round 0 only snapshots,
// later rounds apply the outer step with min_gap >= 1 and every outer
// displacement bounded by alpha * phi.  Built by `make round_example`; run by
// tests/test_gpu_parity.py.  Prints "ROUNDS OK" on success.
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "co2_b200.h"

#define REQUIRE(call)                                                              \
  do {                                                                             \
    co2_status_t _s = (call);                                                      \
    if (_s != CO2_OK) {                                                            \
      std::printf("FAIL %s -> %d: %s\n", #call, (int)_s, co2_last_error());       \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main() {
  const int64_t n = 1 << 20;
  const int g = 2, tau = 4, rounds = 5;
  co2_hyper_t h{1.0, 0.7, 5e-3, 1e-12, tau, 1, 1, 0, 0};
  REQUIRE(co2_hyper_validate(&h));
  cudaStream_t st = nullptr;  // legacy default stream
  co2_aar_t* eng = nullptr;
  REQUIRE(co2_aar_create_local(&eng, g));
  std::vector<co2_worker_t*> ws(g, nullptr);
  for (int i = 0; i < g; ++i) {
    REQUIRE(co2_worker_create(&ws[i], CO2_MODE_F32, n, nullptr, 1, st));
    // x_{0,0}: synthetic draws for this worker (x_end stream)
    REQUIRE(co2_synth(CO2_MODE_F32, 7, i, 0, n, nullptr, nullptr, nullptr,
                      co2_worker_buffer(ws[i], CO2_BUF_PARAMS), nullptr, st));
  }
  int bad = 0;
  for (int t = 0; t < rounds; ++t) {
    for (int i = 0; i < g; ++i) {
      void* params = co2_worker_buffer(ws[i], CO2_BUF_PARAMS);
      REQUIRE(co2_worker_snapshot_start(ws[i], st));
      for (int k = 0; k < tau; ++k) {
        REQUIRE(co2_synthetic_inner_step(CO2_DTYPE_F32, n, params, 1e-3, 1.0, 7, i,
                                         (int64_t)t * tau + k, 1, st));
        if (k == 0) REQUIRE(co2_worker_snapshot_first(ws[i], st));
      }
    }
    co2_round_result_t r{};
    REQUIRE(co2_round(ws.data(), g, eng, &h, st, /*sync=*/1, &r));
    std::printf("round %d: outer_applied=%d min_gap=%.6g max_outer_step=%.6g\n", t,
                r.outer_applied, r.min_gap, r.max_outer_step);
    if (t == 0 && r.outer_applied != 0) ++bad;
    if (t > 0 && (r.outer_applied != 1 || !(r.min_gap >= 1.0) ||
                  !(r.max_outer_step <= h.alpha * h.phi * (1 + 1e-6))))
      ++bad;
  }
  co2_round_result_t r1{};
  co2_status_t bad_call = co2_round(ws.data(), 1, eng, &h, st, 1, &r1);
  if (bad_call != CO2_ERR_VALIDATION) ++bad;  // worker count must match the engine
  for (co2_worker_t* w : ws) REQUIRE(co2_worker_destroy(w));
  REQUIRE(co2_aar_destroy(eng));
  std::printf(bad ? "ROUNDS FAILED %d\n" : "ROUNDS OK\n", bad);
  return bad ? 1 : 0;
}
