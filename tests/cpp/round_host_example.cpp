// C++ host driver of the "inner loop on the CPU, outer round on the GPU"
// drop-in (co2_round_host): the reference's problems and
// run_inner_loop stay host code (here: tau steps of x <- x - lr * (x - target)
// on a quadratic, in plain C++), only the InnerTrace (x_{t,1}, x_{t,tau})
// goes to the GPU each round, and the next inner loop starts from the
// x_{t+1,0} that comes back.  The outer state stays resident in the worker.
// Checks: the rounds follow the reference's contract (round 0 only
// snapshots; then min_gap >= 1 and every outer displacement <= alpha*phi),
// and a second set of workers driven by uploading the same traces by hand
// and calling co2_round gives bit-identical params every round.  Built by
// `make round_host_example`; run by tests/test_gpu_parity.py.  Prints
// "HOST ROUNDS OK" on success.
#include <cmath>
#include <cstdio>
#include <cstring>
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
#define CUDA(call)                                                                 \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      std::printf("FAIL %s: %s\n", #call, cudaGetErrorString(_e));               \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main() {
  const int64_t n = 200003;  // ragged: not a multiple of the vector width
  const int g = 2, tau = 3, rounds = 5;
  const double lr = 0.05;
  co2_hyper_t h{1.0, 0.7, 5e-3, 1e-12, tau, 1, 1, 0, 0};
  REQUIRE(co2_hyper_validate(&h));
  cudaStream_t st = nullptr;
  co2_aar_t *ea = nullptr, *eb = nullptr;
  REQUIRE(co2_aar_create_local(&ea, g));  // driven by co2_round_host
  REQUIRE(co2_aar_create_local(&eb, g));  // driven by hand uploads + co2_round
  const size_t bytes = sizeof(float) * (size_t)n;
  // host: each worker's params, target, and the pinned trace / result buffers
  std::vector<std::vector<float>> x(g, std::vector<float>(n)), target(g, std::vector<float>(n));
  std::vector<float*> first(g), end(g), next(g);
  for (int i = 0; i < g; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      x[i][j] = 0.01f * std::sin(0.001f * (float)(j + 17 * i));
      target[i][j] = 0.02f * std::cos(0.0007f * (float)(j * (i + 1)));
    }
    CUDA(cudaMallocHost(&first[i], bytes));
    CUDA(cudaMallocHost(&end[i], bytes));
    CUDA(cudaMallocHost(&next[i], bytes));
  }
  std::vector<co2_worker_t*> wa(g, nullptr), wb(g, nullptr);
  for (int i = 0; i < g; ++i) {
    void* d = nullptr;
    CUDA(cudaMalloc(&d, bytes));
    CUDA(cudaMemcpy(d, x[i].data(), bytes, cudaMemcpyHostToDevice));
    REQUIRE(co2_worker_create(&wa[i], CO2_MODE_F32, n, d, 1, st));
    REQUIRE(co2_worker_create(&wb[i], CO2_MODE_F32, n, d, 1, st));
    CUDA(cudaDeviceSynchronize());
    CUDA(cudaFree(d));
    REQUIRE(co2_worker_snapshot_start(wa[i], st));  // x_{0,0} anchor on the device
    REQUIRE(co2_worker_snapshot_start(wb[i], st));
  }
  std::vector<float> check(n);
  int bad = 0;
  for (int t = 0; t < rounds; ++t) {
    for (int i = 0; i < g; ++i) {  // the reference's inner loop, on the CPU
      for (int k = 0; k < tau; ++k) {
        for (int64_t j = 0; j < n; ++j) x[i][j] -= (float)lr * (x[i][j] - target[i][j]);
        if (k == 0) std::memcpy(first[i], x[i].data(), bytes);  // InnerTrace::x_first
      }
      std::memcpy(end[i], x[i].data(), bytes);  // InnerTrace::x_end
    }
    co2_round_result_t r{};
    REQUIRE(co2_round_host(wa.data(), g, ea, &h, (const void* const*)first.data(),
                           (const void* const*)end.data(), (void* const*)next.data(), st,
                           /*sync=*/1, &r));
    for (int i = 0; i < g; ++i) {  // the same traces by hand, then co2_round
      CUDA(cudaMemcpy(co2_worker_buffer(wb[i], CO2_BUF_XFIRST), first[i], bytes,
                      cudaMemcpyHostToDevice));
      CUDA(cudaMemcpy(co2_worker_buffer(wb[i], CO2_BUF_PARAMS), end[i], bytes,
                      cudaMemcpyHostToDevice));
    }
    co2_round_result_t rb{};
    REQUIRE(co2_round(wb.data(), g, eb, &h, st, 1, &rb));
    for (int i = 0; i < g; ++i) {
      CUDA(cudaMemcpy(check.data(), co2_worker_buffer(wb[i], CO2_BUF_PARAMS), bytes,
                      cudaMemcpyDeviceToHost));
      if (std::memcmp(check.data(), next[i], bytes) != 0) ++bad;
      std::memcpy(x[i].data(), next[i], bytes);  // the next inner loop starts from x_{t+1,0}
    }
    std::printf("round %d: outer_applied=%d min_gap=%.6g max_outer_step=%.6g\n", t,
                r.outer_applied, r.min_gap, r.max_outer_step);
    if (t == 0 && r.outer_applied != 0) ++bad;
    if (t > 0 && (r.outer_applied != 1 || !(r.min_gap >= 1.0) ||
                  !(r.max_outer_step <= h.alpha * h.phi * (1 + 1e-6))))
      ++bad;
    if (r.min_gap != rb.min_gap || r.max_outer_step != rb.max_outer_step) ++bad;
  }
  for (int i = 0; i < g; ++i) {
    REQUIRE(co2_worker_destroy(wa[i]));
    REQUIRE(co2_worker_destroy(wb[i]));
    cudaFreeHost(first[i]);
    cudaFreeHost(end[i]);
    cudaFreeHost(next[i]);
  }
  REQUIRE(co2_aar_destroy(ea));
  REQUIRE(co2_aar_destroy(eb));
  std::printf(bad ? "HOST ROUNDS FAILED %d\n" : "HOST ROUNDS OK\n", bad);
  return bad ? 1 : 0;
}
