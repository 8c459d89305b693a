// C++ facade test: the reference's outer-op unit tests
// (proj/tests/test_outer_algorithms.cpp:85-168, proj/tests/test_param_ops.cpp:
// 30-52,113-145) rerun through include/co2_b200.hpp on the GPU.  Built by
// `make facade_test`; run by tests/test_gpu_parity.py.  Prints one line per
// case and exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "co2_b200.hpp"

using namespace co2b200;

static int g_fail = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);      \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

template <class E, class F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static DeviceVector vec(std::vector<double> v) { return DeviceVector::from_host(v); }

int main() {
  {  // staleness gap compares displacement against the first inner step
    auto gap = staleness_gap(vec({1.6, 0.3}), vec({1.0, 0.2}), vec({1.2, 0.3}), 2, 1e-12).to_host();
    CHECK(std::fabs(gap[0] - (0.6 / 0.4 + 1.0)) <= 1e-15 * (0.6 / 0.4 + 1.0));
    CHECK(std::fabs(gap[1] - (0.1 / 0.2 + 1.0)) <= 1e-15 * (0.1 / 0.2 + 1.0));
    std::printf("ok staleness_gap\n");
  }
  {  // a motionless coordinate falls back to the epsilon floor
    auto gap = staleness_gap(vec({2.0, 1.0}), vec({1.0, 1.0}), vec({1.0, 1.0}), 4, 0.5).to_host();
    CHECK(gap[0] == 1.0 / 0.5 + 1.0);
    CHECK(gap[1] == 1.0);
    std::printf("ok epsilon floor\n");
  }
  {  // penalized momentum divides the displacement by the gap
    auto mp = vec({1.0, -2.0}), g = vec({2.0, 1.0}), d = vec({0.5, 0.3});
    auto m = penalized_momentum_update(mp, 0.5, g, d, true).to_host();
    CHECK(m[0] == 0.5 * 1.0 + 0.5 / 2.0);
    CHECK(m[1] == 0.5 * -2.0 + 0.3);
    auto raw = penalized_momentum_update(mp, 0.5, g, d, false).to_host();
    CHECK(raw[0] == 1.0);
    CHECK(raw[1] == -0.7);
    auto bad = vec({0.5, 1.0});
    CHECK(throws<validation_error>([&] { penalized_momentum_update(mp, 0.5, bad, d, true); }));
    std::printf("ok penalized momentum\n");
  }
  {  // outer_iterate applies the clipped momentum step
    auto x = vec({1.0, -1.0, 0.0}), m = vec({4.0, -0.25, -9.0});
    auto next = outer_iterate(x, 0.5, m, 1.0, true).to_host();
    CHECK(next[0] == 1.0 - 0.5 * 1.0);
    CHECK(next[1] == -1.0 + 0.5 * 0.25);
    CHECK(next[2] == 0.5);
    auto raw = outer_iterate(x, 0.5, m, 1.0, false).to_host();
    CHECK(raw[0] == -1.0);
    CHECK(raw[2] == 4.5);
    std::printf("ok outer_iterate\n");
  }
  {  // hyperparameter validation
    Co2Hyper h;
    h.validate();
    h.alpha = 0.0;
    CHECK(throws<validation_error>([&] { h.validate(); }));
    h.alpha = 1.0;
    h.beta = 1.0;
    CHECK(throws<validation_error>([&] { h.validate(); }));
    h.beta = 0.5;
    h.phi = 0.0;
    CHECK(throws<validation_error>([&] { h.validate(); }));
    h.phi = 1.0;
    h.epsilon = 0.0;
    CHECK(throws<validation_error>([&] { h.validate(); }));
    std::printf("ok hyper validation\n");
  }
  {  // average matches a frozen fixed-order sum oracle bit for bit
    std::vector<DeviceVector> in;
    in.push_back(vec({0.5442868880568308, 1.8113273945956503, 0.19139323188558377,
                      1.6248311340530925, 0.40218505048593167, 0.04286966237077339}));
    in.push_back(vec({0.6314264412370334, 1.9654648029382469, 0.3630702349745145,
                      -1.6270775115457816, 1.0069351598601868, 0.9299044643529717}));
    in.push_back(vec({1.234339331698358, -1.746282902040115, 1.2644511896284585,
                      -0.7586432236672516, -1.2602236517597354, -0.861636910493905}));
    in.push_back(vec({-0.4532469812019473, -1.6901608867535085, -1.676126903631042,
                      1.4676310219404995, -0.02718374543101465, -1.0251692135856851}));
    in.push_back(vec({1.247027127420412, 0.8302750132245422, -1.4892671475422357,
                      1.808391263414844, 1.8002180507247614, -1.8361414984061626}));
    std::vector<double> expected = {0.6407665614421374,  0.2341246843929632,
                                    -0.2692958789369442, 0.5030265368390806,
                                    0.38438617277602594, -0.5500346991524016};
    auto got = average(in).to_host();
    for (size_t i = 0; i < expected.size(); ++i) CHECK(got[i] == expected[i]);
    std::vector<DeviceVector> withinf;
    withinf.push_back(vec({1.0, INFINITY}));
    withinf.push_back(vec({1.0, 2.0}));
    CHECK(throws<numeric_error>([&] { average(withinf); }));
    std::printf("ok average\n");
  }
  {  // clip_elementwise clamps to the band and rejects non-finite input
    auto c = clip_elementwise(vec({-3.0, -0.5, 0.0, 0.25, 7.0}), 0.5).to_host();
    CHECK(c[0] == -0.5 && c[1] == -0.5 && c[2] == 0.0 && c[3] == 0.25 && c[4] == 0.5);
    CHECK(throws<validation_error>([&] { clip_elementwise(vec({1.0}), 0.0); }));
    CHECK(throws<numeric_error>([&] { clip_elementwise(vec({NAN}), 1.0); }));
    std::printf("ok clip\n");
  }
  {  // ensure_finite names the failing context (test_param_ops.cpp:162-170)
    ensure_finite(vec({1.0, 2.0}), "outer momentum");
    bool named = false;
    try {
      ensure_finite(vec({1.0, NAN}), "outer momentum");
    } catch (const numeric_error& e) {
      named = std::string(e.what()).find("outer momentum") != std::string::npos;
    }
    CHECK(named);
    std::printf("ok ensure_finite\n");
  }
  {  // elementwise_abs_diff / l2_norm (test_param_ops.cpp:147-160)
    auto d = elementwise_abs_diff(vec({1.0, -2.0, 3.5}), vec({2.5, -2.0, -1.0})).to_host();
    CHECK(d[0] == 1.5 && d[1] == 0.0 && d[2] == 4.5);
    CHECK(throws<validation_error>([&] { elementwise_abs_diff(vec({1.0}), vec({1.0, 2.0})); }));
    CHECK(throws<numeric_error>([&] { elementwise_abs_diff(vec({INFINITY}), vec({1.0})); }));
    CHECK(l2_norm(vec({3.0, 4.0})) == 5.0);
    CHECK(l2_norm(vec({0.0, 0.0, 0.0})) == 0.0);
    CHECK(throws<numeric_error>([&] { l2_norm(vec({1e300, 1e300})); }));
    std::printf("ok elementwise_abs_diff / l2_norm\n");
  }
  {  // overlap ratio (timing_model.cpp:36-43 via the ABI)
    CHECK(overlap_ratio(2, 0.25, 1.0) == 0.5);
    CHECK(overlap_ratio(8, 0.25, 1.0) == 1.0);
    CHECK(throws<validation_error>([&] { overlap_ratio(0, 0.1, 1.0); }));
    std::printf("ok overlap_ratio\n");
  }
  {  // fused step and the global-norm clip extension (fp64, 3 coordinates)
    Context& ctx = Context::get();
    Co2Hyper h;
    h.phi = 0.1;
    auto x = vec({1.0, 2.0, 3.0}), p0 = vec({0.5, 2.5, 2.0}), p1 = vec({0.6, 2.4, 2.2});
    auto xb = vec({0.2, 2.9, 1.5});
    auto m1 = vec({0.0, 0.0, 0.0}), m2 = vec({0.0, 0.0, 0.0});
    DeviceVector a1(3, CO2_DTYPE_F64), a2(3, CO2_DTYPE_F64);
    OuterStepBuffers b{x.data(), p0.data(), p1.data(), xb.data(), m1.data(), a1.data(),
                       nullptr, nullptr};
    outer_step(CO2_MODE_F64, 3, b, 1, h, 1, ctx.ws, ctx.stream);
    finish_step(ctx.ws, ctx.stream);
    b.momentum = m2.data();
    b.anchor_out = a2.data();
    const double norm = outer_step_global_clip(CO2_MODE_F64, 3, b, 1, h, 1, ctx.ws, ctx.stream);
    co2_diag_t d = finish_step(ctx.ws, ctx.stream);
    auto mv = m2.to_host(), xg = a2.to_host(), xc = a1.to_host();
    CHECK(mv == m1.to_host());  // m' does not depend on the clip
    const double nn = std::sqrt(mv[0] * mv[0] + mv[1] * mv[1] + mv[2] * mv[2]);
    CHECK(std::fabs(norm - nn) <= 1e-15 * nn);
    CHECK(norm > 0.1 && d.n_clipped == 3);
    for (int j = 0; j < 3; ++j) {
      const double xs[3] = {1.0, 2.0, 3.0};
      CHECK(xg[j] == xs[j] - 1.0 * (mv[j] * (0.1 / norm)));
      CHECK(xc[j] == xs[j] - std::fmin(std::fmax(mv[j], -0.1), 0.1));
    }
    std::printf("ok outer_step / outer_step_global_clip\n");
  }
  std::printf(g_fail ? "FACADE FAILED %d\n" : "FACADE OK\n", g_fail);
  return g_fail ? 1 : 0;
}
