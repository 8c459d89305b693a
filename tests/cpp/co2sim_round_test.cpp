// Drop-in test of the reference-shaped round API (include/co2sim_b200.hpp):
// proj/fixtures/co2_dim1.json replayed through
//   co2sim::co2_round(std::vector<WorkerState>&, std::vector<OuterState>&,
//                     const std::vector<InnerTrace>&, int, CollectiveEngine&,
//                     Clock&, const Co2Hyper&)
// exactly as the reference's Simulation::step drives it
// (proj/src/outer_algorithms.cpp:422-512), with the reference's dim-1
// quadratic full-shard inner loop (proj/src/inner_loop.cpp:64-103,
// proj/src/problems.cpp:60-69,102-126) on the host in fp64.  The fixture's
// tolerance is 0: every value is compared with ==.  Then the engine audit
// (proj/tests/test_collective.cpp:43-207) and the ghost-consistent branch.
// Built by `make co2sim_round_test` (-ffp-contract=off); run by
// tests/test_gpu_parity.py.  Exits non-zero on the first failure.
#include <cstdio>
#include <vector>

#include "co2sim_b200.hpp"

using namespace co2sim;

static int g_fail = 0;
#define CHECK(cond)                                                 \
  do {                                                              \
    if (!(cond)) {                                                  \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);    \
      ++g_fail;                                                     \
    }                                                               \
  } while (0)

static double one(const ParamVector& v) { return v.to_host().at(0); }
static ParamVector dev(double x) { return ParamVector::from_host({x}); }

// co2_dim1 (proj/fixtures/co2_dim1.json:1-21): features all [1.0], targets
// [0, 2, 2, 4], shards [[0, 1], [2, 3]], init [0.0], tau 2, constant lr .25.
static const double kTargets[4] = {0.0, 2.0, 2.0, 4.0};
static const int kShards[2][2] = {{0, 1}, {2, 3}};

// accumulate() over the shard rows in order, then / rows (problems.cpp:60-69).
static double grad(int w, double x) {
  double g = 0.0;
  for (int r : kShards[w]) {
    const double dot = 1.0 * x;
    const double res = dot - kTargets[r];
    g = g + res * 1.0;
  }
  return g / 2.0;
}

static InnerTrace inner(int w, double& x, int tau, double lr) {
  InnerTrace tr;
  tr.x_start = dev(x);
  for (int k = 0; k < tau; ++k) {
    x = x - lr * grad(w, x);
    if (k == 0) tr.x_first = dev(x);
  }
  tr.x_end = dev(x);
  tr.steps = tau;
  return tr;
}

int main() {
  const int G = 2, tau = 2;
  const double lr = 0.25;
  Co2Hyper hyper;
  hyper.alpha = 0.5;
  hyper.beta = 0.5;
  hyper.phi = 0.125;
  hyper.epsilon = 1e-12;
  ClusterSpec spec;
  spec.workers = G;  // zero-cost comm: the fixture harness default (harness.cpp:401-403)
  {
    CollectiveEngine engine(spec);
    Clock clock;
    std::vector<WorkerState> workers(G);
    std::vector<OuterState> outer;
    std::vector<double> x(G, 0.0);
    for (int i = 0; i < G; ++i) {
      workers[i].index = i;
      workers[i].params = dev(0.0);
      outer.push_back(OuterState::initial(1, CO2_DTYPE_F64));
    }
    // round 0 (fixture "rounds"[0])
    std::vector<InnerTrace> traces;
    for (int i = 0; i < G; ++i) {
      traces.push_back(inner(i, x[i], tau, lr));
      workers[i].params = dev(x[i]);
    }
    CHECK(one(traces[0].x_first) == 0.25 && one(traces[1].x_first) == 0.75);
    CHECK(one(traces[0].x_end) == 0.4375 && one(traces[1].x_end) == 1.3125);
    RoundResult r0 = co2_round(workers, outer, traces, tau, engine, clock, hyper);
    CHECK(!r0.outer_applied && r0.consumed_average.size() == 0);
    CHECK(one(workers[0].params) == 0.4375 && one(workers[1].params) == 1.3125);
    CHECK(outer[0].t == 1 && outer[0].pending && engine.live_handles() == 1);
    // round 1 (fixture "rounds"[1])
    traces.clear();
    for (int i = 0; i < G; ++i) {
      x[i] = one(workers[i].params);
      traces.push_back(inner(i, x[i], tau, lr));
      workers[i].params = dev(x[i]);
    }
    CHECK(one(traces[0].x_first) == 0.578125 && one(traces[1].x_first) == 1.734375);
    CHECK(one(traces[0].x_end) == 0.68359375 && one(traces[1].x_end) == 2.05078125);
    const std::uint64_t consumed = *outer[0].pending;
    RoundResult r1 = co2_round(workers, outer, traces, tau, engine, clock, hyper);
    CHECK(r1.outer_applied);
    CHECK(one(r1.consumed_average) == 0.875);
    CHECK(one(workers[0].params) == 0.5 && one(workers[1].params) == 1.375);
    for (int i = 0; i < G; ++i) {
      CHECK(one(outer[i].momentum) == -0.4666666666666667);
      CHECK(one(outer[i].gap) == 1.875);
      CHECK(outer[i].t == 2);
    }
    CHECK(r1.min_gap == 1.875);
    CHECK(r1.max_outer_step == 0.125 * 0.5);  // clip active: alpha * phi
    // engine audit (collective.hpp:38-50; test_collective.cpp:43-207)
    CollectiveEngine::HandleInfo info = engine.info(consumed);
    CHECK(info.consumed && info.polled && info.contributions == G && info.completion_logged);
    CHECK(info.stall >= 0.0 && (info.stall == 0.0 || !info.last_poll || info.stall < 1e-4));
    CHECK(r1.stall_seconds == info.stall);
    CHECK(clock.now >= info.stall);
    CHECK(engine.live_handles() == 1 && engine.handle_count() == 2);
    bool threw = false;
    try {
      (void)engine.wait(consumed, clock);
    } catch (const validation_error& e) {
      threw = std::string(e.what()).find("already consumed") != std::string::npos;
    }
    CHECK(threw);
    int launches = 0, waits = 0, completes = 0;
    for (const ReduceEvent& e : engine.events()) {
      launches += e.event == "launch";
      waits += e.event == "wait";
      completes += e.event == "complete";
    }
    CHECK(launches == 2 && waits == 1 && completes == 2);
    // overlap window: a third live reduce is refused (collective.cpp:39-42)
    std::vector<ParamVector> c;
    c.push_back(dev(1.0));
    c.push_back(dev(2.0));
    (void)engine.launch_all_reduce(c, clock);
    threw = false;
    try {
      (void)engine.launch_all_reduce(c, clock);
    } catch (const validation_error& e) {
      threw = std::string(e.what()).find("overlap window exceeded") != std::string::npos;
    }
    CHECK(threw);
    // contribution count must match the cluster (collective.cpp:33-38)
    threw = false;
    try {
      std::vector<ParamVector> one_only;
      one_only.push_back(dev(1.0));
      (void)engine.launch_all_reduce(one_only, clock);
    } catch (const validation_error&) {
      threw = true;
    }
    CHECK(threw);
    std::printf("ok co2_dim1 through co2sim::co2_round (tolerance 0)\n");
  }
  {  // ghost-consistent branch: identical workers after the first update
    hyper.ghost_consistent = true;
    CollectiveEngine engine(spec);
    Clock clock;
    std::vector<WorkerState> workers(G);
    std::vector<OuterState> outer;
    std::vector<double> x(G, 0.0);
    for (int i = 0; i < G; ++i) {
      workers[i].params = dev(0.0);
      outer.push_back(OuterState::initial(1, CO2_DTYPE_F64));
    }
    for (int t = 0; t < 3; ++t) {
      std::vector<InnerTrace> traces;
      for (int i = 0; i < G; ++i) {
        x[i] = one(workers[i].params);
        traces.push_back(inner(i, x[i], tau, lr));
        workers[i].params = dev(x[i]);
      }
      RoundResult r = co2_round(workers, outer, traces, tau, engine, clock, hyper);
      CHECK(r.outer_applied == (t > 0));
      if (t > 0) {
        CHECK(one(workers[0].params) == one(workers[1].params));
        CHECK(one(outer[0].momentum) == one(outer[1].momentum));
      }
    }
    std::printf("ok ghost-consistent co2sim::co2_round\n");
  }
  {  // validation before any launch: a bad hyper throws the reference message
    Co2Hyper bad;
    bad.beta = 1.0;
    CollectiveEngine engine(spec);
    Clock clock;
    std::vector<WorkerState> workers(G);
    std::vector<OuterState> outer(G);
    std::vector<InnerTrace> traces(G);
    bool threw = false;
    try {
      (void)co2_round(workers, outer, traces, tau, engine, clock, bad);
    } catch (const validation_error&) {
      threw = true;
    }
    CHECK(threw && engine.handle_count() == 0);
    std::printf("ok hyper validated first\n");
  }
  if (g_fail) {
    std::printf("%d failure(s)\n", g_fail);
    return 1;
  }
  std::printf("co2sim round facade: all passed\n");
  return 0;
}
