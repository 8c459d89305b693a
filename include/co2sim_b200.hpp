// co2sim_b200.hpp -- drop-in for the reference's round-level C++ API.
//
// Namespace co2sim with the reference's names and signatures for the CO2
// round path, over device buffers (header-only, on top of co2_b200.hpp and
// the C ABI):
//
//   Clock                      proj/include/co2sim/collective.hpp:18-22
//   ReduceEvent                collective.hpp:24-29
//   CollectiveEngine           collective.hpp:31-93 (launch_all_reduce,
//                              is_completed, wait, info, events, total_stall,
//                              reduce_time, live_handles, handle_count)
//   ClusterSpec                proj/include/co2sim/timing_model.hpp:14-25
//   WorkerState, InnerTrace    proj/include/co2sim/inner_loop.hpp:40-61
//   OuterState, RoundResult    proj/include/co2sim/outer_algorithms.hpp:52-69
//   co2_round                  outer_algorithms.hpp:77-81
//   staleness_gap, penalized_momentum_update, outer_iterate, average,
//   clip_elementwise, ensure_finite, Co2Hyper, validation_error,
//   numeric_error              re-exported from co2_b200.hpp
//
// ParamVector is co2b200::DeviceVector: an owning flat device buffer (fp64
// reproduces the reference bit for bit; fp32 is the same-op-order fp32
// restatement).  Value semantics as in the reference: every call returns
// after its device work finished, errors surface as the reference's
// exceptions with its messages, and co2_round's per-worker body is ONE fused
// kernel (co2_outer_step) instead of the reference's unfused passes.
//
// Time: the reference's Clock is simulated.  Here launch / completion times
// are the device's (seconds since the engine was created), is_completed is
// a non-blocking event query, and wait() advances the caller's Clock by the
// MEASURED stall (device time the consumer spent waiting on the reduce).
//
// Transports: the ClusterSpec constructor gives the LOCAL engine (all
// spec.workers simulated workers on this GPU, the fixed-order average
// kernel); CollectiveEngine::nccl gives one rank per GPU over NCCL (the
// fixed-order slice-exchange algorithm by default).  The overlapped
// production path with ping-pong device state is co2_round over
// co2_worker_t (co2_b200.h); this facade is the drop-in for code written
// against the reference's value-semantics API.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <limits>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "co2_b200.hpp"

namespace co2sim {

using co2b200::Co2Hyper;
using co2b200::numeric_error;
using co2b200::validation_error;
using ParamVector = co2b200::DeviceVector;
using co2b200::average;
using co2b200::clip_elementwise;
using co2b200::ensure_finite;
using co2b200::outer_iterate;
using co2b200::penalized_momentum_update;
using co2b200::staleness_gap;

namespace detail {
inline void check(co2_status_t s) { co2b200::check(s); }
inline cudaStream_t stream() { return co2b200::Context::get().stream; }
inline void sync() { co2b200::cuda_check(cudaStreamSynchronize(stream()), "sync"); }
inline void copy(ParamVector& dst, const ParamVector& src) {
  if (dst.size() != src.size() || dst.dtype() != src.dtype()) dst = ParamVector(src.size(), src.dtype());
  if (src.bytes())
    co2b200::cuda_check(cudaMemcpyAsync(dst.data(), src.data(), src.bytes(),
                                        cudaMemcpyDeviceToDevice, stream()),
                        "D2D");
}
inline ParamVector filled(int64_t n, co2_dtype_t dt, double v) {
  ParamVector out(n, dt);
  std::vector<double> h((size_t)n, v);
  ParamVector tmp = ParamVector::from_host(h);
  if (dt == CO2_DTYPE_F64) return tmp;
  check(co2_convert(dt, out.data(), CO2_DTYPE_F64, tmp.data(), n, stream()));
  sync();
  return out;
}
}  // namespace detail

// Simulated-time clock of the reference (collective.cpp:20-25): advancing
// is the only mutation and never goes backwards.
struct Clock {
  double now = 0.0;
  void advance(double dt) {
    if (!(dt >= 0.0) || dt == std::numeric_limits<double>::infinity())
      throw validation_error("clock: advance must be non-negative and finite");
    now += dt;
  }
};

struct ReduceEvent {
  std::string event;  // "launch" | "complete" | "wait"
  std::uint64_t handle_id = 0;
  double t_sim = 0.0;
  double stall = 0.0;
};

struct ClusterSpec {
  int workers = 1;
  int gpus_per_node = 8;
  double t_comp = 0.0;
  double t_outer = 0.0;
  double param_bytes = 0.0;
  double inter_bandwidth = 1.0;
  double latency = 0.0;
  std::optional<double> measured_override;

  co2_cluster_t c() const {
    co2_cluster_t s{workers, gpus_per_node, t_comp, t_outer, param_bytes, inter_bandwidth,
                    latency, measured_override ? 1 : 0,
                    measured_override ? *measured_override : 0.0};
    return s;
  }
  void validate() const {
    co2_cluster_t s = c();
    double t = 0.0;
    detail::check(co2_allreduce_time(&s, &t));
  }
};

inline double allreduce_time(const ClusterSpec& spec) {
  co2_cluster_t s = spec.c();
  double t = 0.0;
  detail::check(co2_allreduce_time(&s, &t));
  return t;
}

enum class CommMode { simulated, threaded };

class CollectiveEngine {
 public:
  struct HandleInfo {
    double launch_time = 0.0;
    double completion_time = 0.0;
    int contributions = 0;
    bool consumed = false;
    bool polled = false;
    bool last_poll = false;
    bool completion_logged = false;
    double stall = 0.0;
  };

  // LOCAL transport: spec.workers simulated workers on this GPU.  Both
  // CommModes produce the same fixed-order average (the reference's
  // threaded mode only moves its arithmetic off the caller, collective.hpp:
  // 31-37); here the reduce always runs on the engine's own stream.
  explicit CollectiveEngine(const ClusterSpec& spec, CommMode mode = CommMode::simulated)
      : workers_(spec.workers), mode_(mode), comm_model_(allreduce_time(spec)) {
    detail::check(co2_aar_create_local(&e_, spec.workers));
  }

  // One rank per GPU over NCCL (ids from unique_id() on rank 0, shared by
  // the caller's own bootstrap).  contributions = this rank's single buffer.
  static CollectiveEngine nccl(const uint8_t id[CO2_NCCL_ID_BYTES], int rank, int world,
                               int algo = CO2_NCCL_FIXED_ORDER) {
    CollectiveEngine ce;
    ce.workers_ = world;
    ce.per_rank_ = true;
    detail::check(co2_aar_create_nccl(&ce.e_, id, rank, world, 0));
    detail::check(co2_aar_set_nccl_algo(ce.e_, algo));
    return ce;
  }
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(CO2_NCCL_ID_BYTES);
    detail::check(co2_nccl_unique_id(id.data()));
    return id;
  }

  CollectiveEngine(CollectiveEngine&& o) noexcept { *this = std::move(o); }
  CollectiveEngine& operator=(CollectiveEngine&& o) noexcept {
    std::swap(e_, o.e_);
    workers_ = o.workers_;
    per_rank_ = o.per_rank_;
    mode_ = o.mode_;
    comm_model_ = o.comm_model_;
    results_.swap(o.results_);
    return *this;
  }
  CollectiveEngine(const CollectiveEngine&) = delete;
  CollectiveEngine& operator=(const CollectiveEngine&) = delete;
  ~CollectiveEngine() {
    if (e_) co2_aar_destroy(e_);
  }

  // launch_all_reduce (collective.cpp:31-58).  The contributions may be
  // overwritten as soon as this returns (the reference snapshots them): the
  // facade stream's later work is ordered after the reduce.
  std::uint64_t launch_all_reduce(const std::vector<ParamVector>& contributions, Clock& clock) {
    (void)clock;
    const int expect = per_rank_ ? 1 : workers_;
    if ((int)contributions.size() != expect)
      throw validation_error("launch_all_reduce: contribution count " +
                             std::to_string(contributions.size()) +
                             " does not match worker count " + std::to_string(expect));
    for (const ParamVector& c : contributions)
      if (c.size() != contributions.front().size() || c.dtype() != contributions.front().dtype())
        throw validation_error("average: contribution dimensions differ");
    const ParamVector& c0 = contributions.front();
    ParamVector result(c0.size(), c0.dtype());
    std::vector<const void*> ptrs;
    if (per_rank_) {  // in-place transport: reduce a snapshot copy
      detail::copy(result, c0);
      ptrs.push_back(result.data());
    } else {
      for (const ParamVector& c : contributions) ptrs.push_back(c.data());
    }
    std::uint64_t h = 0;
    detail::check(co2_aar_launch(e_, c0.dtype(), ptrs.data(), result.data(), c0.size(),
                                 detail::stream(), &h));
    if (!per_rank_) detail::check(co2_aar_order_after(e_, h, detail::stream()));
    results_.emplace(h, std::move(result));
    return h;
  }

  // is_completed (collective.cpp:73-86): never blocks.
  bool is_completed(std::uint64_t handle, const Clock& clock) {
    (void)clock;
    int32_t d = 0;
    detail::check(co2_aar_poll(e_, handle, &d));
    return d != 0;
  }

  // wait (collective.cpp:88-105): consumes the handle, advances the clock by
  // the measured stall and returns the average.
  ParamVector wait(std::uint64_t handle, Clock& clock) {
    detail::check(co2_aar_wait(e_, handle, detail::stream()));
    detail::sync();
    double stall = 0.0;
    detail::check(co2_aar_stall(e_, handle, &stall, nullptr));  // also the reduce's flags
    clock.advance(stall);
    auto it = results_.find(handle);
    ParamVector out = std::move(it->second);
    results_.erase(it);
    return out;
  }

  double reduce_time() const { return comm_model_; }  // the modelled cost (timing_model)
  double total_stall() const {
    double s = 0.0;
    detail::check(co2_aar_totals(e_, &s, nullptr));
    return s;
  }
  std::size_t live_handles() const {
    int32_t v = 0;
    detail::check(co2_aar_live(e_, &v));
    return (std::size_t)v;
  }
  std::size_t handle_count() const {
    uint64_t c = 0;
    detail::check(co2_aar_totals(e_, nullptr, &c));
    return (std::size_t)c;
  }
  HandleInfo info(std::uint64_t handle) const {
    co2_handle_info_t r{};
    detail::check(co2_aar_info(e_, handle, &r));
    HandleInfo h;
    h.launch_time = r.launch_time;
    h.completion_time = r.completion_time;
    h.contributions = r.contributions;
    h.consumed = r.consumed != 0;
    h.polled = r.polled != 0;
    h.last_poll = r.last_poll != 0;
    h.completion_logged = r.completion_logged != 0;
    h.stall = r.consumed ? r.stall : 0.0;
    return h;
  }
  std::vector<ReduceEvent> events() const {
    int64_t cnt = 0;
    detail::check(co2_aar_events(e_, nullptr, 0, &cnt));
    std::vector<co2_event_t> raw((size_t)(cnt > 0 ? cnt : 1));
    detail::check(co2_aar_events(e_, raw.data(), cnt, &cnt));
    static const char* kinds[] = {"launch", "complete", "wait"};
    std::vector<ReduceEvent> out;
    for (int64_t i = 0; i < cnt; ++i)
      out.push_back(ReduceEvent{kinds[raw[i].kind], raw[i].handle, raw[i].t, raw[i].stall});
    return out;
  }
  co2_aar_t* handle() { return e_; }

 private:
  CollectiveEngine() = default;
  co2_aar_t* e_ = nullptr;
  int workers_ = 1;
  bool per_rank_ = false;
  CommMode mode_ = CommMode::simulated;
  double comm_model_ = 0.0;
  std::map<std::uint64_t, ParamVector> results_;
};

struct WorkerState {
  int index = 0;
  ParamVector params;
};

struct InnerTrace {
  ParamVector x_start;  // x_{t,0}
  ParamVector x_first;  // x_{t,1}
  ParamVector x_end;    // x_{t,tau}
  int steps = 0;
};

struct OuterState {
  int t = 0;
  ParamVector momentum;  // zeros until the first outer update
  ParamVector gap;       // ones until first computed
  ParamVector prev_x0, prev_x1;
  ParamVector anchor;
  std::optional<std::uint64_t> pending;

  // Simulation's initial state (outer_algorithms.cpp:416-418).
  static OuterState initial(int64_t n, co2_dtype_t dt) {
    OuterState s;
    s.momentum = detail::filled(n, dt, 0.0);
    s.gap = detail::filled(n, dt, 1.0);
    return s;
  }
};

struct RoundResult {
  double stall_seconds = 0.0;
  bool outer_applied = false;
  double min_gap = std::numeric_limits<double>::infinity();
  double max_outer_step = 0.0;
  ParamVector consumed_average;  // empty when no reduce was consumed
};

namespace detail {
inline std::uint64_t shared_pending(const std::vector<OuterState>& outer) {
  // outer_algorithms.cpp:22-33
  if (!outer.front().pending) throw validation_error("outer round: no pending reduce to consume");
  const std::uint64_t h = *outer.front().pending;
  for (const OuterState& st : outer)
    if (!st.pending || *st.pending != h)
      throw validation_error("outer round: pending handles diverged");
  return h;
}

inline co2_mode_t mode_of(co2_dtype_t dt) {
  if (dt == CO2_DTYPE_F64) return CO2_MODE_F64;
  if (dt == CO2_DTYPE_F32) return CO2_MODE_F32;
  throw validation_error("co2_round: facade vectors must be fp64 or fp32 (bf16-mixed state: "
                         "use co2_worker_t)");
}

// The per-worker body (outer_algorithms.cpp:186-196) as one fused kernel:
// gap, Delta = prev_x0 - avg, penalized momentum, clipped outer iterate,
// min gap and max |x' - x_t0|.  m is updated in place; next and lam are
// written; throws the reference's first error for this worker.
inline void fused_body(const ParamVector& x_t0, const ParamVector& prev_x0,
                       const ParamVector& prev_x1, const ParamVector& avg, ParamVector& m,
                       ParamVector& next, ParamVector& lam, int tau, const Co2Hyper& hyper,
                       RoundResult& res) {
  const int64_t n = x_t0.size();
  for (const ParamVector* v : {&prev_x0, &prev_x1, &avg, (const ParamVector*)&m})
    if (v->size() != n || v->dtype() != x_t0.dtype())
      throw validation_error("staleness_gap: dimensions differ");
  if (next.size() != n || next.dtype() != x_t0.dtype()) next = ParamVector(n, x_t0.dtype());
  if (lam.size() != n || lam.dtype() != x_t0.dtype()) lam = ParamVector(n, x_t0.dtype());
  co2b200::Context& c = co2b200::Context::get();
  const co2_hyper_t h = hyper.c(tau);
  check(co2_outer_step(mode_of(x_t0.dtype()), n, x_t0.data(), prev_x0.data(), prev_x1.data(),
                       avg.data(), 1, m.data(), nullptr, next.data(), lam.data(), &h, c.ws,
                       c.stream));
  co2_diag_t d{};
  check(co2_diag_fetch(c.ws, &d, c.stream));  // throws staleness / momentum / iterate errors
  res.min_gap = d.min_gap < res.min_gap ? d.min_gap : res.min_gap;
  res.max_outer_step = d.max_outer_step > res.max_outer_step ? d.max_outer_step
                                                             : res.max_outer_step;
}
}  // namespace detail

// co2_round (outer_algorithms.hpp:77-81, outer_algorithms.cpp:110-211).
inline RoundResult co2_round(std::vector<WorkerState>& workers, std::vector<OuterState>& outer,
                             const std::vector<InnerTrace>& traces, int tau,
                             CollectiveEngine& engine, Clock& clock, const Co2Hyper& hyper) {
  hyper.validate();
  const std::size_t g = workers.size();
  if (outer.size() != g || traces.size() != g)
    throw validation_error("co2_round: workers, outer states and traces differ in count");
  RoundResult res;
  if (tau < 1) throw validation_error("staleness_gap: tau must be >= 1");

  std::vector<ParamVector> params;  // collect_params (views are copied: value semantics)
  for (WorkerState& w : workers) {
    ParamVector p;
    detail::copy(p, w.params);
    params.push_back(std::move(p));
  }
  const std::uint64_t launched = engine.launch_all_reduce(params, clock);

  if (outer.front().t == 0) {  // :123-151
    if (hyper.ghost_consistent) {
      std::vector<ParamVector> starts, firsts;
      for (const InnerTrace& tr : traces) {
        ParamVector a, b;
        detail::copy(a, tr.x_start);
        detail::copy(b, tr.x_first);
        starts.push_back(std::move(a));
        firsts.push_back(std::move(b));
      }
      ParamVector bar0 = average(starts), bar1 = average(firsts);
      for (std::size_t i = 0; i < g; ++i) {
        detail::copy(outer[i].prev_x0, bar0);
        detail::copy(outer[i].prev_x1, bar1);
      }
    } else {
      for (std::size_t i = 0; i < g; ++i) {
        detail::copy(outer[i].prev_x0, traces[i].x_start);
        detail::copy(outer[i].prev_x1, traces[i].x_first);
      }
    }
    for (std::size_t i = 0; i < g; ++i) {
      outer[i].pending = launched;
      outer[i].t = 1;
    }
    detail::sync();
    return res;
  }

  const std::uint64_t prev = detail::shared_pending(outer);  // :153-159
  engine.is_completed(prev, clock);
  ParamVector avg = engine.wait(prev, clock);
  res.stall_seconds = engine.info(prev).stall;
  detail::copy(res.consumed_average, avg);

  if (hyper.ghost_consistent) {  // :161-184
    std::vector<ParamVector> starts, firsts;
    for (const InnerTrace& tr : traces) {
      ParamVector a, b;
      detail::copy(a, tr.x_start);
      detail::copy(b, tr.x_first);
      starts.push_back(std::move(a));
      firsts.push_back(std::move(b));
    }
    ParamVector bar0 = average(starts), bar1 = average(firsts);
    ParamVector m, next, lam;
    detail::copy(m, outer.front().momentum);
    detail::fused_body(bar0, outer.front().prev_x0, outer.front().prev_x1, avg, m, next, lam, tau,
                       hyper, res);
    for (std::size_t i = 0; i < g; ++i) {
      detail::copy(outer[i].momentum, m);
      detail::copy(outer[i].gap, lam);
      detail::copy(outer[i].prev_x0, bar0);
      detail::copy(outer[i].prev_x1, bar1);
      detail::copy(workers[i].params, next);
    }
  } else {  // :185-203
    for (std::size_t i = 0; i < g; ++i) {
      ParamVector next, lam;
      detail::fused_body(traces[i].x_start, outer[i].prev_x0, outer[i].prev_x1, avg,
                         outer[i].momentum, next, lam, tau, hyper, res);
      outer[i].gap = std::move(lam);
      detail::copy(outer[i].prev_x0, traces[i].x_start);
      detail::copy(outer[i].prev_x1, traces[i].x_first);
      workers[i].params = std::move(next);
    }
  }
  for (std::size_t i = 0; i < g; ++i) {
    outer[i].pending = launched;
    outer[i].t += 1;
  }
  res.outer_applied = true;
  detail::sync();
  return res;
}

}  // namespace co2sim
