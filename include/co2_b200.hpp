// co2_b200.hpp -- header-only C++ facade over the C ABI (co2_b200.h).
//
// Re-exposes the reference's C++ operator API (namespace co2sim in
// /root/reference/proj/include/co2sim/) with the same names, argument order
// and exception types, replacing `ParamVector` (an owning fp64 Eigen vector)
// by `DeviceVector`, an owning device buffer of fp64 / fp32 / bf16:
//
//   validation_error, numeric_error   errors.hpp:8-20
//   Co2Hyper::validate                outer_algorithms.hpp:17-30
//   staleness_gap                     outer_algorithms.hpp:37-38
//   penalized_momentum_update         outer_algorithms.hpp:43-46
//   outer_iterate                     outer_algorithms.hpp:49-50
//   average, clip_elementwise         param_ops.hpp:16-24
//   allreduce_time, overlap_ratio     timing_model.hpp:27-35
//
// Value semantics as in the reference: inputs by const&, each op returns a
// fresh DeviceVector.  Ops run on the facade's stream and synchronize before
// returning so numeric errors surface as exceptions, exactly where the
// reference throws.  The fused co2::outer_step is the production entry.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "co2_b200.h"

namespace co2b200 {

class validation_error : public std::runtime_error {
 public:
  explicit validation_error(const std::string& w) : std::runtime_error(w) {}
};
class numeric_error : public std::runtime_error {
 public:
  explicit numeric_error(const std::string& w) : std::runtime_error(w) {}
};
class device_error : public std::runtime_error {
 public:
  explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(co2_status_t s) {
  if (s == CO2_OK) return;
  std::string msg = co2_last_error();
  if (s == CO2_ERR_VALIDATION) throw validation_error(msg);
  if (s == CO2_ERR_NUMERIC) throw numeric_error(msg);
  throw device_error(msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw device_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline size_t dtype_size(co2_dtype_t d) {
  return d == CO2_DTYPE_F64 ? 8 : (d == CO2_DTYPE_F32 ? 4 : 2);
}

// Owning flat device buffer: the ParamVector stand-in.
class DeviceVector {
 public:
  DeviceVector() = default;
  DeviceVector(int64_t n, co2_dtype_t dt) : n_(n), dt_(dt) {
    cuda_check(cudaMalloc(&p_, bytes() ? bytes() : 16), "cudaMalloc");
  }
  static DeviceVector from_host(const std::vector<double>& v) {
    DeviceVector d((int64_t)v.size(), CO2_DTYPE_F64);
    cuda_check(cudaMemcpy(d.p_, v.data(), d.bytes(), cudaMemcpyHostToDevice), "H2D");
    return d;
  }
  std::vector<double> to_host() const {  // fp64 vectors only
    if (dt_ != CO2_DTYPE_F64) throw validation_error("to_host: fp64 vectors only");
    std::vector<double> v((size_t)n_);
    cuda_check(cudaMemcpy(v.data(), p_, bytes(), cudaMemcpyDeviceToHost), "D2H");
    return v;
  }
  DeviceVector(const DeviceVector& o) : DeviceVector(o.n_, o.dt_) {
    cuda_check(cudaMemcpy(p_, o.p_, bytes(), cudaMemcpyDeviceToDevice), "D2D");
  }
  DeviceVector(DeviceVector&& o) noexcept
      : p_(std::exchange(o.p_, nullptr)), n_(o.n_), dt_(o.dt_) {}
  DeviceVector& operator=(DeviceVector o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(dt_, o.dt_);
    return *this;
  }
  ~DeviceVector() {
    if (p_) cudaFree(p_);
  }
  int64_t size() const { return n_; }
  co2_dtype_t dtype() const { return dt_; }
  size_t bytes() const { return (size_t)n_ * dtype_size(dt_); }
  void* data() { return p_; }
  const void* data() const { return p_; }

 private:
  void* p_ = nullptr;
  int64_t n_ = 0;
  co2_dtype_t dt_ = CO2_DTYPE_F64;
};

// Shared per-thread workspace + default stream for the synchronous ops.
struct Context {
  void* ws = nullptr;
  cudaStream_t stream = nullptr;
  Context() {
    cuda_check(cudaMalloc(&ws, co2_workspace_bytes()), "cudaMalloc(ws)");
    check(co2_workspace_init(ws, nullptr));
    cuda_check(cudaDeviceSynchronize(), "sync");
  }
  ~Context() {
    if (ws) cudaFree(ws);
  }
  static Context& get() {
    static thread_local Context c;
    return c;
  }
  void finish() {
    co2_diag_t d;
    check(co2_diag_fetch(ws, &d, stream));
  }
};

struct Co2Hyper {
  double alpha = 1.0;
  double beta = 0.7;
  double phi = 1.0;
  double epsilon = 1e-12;
  bool penalty = true;
  bool clip = true;
  bool ghost_consistent = false;

  co2_hyper_t c(int tau = 1) const {
    co2_hyper_t h{alpha, beta, phi, epsilon, tau, (uint8_t)penalty, (uint8_t)clip,
                  (uint8_t)ghost_consistent, 0};
    return h;
  }
  void validate() const {
    co2_hyper_t h = c();
    check(co2_hyper_validate(&h));
  }
};

inline void same_size(const DeviceVector& a, const DeviceVector& b, const char* msg) {
  if (a.size() != b.size() || a.dtype() != b.dtype()) throw validation_error(msg);
}

inline DeviceVector staleness_gap(const DeviceVector& x_t0, const DeviceVector& prev_x0,
                                  const DeviceVector& prev_x1, int tau, double epsilon) {
  if (tau < 1) throw validation_error("staleness_gap: tau must be >= 1");
  if (!(epsilon > 0.0)) throw validation_error("staleness_gap: epsilon must be positive");
  same_size(x_t0, prev_x0, "staleness_gap: dimensions differ");
  same_size(prev_x0, prev_x1, "staleness_gap: dimensions differ");
  Context& c = Context::get();
  DeviceVector gap(x_t0.size(), x_t0.dtype());
  check(co2_staleness_gap(x_t0.dtype(), x_t0.size(), x_t0.data(), prev_x0.data(), prev_x1.data(),
                          tau, epsilon, gap.data(), c.ws, c.stream));
  c.finish();
  return gap;
}

inline DeviceVector penalized_momentum_update(const DeviceVector& m_prev, double beta,
                                              const DeviceVector& gap, const DeviceVector& delta,
                                              bool penalty_enabled) {
  if (beta < 0.0 || beta >= 1.0)
    throw validation_error("momentum update: beta must lie in [0, 1)");
  same_size(m_prev, delta, "momentum update: dimensions differ");
  if (penalty_enabled) same_size(gap, delta, "momentum update: gap dimension differs");
  Context& c = Context::get();
  DeviceVector m(m_prev.size(), m_prev.dtype());
  check(co2_penalized_momentum(m_prev.dtype(), m_prev.size(), m_prev.data(), beta,
                               penalty_enabled ? gap.data() : delta.data(), delta.data(),
                               penalty_enabled, m.data(), c.ws, c.stream));
  c.finish();
  return m;
}

inline DeviceVector outer_iterate(const DeviceVector& x_t0, double alpha, const DeviceVector& m,
                                  double phi, bool clip_enabled) {
  if (!(alpha > 0.0)) throw validation_error("outer_iterate: alpha must be positive");
  same_size(x_t0, m, "outer_iterate: dimensions differ");
  Context& c = Context::get();
  DeviceVector x(x_t0.size(), x_t0.dtype());
  check(co2_outer_iterate(x_t0.dtype(), x_t0.size(), x_t0.data(), alpha, m.data(), phi,
                          clip_enabled, x.data(), c.ws, c.stream));
  c.finish();
  return x;
}

inline DeviceVector clip_elementwise(const DeviceVector& v, double phi) {
  Context& c = Context::get();
  DeviceVector out(v.size(), v.dtype());
  check(co2_clip_elementwise(v.dtype(), v.size(), v.data(), phi, out.data(), c.ws, c.stream));
  c.finish();
  return out;
}

inline DeviceVector average(const std::vector<DeviceVector>& contributions) {
  if (contributions.empty()) throw validation_error("average: empty contribution list");
  for (const DeviceVector& v : contributions)
    same_size(v, contributions.front(), "average: contribution dimensions differ");
  Context& c = Context::get();
  std::vector<const void*> ptrs;
  for (const DeviceVector& v : contributions) ptrs.push_back(v.data());
  DeviceVector out(contributions.front().size(), contributions.front().dtype());
  check(co2_average(out.dtype(), (int32_t)ptrs.size(), ptrs.data(), out.size(), out.data(), c.ws,
                    c.stream));
  c.finish();
  return out;
}

// ensure_finite (param_ops.hpp:14): numeric_error "non-finite value in " +
// context.
inline void ensure_finite(const DeviceVector& v, const std::string& context) {
  Context& c = Context::get();
  check(co2_ensure_finite(v.dtype(), v.size(), v.data(), context.c_str(), c.ws, c.stream));
}

// elementwise_abs_diff / l2_norm (param_ops.hpp:26-30).
inline DeviceVector elementwise_abs_diff(const DeviceVector& a, const DeviceVector& b) {
  if (a.size() != b.size() || a.dtype() != b.dtype())
    throw validation_error("elementwise_abs_diff: dimensions differ");
  Context& c = Context::get();
  DeviceVector out(a.size(), a.dtype());
  check(co2_elementwise_abs_diff(a.dtype(), a.size(), a.data(), b.data(), out.data(), c.ws,
                                 c.stream));
  return out;
}

inline double l2_norm(const DeviceVector& v) {
  Context& c = Context::get();
  double r = 0.0;
  check(co2_l2_norm(v.dtype(), v.size(), v.data(), &r, c.ws, c.stream));
  return r;
}

inline double overlap_ratio(int tau, double t_comp, double t_comm) {
  double r = 0.0;
  check(co2_overlap_ratio(tau, t_comp, t_comm, &r));
  return r;
}

// Fused production entry: one HBM pass for the whole per-worker body
// (outer_algorithms.cpp:186-196), asynchronous on `stream`; the returned
// status is checked after the caller synchronizes via finish_step().
struct OuterStepBuffers {
  const void* x_t0;
  const void* prev_x0;
  const void* prev_x1;
  const void* xbar;
  void* momentum;
  void* anchor_out;
  void* params_out;
  void* gap_out;
};

inline void outer_step(co2_mode_t mode, int64_t n, const OuterStepBuffers& b, int xbar_divisor,
                       const Co2Hyper& hyper, int tau, void* workspace, cudaStream_t stream) {
  co2_hyper_t h = hyper.c(tau);
  check(co2_outer_step(mode, n, b.x_t0, b.prev_x0, b.prev_x1, b.xbar, xbar_divisor, b.momentum,
                       b.anchor_out, b.params_out, b.gap_out, &h, workspace, stream));
}

inline co2_diag_t finish_step(void* workspace, cudaStream_t stream) {
  co2_diag_t d;
  check(co2_diag_fetch(workspace, &d, stream));
  return d;
}

// EXTENSION, not a reference API: the same step with a global-norm clip of
// m' (co2_outer_step_global_clip).  Returns ||m'||_2 after synchronizing;
// finish_step() then reports the diagnostics.
inline double outer_step_global_clip(co2_mode_t mode, int64_t n, const OuterStepBuffers& b,
                                     int xbar_divisor, const Co2Hyper& hyper, int tau,
                                     void* workspace, cudaStream_t stream) {
  co2_hyper_t h = hyper.c(tau);
  check(co2_outer_step_global_clip(mode, n, b.x_t0, b.prev_x0, b.prev_x1, b.xbar, xbar_divisor,
                                   b.momentum, b.anchor_out, b.params_out, b.gap_out, &h,
                                   workspace, stream));
  double norm = 0.0;
  check(co2_global_clip_norm_fetch(workspace, &norm, stream));
  return norm;
}

}  // namespace co2b200
