// C ABI glue: error reporting, validation with the reference's messages,
// workspace / diagnostics, the fused step's entry points (device and
// host-buffer forms) and the analytic timing model.
#include <atomic>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace co2 {

static thread_local char g_err[512];

co2_status_t fail(co2_status_t code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

co2_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(CO2_ERR_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e),
              cudaGetErrorString(e), what);
}

int sm_count() {
  static std::atomic<int> cache[64];  // zero-initialised (static storage)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

}  // namespace co2

using namespace co2;

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" const char* co2_last_error(void) { return g_err; }
extern "C" int32_t co2_abi_version(void) { return CO2_ABI_VERSION; }

extern "C" co2_status_t co2_hyper_validate(const co2_hyper_t* h) {
  // Co2Hyper::validate, proj/src/outer_algorithms.cpp:37-46
  if (!h) return fail(CO2_ERR_VALIDATION, "hyper: null");
  if (!(h->alpha > 0.0)) return fail(CO2_ERR_VALIDATION, "hyper: alpha must be positive");
  if (h->beta < 0.0 || h->beta >= 1.0)
    return fail(CO2_ERR_VALIDATION, "hyper: beta must lie in [0, 1)");
  if (!(h->phi > 0.0)) return fail(CO2_ERR_VALIDATION, "hyper: phi must be positive");
  if (!(h->epsilon > 0.0)) return fail(CO2_ERR_VALIDATION, "hyper: epsilon must be positive");
  return CO2_OK;
}

extern "C" size_t co2_workspace_bytes(void) { return kWsBytes; }

extern "C" co2_status_t co2_workspace_init(void* ws, void* stream) {
  if (!ws) return fail(CO2_ERR_VALIDATION, "null workspace");
  CO2_CUDA(cudaMemsetAsync(ws, 0, kWsBytes, S(stream)));
  return CO2_OK;
}

extern "C" co2_status_t co2_diag_status(const co2_diag_t* d) {
  // Reference error precedence: staleness_gap numeric
  // (outer_algorithms.cpp:62) -> gap<1 validation (:81-83) -> momentum
  // numeric (:88) -> clip input numeric (param_ops.cpp:41) -> outer_iterate
  // numeric (outer_algorithms.cpp:106) -> average numeric (param_ops.cpp:31).
  uint32_t f = d->flags;
  if (f & CO2_FLAG_GAP_NONFINITE) return fail(CO2_ERR_NUMERIC, "non-finite value in staleness_gap");
  if (f & CO2_FLAG_GAP_BELOW_ONE)
    return fail(CO2_ERR_VALIDATION, "momentum update: gap coordinate below 1");
  if (f & CO2_FLAG_M_NONFINITE) return fail(CO2_ERR_NUMERIC, "non-finite value in momentum update");
  if (f & CO2_FLAG_NORM_NONFINITE)
    return fail(CO2_ERR_NUMERIC, "non-finite value in global clip norm");
  if (f & CO2_FLAG_CLIP_NONFINITE)
    return fail(CO2_ERR_NUMERIC, "non-finite value in clip_elementwise input");
  if (f & CO2_FLAG_X_NONFINITE) return fail(CO2_ERR_NUMERIC, "non-finite value in outer_iterate");
  if (f & CO2_FLAG_AVG_NONFINITE) return fail(CO2_ERR_NUMERIC, "non-finite value in average");
  if (f & CO2_FLAG_SLOWMO_M) return fail(CO2_ERR_NUMERIC, "non-finite value in slowmo momentum");
  if (f & CO2_FLAG_SLOWMO_X)
    return fail(CO2_ERR_NUMERIC, "non-finite value in slowmo outer iterate");
  if (f & CO2_FLAG_OVERLAP) return fail(CO2_ERR_NUMERIC, "non-finite value in overlap correction");
  if (f & CO2_FLAG_NONFINITE_INPUT) return fail(CO2_ERR_NUMERIC, "non-finite value");
  return CO2_OK;
}

extern "C" co2_status_t co2_diag_fetch_async(const void* ws, co2_diag_t* out, void* stream) {
  if (!ws || !out) return fail(CO2_ERR_VALIDATION, "null workspace or output");
  const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws);
  CO2_CUDA(cudaMemcpyAsync(out, &hdr->diag, sizeof(co2_diag_t), cudaMemcpyDeviceToHost, S(stream)));
  return CO2_OK;
}

extern "C" co2_status_t co2_diag_fetch(const void* ws, co2_diag_t* out, void* stream) {
  CO2_TRY(co2_diag_fetch_async(ws, out, stream));
  CO2_CUDA(cudaStreamSynchronize(S(stream)));
  return co2_diag_status(out);
}

static co2_status_t validate_step(co2_mode_t mode, int64_t n, const void* x_t0, const void* p0,
                                  const void* p1, const void* xbar, int32_t divisor,
                                  const void* m, const co2_hyper_t* h) {
  // co2_round validates the hyper first (outer_algorithms.cpp:115), then
  // staleness_gap its own scalars (:50-53).
  CO2_TRY(co2_hyper_validate(h));
  if (h->tau < 1) return fail(CO2_ERR_VALIDATION, "staleness_gap: tau must be >= 1");
  if (mode != CO2_MODE_F64 && mode != CO2_MODE_F32 && mode != CO2_MODE_BF16_MIXED)
    return fail(CO2_ERR_VALIDATION, "outer step: unknown mode %d", (int)mode);
  if (n < 0) return fail(CO2_ERR_VALIDATION, "staleness_gap: dimensions differ");
  if (divisor < 1) return fail(CO2_ERR_VALIDATION, "outer step: xbar divisor must be >= 1");
  if (n > 0 && (!x_t0 || !p0 || !p1 || !xbar || !m))
    return fail(CO2_ERR_VALIDATION, "outer step: null input buffer");
  return CO2_OK;
}

extern "C" co2_status_t co2_outer_step(co2_mode_t mode, int64_t n, const void* x_t0,
                                       const void* p0, const void* p1, const void* xbar,
                                       int32_t divisor, void* m, void* anchor, void* params,
                                       void* gap, const co2_hyper_t* h, void* ws, void* stream) {
  CO2_TRY(validate_step(mode, n, x_t0, p0, p1, xbar, divisor, m, h));
  if (!ws) return fail(CO2_ERR_VALIDATION, "null workspace");
  return outer_step_impl(mode, n, x_t0, p0, p1, xbar, divisor, m, anchor, params, gap, h, ws,
                         S(stream));
}

extern "C" co2_status_t co2_outer_step_global_clip(co2_mode_t mode, int64_t n, const void* x_t0,
                                                   const void* p0, const void* p1,
                                                   const void* xbar, int32_t divisor, void* m,
                                                   void* anchor, void* params, void* gap,
                                                   const co2_hyper_t* h, void* ws, void* stream) {
  CO2_TRY(validate_step(mode, n, x_t0, p0, p1, xbar, divisor, m, h));
  if (!ws) return fail(CO2_ERR_VALIDATION, "null workspace");
  return outer_step_global_clip_impl(mode, n, x_t0, p0, p1, xbar, divisor, m, anchor, params,
                                     gap, h, ws, S(stream));
}

extern "C" co2_status_t co2_global_clip_norm_fetch(const void* ws, double* out, void* stream) {
  if (!ws || !out) return fail(CO2_ERR_VALIDATION, "null workspace or output");
  const WsHeader* hdr = reinterpret_cast<const WsHeader*>(ws);
  CO2_CUDA(cudaMemcpyAsync(out, &hdr->gnorm, sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
  CO2_CUDA(cudaStreamSynchronize(S(stream)));
  return CO2_OK;
}

extern "C" int64_t co2_global_clip_chunk(co2_mode_t mode, int64_t n) {
  const int V = mode == CO2_MODE_F64 ? 2 : (mode == CO2_MODE_F32 ? 4 : 8);
  return gc_chunk(n, V);
}

// ---------------------------------------------------------------------------
// Host-buffer form: chunked H2D -> fused step -> D2H pipeline over a cached
// per-device staging pool (grown on demand, never shrunk).
namespace {

struct StageSlot {
  cudaStream_t stream = nullptr;
  void* buf = nullptr;  // x_t0 | p0 | m (state) ; p1 | xbar (low) ; params (low) ; ws
  size_t bytes = 0;
};

// One staging pool per device (streams and buffers belong to it); calls on
// the same device serialise on its mutex, calls on different devices run
// concurrently.
struct StagePool {
  std::mutex mu;
  std::vector<StageSlot> slots;
  co2_diag_t* host_diags = nullptr;  // pinned
  size_t host_diag_cap = 0;
};

constexpr int kMaxDevices = 64;

StagePool& pool(int dev) {
  static StagePool p[kMaxDevices];
  return p[dev];
}

}  // namespace

extern "C" co2_status_t co2_outer_step_host(co2_mode_t mode, int64_t n, const void* x_t0,
                                            const void* p0, const void* p1, const void* xbar,
                                            int32_t divisor, void* m, void* anchor, void* params,
                                            const co2_hyper_t* h, int64_t chunk, int32_t nstreams,
                                            co2_diag_t* diag_out) {
  CO2_TRY(validate_step(mode, n, x_t0, p0, p1, xbar, divisor, m, h));
  if (nstreams < 1) nstreams = 1;
  if (nstreams > 4) nstreams = 4;
  if (chunk <= 0) chunk = 16 << 20;
  chunk = (chunk + 7) / 8 * 8;  // keep every chunk offset 16-byte aligned
  const size_t sb = state_bytes(mode), lb = low_bytes(mode);
  const size_t per = 3 * sb + 3 * lb;  // x_t0, p0, m, p1, xbar, params
  auto align = [](size_t v) { return (v + 255) / 256 * 256; };
  const size_t need = align(3 * sb * chunk) + align(3 * lb * chunk) + kWsBytes + 1024;
  (void)per;
  int dev = 0;
  CO2_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices)
    return fail(CO2_ERR_VALIDATION, "outer_step_host: device %d out of range", dev);
  StagePool& P = pool(dev);
  std::lock_guard<std::mutex> lock(P.mu);
  while ((int)P.slots.size() < nstreams) {
    StageSlot s;
    CO2_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    P.slots.push_back(s);
  }
  for (int i = 0; i < nstreams; ++i) {
    StageSlot& s = P.slots[i];
    if (s.bytes < need) {
      if (s.buf) CO2_CUDA(cudaFree(s.buf));
      CO2_CUDA(cudaMalloc(&s.buf, need));
      s.bytes = need;
      // The workspace sits at offset 0 so its self-resetting ticket survives
      // calls with other modes / chunk sizes that reuse this buffer.
      CO2_CUDA(cudaMemsetAsync(s.buf, 0, kWsBytes, s.stream));
    }
  }
  const int64_t nchunks = n == 0 ? 0 : (n + chunk - 1) / chunk;
  if ((size_t)nchunks > P.host_diag_cap) {
    if (P.host_diags) cudaFreeHost(P.host_diags);
    size_t cap = std::max<size_t>(64, (size_t)nchunks);
    CO2_CUDA(cudaMallocHost(&P.host_diags, cap * sizeof(co2_diag_t)));
    P.host_diag_cap = cap;
  }
  auto H = [](const void* p, size_t off) { return static_cast<const char*>(p) + off; };
  auto Hm = [](void* p, size_t off) { return static_cast<char*>(p) + off; };
  for (int64_t c = 0; c < nchunks; ++c) {
    StageSlot& s = P.slots[c % nstreams];
    const int64_t j0 = c * chunk;
    const int64_t len = std::min<int64_t>(chunk, n - j0);
    void* ws = s.buf;
    char* base = static_cast<char*>(s.buf) + align(kWsBytes);
    char* dx = base;
    char* dp0 = dx + sb * chunk;
    char* dm = dp0 + sb * chunk;
    char* dp1 = base + align(3 * sb * chunk);
    char* dxb = dp1 + lb * chunk;
    char* dpr = dxb + lb * chunk;
    const size_t so = sb * j0, lo = lb * j0, sl = sb * len, ll = lb * len;
    CO2_CUDA(cudaMemcpyAsync(dx, H(x_t0, so), sl, cudaMemcpyHostToDevice, s.stream));
    CO2_CUDA(cudaMemcpyAsync(dp0, H(p0, so), sl, cudaMemcpyHostToDevice, s.stream));
    CO2_CUDA(cudaMemcpyAsync(dm, H(m, so), sl, cudaMemcpyHostToDevice, s.stream));
    CO2_CUDA(cudaMemcpyAsync(dp1, H(p1, lo), ll, cudaMemcpyHostToDevice, s.stream));
    CO2_CUDA(cudaMemcpyAsync(dxb, H(xbar, lo), ll, cudaMemcpyHostToDevice, s.stream));
    // anchor is produced in place over the staged prev_x0 (aliasing allowed).
    CO2_TRY(outer_step_impl(mode, len, dx, dp0, dp1, dxb, divisor, dm, anchor ? dp0 : nullptr,
                            params ? dpr : nullptr, nullptr, h, ws, s.stream));
    CO2_CUDA(cudaMemcpyAsync(&P.host_diags[c], &ws_header(ws)->diag, sizeof(co2_diag_t),
                             cudaMemcpyDeviceToHost, s.stream));
    CO2_CUDA(cudaMemcpyAsync(Hm(m, so), dm, sl, cudaMemcpyDeviceToHost, s.stream));
    if (anchor) CO2_CUDA(cudaMemcpyAsync(Hm(anchor, so), dp0, sl, cudaMemcpyDeviceToHost, s.stream));
    if (params) CO2_CUDA(cudaMemcpyAsync(Hm(params, lo), dpr, ll, cudaMemcpyDeviceToHost, s.stream));
  }
  for (int i = 0; i < nstreams; ++i) CO2_CUDA(cudaStreamSynchronize(P.slots[i].stream));
  co2_diag_t d{INFINITY, 0.0, 0, 0, 0u, 0u};
  for (int64_t c = 0; c < nchunks; ++c) {
    const co2_diag_t& q = P.host_diags[c];
    d.min_gap = q.min_gap < d.min_gap ? q.min_gap : d.min_gap;
    d.max_outer_step = q.max_outer_step > d.max_outer_step ? q.max_outer_step : d.max_outer_step;
    d.n_clipped += q.n_clipped;
    d.n_floored += q.n_floored;
    d.flags |= q.flags;
  }
  if (diag_out) *diag_out = d;
  return co2_diag_status(&d);
}

// ---------------------------------------------------------------------------
// Analytic timing model (proj/src/timing_model.cpp).  Host arithmetic, used to
// predict the measured schedule, not a fallback for any device work.
extern "C" co2_status_t co2_cluster_validate(const co2_cluster_t* s) {
  // ClusterSpec::validate, timing_model.cpp:10-25
  if (s->workers < 1) return fail(CO2_ERR_VALIDATION, "cluster: workers must be >= 1");
  if (s->gpus_per_node < 1) return fail(CO2_ERR_VALIDATION, "cluster: gpus_per_node must be >= 1");
  if (s->t_comp < 0.0) return fail(CO2_ERR_VALIDATION, "cluster: negative t_comp");
  if (s->t_outer < 0.0) return fail(CO2_ERR_VALIDATION, "cluster: negative t_outer");
  if (s->param_bytes < 0.0) return fail(CO2_ERR_VALIDATION, "cluster: negative param_bytes");
  if (!(s->inter_bandwidth > 0.0))
    return fail(CO2_ERR_VALIDATION, "cluster: inter_bandwidth must be positive");
  if (s->latency < 0.0) return fail(CO2_ERR_VALIDATION, "cluster: negative latency");
  if (s->has_measured_override && s->measured_override < 0.0)
    return fail(CO2_ERR_VALIDATION, "cluster: negative measured_override");
  return CO2_OK;
}

extern "C" co2_status_t co2_allreduce_time(const co2_cluster_t* s, double* out) {
  // timing_model.cpp:27-34
  CO2_TRY(co2_cluster_validate(s));
  if (s->workers < 2) {
    *out = 0.0;
    return CO2_OK;
  }
  if (s->has_measured_override) {
    *out = s->measured_override;
    return CO2_OK;
  }
  double g = (double)s->workers;
  *out = 2.0 * (g - 1.0) * s->latency + 2.0 * ((g - 1.0) / g) * s->param_bytes / s->inter_bandwidth;
  return CO2_OK;
}

extern "C" co2_status_t co2_overlap_ratio(int32_t tau, double t_comp, double t_comm, double* out) {
  // timing_model.cpp:36-43
  if (tau < 1) return fail(CO2_ERR_VALIDATION, "overlap_ratio: tau must be >= 1");
  if (t_comp < 0.0 || t_comm < 0.0) return fail(CO2_ERR_VALIDATION, "overlap_ratio: negative time");
  if (t_comm <= 0.0) {
    *out = 1.0;
    return CO2_OK;
  }
  double r = tau * t_comp / t_comm;
  *out = r < 1.0 ? r : 1.0;
  return CO2_OK;
}

extern "C" co2_status_t co2_simulate_timeline(int32_t kind, const co2_cluster_t* s, int32_t tau,
                                              int32_t rounds, int32_t batch_size,
                                              co2_timeline_t* out,
                                              co2_round_timing_t* per_round) {
  // simulate_timeline, timing_model.cpp:76-173: co2 / slowmo / local_sgd /
  // overlap_local_sgd / sync_sgd (AlgorithmKind order, algorithm_kind.hpp:9)
  CO2_TRY(co2_cluster_validate(s));
  if (kind < CO2_ALG_CO2 || kind > CO2_ALG_SYNC_SGD)
    return fail(CO2_ERR_VALIDATION, "simulate_timeline: unknown algorithm %d", (int)kind);
  if (tau < 1) return fail(CO2_ERR_VALIDATION, "simulate_timeline: tau must be >= 1");
  if (rounds < 1) return fail(CO2_ERR_VALIDATION, "simulate_timeline: rounds must be >= 1");
  if (batch_size < 1) return fail(CO2_ERR_VALIDATION, "simulate_timeline: batch_size must be >= 1");
  if (!out) return fail(CO2_ERR_VALIDATION, "simulate_timeline: null output");
  double comm = 0.0;
  CO2_TRY(co2_allreduce_time(s, &comm));
  double now = 0.0, total_stall = 0.0, waited = 0.0, pending = 0.0;
  bool has_pending = false;
  for (int t = 0; t < rounds; ++t) {
    co2_round_timing_t rt{t, now, 0.0, 0.0};
    switch (kind) {
      case CO2_ALG_CO2: {
        now += tau * s->t_comp;
        const double launched = now + comm;
        if (t == 0) {  // the first round skips the outer update
          pending = launched;
          has_pending = true;
          break;
        }
        const double stall = std::max(0.0, pending - now);
        now += stall;
        rt.stall = stall;
        total_stall += stall;
        waited += comm;
        pending = launched;
        now += s->t_outer;
        break;
      }
      case CO2_ALG_SLOWMO:
      case CO2_ALG_LOCAL_SGD:  // blocking reduce every round
        now += tau * s->t_comp;
        rt.stall = comm;
        total_stall += comm;
        waited += comm;
        now += comm;
        now += s->t_outer;
        break;
      case CO2_ALG_OVERLAP_LOCAL_SGD:
        now += tau * s->t_comp;
        if (has_pending) {
          const double stall = std::max(0.0, pending - now);
          now += stall;
          rt.stall = stall;
          total_stall += stall;
          waited += comm;
          has_pending = false;
        }
        if (comm > 0.0) {  // an instant reduce is consumed in its own round
          pending = now + comm;
          has_pending = true;
        }
        now += s->t_outer;
        break;
      default:  // CO2_ALG_SYNC_SGD: compute and reduce serialised per step
        for (int k = 0; k < tau; ++k) {
          now += s->t_comp;
          rt.stall += comm;
          total_stall += comm;
          waited += comm;
          now += comm;
        }
        break;
    }
    rt.end = now;
    if (per_round) per_round[t] = rt;
  }
  out->workers = s->workers;
  out->tau = tau;
  out->rounds = rounds;
  out->batch_size = batch_size;
  out->comm_time = comm;
  out->wall_time = now;
  out->total_stall = total_stall;
  out->overlap_ratio_achieved = waited > 0.0 ? 1.0 - total_stall / waited : 1.0;
  const double work = (double)rounds * tau * s->workers * batch_size;
  out->throughput = now > 0.0 ? work / now : 0.0;
  return CO2_OK;
}

extern "C" co2_status_t co2_simulate_timeline_co2(const co2_cluster_t* s, int32_t tau,
                                                  int32_t rounds, int32_t batch_size,
                                                  co2_timeline_t* out,
                                                  co2_round_timing_t* per_round) {
  return co2_simulate_timeline(CO2_ALG_CO2, s, tau, rounds, batch_size, out, per_round);
}

extern "C" co2_status_t co2_scalability_ratio(double throughput_small, double throughput_large,
                                              double workers_small, double workers_large,
                                              double* out) {
  // scalability_ratio, timing_model.cpp:45-53
  if (!(throughput_small > 0.0) || !(workers_small > 0.0) || !(workers_large > 0.0))
    return fail(CO2_ERR_VALIDATION, "scalability_ratio: non-positive input");
  if (!out) return fail(CO2_ERR_VALIDATION, "scalability_ratio: null output");
  *out = (throughput_large / throughput_small) / (workers_large / workers_small);
  return CO2_OK;
}
