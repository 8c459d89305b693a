// One-step-stale all-reduce engine (CollectiveEngine) and the co2_round
// driver over device-resident worker state.
//
// Reference: proj/include/co2sim/collective.hpp:54-93, proj/src/collective.cpp
// (simulated clock + std::async average) and proj/src/outer_algorithms.cpp:
// 110-211 (co2_round).  Here the "launch" is a real collective on a
// dedicated high-priority comm stream fenced by an event after the producer's
// work, "poll" is cudaEventQuery, and "wait" makes the consumer stream wait on
// the completion event -- the host never blocks on the reduce.  Stall is the
// device time between the consumer reaching the wait and the reduce finishing
// (events straddling cudaStreamWaitEvent), the measured counterpart of the
// reference's `stall = max(0, completion - now)` (collective.cpp:93).
#include <cuda.h>  // CUdeviceptr / CUresult for the driver entry point below
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <limits>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

using namespace co2;

#define CO2_NCCL(call)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (call);                                                             \
    if (_r != ncclSuccess)                                                                \
      return ::co2::fail(CO2_ERR_NCCL, "NCCL error %s in %s", ncclGetErrorString(_r), #call); \
  } while (0)

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

namespace {

enum { T_NCCL = 0, T_LOCAL = 1, T_P2P = 2 };

struct Handle {
  cudaEvent_t start = nullptr, done = nullptr, wait_begin = nullptr, wait_end = nullptr;
  // Kernel-timed handle (single-launch LOCAL round): the kernel writes its
  // own start / end %globaltimer and the average's diagnostics into the
  // engine's DEVICE slot of the handle, fetched into the pinned slot (`ts`,
  // `diag`) only when the handle is cached; completion is the non-timing
  // event `fin`.  A timing event record costs the stream ~2.5 us and the
  // mapped host writes + system fence at a kernel's end ~2.3 us
  // (profiles/r02/c1/), against a ~31 us C1 round kernel; a non-timing
  // record costs nothing measurable.
  cudaEvent_t fin = nullptr;
  bool ktimed = false;
  uint64_t* ts = nullptr;
  uint64_t* ts_dev = nullptr;
  co2_diag_t* diag_dev = nullptr;
  bool consumed = false, polled = false, last_poll = false, completion_logged = false;
  bool waited = false;
  // Stream-ordered consume (single-launch LOCAL round): the reduce completed
  // on the consumer's own stream, so the wait cannot stall and records no
  // events; its end is the start event of handle `wait_alias` (recorded at
  // the same stream position).  -1: an ordinary wait (wait_begin/wait_end).
  int64_t wait_alias = -1;
  cudaStream_t done_stream = nullptr;  // the stream `done` was recorded on
  int contributions = 0;
  co2_diag_t* diag = nullptr;  // LOCAL: pinned copy of the average's flags (pool slot)
  uint32_t* p2p_error = nullptr;  // P2P: pinned copy of the signal area's error word (pool slot)
  // After kRing newer launches a handle's events are recycled; its device
  // times and status are cached first (the reference keeps every record).
  bool cached = false, cached_wait = false;
  double c_start = 0, c_done = 0, c_wait_end = 0, c_stall = 0, c_comm = 0;
  uint32_t c_flags = 0, c_err = 0;
};

constexpr size_t kRing = 256;
constexpr int kMaxNcclRanks = 64;  // fixed-order average: co2_average's contribution cap

// A buffer registered with the P2P transport: the same logical buffer on
// every rank (rank-indexed device pointers, peers opened via CUDA IPC).
struct P2PBuffer {
  const void* local = nullptr;
  std::vector<void*> ptrs;
  std::vector<std::pair<int, std::string>> keys;  // opened peer allocations it holds
};

ncclDataType_t nccl_dtype(co2_dtype_t d) {
  return d == CO2_DTYPE_F64 ? ncclFloat64 : (d == CO2_DTYPE_F32 ? ncclFloat32 : ncclBfloat16);
}

}  // namespace

struct co2_aar {
  int transport = T_LOCAL;
  int rank = 0, world = 1, workers = 1;
  ncclComm_t comm = nullptr;
  ncclComm_t comm2 = nullptr;  // blocking collectives issued on the caller's stream
  // NCCL algorithm: false (default) = fixed-order average (send/recv slice
  // exchange + ascending-rank sum kernel + send/recv all-gather), bitwise
  // the reference's average() at any world size; true = ncclAllReduce /
  // ncclReduceScatter sums in the storage dtype (ring / tree order, rounded
  // per hop), divided by G in the consumer.
  bool nccl_sum = false;
  // staging of the slices received from peers: [0] comm stream, [1] the
  // caller's stream (sharded x_{t,1}); a second workspace for [1]'s sum kernel
  void* stage[2] = {nullptr, nullptr};
  size_t stage_bytes[2] = {0, 0};
  void* ws2 = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t epoch = nullptr;
  void* ws = nullptr;
  int live = 0;
  std::vector<Handle> handles;
  // P2P transport
  int ctas = 0;
  int slice_ctas = 0;  // sharded slice reduce; 0 = one CTA per SM
  uint32_t p2p_epoch = 0;      // ready flags of every P2P reduce launch (average and slice)
  uint32_t p2p_done = 0;       // cumulative exit-barrier target of the average kernel
  // Adaptive reduce occupancy (co2_aar_set_adaptive / CO2_P2P_ADAPT=1): the
  // P2P all-reduce's CTA count follows the measured slack of the consumed
  // reduces, between ctas_min and ctas_max; adapt_next = first handle not
  // yet used for a decision.
  bool adaptive = false;
  int ctas_min = 16, ctas_max = 148;
  size_t adapt_next = 0;
  bool fused = false;        // worker-local rounds use the fused all-reduce + step kernel
  uint32_t fused_epoch = 0;  // exit barrier (done3) of the fused all-reduce + step
  uint32_t shard_epoch = 0;  // exit barrier (done2) of the sharded P2P step: per engine,
                             // since the counter lives in the engine's signal area
  void* signals = nullptr;        // this rank's signal area (cudaMalloc, IPC-exported)
  std::vector<void*> peer_signals;  // rank-indexed (opened IPC pointers; own = signals)
  std::vector<P2PBuffer> p2p_bufs;
  // Opened peer allocations, keyed by (peer rank, IPC handle bytes) and
  // reference-counted: several registered buffers may share one allocation.
  struct Opened {
    void* base = nullptr;
    int refs = 0;
  };
  std::map<std::pair<int, std::string>, Opened> opened;
  // pinned per-launch slots (ring) and the reusable producer fence
  co2_diag_t* pin_diag = nullptr;
  co2_diag_t* pin_diag_dev = nullptr;  // device mapping of pin_diag
  uint32_t* pin_err = nullptr;
  uint64_t* pin_ts = nullptr;      // kernel-timed handles: [start, end] globaltimer ns
  uint64_t* dev_ts = nullptr;      // ... written by the kernel here (device ring)
  co2_diag_t* dev_diag = nullptr;  // ... and the average's diagnostics
  cudaStream_t aux_stream = nullptr;  // fetches of the device slots
  uint64_t epoch_ns = 0;           // %globaltimer read right after the epoch event
  cudaEvent_t fence = nullptr;
};

// Comm-stream readbacks (the P2P barrier error word, a reduce's diagnostics)
// as a one-thread kernel storing into device-mapped pinned memory, not a
// cudaMemcpyAsync: a D2H copy on the comm stream waits for the reduce in
// the copy engine's queue, and the compute stream's own D2H copies queued
// behind it then wait for the reduce too -- a stall the wait events never
// see (C3 N=4: 0.6-1.7 ms per round on some ranks, profiles/r02/tune/ce_hol/).
__global__ void co2_copy_words_kernel(const uint32_t* src, uint32_t* dst, int nwords) {
  for (int i = 0; i < nwords; ++i) dst[i] = *reinterpret_cast<const volatile uint32_t*>(src + i);
}

static co2_status_t copy_words_to_host(const void* src_dev, void* dst_host, size_t bytes,
                                       cudaStream_t st) {
  void* dst_dev = nullptr;
  CO2_CUDA(cudaHostGetDevicePointer(&dst_dev, dst_host, 0));
  co2_copy_words_kernel<<<1, 1, 0, st>>>(static_cast<const uint32_t*>(src_dev),
                                         static_cast<uint32_t*>(dst_dev), (int)(bytes / 4));
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

// A workspace's diagnostics into a pinned host slot (engine-internal: the
// slots are cudaMallocHost'd, so mapped), without the copy engine.
static co2_status_t diag_to_host(const void* ws, co2_diag_t* host, void* stream) {
  return copy_words_to_host(&ws_header(const_cast<void*>(ws))->diag, host, sizeof(co2_diag_t),
                            S(stream));
}

__global__ void co2_globaltimer_kernel(uint64_t* out) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

static co2_status_t engine_common_init(co2_aar* e) {
  int lo = 0, hi = 0;
  CO2_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // The comm stream runs at the highest priority so the reduce's CTAs are
  // scheduled ahead of queued step CTAs.  CO2_COMM_PRIORITY=low inverts it:
  // the reduce then starves behind the 32-wave step grid and 28-37 % of it
  // is exposed (profiles/r01/bench/comm_priority.txt).
  const char* pr = getenv("CO2_COMM_PRIORITY");
  const int prio = (pr && strcmp(pr, "low") == 0) ? lo : hi;
  CO2_CUDA(cudaStreamCreateWithPriority(&e->comm_stream, cudaStreamNonBlocking, prio));
  CO2_CUDA(cudaEventCreate(&e->epoch));
  CO2_CUDA(cudaEventRecord(e->epoch, e->comm_stream));
  {  // the epoch on the %globaltimer clock, for kernel-timed handles
    uint64_t* d = nullptr;
    CO2_CUDA(cudaMalloc(&d, sizeof(uint64_t)));
    co2_globaltimer_kernel<<<1, 1, 0, e->comm_stream>>>(d);
    cudaError_t ce = cudaMemcpyAsync(&e->epoch_ns, d, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                     e->comm_stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->comm_stream);
    cudaFree(d);
    if (ce != cudaSuccess) return cuda_fail(ce, "epoch globaltimer");
  }
  CO2_CUDA(cudaMalloc(&e->ws, co2_workspace_bytes()));
  CO2_CUDA(cudaMemsetAsync(e->ws, 0, co2_workspace_bytes(), e->comm_stream));
  return CO2_OK;
}

extern "C" co2_status_t co2_nccl_unique_id(uint8_t id_out[CO2_NCCL_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == CO2_NCCL_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  CO2_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof id);
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_create_nccl(co2_aar_t** out, const uint8_t id[CO2_NCCL_ID_BYTES],
                                            int32_t rank, int32_t world, int32_t max_ctas) {
  if (!out) return fail(CO2_ERR_VALIDATION, "aar: null output handle");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(CO2_ERR_VALIDATION, "aar: bad rank %d / world %d", rank, world);
  co2_aar* e = new co2_aar();
  e->transport = T_NCCL;
  e->rank = rank;
  e->world = world;
  e->workers = world;
  e->nccl_sum = world > kMaxNcclRanks;  // beyond the average kernel's fan-in
  co2_status_t s = engine_common_init(e);
  if (s != CO2_OK) {
    delete e;
    return s;
  }
  if (world > 1) {
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (max_ctas > 0) cfg.maxCTAs = max_ctas;
    ncclResult_t r = ncclCommInitRankConfig(&e->comm, world, uid, rank, &cfg);
    if (r != ncclSuccess) {
      delete e;
      return fail(CO2_ERR_NCCL, "NCCL error %s in ncclCommInitRankConfig", ncclGetErrorString(r));
    }
  }
  *out = e;
  return CO2_OK;
}

// Base of the allocation containing p (driver cuMemGetAddressRange, reached
// through the runtime's entry-point query so the library needs no -lcuda).
static co2_status_t alloc_base(const void* p, char** base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CO2_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      return fail(CO2_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    fn = reinterpret_cast<Fn>(f);
  }
  CUdeviceptr b = 0;
  size_t size = 0;
  if (fn(&b, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    return fail(CO2_ERR_VALIDATION, "ipc export: not a device allocation");
  *base = reinterpret_cast<char*>(b);
  return CO2_OK;
}

extern "C" co2_status_t co2_ipc_export(const void* dev_ptr, uint8_t handle_out[CO2_IPC_HANDLE_BYTES]) {
  static_assert(sizeof(cudaIpcMemHandle_t) + sizeof(int64_t) == CO2_IPC_HANDLE_BYTES,
                "IPC handle size");
  if (!dev_ptr) return fail(CO2_ERR_VALIDATION, "ipc export: null pointer");
  char* base = nullptr;
  CO2_TRY(alloc_base(dev_ptr, &base));
  cudaIpcMemHandle_t h;
  CO2_CUDA(cudaIpcGetMemHandle(&h, base));
  const int64_t off = static_cast<const char*>(dev_ptr) - base;
  memcpy(handle_out, &h, sizeof h);
  memcpy(handle_out + sizeof h, &off, sizeof off);
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_create_p2p(co2_aar_t** out, int32_t rank, int32_t world,
                                           int32_t ctas) {
  if (!out) return fail(CO2_ERR_VALIDATION, "aar: null output handle");
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    return fail(CO2_ERR_VALIDATION, "aar: bad rank %d / world %d (p2p supports <= 8)", rank,
                world);
  co2_aar* e = new co2_aar();
  e->transport = T_P2P;
  e->rank = rank;
  e->world = world;
  e->workers = world;
  // 96 CTAs of 256 threads while the reduce shares HBM and SMs with the
  // 32-wave fused outer step (bench.py --max-ctas sweeps): fewer starve the
  // reduce, more steal SM slots from the step.  With the 64-register reduce
  // kernel, C3 N=4 at 64 CTAs leaves 27 % of the reduce exposed (5.68e11
  // params/s) against 2.3 % at 96 (7.10e11); N=2 is best at 96.  At N=4 the
  // reduce is about as long as the step it hides behind: 96 CTAs left
  // 0.05-12 % of it exposed from box to box, 128 / 148 measure the same
  // params/s and stayed at 0.05 % (profiles/r02/tune/c3_p2p_ctas_r6/,
  // profiles/r02/final*/), so from 4 ranks on it gets 128 (8 ranks,
  // unmeasured here, move 7/8 of the replica per rank instead of 3/4).
  e->ctas = ctas > 0 ? ctas : (world <= 2 ? 96 : 128);
  {
    const char* ad = getenv("CO2_P2P_ADAPT");
    e->adaptive = ad && atoi(ad) == 1;
  }
  // The sharded slice reduce runs beside a step that touches 1/world of the
  // parameters, so it wants the whole chip: 0 = the launcher's per-world
  // default (C4 N=4: 592 CTAs 49.0 ms/round vs 64 CTAs 61.7,
  // profiles/r01/bench/c4_ctas_sweep.txt).
  e->slice_ctas = ctas;
  co2_status_t s = engine_common_init(e);
  if (s == CO2_OK) {
    cudaError_t ce = cudaMalloc(&e->signals, p2p_signal_bytes());
    if (ce == cudaSuccess) ce = cudaMemset(e->signals, 0, p2p_signal_bytes());
    if (ce == cudaSuccess) {
      // barrier spin budget (Signals::timeout_ms): CO2_P2P_TIMEOUT_MS, else 10 s
      const char* env = getenv("CO2_P2P_TIMEOUT_MS");
      const long v = env ? atol(env) : 10000;
      const uint32_t ms = (uint32_t)(v < 1 ? 1 : (v > 3600000 ? 3600000 : v));
      ce = cudaMemcpy(static_cast<char*>(e->signals) + p2p_signal_timeout_offset(), &ms,
                      sizeof ms, cudaMemcpyHostToDevice);
    }
    if (ce != cudaSuccess) s = cuda_fail(ce, "cudaMalloc(signals)");
  }
  if (s != CO2_OK) {
    co2_aar_destroy(e);
    return s;
  }
  *out = e;
  return CO2_OK;
}

extern "C" void* co2_aar_signal_buffer(co2_aar_t* e) { return e ? e->signals : nullptr; }

extern "C" co2_status_t co2_aar_set_adaptive(co2_aar_t* e, int32_t on) {
  if (!e || e->transport != T_P2P)
    return fail(CO2_ERR_VALIDATION, "set_adaptive: not a P2P engine");
  e->adaptive = on != 0;
  e->adapt_next = e->handles.size();
  return CO2_OK;
}

extern "C" int32_t co2_aar_ctas(const co2_aar_t* e) { return e ? e->ctas : 0; }

extern "C" co2_status_t co2_aar_set_fused(co2_aar_t* e, int32_t on) {
  if (!e || e->transport != T_P2P)
    return fail(CO2_ERR_VALIDATION, "fused schedule: P2P transport only");
  e->fused = on != 0;
  return CO2_OK;
}

// Drop one reference to each opened peer allocation in `keys`.
static co2_status_t release_keys(co2_aar* e, const std::vector<std::pair<int, std::string>>& keys) {
  for (const auto& key : keys) {
    auto it = e->opened.find(key);
    if (it == e->opened.end()) continue;
    if (--it->second.refs == 0) {
      void* base = it->second.base;
      e->opened.erase(it);
      CO2_CUDA(cudaIpcCloseMemHandle(base));
    }
  }
  return CO2_OK;
}

static co2_status_t open_peers(co2_aar* e, const void* local, const uint8_t* handles,
                               std::vector<void*>* out,
                               std::vector<std::pair<int, std::string>>* keys = nullptr) {
  out->assign(e->world, nullptr);
  for (int p = 0; p < e->world; ++p) {
    if (p == e->rank) {
      (*out)[p] = const_cast<void*>(local);
      continue;
    }
    const uint8_t* rec = handles + (size_t)p * CO2_IPC_HANDLE_BYTES;
    cudaIpcMemHandle_t h;
    int64_t off = 0;
    memcpy(&h, rec, sizeof h);
    memcpy(&off, rec + sizeof h, sizeof off);
    auto key = std::make_pair(p, std::string(reinterpret_cast<const char*>(rec), sizeof h));
    co2_aar::Opened& o = e->opened[key];
    if (o.refs == 0) {
      void* base = nullptr;
      cudaError_t ce = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
      if (ce != cudaSuccess) {
        e->opened.erase(key);
        return cuda_fail(ce, "cudaIpcOpenMemHandle");
      }
      o.base = base;
    }
    o.refs += 1;
    if (keys) keys->push_back(key);
    (*out)[p] = static_cast<char*>(o.base) + off;
  }
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_p2p_attach_signals(co2_aar_t* e, const uint8_t* handles) {
  if (!e || e->transport != T_P2P) return fail(CO2_ERR_VALIDATION, "attach: not a P2P engine");
  return open_peers(e, e->signals, handles, &e->peer_signals);
}

extern "C" co2_status_t co2_aar_p2p_attach(co2_aar_t* e, const void* local,
                                           const uint8_t* handles) {
  if (!e || e->transport != T_P2P) return fail(CO2_ERR_VALIDATION, "attach: not a P2P engine");
  if (!local) return fail(CO2_ERR_VALIDATION, "attach: null buffer");
  P2PBuffer b;
  b.local = local;
  co2_status_t st = open_peers(e, local, handles, &b.ptrs, &b.keys);
  if (st != CO2_OK) {
    release_keys(e, b.keys);  // keep the first error's message
    return st;
  }
  e->p2p_bufs.push_back(b);
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_p2p_detach(co2_aar_t* e, const void* local) {
  if (!e || e->transport != T_P2P) return fail(CO2_ERR_VALIDATION, "detach: not a P2P engine");
  for (size_t i = 0; i < e->p2p_bufs.size(); ++i) {
    if (e->p2p_bufs[i].local != local) continue;
    // No kernel may still touch the peers' memory: besides the reduces on
    // the comm stream, the fused all-reduce step and the sharded P2P step
    // run on the caller's stream(s), so wait for the whole device.
    CO2_CUDA(cudaDeviceSynchronize());
    const std::vector<std::pair<int, std::string>> keys = e->p2p_bufs[i].keys;
    e->p2p_bufs.erase(e->p2p_bufs.begin() + (std::ptrdiff_t)i);
    return release_keys(e, keys);
  }
  return fail(CO2_ERR_VALIDATION, "detach: buffer not registered for P2P");
}

extern "C" co2_status_t co2_aar_create_local(co2_aar_t** out, int32_t workers) {
  if (!out) return fail(CO2_ERR_VALIDATION, "aar: null output handle");
  if (workers < 1 || workers > 64)
    return fail(CO2_ERR_VALIDATION, "aar: local workers must lie in [1, 64]");
  co2_aar* e = new co2_aar();
  e->transport = T_LOCAL;
  e->workers = workers;
  co2_status_t s = engine_common_init(e);
  if (s != CO2_OK) {
    delete e;
    return s;
  }
  *out = e;
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_destroy(co2_aar_t* e) {
  if (!e) return CO2_OK;
  cudaDeviceSynchronize();  // kernels on any stream may use the peer mappings
  for (Handle& h : e->handles) {
    for (cudaEvent_t ev : {h.start, h.done, h.wait_begin, h.wait_end, h.fin})
      if (ev) cudaEventDestroy(ev);
  }
  if (e->pin_diag) cudaFreeHost(e->pin_diag);
  if (e->pin_err) cudaFreeHost(e->pin_err);
  if (e->pin_ts) cudaFreeHost(e->pin_ts);
  if (e->dev_ts) cudaFree(e->dev_ts);
  if (e->dev_diag) cudaFree(e->dev_diag);
  if (e->aux_stream) cudaStreamDestroy(e->aux_stream);
  if (e->fence) cudaEventDestroy(e->fence);
  if (e->comm2) ncclCommDestroy(e->comm2);
  if (e->comm) ncclCommDestroy(e->comm);
  if (e->ws) cudaFree(e->ws);
  if (e->ws2) cudaFree(e->ws2);
  for (void* p : e->stage)
    if (p) cudaFree(p);
  for (auto& kv : e->opened) cudaIpcCloseMemHandle(kv.second.base);
  if (e->signals) cudaFree(e->signals);
  if (e->epoch) cudaEventDestroy(e->epoch);
  if (e->comm_stream) cudaStreamDestroy(e->comm_stream);
  delete e;
  return CO2_OK;
}

extern "C" int32_t co2_aar_world(const co2_aar_t* e) { return e ? e->workers : 0; }

static co2_status_t record_for(co2_aar* e, uint64_t h, Handle** out) {
  if (!e || h >= e->handles.size()) return fail(CO2_ERR_VALIDATION, "unknown reduce handle");
  *out = &e->handles[h];
  return CO2_OK;
}

// ---- NCCL fixed-order average (the default NCCL algorithm) ---------------
// The reference's average() (proj/src/param_ops.cpp:16-33) sums the
// contributions in ascending worker order and divides once.  A ring or tree
// all-reduce sums in a topology-dependent order and, in bf16, rounds after
// every hop.  This decomposition keeps the ring's NVLink volume, (G-1)/G of
// the buffer in and out per rank, but fixes the order:
//   1. slice exchange: rank r sends slice p of its buffer to rank p and
//      receives slice r of every peer's buffer into staging (grouped
//      ncclSend / ncclRecv, an all-to-all);
//   2. the fixed-order average kernel (co2_average) over the G copies of
//      slice r, ascending rank order, one division, written to `dst`;
//   3. (all-reduce only) slice all-gather with grouped send / recv.
// Slices are ceil(n/G) rounded up to 8 elements (16-byte aligned in every
// dtype); the last ones may be short or empty.
static int64_t nccl_slice(int64_t n, int world) { return ((n + world - 1) / world + 7) / 8 * 8; }

static co2_status_t stage_reserve(co2_aar* e, int which, size_t bytes) {
  if (e->stage_bytes[which] >= bytes) return CO2_OK;
  if (e->stage[which]) CO2_CUDA(cudaFree(e->stage[which]));
  e->stage[which] = nullptr;
  e->stage_bytes[which] = 0;
  CO2_CUDA(cudaMalloc(&e->stage[which], bytes));
  e->stage_bytes[which] = bytes;
  return CO2_OK;
}

// Steps 1-2: average of slice `rank` of every rank's `src` (n elements,
// slices of `slice`) into dst (len_r elements).  `which` selects the staging
// buffer / workspace pair of the stream.
static co2_status_t nccl_fixed_rs(co2_aar* e, ncclComm_t comm, int which, co2_dtype_t dt,
                                  const void* src, int64_t n, int64_t slice, void* dst,
                                  void* ws, cudaStream_t st) {
  const int G = e->world, r = e->rank;
  const size_t es = dtype_bytes(dt);
  auto lo = [&](int p) { return std::min<int64_t>((int64_t)p * slice, n); };
  auto len = [&](int p) { return std::max<int64_t>(0, std::min<int64_t>(slice, n - lo(p))); };
  const int64_t mine = len(r);
  CO2_TRY(stage_reserve(e, which, es * (size_t)slice * (size_t)G + 16));
  char* stg = static_cast<char*>(e->stage[which]);
  const char* s8 = static_cast<const char*>(src);
  if (n == slice * G) {
    // Equal slices: NCCL's all-to-all collective (one kernel over every
    // peer) moves the same bytes as the grouped send / recv below.
    CO2_NCCL(ncclAlltoAll(s8, stg, (size_t)slice, nccl_dtype(dt), comm, st));
  } else {
    CO2_NCCL(ncclGroupStart());
    for (int p = 0; p < G; ++p) {
      if (p == r) continue;
      if (len(p) > 0)
        CO2_NCCL(ncclSend(s8 + es * lo(p), (size_t)len(p), nccl_dtype(dt), p, comm, st));
      if (mine > 0)
        CO2_NCCL(ncclRecv(stg + es * (size_t)slice * p, (size_t)mine, nccl_dtype(dt), p, comm, st));
    }
    CO2_NCCL(ncclGroupEnd());
  }
  const void* parts[kMaxNcclRanks];
  for (int p = 0; p < G; ++p)
    parts[p] = p == r ? static_cast<const void*>(s8 + es * lo(r))
                      : static_cast<const void*>(stg + es * (size_t)slice * p);
  return co2_average(dt, G, parts, mine, dst, ws, st);
}

// Step 3: every rank's slice of `buf` into every rank (in place).
static co2_status_t nccl_fixed_ag(co2_aar* e, ncclComm_t comm, co2_dtype_t dt, void* buf,
                                  int64_t n, int64_t slice, cudaStream_t st) {
  const int G = e->world, r = e->rank;
  const size_t es = dtype_bytes(dt);
  auto lo = [&](int p) { return std::min<int64_t>((int64_t)p * slice, n); };
  auto len = [&](int p) { return std::max<int64_t>(0, std::min<int64_t>(slice, n - lo(p))); };
  char* b8 = static_cast<char*>(buf);
  if (n == slice * G) {  // equal slices: the in-place all-gather collective
    CO2_NCCL(ncclAllGather(b8 + es * lo(r), b8, (size_t)slice, nccl_dtype(dt), comm, st));
    return CO2_OK;
  }
  CO2_NCCL(ncclGroupStart());
  for (int p = 0; p < G; ++p) {
    if (p == r) continue;
    if (len(r) > 0) CO2_NCCL(ncclSend(b8 + es * lo(r), (size_t)len(r), nccl_dtype(dt), p, comm, st));
    if (len(p) > 0) CO2_NCCL(ncclRecv(b8 + es * lo(p), (size_t)len(p), nccl_dtype(dt), p, comm, st));
  }
  CO2_NCCL(ncclGroupEnd());
  return CO2_OK;
}

// Consumers divide the delivered reduce by this: NCCL's sum algorithm
// delivers the worker sum; every other path delivers the average itself.
static int32_t reduce_divisor(const co2_aar* e) {
  return (e->transport == T_NCCL && e->nccl_sum) ? e->world : 1;
}

extern "C" co2_status_t co2_aar_set_nccl_algo(co2_aar_t* e, int32_t algo) {
  if (!e || e->transport != T_NCCL)
    return fail(CO2_ERR_VALIDATION, "nccl algorithm: NCCL transport only");
  if (algo != CO2_NCCL_FIXED_ORDER && algo != CO2_NCCL_SUM)
    return fail(CO2_ERR_VALIDATION, "nccl algorithm: unknown value %d", (int)algo);
  if (algo == CO2_NCCL_FIXED_ORDER && e->world > kMaxNcclRanks)
    return fail(CO2_ERR_VALIDATION, "nccl algorithm: fixed order supports <= %d ranks",
                kMaxNcclRanks);
  if (e->live > 0)
    return fail(CO2_ERR_VALIDATION, "nccl algorithm: cannot change with reduces in flight");
  e->nccl_sum = algo == CO2_NCCL_SUM;
  return CO2_OK;
}

static double ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e-3;
}

// The event a handle completes on (poll / wait / synchronize).
static cudaEvent_t sync_event(const Handle& h) { return h.ktimed ? h.fin : h.done; }

// Kernel-timed handle: wait for it, then copy its device slots (times, the
// average's diagnostics) into its pinned slots.
static co2_status_t fetch_slots(co2_aar* e, const Handle& h) {
  CO2_CUDA(cudaEventSynchronize(h.fin));
  // kernel copies, not cudaMemcpyAsync: a D2H copy could queue in the copy
  // engine behind a caller's D2H that waits for a later round
  CO2_TRY(copy_words_to_host(h.ts_dev, h.ts, 2 * sizeof(uint64_t), e->aux_stream));
  CO2_TRY(copy_words_to_host(h.diag_dev, h.diag, sizeof(co2_diag_t), e->aux_stream));
  CO2_CUDA(cudaStreamSynchronize(e->aux_stream));
  return CO2_OK;
}

// Launch time (s since the epoch) of a completed handle.
static co2_status_t start_time(co2_aar* e, const Handle& h, double* t) {
  if (h.cached) {
    *t = h.c_start;
  } else if (h.ktimed) {
    CO2_TRY(fetch_slots(e, h));
    *t = (double)(int64_t)(h.ts[0] - e->epoch_ns) * 1e-9;
  } else {
    CO2_CUDA(cudaEventSynchronize(h.start));
    *t = ms_between(e->epoch, h.start);
  }
  return CO2_OK;
}

// Cache a finished handle's device times and status (blocking) ...
static co2_status_t cache_done(co2_aar* e, Handle& h) {
  if (h.cached) return CO2_OK;
  if (h.ktimed)
    CO2_TRY(fetch_slots(e, h));
  else
    CO2_CUDA(cudaEventSynchronize(h.done));
  if (h.ktimed) {
    h.c_start = (double)(int64_t)(h.ts[0] - e->epoch_ns) * 1e-9;
    h.c_done = (double)(int64_t)(h.ts[1] - e->epoch_ns) * 1e-9;
    h.c_comm = (double)(int64_t)(h.ts[1] - h.ts[0]) * 1e-9;
  } else {
    h.c_start = ms_between(e->epoch, h.start);
    h.c_done = ms_between(e->epoch, h.done);
    h.c_comm = ms_between(h.start, h.done);
  }
  h.c_flags = h.diag ? h.diag->flags : 0;
  h.c_err = h.p2p_error ? *h.p2p_error : 0;
  h.cached = true;
  return CO2_OK;
}

// ... and, once it has been waited, its wait times (blocking).
static co2_status_t cache_wait(co2_aar* e, Handle& h) {
  if (!h.waited || h.cached_wait) return CO2_OK;
  if (h.wait_alias >= 0) {  // stream-ordered consume: ends where handle wait_alias starts
    CO2_TRY(start_time(e, e->handles[(size_t)h.wait_alias], &h.c_wait_end));
    h.c_stall = 0.0;
  } else {
    CO2_CUDA(cudaEventSynchronize(h.wait_end));
    h.c_stall = ms_between(h.wait_begin, h.wait_end);
    h.c_wait_end = ms_between(e->epoch, h.wait_end);
  }
  h.cached_wait = true;
  return CO2_OK;
}

// Both; handles older than kRing launches are cached this way before their
// events are recycled (at most two are ever live).
static co2_status_t cache_handle(co2_aar* e, Handle& h) {
  CO2_TRY(cache_done(e, h));
  return cache_wait(e, h);
}

// Non-blocking variant for info(): caches only what has already completed.
static co2_status_t cache_handle_if_ready(co2_aar* e, Handle& h) {
  if (!h.cached && cudaEventQuery(sync_event(h)) != cudaSuccess) return CO2_OK;
  CO2_TRY(cache_done(e, h));
  if (!h.waited || h.cached_wait) return CO2_OK;
  if (h.wait_alias >= 0) {
    const Handle& a = e->handles[(size_t)h.wait_alias];
    if (!a.cached && cudaEventQuery(a.ktimed ? a.fin : a.start) != cudaSuccess) return CO2_OK;
  } else if (cudaEventQuery(h.wait_end) != cudaSuccess) {
    return CO2_OK;
  }
  return cache_wait(e, h);
}

// A new handle: events (recycled from the handle kRing launches back) and
// pinned diagnostic slots from the engine's ring.
static co2_status_t new_handle(co2_aar* e, Handle* h) {
  const size_t id = e->handles.size();
  if (!e->pin_diag) {
    CO2_CUDA(cudaMallocHost(&e->pin_diag, kRing * sizeof(co2_diag_t)));
    CO2_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->pin_diag_dev), e->pin_diag, 0));
    CO2_CUDA(cudaMallocHost(&e->pin_err, kRing * sizeof(uint32_t)));
    CO2_CUDA(cudaMallocHost(&e->pin_ts, 2 * kRing * sizeof(uint64_t)));
    CO2_CUDA(cudaMalloc(&e->dev_ts, 2 * kRing * sizeof(uint64_t)));
    CO2_CUDA(cudaMalloc(&e->dev_diag, kRing * sizeof(co2_diag_t)));
    CO2_CUDA(cudaStreamCreateWithFlags(&e->aux_stream, cudaStreamNonBlocking));
    CO2_CUDA(cudaEventCreateWithFlags(&e->fence, cudaEventDisableTiming));
  }
  if (id >= kRing) {
    Handle& old = e->handles[id - kRing];
    if (!old.consumed) return fail(CO2_ERR_VALIDATION, "aar: handle ring overrun");
    CO2_TRY(cache_handle(e, old));
    h->start = old.start;
    h->done = old.done;
    h->wait_begin = old.wait_begin;
    h->wait_end = old.wait_end;
    h->fin = old.fin;
    old.start = old.done = old.wait_begin = old.wait_end = old.fin = nullptr;
    old.ts = nullptr;
    old.ts_dev = nullptr;
    old.diag_dev = nullptr;
    old.diag = nullptr;
    old.p2p_error = nullptr;
  } else {
    CO2_CUDA(cudaEventCreateWithFlags(&h->start, cudaEventDefault));
    CO2_CUDA(cudaEventCreateWithFlags(&h->done, cudaEventDefault));
    CO2_CUDA(cudaEventCreateWithFlags(&h->wait_begin, cudaEventDefault));
    CO2_CUDA(cudaEventCreateWithFlags(&h->wait_end, cudaEventDefault));
    CO2_CUDA(cudaEventCreateWithFlags(&h->fin, cudaEventDisableTiming));
  }
  h->diag = &e->pin_diag[id % kRing];
  h->p2p_error = &e->pin_err[id % kRing];
  h->ts = &e->pin_ts[2 * (id % kRing)];
  h->ts[0] = h->ts[1] = 0;
  h->ts_dev = e->dev_ts + 2 * (id % kRing);
  h->diag_dev = e->dev_diag + id % kRing;
  h->diag->flags = 0;
  *h->p2p_error = 0;
  return CO2_OK;
}

// kind 0: all-reduce (NCCL in place / LOCAL average); kind 1: reduce-scatter
// (sum) of the full buffer bufs[0] (n = world * shard) into out (one shard).
// Adaptive reduce occupancy.  From the newest consumed reduce whose device
// times are known (never blocking): it stalled the consumer (> 1 % of its
// duration) -> more CTAs; it finished with slack to spare before the consumer
// reached its wait (> half its duration) -> fewer, so the reduce takes fewer
// SMs from the compute it overlaps.  The CTA count does not change results
// (every element's fixed-order sum is the same) and ranks may differ (the
// exit barrier counts ranks, not CTAs).  It never blocks, so when the host
// enqueues rounds far ahead of the GPU it decides rarely; measured no gain
// on the bench or the tau sweep (profiles/r02/tune/adaptive/), hence opt-in.
static co2_status_t adapt_ctas(co2_aar* e) {
  for (size_t i = e->handles.size(); i-- > e->adapt_next;) {
    Handle& h = e->handles[i];
    if (!h.waited) continue;
    CO2_TRY(cache_handle_if_ready(e, h));
    if (!h.cached || !h.cached_wait) continue;
    e->adapt_next = i + 1;
    const double comm = h.c_comm, stall = h.c_stall;
    const double slack = (h.c_wait_end - stall) - h.c_done;  // wait begin - completion
    int c = e->ctas;
    if (stall > 0.01 * comm)
      c = c + c / 4 + 4;
    else if (slack > 0.5 * comm)
      c = c - c / 8 - 1;
    e->ctas = c < e->ctas_min ? e->ctas_min : (c > e->ctas_max ? e->ctas_max : c);
    break;
  }
  return CO2_OK;
}

static co2_status_t launch_impl(co2_aar_t* e, int kind, co2_dtype_t dt, const void* const* bufs,
                                void* out, int64_t n, void* producer, uint64_t* handle_out) {
  // launch_all_reduce, collective.cpp:31-58
  if (!e) return fail(CO2_ERR_VALIDATION, "aar: null engine");
  if (e->live >= 2)
    return fail(CO2_ERR_VALIDATION,
                "launch_all_reduce: overlap window exceeded, two reduces already live");
  if (n < 0) return fail(CO2_ERR_VALIDATION, "launch_all_reduce: negative size");
  Handle h;
  CO2_TRY(new_handle(e, &h));
  h.contributions = e->workers;
  // Fence: the reduce reads x_{t,tau} only after the producer wrote it.
  CO2_CUDA(cudaEventRecord(e->fence, S(producer)));
  CO2_CUDA(cudaStreamWaitEvent(e->comm_stream, e->fence, 0));
  CO2_CUDA(cudaEventRecord(h.start, e->comm_stream));
  if (kind == 1) {
    if (e->transport != T_NCCL)
      return fail(CO2_ERR_VALIDATION, "reduce-scatter: NCCL transport only");
    const int64_t shard = n / e->world;
    if (e->world > 1 && shard > 0 && !e->nccl_sum) {
      CO2_TRY(nccl_fixed_rs(e, e->comm, 0, dt, bufs[0], n, shard, out, e->ws, e->comm_stream));
      CO2_TRY(copy_words_to_host(&ws_header(e->ws)->diag, h.diag, sizeof(co2_diag_t),
                                 e->comm_stream));
    } else if (e->world > 1 && shard > 0)
      CO2_NCCL(ncclReduceScatter(bufs[0], out, (size_t)shard, nccl_dtype(dt), ncclSum, e->comm,
                                 e->comm_stream));
    else if (shard > 0)
      CO2_CUDA(cudaMemcpyAsync(out, bufs[0], dtype_bytes(dt) * (size_t)shard,
                               cudaMemcpyDeviceToDevice, e->comm_stream));
  } else if (e->transport == T_P2P) {
    if (out && out != bufs[0])
      return fail(CO2_ERR_VALIDATION, "launch_all_reduce: P2P transport reduces in place");
    const P2PBuffer* pb = nullptr;
    for (const P2PBuffer& b : e->p2p_bufs)
      if (b.local == bufs[0]) pb = &b;
    if (!pb) return fail(CO2_ERR_VALIDATION, "launch_all_reduce: buffer not registered for P2P");
    if (e->world > 1 && (int)e->peer_signals.size() != e->world)
      return fail(CO2_ERR_VALIDATION, "launch_all_reduce: P2P signals not attached");
    if (e->world > 1 && n > 0) {
      if (e->adaptive) CO2_TRY(adapt_ctas(e));
      e->p2p_epoch += 1;
      CO2_TRY(p2p_average_launch(dt, pb->ptrs.data(), e->peer_signals.data(), e->world, e->rank,
                                 n, e->p2p_epoch, &e->p2p_done, e->ctas, e->comm_stream));
      // the kernel records a timed-out barrier in the signal area's error word
      CO2_TRY(copy_words_to_host(static_cast<char*>(e->signals) + p2p_signal_error_offset(),
                                 h.p2p_error, 4, e->comm_stream));
    }
  } else if (e->transport == T_NCCL) {
    if (out && out != bufs[0])
      return fail(CO2_ERR_VALIDATION, "launch_all_reduce: NCCL transport reduces in place");
    if (e->world > 1 && n > 0 && !e->nccl_sum) {
      const int64_t slice = nccl_slice(n, e->world);
      void* buf = const_cast<void*>(bufs[0]);
      void* mine = static_cast<char*>(buf) +
                   dtype_bytes(dt) * (size_t)std::min<int64_t>((int64_t)e->rank * slice, n);
      CO2_TRY(nccl_fixed_rs(e, e->comm, 0, dt, buf, n, slice, mine, e->ws, e->comm_stream));
      CO2_TRY(copy_words_to_host(&ws_header(e->ws)->diag, h.diag, sizeof(co2_diag_t),
                                 e->comm_stream));
      CO2_TRY(nccl_fixed_ag(e, e->comm, dt, buf, n, slice, e->comm_stream));
    } else if (e->world > 1 && n > 0) {
      CO2_NCCL(ncclAllReduce(bufs[0], const_cast<void*>(bufs[0]), (size_t)n, nccl_dtype(dt), ncclSum,
                             e->comm, e->comm_stream));
    }
  } else {
    CO2_TRY(co2_average(dt, e->workers, bufs, n, out, e->ws, e->comm_stream));
    CO2_TRY(copy_words_to_host(&ws_header(e->ws)->diag, h.diag, sizeof(co2_diag_t),
                               e->comm_stream));
  }
  CO2_CUDA(cudaEventRecord(h.done, e->comm_stream));
  h.done_stream = e->comm_stream;
  e->handles.push_back(h);
  e->live += 1;
  *handle_out = e->handles.size() - 1;
  return CO2_OK;
}

static const P2PBuffer* find_p2p(const co2_aar* e, const void* local) {
  for (const P2PBuffer& b : e->p2p_bufs)
    if (b.local == local) return &b;
  return nullptr;
}

// P2P sharded layout: one handle covering the deterministic slice averages of
// x_{t,tau} (src0) and x_{t,1} (src1) into local slices dst0 / dst1.
static co2_status_t launch_slice(co2_aar* e, co2_dtype_t dt, const void* src0, const void* src1,
                                 void* dst0, void* dst1, int64_t lo, int64_t len, void* producer,
                                 uint64_t* handle_out) {
  if (e->live >= 2)
    return fail(CO2_ERR_VALIDATION,
                "launch_all_reduce: overlap window exceeded, two reduces already live");
  const P2PBuffer* b0 = find_p2p(e, src0);
  const P2PBuffer* b1 = find_p2p(e, src1);
  if (!b0 || !b1) return fail(CO2_ERR_VALIDATION, "slice reduce: buffer not registered for P2P");
  if ((int)e->peer_signals.size() != e->world)
    return fail(CO2_ERR_VALIDATION, "slice reduce: P2P signals not attached");
  Handle h;
  CO2_TRY(new_handle(e, &h));
  h.contributions = e->workers;
  CO2_CUDA(cudaEventRecord(e->fence, S(producer)));
  CO2_CUDA(cudaStreamWaitEvent(e->comm_stream, e->fence, 0));
  CO2_CUDA(cudaEventRecord(h.start, e->comm_stream));
  e->p2p_epoch += 1;
  CO2_TRY(p2p_slice_average_launch(dt, 2, b0->ptrs.data(), b1->ptrs.data(), dst0, dst1,
                                   e->peer_signals.data(), e->world, e->rank, lo, len,
                                   e->p2p_epoch, e->slice_ctas, e->comm_stream));
  CO2_TRY(copy_words_to_host(static_cast<char*>(e->signals) + p2p_signal_error_offset(),
                             h.p2p_error, 4, e->comm_stream));
  CO2_CUDA(cudaEventRecord(h.done, e->comm_stream));
  h.done_stream = e->comm_stream;
  e->handles.push_back(h);
  e->live += 1;
  *handle_out = e->handles.size() - 1;
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_launch(co2_aar_t* e, co2_dtype_t dt, const void* const* bufs,
                                       void* out, int64_t n, void* producer, uint64_t* handle_out) {
  return launch_impl(e, 0, dt, bufs, out, n, producer, handle_out);
}

extern "C" co2_status_t co2_aar_poll(co2_aar_t* e, uint64_t handle, int32_t* done) {
  // is_completed, collective.cpp:74-86 (never blocks)
  Handle* h = nullptr;
  CO2_TRY(record_for(e, handle, &h));
  if (h->consumed) return fail(CO2_ERR_VALIDATION, "is_completed: handle already consumed");
  cudaError_t q = cudaEventQuery(sync_event(*h));
  if (q != cudaSuccess && q != cudaErrorNotReady) return cuda_fail(q, "cudaEventQuery");
  bool d = q == cudaSuccess;
  h->polled = true;
  h->last_poll = d;
  if (d) h->completion_logged = true;
  *done = d ? 1 : 0;
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_wait(co2_aar_t* e, uint64_t handle, void* consumer) {
  // wait, collective.cpp:88-105: consume once; the consumer stream (not the
  // host) waits for completion.
  Handle* h = nullptr;
  CO2_TRY(record_for(e, handle, &h));
  if (h->consumed) return fail(CO2_ERR_VALIDATION, "wait: handle already consumed");
  CO2_CUDA(cudaEventRecord(h->wait_begin, S(consumer)));
  CO2_CUDA(cudaStreamWaitEvent(S(consumer), sync_event(*h), 0));
  CO2_CUDA(cudaEventRecord(h->wait_end, S(consumer)));
  h->consumed = true;
  h->waited = true;
  e->live -= 1;
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_order_after(co2_aar_t* e, uint64_t handle, void* stream) {
  // Orders `stream`'s later work after the reduce without consuming it: the
  // reference's launch snapshots its contributions (collective.cpp:44-50),
  // so a value-semantics caller may overwrite them right after the launch.
  Handle* h = nullptr;
  CO2_TRY(record_for(e, handle, &h));
  if (h->consumed) return fail(CO2_ERR_VALIDATION, "order_after: handle already consumed");
  CO2_CUDA(cudaStreamWaitEvent(S(stream), sync_event(*h), 0));
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_stall(co2_aar_t* e, uint64_t handle, double* stall,
                                      double* comm) {
  Handle* h = nullptr;
  CO2_TRY(record_for(e, handle, &h));
  if (!h->waited) return fail(CO2_ERR_VALIDATION, "stall: handle not waited yet");
  CO2_TRY(cache_handle(e, *h));
  if (stall) *stall = h->c_stall;
  if (comm) *comm = h->c_comm;
  if (h->c_flags) {
    co2_diag_t d{};
    d.flags = h->c_flags;
    return co2_diag_status(&d);
  }
  if (h->c_err)
    return fail(CO2_ERR_CUDA, "p2p all-reduce: cross-GPU barrier timed out (code %u)", h->c_err);
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_live(const co2_aar_t* e, int32_t* live) {
  if (!e) return fail(CO2_ERR_VALIDATION, "aar: null engine");
  *live = e->live;
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_info(co2_aar_t* e, uint64_t handle, co2_handle_info_t* out) {
  Handle* h = nullptr;
  CO2_TRY(record_for(e, handle, &h));
  if (!out) return fail(CO2_ERR_VALIDATION, "info: null output");
  const double nan = std::numeric_limits<double>::quiet_NaN();
  co2_handle_info_t r{handle, nan, nan, nan, nan, 0, h->consumed ? 1 : 0, h->contributions,
                      h->polled ? 1 : 0, h->last_poll ? 1 : 0, 0};
  CO2_TRY(cache_handle_if_ready(e, *h));
  if (h->cached) {
    r.launch_time = h->c_start;
    r.completion_time = h->c_done;
    r.comm = h->c_comm;
    r.completed = 1;
    if (h->cached_wait) r.stall = h->c_stall;
  }
  // log_completion (collective.cpp:66-71): a successful poll or the wait
  r.completion_logged = (h->completion_logged || h->consumed) ? 1 : 0;
  *out = r;
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_totals(co2_aar_t* e, double* total_stall, uint64_t* count) {
  if (!e) return fail(CO2_ERR_VALIDATION, "aar: null engine");
  double t = 0.0;
  for (Handle& h : e->handles)
    if (h.waited) {
      CO2_TRY(cache_handle(e, h));
      t += h.c_stall;
    }
  if (total_stall) *total_stall = t;
  if (count) *count = e->handles.size();
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_allreduce_blocking(co2_aar_t* e, co2_dtype_t dt, void* buf,
                                                   int64_t n, void* stream) {
  if (!e) return fail(CO2_ERR_VALIDATION, "aar: null engine");
  if (e->transport != T_NCCL)
    return fail(CO2_ERR_VALIDATION, "allreduce_blocking: NCCL transport only");
  if (e->world > 1 && n > 0)
    CO2_NCCL(ncclAllReduce(buf, buf, (size_t)n, nccl_dtype(dt), ncclSum, e->comm, S(stream)));
  return CO2_OK;
}

extern "C" co2_status_t co2_aar_events(co2_aar_t* e, co2_event_t* out, int64_t cap,
                                       int64_t* count) {
  // Event log of collective.hpp:24-29 from device timestamps.
  if (!e) return fail(CO2_ERR_VALIDATION, "aar: null engine");
  int64_t k = 0;
  auto push = [&](int kind, uint64_t id, double t, double stall) {
    if (k < cap && out) out[k] = co2_event_t{kind, 0, id, t, stall};
    ++k;
  };
  for (uint64_t i = 0; i < e->handles.size(); ++i) {
    Handle& h = e->handles[i];
    CO2_TRY(cache_handle(e, h));  // blocks until the handle (and its wait) completed
    push(0, i, h.c_start, 0.0);
    push(1, i, h.c_done, 0.0);
    if (h.waited) push(2, i, h.c_wait_end, h.c_stall);
  }
  *count = k;
  return CO2_OK;
}

// ===================================================================== worker
struct co2_worker {
  co2_mode_t mode = CO2_MODE_F32;
  int64_t n = 0;
  int t = 0;
  int cur = 0;
  void* params[2] = {nullptr, nullptr};
  void* anchor = nullptr;
  void* xfirst = nullptr;
  void* prev_x0 = nullptr;
  void* prev_x1 = nullptr;
  void* m = nullptr;
  void* gap = nullptr;
  void* avg[2] = {nullptr, nullptr};  // LOCAL transport consumed averages
  void* tmp_state = nullptr;          // ghost: bar0
  void* tmp_low = nullptr;            // ghost: bar1
  void* xbar = nullptr;               // last consumed reduce (for CO2_BUF_XBAR)
  // RoundResult::consumed_average on the in-place transports (NCCL / P2P):
  // the step copies the reduce it consumes here (co2_worker_keep_average).
  void* avg_keep = nullptr;
  bool keep_avg = false;
  void* ws = nullptr;
  co2_diag_t* host_diag = nullptr;  // pinned
  // the last round's diagnostics are only in the workspace header (the
  // single-launch LOCAL round): co2_round_finish fetches them first
  bool diag_on_device = false;
  // fused P2P schedule: pinned copy of the engine's signal error word, read
  // back after every fused round (a timed-out barrier means the consumed
  // average is incomplete); checked by co2_round_finish and the next round
  uint32_t* fused_err = nullptr;
  bool has_pending = false;
  uint64_t pending = 0;
  uint64_t consumed = 0;
  bool has_consumed = false;
  // optional device timing of the fused launch (ring of event pairs)
  std::vector<cudaEvent_t> tev;  // 2 * cap
  int64_t tev_recorded = 0, tev_read = 0;
  int clip_mode = CO2_CLIP_COORDINATE;  // CO2_CLIP_GLOBAL_NORM: the extension
};

static co2_status_t step_launch(co2_worker* w, co2_mode_t mode, int64_t n, const void* x_t0,
                                const void* p0, const void* p1, const void* xbar,
                                int32_t divisor, void* m, void* anchor, void* params, void* gap,
                                const co2_hyper_t* h, cudaStream_t st, void* xbar_out = nullptr) {
  const int64_t cap = (int64_t)w->tev.size() / 2;
  const int64_t slot = cap ? w->tev_recorded % cap : 0;
  if (cap) CO2_CUDA(cudaEventRecord(w->tev[2 * slot], st));
  if (w->clip_mode == CO2_CLIP_GLOBAL_NORM)
    CO2_TRY(outer_step_global_clip_impl(mode, n, x_t0, p0, p1, xbar, divisor, m, anchor, params,
                                        gap, h, w->ws, st, xbar_out));
  else
    CO2_TRY(outer_step_impl(mode, n, x_t0, p0, p1, xbar, divisor, m, anchor, params, gap, h,
                            w->ws, st, xbar_out));
  if (cap) {
    CO2_CUDA(cudaEventRecord(w->tev[2 * slot + 1], st));
    w->tev_recorded += 1;
  }
  return CO2_OK;
}

static co2_status_t walloc(void** p, size_t bytes) {
  CO2_CUDA(cudaMalloc(p, bytes ? bytes : 16));
  return CO2_OK;
}

extern "C" co2_status_t co2_worker_create(co2_worker_t** out, co2_mode_t mode, int64_t n,
                                          const void* init, int32_t keep_gap, void* stream) {
  if (n < 0) return fail(CO2_ERR_VALIDATION, "worker: negative dimension");
  if (mode != CO2_MODE_F64 && mode != CO2_MODE_F32 && mode != CO2_MODE_BF16_MIXED)
    return fail(CO2_ERR_VALIDATION, "worker: unknown mode %d", (int)mode);
  co2_worker* w = new co2_worker();
  w->mode = mode;
  w->n = n;
  const size_t sb = state_bytes(mode) * n, lb = low_bytes(mode) * n;
  co2_status_t s = CO2_OK;
  auto A = [&](void** p, size_t b) {
    if (s == CO2_OK) s = walloc(p, b);
  };
  A(&w->params[0], lb);
  A(&w->params[1], lb);
  A(&w->anchor, sb);
  A(&w->xfirst, lb);
  A(&w->prev_x0, sb);
  A(&w->prev_x1, lb);
  A(&w->m, sb);
  if (keep_gap) A(&w->gap, sb);
  A(&w->ws, co2_workspace_bytes());
  if (s != CO2_OK) {
    co2_worker_destroy(w);
    return s;
  }
  cudaStream_t st = S(stream);
  CO2_CUDA(cudaMallocHost(&w->host_diag, sizeof(co2_diag_t)));
  CO2_CUDA(cudaMemsetAsync(w->ws, 0, co2_workspace_bytes(), st));
  // OuterState init, outer_algorithms.cpp:416-418: momentum zeros, gap ones.
  CO2_CUDA(cudaMemsetAsync(w->m, 0, sb ? sb : 1, st));
  if (init) {
    CO2_CUDA(cudaMemcpyAsync(w->params[0], init, lb, cudaMemcpyDeviceToDevice, st));
  } else {
    CO2_CUDA(cudaMemsetAsync(w->params[0], 0, lb ? lb : 1, st));
  }
  if (w->gap && n > 0) {
    if (mode == CO2_MODE_F64) {
      std::vector<double> ones(n, 1.0);
      CO2_CUDA(cudaMemcpy(w->gap, ones.data(), sb, cudaMemcpyHostToDevice));
    } else {
      CO2_TRY(co2_fill_u32(w->gap, 0x3f800000u, n, stream));
    }
  }
  *out = w;
  return CO2_OK;
}

extern "C" co2_status_t co2_worker_destroy(co2_worker_t* w) {
  if (!w) return CO2_OK;
  for (void* p : {w->params[0], w->params[1], w->anchor, w->xfirst, w->prev_x0, w->prev_x1, w->m,
                  w->gap, w->avg[0], w->avg[1], w->tmp_state, w->tmp_low, w->avg_keep, w->ws})
    if (p) cudaFree(p);
  if (w->host_diag) cudaFreeHost(w->host_diag);
  if (w->fused_err) cudaFreeHost(w->fused_err);
  for (cudaEvent_t ev : w->tev) cudaEventDestroy(ev);
  delete w;
  return CO2_OK;
}

extern "C" co2_status_t co2_worker_enable_timing(co2_worker_t* w, int32_t cap) {
  if (!w || cap < 1) return fail(CO2_ERR_VALIDATION, "timing: bad arguments");
  for (cudaEvent_t ev : w->tev) cudaEventDestroy(ev);
  w->tev.assign(2 * (size_t)cap, nullptr);
  for (cudaEvent_t& ev : w->tev) CO2_CUDA(cudaEventCreate(&ev));
  w->tev_recorded = w->tev_read = 0;
  return CO2_OK;
}

extern "C" co2_status_t co2_worker_step_times(co2_worker_t* w, double* out, int32_t cap,
                                              int32_t* count) {
  if (!w) return fail(CO2_ERR_VALIDATION, "timing: null worker");
  const int64_t ring = (int64_t)w->tev.size() / 2;
  int64_t first = w->tev_read;
  if (ring && w->tev_recorded - first > ring) first = w->tev_recorded - ring;  // overwritten
  int32_t k = 0;
  for (int64_t i = first; ring && i < w->tev_recorded && k < cap; ++i) {
    const int64_t s = i % ring;
    CO2_CUDA(cudaEventSynchronize(w->tev[2 * s + 1]));
    float ms = 0.f;
    CO2_CUDA(cudaEventElapsedTime(&ms, w->tev[2 * s], w->tev[2 * s + 1]));
    if (out) out[k] = ms * 1e-3;
    ++k;
  }
  w->tev_read = w->tev_recorded;
  *count = k;
  return CO2_OK;
}

extern "C" void* co2_worker_buffer(co2_worker_t* w, int32_t which) {
  if (!w) return nullptr;
  switch (which) {
    case CO2_BUF_PARAMS: return w->params[w->cur];
    case CO2_BUF_ANCHOR: return w->anchor;
    case CO2_BUF_XFIRST: return w->xfirst;
    case CO2_BUF_PREV_X0: return w->prev_x0;
    case CO2_BUF_PREV_X1: return w->prev_x1;
    case CO2_BUF_MOMENTUM: return w->m;
    case CO2_BUF_GAP: return w->gap;
    case CO2_BUF_XBAR: return w->xbar;
    case CO2_BUF_PARAMS_ALT: return w->params[1 - w->cur];
  }
  return nullptr;
}

extern "C" co2_status_t co2_worker_set_clip_mode(co2_worker_t* w, int32_t mode) {
  if (!w) return fail(CO2_ERR_VALIDATION, "worker: null handle");
  if (mode != CO2_CLIP_COORDINATE && mode != CO2_CLIP_GLOBAL_NORM)
    return fail(CO2_ERR_VALIDATION, "worker: unknown clip mode %d", (int)mode);
  w->clip_mode = mode;
  return CO2_OK;
}

extern "C" co2_status_t co2_worker_keep_average(co2_worker_t* w, int32_t on) {
  if (!w) return fail(CO2_ERR_VALIDATION, "worker: null handle");
  w->keep_avg = on != 0;
  if (w->keep_avg && !w->avg_keep) CO2_TRY(walloc(&w->avg_keep, low_bytes(w->mode) * w->n));
  return CO2_OK;
}

extern "C" int32_t co2_worker_round(const co2_worker_t* w) { return w ? w->t : -1; }

extern "C" co2_status_t co2_worker_snapshot_start(co2_worker_t* w, void* stream) {
  // InnerTrace::x_start = params (inner_loop.cpp:73).  For t >= 1 the outer
  // step already wrote x_{t,0} into the anchor (fused snapshot capture).
  if (!w) return fail(CO2_ERR_VALIDATION, "worker: null");
  if (w->t > 0) return CO2_OK;
  return co2_convert(state_dtype(w->mode), w->anchor, low_dtype(w->mode), w->params[w->cur], w->n,
                     stream);
}

extern "C" co2_status_t co2_worker_snapshot_first(co2_worker_t* w, void* stream) {
  // InnerTrace::x_first = params after inner step 0 (inner_loop.cpp:96-98).
  if (!w) return fail(CO2_ERR_VALIDATION, "worker: null");
  return co2_convert(low_dtype(w->mode), w->xfirst, low_dtype(w->mode), w->params[w->cur], w->n,
                     stream);
}

static co2_status_t copy_dev(void* d, const void* s, size_t bytes, cudaStream_t st) {
  if (bytes) CO2_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, st));
  return CO2_OK;
}

extern "C" co2_status_t co2_round_finish(co2_worker_t* const* ws, int32_t g, void* stream,
                                         co2_round_result_t* res) {
  if (!ws || !res || g < 1) return fail(CO2_ERR_VALIDATION, "co2_round_finish: bad arguments");
  for (int i = 0; i < g; ++i)
    if (!ws[i]) return fail(CO2_ERR_VALIDATION, "co2_round_finish: null worker");
  for (int i = 0; i < g; ++i)
    if (ws[i]->diag_on_device) {
      CO2_TRY(diag_to_host(ws[i]->ws, ws[i]->host_diag, stream));
      ws[i]->diag_on_device = false;
    }
  CO2_CUDA(cudaStreamSynchronize(S(stream)));
  co2_round_result_t r = *res;
  r.min_gap = INFINITY;
  r.max_outer_step = 0.0;
  r.n_clipped = 0;
  r.n_floored = 0;
  co2_status_t first = CO2_OK;
  char msg[512] = {0};
  for (int i = 0; i < g; ++i)
    if (ws[i]->fused_err && *ws[i]->fused_err)
      return fail(CO2_ERR_CUDA, "p2p fused step: cross-GPU barrier timed out (code %u)",
                  *ws[i]->fused_err);
  for (int i = 0; i < g; ++i) {  // worker order = the reference's error order (cpp:186)
    const co2_diag_t& d = *ws[i]->host_diag;
    r.min_gap = d.min_gap < r.min_gap ? d.min_gap : r.min_gap;
    r.max_outer_step = d.max_outer_step > r.max_outer_step ? d.max_outer_step : r.max_outer_step;
    r.n_clipped += d.n_clipped;
    r.n_floored += d.n_floored;
    if (first == CO2_OK && d.flags) {
      first = co2_diag_status(&d);
      snprintf(msg, sizeof msg, "%s", co2_last_error());
    }
  }
  *res = r;
  if (first != CO2_OK) return fail(first, "%s", msg);
  return CO2_OK;
}

extern "C" co2_status_t co2_round_host(co2_worker_t* const* ws, int32_t g, co2_aar_t* e,
                                       const co2_hyper_t* hyper,
                                       const void* const* x_first_host,
                                       const void* const* x_end_host, void* const* x_next_host,
                                       void* stream, int32_t sync, co2_round_result_t* res) {
  if (!ws || g < 1 || !x_end_host || !x_next_host)
    return fail(CO2_ERR_VALIDATION, "co2_round_host: bad arguments");
  cudaStream_t st = S(stream);
  for (int i = 0; i < g; ++i) {
    co2_worker* w = ws[i];
    if (!w || !x_end_host[i] || !x_next_host[i])
      return fail(CO2_ERR_VALIDATION, "co2_round_host: null worker or host buffer");
    const size_t lb = low_bytes(w->mode) * (size_t)w->n;
    if (!lb) continue;
    if (x_first_host && x_first_host[i])  // InnerTrace::x_first (inner_loop.cpp:96-98)
      CO2_CUDA(cudaMemcpyAsync(w->xfirst, x_first_host[i], lb, cudaMemcpyHostToDevice, st));
    // InnerTrace::x_end: the params the round reduces and steps from (:110)
    CO2_CUDA(cudaMemcpyAsync(w->params[w->cur], x_end_host[i], lb, cudaMemcpyHostToDevice, st));
  }
  co2_round_result_t r{};
  const co2_status_t s0 = co2_round(ws, g, e, hyper, stream, sync, &r);
  if (res) *res = r;
  if (s0 != CO2_OK && s0 != CO2_ERR_NUMERIC) return s0;
  for (int i = 0; i < g; ++i) {  // the next inner loop's start
    co2_worker* w = ws[i];
    const size_t lb = low_bytes(w->mode) * (size_t)w->n;
    if (lb)
      CO2_CUDA(cudaMemcpyAsync(x_next_host[i], w->params[w->cur], lb, cudaMemcpyDeviceToHost, st));
  }
  if (sync) CO2_CUDA(cudaStreamSynchronize(st));
  return s0;
}

extern "C" co2_status_t co2_round_drain(co2_worker_t* const* ws, int32_t g, co2_aar_t* e,
                                        void* stream) {
  if (!ws || g < 1 || !e) return fail(CO2_ERR_VALIDATION, "co2_round_drain: bad arguments");
  if (!ws[0]->has_pending) return CO2_OK;
  const uint64_t h = ws[0]->pending;
  CO2_TRY(co2_aar_wait(e, h, stream));
  for (int i = 0; i < g; ++i) ws[i]->has_pending = false;
  return CO2_OK;
}

// Argument checks shared by the round drivers: engine, worker array and
// every worker handle non-null, g >= 1.
static co2_status_t check_round_args(co2_worker_t* const* ws, int32_t g, const co2_aar* e,
                                     const char* who) {
  if (!e || !ws || g < 1) return fail(CO2_ERR_VALIDATION, "%s: bad arguments", who);
  for (int i = 0; i < g; ++i)
    if (!ws[i]) return fail(CO2_ERR_VALIDATION, "%s: null worker", who);
  return CO2_OK;
}

// Single-launch LOCAL round (C1): rounds t >= 1 of the
// worker-local branch with up to kMaxLocalRound simulated workers run as one
// kernel that both averages this round's x_{t,tau} (the launch) and applies
// every worker's step on the previous average (the consume) -- see
// local_round_kernel.  CO2_LOCAL_ROUND=split keeps the two-kernel schedule.
static bool local_round_fused_enabled() {
  static const bool on = [] {
    const char* v = getenv("CO2_LOCAL_ROUND");
    return !(v && strcmp(v, "split") == 0);
  }();
  return on;
}

static co2_status_t local_round_fused(co2_worker_t* const* ws, int32_t g, co2_aar* e,
                                      const co2_hyper_t* hyper, void* stream, int32_t sync,
                                      co2_round_result_t* res) {
  co2_worker* w0 = ws[0];
  cudaStream_t st = S(stream);
  if (!w0->has_pending)  // shared_pending, outer_algorithms.cpp:22-26
    return fail(CO2_ERR_VALIDATION, "outer round: no pending reduce to consume");
  if (e->live >= 2)
    return fail(CO2_ERR_VALIDATION,
                "launch_all_reduce: overlap window exceeded, two reduces already live");
  const uint64_t prev = w0->pending;
  int32_t done = 0;
  CO2_TRY(co2_aar_poll(e, prev, &done));  // :155-157
  // wait (collective.cpp:88-105).  A reduce that completed on this stream
  // (the previous single-launch round) is ordered before this round by the
  // stream itself: consume it without a cross-stream wait or its two timing
  // events (each timing event record costs the stream ~2.5 us, measured
  // beside a ~35 us C1 round; profiles/r02/c1/), stall 0, its wait time the
  // start of the handle launched below.  Otherwise (round 1: the reduce ran
  // on the comm stream) the ordinary wait.
  Handle& ph = e->handles[prev];
  const bool ordered = ph.done_stream == st && !ph.consumed;
  if (ordered) {
    ph.consumed = true;
    ph.waited = true;
    ph.wait_alias = (int64_t)e->handles.size();  // the handle new_handle adds next
    e->live -= 1;
  } else {
    CO2_TRY(co2_aar_wait(e, prev, stream));
  }
  const int t = w0->t;
  void* xbar = w0->avg[(t - 1) % 2];
  void* avg_out = w0->avg[t % 2];
  const void *x0[kMaxLocalRound], *p0[kMaxLocalRound], *p1[kMaxLocalRound],
      *cur[kMaxLocalRound];
  void *m[kMaxLocalRound], *an[kMaxLocalRound], *pr[kMaxLocalRound], *gp[kMaxLocalRound],
      *wsp[kMaxLocalRound];
  for (int i = 0; i < g; ++i) {
    co2_worker* w = ws[i];
    x0[i] = w->anchor;
    p0[i] = w->prev_x0;
    p1[i] = w->prev_x1;
    cur[i] = w->params[w->cur];
    m[i] = w->m;
    an[i] = w->prev_x0;  // x_{t+1,0} over prev_x0 (the rotation swaps it in)
    pr[i] = w->params[1 - w->cur];
    gp[i] = w->gap;
    wsp[i] = w->ws;
  }
  Handle h;
  CO2_TRY(new_handle(e, &h));
  h.contributions = g;
  const size_t slot = e->handles.size() % kRing;
  // Kernel-timed: the kernel stamps its own start / end into the handle's
  // pinned slot and completion is a non-timing event, so the round adds no
  // timing event to the stream (the worker's optional step timing still does).
  h.ktimed = true;
  const int64_t cap = (int64_t)w0->tev.size() / 2;
  const int64_t tslot = cap ? w0->tev_recorded % cap : 0;
  if (cap) CO2_CUDA(cudaEventRecord(w0->tev[2 * tslot], st));
  CO2_TRY(local_round_impl(w0->mode, g, w0->n, x0, p0, p1, m, an, pr, gp, cur, wsp, nullptr,
                           e->dev_diag + slot, xbar, avg_out, hyper,
                           reinterpret_cast<unsigned long long*>(e->dev_ts + 2 * slot), st));
  for (int i = 0; i < g; ++i) ws[i]->diag_on_device = true;  // co2_round_finish fetches
  if (cap) {
    CO2_CUDA(cudaEventRecord(w0->tev[2 * tslot + 1], st));
    w0->tev_recorded += 1;
  }
  CO2_CUDA(cudaEventRecord(h.fin, st));
  h.done_stream = st;
  e->handles.push_back(h);
  e->live += 1;
  const uint64_t launched = e->handles.size() - 1;
  for (int i = 0; i < g; ++i) {
    co2_worker* w = ws[i];
    std::swap(w->anchor, w->prev_x0);  // anchor <- x_{t+1,0}; prev_x0 <- x_{t,0}
    std::swap(w->prev_x1, w->xfirst);  // prev_x1 <- x_{t,1}
    w->cur = 1 - w->cur;
    w->xbar = xbar;
    w->consumed = prev;
    w->has_consumed = true;
    w->pending = launched;
    w->t += 1;
  }
  co2_round_result_t r{};
  r.min_gap = INFINITY;
  r.outer_applied = 1;
  if (sync) {
    co2_status_t s1 = co2_round_finish(ws, g, stream, &r);
    double stall = 0.0;
    co2_status_t s2 = co2_aar_stall(e, prev, &stall, nullptr);
    r.stall_seconds = stall;
    if (res) *res = r;
    if (s1 != CO2_OK) return s1;
    return s2;
  }
  if (res) *res = r;
  return CO2_OK;
}

extern "C" co2_status_t co2_round(co2_worker_t* const* ws, int32_t g, co2_aar_t* e,
                                  const co2_hyper_t* hyper, void* stream, int32_t sync,
                                  co2_round_result_t* res) {
  // co2_round, proj/src/outer_algorithms.cpp:110-211
  CO2_TRY(co2_hyper_validate(hyper));  // :115
  CO2_TRY(check_round_args(ws, g, e, "co2_round"));
  if (hyper->tau < 1) return fail(CO2_ERR_VALIDATION, "staleness_gap: tau must be >= 1");
  if (g != (e->transport == T_LOCAL ? e->workers : 1))
    return fail(CO2_ERR_VALIDATION,
                "launch_all_reduce: contribution count %d does not match worker count %d", g,
                e->transport == T_LOCAL ? e->workers : 1);
  co2_worker* w0 = ws[0];
  const co2_mode_t mode = w0->mode;
  const int64_t n = w0->n;
  for (int i = 0; i < g; ++i) {
    if (ws[i]->mode != mode || ws[i]->n != n)
      return fail(CO2_ERR_VALIDATION, "staleness_gap: dimensions differ");
    if (ws[i]->t != w0->t || ws[i]->has_pending != w0->has_pending ||
        (w0->has_pending && ws[i]->pending != w0->pending))
      return fail(CO2_ERR_VALIDATION, "outer round: pending handles diverged");
  }
  if (hyper->ghost_consistent && e->transport != T_LOCAL && e->world > 1)
    return fail(CO2_ERR_VALIDATION,
                "co2_round: ghost-consistent mode over NCCL runs in the sharded driver");
  cudaStream_t st = S(stream);
  const co2_dtype_t sdt = state_dtype(mode), ldt = low_dtype(mode);
  const size_t sb = state_bytes(mode) * n, lb = low_bytes(mode) * n;
  const bool local = e->transport == T_LOCAL;
  co2_round_result_t r{};
  r.min_gap = INFINITY;
  if (local && w0->t > 0 && !hyper->ghost_consistent && g <= kMaxLocalRound && w0->avg[0] &&
      local_round_fused_enabled()) {
    bool coord = true;
    for (int i = 0; i < g; ++i) coord = coord && ws[i]->clip_mode == CO2_CLIP_COORDINATE;
    if (coord) return local_round_fused(ws, g, e, hyper, stream, sync, res);
  }

  // 1. Launch the reduce of x_{t,tau} (:120).
  if (local && !w0->avg[0]) {
    CO2_TRY(walloc(&w0->avg[0], lb));
    CO2_TRY(walloc(&w0->avg[1], lb));
  }
  if (w0->t == 0) {
    // Round 0 keeps x_{1,0} = x_{0,tau} worker-local, but the reduce about
    // to be launched owns params[cur] (NCCL reduces it in place): copy the
    // params to the other buffer first, so the launch fence orders the copy
    // before the collective touches the buffer.
    for (int i = 0; i < g; ++i)
      CO2_TRY(copy_dev(ws[i]->params[1 - ws[i]->cur], ws[i]->params[ws[i]->cur], lb, st));
  }
  if (w0->t > 0 && e->transport == T_P2P && e->fused && !hyper->ghost_consistent) {
    // Fused schedule (t >= 1): ONE kernel consumes the average reduced by the
    // previous launch (in params[1-cur]) for the outer step AND averages this
    // round's x_{t,tau} (params[cur]) over NVLink for the next round -- the
    // compute and the collective share the HBM stream instead of competing
    // as two kernels on two streams.
    co2_worker* w = w0;
    if (w->clip_mode != CO2_CLIP_COORDINATE)
      return fail(CO2_ERR_VALIDATION,
                  "global-norm clip: not available with the fused all-reduce schedule");
    if (!w->fused_err) {
      CO2_CUDA(cudaMallocHost(&w->fused_err, sizeof(uint32_t)));
      *w->fused_err = 0;
    }
    if (*w->fused_err)  // an earlier async round's barrier timed out
      return fail(CO2_ERR_CUDA, "p2p fused step: cross-GPU barrier timed out (code %u)",
                  *w->fused_err);
    if (w->has_pending) {  // the round-0 reduce (standalone P2P kernel)
      int32_t done = 0;
      CO2_TRY(co2_aar_poll(e, w->pending, &done));
      CO2_TRY(co2_aar_wait(e, w->pending, stream));
      w->has_pending = false;
    }
    const P2PBuffer* pb = find_p2p(e, w->params[w->cur]);
    if (!pb) return fail(CO2_ERR_VALIDATION, "launch_all_reduce: buffer not registered for P2P");
    const int64_t shard = ((n + e->world - 1) / e->world + 7) / 8 * 8;
    const int64_t lo = std::min<int64_t>((int64_t)e->rank * shard, n);
    const int64_t len = std::max<int64_t>(0, std::min<int64_t>(shard, n - lo));
    void* out_params = w->params[1 - w->cur];
    e->fused_epoch += 1;
    const int64_t cap = (int64_t)w->tev.size() / 2;
    const int64_t slot = cap ? w->tev_recorded % cap : 0;
    if (cap) CO2_CUDA(cudaEventRecord(w->tev[2 * slot], st));
    CO2_TRY(outer_step_fused_aar_impl(mode, n, w->anchor, w->prev_x0, w->prev_x1, out_params,
                                      w->m, w->prev_x0, out_params, w->gap, hyper,
                                      pb->ptrs.data(), lo, len, e->peer_signals.data(), e->world,
                                      e->rank, e->fused_epoch, w->ws, st,
                                      w->keep_avg ? w->avg_keep : nullptr));
    if (cap) {
      CO2_CUDA(cudaEventRecord(w->tev[2 * slot + 1], st));
      w->tev_recorded += 1;
    }
    CO2_TRY(diag_to_host(w->ws, w->host_diag, stream));
    CO2_TRY(copy_words_to_host(static_cast<char*>(e->signals) + p2p_signal_error_offset(),
                               w->fused_err, 4, st));
    std::swap(w->anchor, w->prev_x0);
    std::swap(w->prev_x1, w->xfirst);
    w->cur = 1 - w->cur;
    w->xbar = w->keep_avg ? w->avg_keep : nullptr;
    w->t += 1;
    r.outer_applied = 1;
    if (sync) {
      co2_status_t s = co2_round_finish(ws, g, stream, &r);  // checks fused_err too
      if (res) *res = r;
      return s;
    }
    if (res) *res = r;
    return CO2_OK;
  }
  const void* bufs[64];
  for (int i = 0; i < g; ++i) bufs[i] = ws[i]->params[ws[i]->cur];
  void* avg_out = local ? w0->avg[w0->t % 2] : const_cast<void*>(bufs[0]);
  uint64_t launched = 0;
  CO2_TRY(co2_aar_launch(e, ldt, bufs, avg_out, n, stream, &launched));

  if (w0->t == 0) {
    // 2. Round 0 (:122-151): snapshots only; continue on the copied buffer
    // and seed the anchor x_{1,0}.
    for (int i = 0; i < g; ++i) {
      co2_worker* w = ws[i];
      std::swap(w->prev_x0, w->anchor);  // prev_x0 <- x_{0,0}
      std::swap(w->prev_x1, w->xfirst);  // prev_x1 <- x_{0,1}
      w->cur = 1 - w->cur;
    }
    if (hyper->ghost_consistent && g > 1) {  // :133-145 averaged snapshots
      std::vector<const void*> s0(g), s1(g);
      for (int i = 0; i < g; ++i) {
        s0[i] = ws[i]->prev_x0;
        s1[i] = ws[i]->prev_x1;
      }
      if (!w0->tmp_state) CO2_TRY(walloc(&w0->tmp_state, sb));
      if (!w0->tmp_low) CO2_TRY(walloc(&w0->tmp_low, lb));
      CO2_TRY(co2_average(sdt, g, s0.data(), n, w0->tmp_state, w0->ws, stream));
      CO2_TRY(diag_to_host(w0->ws, w0->host_diag, stream));
      CO2_TRY(co2_average(ldt, g, s1.data(), n, w0->tmp_low, w0->ws, stream));
      CO2_TRY(diag_to_host(w0->ws, ws[g - 1]->host_diag, stream));
      for (int i = 0; i < g; ++i) {
        CO2_TRY(copy_dev(ws[i]->prev_x0, w0->tmp_state, sb, st));
        CO2_TRY(copy_dev(ws[i]->prev_x1, w0->tmp_low, lb, st));
      }
    } else {
      for (int i = 0; i < g; ++i) {
        ws[i]->host_diag->flags = 0;
        ws[i]->host_diag->min_gap = INFINITY;
        ws[i]->host_diag->max_outer_step = 0.0;
        ws[i]->host_diag->n_clipped = ws[i]->host_diag->n_floored = 0;
      }
    }
    for (int i = 0; i < g; ++i) {
      co2_worker* w = ws[i];
      CO2_TRY(co2_convert(sdt, w->anchor, ldt, w->params[w->cur], n, stream));  // x_{1,0}
      w->pending = launched;
      w->has_pending = true;
      w->t = 1;
    }
    r.outer_applied = 0;
    if (sync) {
      CO2_CUDA(cudaStreamSynchronize(st));
      if (hyper->ghost_consistent && g > 1) {
        for (co2_diag_t* d : {w0->host_diag, ws[g - 1]->host_diag})
          if (d->flags) return co2_diag_status(d);
      }
    }
    if (res) *res = r;
    return CO2_OK;
  }

  // 3. Rounds t >= 1: poll, then wait on the previous reduce (:153-159).
  if (!w0->has_pending)  // shared_pending, outer_algorithms.cpp:22-26
    return fail(CO2_ERR_VALIDATION, "outer round: no pending reduce to consume");
  const uint64_t prev = w0->pending;
  int32_t done = 0;
  CO2_TRY(co2_aar_poll(e, prev, &done));
  CO2_TRY(co2_aar_wait(e, prev, stream));
  const int t = w0->t;
  void* xbar = local ? w0->avg[(t - 1) % 2] : ws[0]->params[1 - ws[0]->cur];
  // NCCL delivers the worker sum (divided once in the step); LOCAL and P2P
  // deliver the fixed-order average itself.
  const int32_t divisor = reduce_divisor(e);

  if (hyper->ghost_consistent && g > 1) {
    // :161-184 -- one shared state driven by the averaged snapshots.
    std::vector<const void*> s0(g), s1(g);
    for (int i = 0; i < g; ++i) {
      s0[i] = ws[i]->anchor;
      s1[i] = ws[i]->xfirst;
    }
    if (!w0->tmp_state) CO2_TRY(walloc(&w0->tmp_state, sb));
    if (!w0->tmp_low) CO2_TRY(walloc(&w0->tmp_low, lb));
    CO2_TRY(co2_average(sdt, g, s0.data(), n, w0->tmp_state, w0->ws, stream));  // bar0
    CO2_TRY(co2_average(ldt, g, s1.data(), n, w0->tmp_low, ws[g - 1]->ws, stream));  // bar1
    co2_worker* w = w0;
    void* out_params = w->params[1 - w->cur];
    CO2_TRY(step_launch(w, mode, n, w0->tmp_state, w->prev_x0, w->prev_x1, xbar, divisor, w->m,
                        w->prev_x0, out_params, w->gap, hyper, st));
    CO2_TRY(diag_to_host(w->ws, w->host_diag, stream));
    // Rotation: anchor <- x_{t+1,0} (written over prev_x0), prev_x0 <- bar0,
    // prev_x1 <- bar1.
    void* old_anchor = w->anchor;
    w->anchor = w->prev_x0;
    w->prev_x0 = w0->tmp_state;
    w0->tmp_state = old_anchor;
    void* old_p1 = w->prev_x1;
    w->prev_x1 = w0->tmp_low;
    w0->tmp_low = old_p1;
    w->cur = 1 - w->cur;
    for (int i = 1; i < g; ++i) {
      co2_worker* v = ws[i];
      CO2_TRY(copy_dev(v->m, w->m, sb, st));
      if (v->gap && w->gap) CO2_TRY(copy_dev(v->gap, w->gap, sb, st));
      CO2_TRY(copy_dev(v->prev_x0, w->prev_x0, sb, st));
      CO2_TRY(copy_dev(v->prev_x1, w->prev_x1, lb, st));
      CO2_TRY(copy_dev(v->anchor, w->anchor, sb, st));
      v->cur = 1 - v->cur;
      CO2_TRY(copy_dev(v->params[v->cur], w->params[w->cur], lb, st));
      v->host_diag->flags = 0;
      v->host_diag->min_gap = INFINITY;
      v->host_diag->max_outer_step = 0.0;
      v->host_diag->n_clipped = v->host_diag->n_floored = 0;
    }
  } else {
    // :185-203 -- per-worker fused step; rotation is a pointer swap.
    for (int i = 0; i < g; ++i) {
      co2_worker* w = ws[i];
      void* out_params = w->params[1 - w->cur];
      void* xb = local ? xbar : out_params;  // NCCL / P2P: the reduce lives in the other buffer
      void* keep = (!local && w->keep_avg) ? w->avg_keep : nullptr;
      CO2_TRY(step_launch(w, mode, n, w->anchor, w->prev_x0, w->prev_x1, xb, divisor, w->m,
                          w->prev_x0, out_params, w->gap, hyper, st, keep));
      // the sum algorithm delivered the worker sum: keep the average
      if (keep && divisor > 1) CO2_TRY(scale_div_impl(ldt, keep, n, divisor, st));
      CO2_TRY(diag_to_host(w->ws, w->host_diag, stream));
      std::swap(w->anchor, w->prev_x0);  // anchor <- x_{t+1,0}; prev_x0 <- x_{t,0}
      std::swap(w->prev_x1, w->xfirst);  // prev_x1 <- x_{t,1}
      w->cur = 1 - w->cur;
    }
  }
  for (int i = 0; i < g; ++i) {
    // in-place transports overwrite the reduce with x_{t+1,0}: readable only
    // through the keep-average copy
    ws[i]->xbar = local ? xbar : (ws[i]->keep_avg ? ws[i]->avg_keep : nullptr);
    ws[i]->consumed = prev;
    ws[i]->has_consumed = true;
    ws[i]->pending = launched;
    ws[i]->t += 1;
  }
  r.outer_applied = 1;
  if (sync) {
    co2_status_t s = co2_round_finish(ws, g, stream, &r);
    double stall = 0.0;
    co2_status_t s2 = co2_aar_stall(e, prev, &stall, nullptr);
    r.stall_seconds = stall;
    if (res) *res = r;
    if (s != CO2_OK) return s;
    return s2;
  }
  if (res) *res = r;
  return CO2_OK;
}

// ============================================================ sharded (C4)
// Ghost-consistent CO2 (outer_algorithms.cpp:126-145,161-184) with the outer
// state sharded across ranks: every worker shares one outer state, so rank r
// keeps only coordinates [r*shard, (r+1)*shard) of x_{t,0}, prev_x0,
// prev_x1, momentum and gap.
struct co2_sharded {
  co2_mode_t mode = CO2_MODE_F32;
  int64_t n = 0, n_pad = 0, shard = 0, offset = 0, length = 0;
  int world = 1, rank = 0;
  int t = 0, cur = 0;
  void* params[2] = {nullptr, nullptr};  // full, low dtype, n_pad
  void* xfirst = nullptr;                // full, low dtype
  void* anchor = nullptr;                // shard, state
  void* prev_x0 = nullptr;               // shard, state
  void* m = nullptr;                     // shard, state
  void* gap = nullptr;                   // shard, state
  void* p1sum[2] = {nullptr, nullptr};   // shard, low: sum over workers of x_{t,1}
  void* xsum[2] = {nullptr, nullptr};    // shard, low: sum over workers of x_{t,tau}
  void* xbar = nullptr;
  void* ws = nullptr;
  co2_diag_t* host_diag = nullptr;
  cudaEvent_t sync_ev = nullptr;
  bool has_pending = false;
  bool started = false;
  uint64_t pending = 0;
  std::vector<cudaEvent_t> tev;
  int64_t tev_recorded = 0, tev_read = 0;
  // P2P transport: fixed-order slice averages (p1sum / xsum then hold the
  // averages, divisor 1), ping-pong x_{t,1} snapshots read asynchronously,
  // and the fused step's all-gather epoch.
  bool p2p = false;
  void* xfirst2 = nullptr;
  void* xfirst_cur() { return (t % 2 == 0 || !p2p) ? xfirst : xfirst2; }
  void* xfirst_alt() { return (t % 2 == 0) ? xfirst2 : xfirst; }
};

static co2_status_t ensure_comm2(co2_aar* e) {
  if (e->transport != T_NCCL)
    return fail(CO2_ERR_VALIDATION, "sharded outer state: NCCL transport only");
  if (e->world > 1 && !e->comm2) CO2_NCCL(ncclCommSplit(e->comm, 0, e->rank, &e->comm2, nullptr));
  return CO2_OK;
}

// Blocking (stream-ordered) collectives on the caller's stream over comm2.
static co2_status_t rs_blocking(co2_aar* e, co2_dtype_t dt, const void* full, void* shard_out,
                                int64_t shard, cudaStream_t st) {
  if (shard <= 0) return CO2_OK;
  if (e->world > 1 && !e->nccl_sum) {
    if (!e->ws2) {
      CO2_CUDA(cudaMalloc(&e->ws2, co2_workspace_bytes()));
      CO2_CUDA(cudaMemsetAsync(e->ws2, 0, co2_workspace_bytes(), st));
    }
    CO2_TRY(nccl_fixed_rs(e, e->comm2, 1, dt, full, shard * e->world, shard, shard_out, e->ws2,
                          st));
  } else if (e->world > 1)
    CO2_NCCL(ncclReduceScatter(full, shard_out, (size_t)shard, nccl_dtype(dt), ncclSum, e->comm2,
                               st));
  else
    CO2_CUDA(cudaMemcpyAsync(shard_out, full, dtype_bytes(dt) * (size_t)shard,
                             cudaMemcpyDeviceToDevice, st));
  return CO2_OK;
}

static co2_status_t ag_inplace(co2_aar* e, co2_dtype_t dt, void* full, int64_t shard,
                               cudaStream_t st) {
  if (shard <= 0 || e->world == 1) return CO2_OK;
  char* base = static_cast<char*>(full);
  CO2_NCCL(ncclAllGather(base + (size_t)e->rank * shard * dtype_bytes(dt), full, (size_t)shard,
                         nccl_dtype(dt), e->comm2, st));
  return CO2_OK;
}

extern "C" co2_status_t co2_sharded_create(co2_sharded_t** out, co2_mode_t mode, int64_t n,
                                           co2_aar_t* e, const void* init, int32_t keep_gap,
                                           void* stream) {
  if (!e) return fail(CO2_ERR_VALIDATION, "sharded: null engine");
  if (n < 0) return fail(CO2_ERR_VALIDATION, "sharded: negative dimension");
  if (mode != CO2_MODE_F64 && mode != CO2_MODE_F32 && mode != CO2_MODE_BF16_MIXED)
    return fail(CO2_ERR_VALIDATION, "sharded: unknown mode %d", (int)mode);
  const bool p2p = e->transport == T_P2P;
  if (!p2p) CO2_TRY(ensure_comm2(e));
  co2_sharded* s = new co2_sharded();
  s->p2p = p2p;
  s->mode = mode;
  s->n = n;
  s->world = e->world;
  s->rank = e->rank;
  // 8-element (16-byte bf16) aligned shards, equal capacity for NCCL.
  const int64_t per = ((n + s->world - 1) / s->world + 7) / 8 * 8;
  s->shard = per;
  s->n_pad = per * s->world;
  s->offset = (int64_t)s->rank * per;
  s->length = std::max<int64_t>(0, std::min<int64_t>(per, n - s->offset));
  const size_t sb = state_bytes(mode), lb = low_bytes(mode);
  co2_status_t st = CO2_OK;
  auto A = [&](void** p, size_t b) {
    if (st == CO2_OK) st = walloc(p, b);
  };
  A(&s->params[0], lb * s->n_pad);
  A(&s->params[1], lb * s->n_pad);
  A(&s->xfirst, lb * s->n_pad);
  if (p2p) A(&s->xfirst2, lb * s->n_pad);
  A(&s->anchor, sb * per);
  A(&s->prev_x0, sb * per);
  A(&s->m, sb * per);
  if (keep_gap) A(&s->gap, sb * per);
  A(&s->p1sum[0], lb * per);
  A(&s->p1sum[1], lb * per);
  A(&s->xsum[0], lb * per);
  A(&s->xsum[1], lb * per);
  A(&s->ws, co2_workspace_bytes());
  if (st != CO2_OK) {
    co2_sharded_destroy(s);
    return st;
  }
  cudaStream_t cs = S(stream);
  CO2_CUDA(cudaMallocHost(&s->host_diag, sizeof(co2_diag_t)));
  CO2_CUDA(cudaEventCreateWithFlags(&s->sync_ev, cudaEventDisableTiming));
  CO2_CUDA(cudaMemsetAsync(s->ws, 0, co2_workspace_bytes(), cs));
  CO2_CUDA(cudaMemsetAsync(s->m, 0, sb * per, cs));
  CO2_CUDA(cudaMemsetAsync(s->params[0], 0, lb * s->n_pad, cs));
  CO2_CUDA(cudaMemsetAsync(s->params[1], 0, lb * s->n_pad, cs));
  CO2_CUDA(cudaMemsetAsync(s->xfirst, 0, lb * s->n_pad, cs));
  if (init && n > 0) CO2_CUDA(cudaMemcpyAsync(s->params[0], init, lb * n, cudaMemcpyDeviceToDevice, cs));
  if (s->gap && mode == CO2_MODE_F64) {
    std::vector<double> ones(per, 1.0);
    CO2_CUDA(cudaMemcpy(s->gap, ones.data(), sb * per, cudaMemcpyHostToDevice));
  } else if (s->gap) {
    CO2_TRY(co2_fill_u32(s->gap, 0x3f800000u, per, stream));
  }
  *out = s;
  return CO2_OK;
}

extern "C" co2_status_t co2_sharded_destroy(co2_sharded_t* s) {
  if (!s) return CO2_OK;
  for (void* p : {s->params[0], s->params[1], s->xfirst, s->xfirst2, s->anchor, s->prev_x0, s->m, s->gap,
                  s->p1sum[0], s->p1sum[1], s->xsum[0], s->xsum[1], s->ws})
    if (p) cudaFree(p);
  if (s->host_diag) cudaFreeHost(s->host_diag);
  if (s->sync_ev) cudaEventDestroy(s->sync_ev);
  for (cudaEvent_t ev : s->tev) cudaEventDestroy(ev);
  delete s;
  return CO2_OK;
}

extern "C" void* co2_sharded_buffer(co2_sharded_t* s, int32_t which) {
  if (!s) return nullptr;
  switch (which) {
    case CO2_BUF_PARAMS: return s->params[s->cur];
    case CO2_BUF_XFIRST: return s->xfirst_cur();
    case CO2_BUF_PARAMS_ALT: return s->params[1 - s->cur];
    case CO2_BUF_XFIRST_ALT: return s->p2p ? s->xfirst_alt() : nullptr;
    case CO2_BUF_ANCHOR: return s->anchor;
    case CO2_BUF_PREV_X0: return s->prev_x0;
    case CO2_BUF_PREV_X1: return s->t > 0 ? s->p1sum[(s->t - 1) % 2] : nullptr;
    case CO2_BUF_MOMENTUM: return s->m;
    case CO2_BUF_GAP: return s->gap;
    case CO2_BUF_XBAR: return s->xbar;
  }
  return nullptr;
}

extern "C" int64_t co2_sharded_shard(const co2_sharded_t* s, int64_t* offset, int64_t* length) {
  if (!s) return 0;
  if (offset) *offset = s->offset;
  if (length) *length = s->length;
  return s->shard;
}

extern "C" co2_status_t co2_sharded_snapshot_start(co2_sharded_t* s, void* stream) {
  // InnerTrace::x_start (inner_loop.cpp:73).  Round 0 only: every worker
  // starts from the same init, so the ghost snapshot average of :133-145 is
  // the average of identical copies of this shard of x_{0,0}.  For t >= 1 the
  // step itself maintains x_{t,0} (anchor) and prev_x0.
  if (!s) return fail(CO2_ERR_VALIDATION, "sharded: null");
  if (s->t > 0) return CO2_OK;
  CO2_TRY(ghost_init_impl(s->mode, s->length,
                          static_cast<char*>(s->params[s->cur]) + low_bytes(s->mode) * s->offset,
                          s->anchor, s->prev_x0, s->world, S(stream)));
  s->started = true;
  return CO2_OK;
}

extern "C" co2_status_t co2_sharded_snapshot_first(co2_sharded_t* s, void* stream) {
  if (!s) return fail(CO2_ERR_VALIDATION, "sharded: null");
  if (s->n == 0) return CO2_OK;
  CO2_CUDA(cudaMemcpyAsync(s->xfirst_cur(), s->params[s->cur], low_bytes(s->mode) * s->n,
                           cudaMemcpyDeviceToDevice, S(stream)));
  return CO2_OK;
}

extern "C" co2_status_t co2_sharded_enable_timing(co2_sharded_t* s, int32_t cap) {
  if (!s || cap < 1) return fail(CO2_ERR_VALIDATION, "timing: bad arguments");
  for (cudaEvent_t ev : s->tev) cudaEventDestroy(ev);
  s->tev.assign(2 * (size_t)cap, nullptr);
  for (cudaEvent_t& ev : s->tev) CO2_CUDA(cudaEventCreate(&ev));
  s->tev_recorded = s->tev_read = 0;
  return CO2_OK;
}

extern "C" co2_status_t co2_sharded_step_times(co2_sharded_t* s, double* out, int32_t cap,
                                               int32_t* count) {
  if (!s) return fail(CO2_ERR_VALIDATION, "timing: null");
  const int64_t ring = (int64_t)s->tev.size() / 2;
  int64_t first = s->tev_read;
  if (ring && s->tev_recorded - first > ring) first = s->tev_recorded - ring;
  int32_t k = 0;
  for (int64_t i = first; ring && i < s->tev_recorded && k < cap; ++i) {
    const int64_t sl = i % ring;
    CO2_CUDA(cudaEventSynchronize(s->tev[2 * sl + 1]));
    float ms = 0.f;
    CO2_CUDA(cudaEventElapsedTime(&ms, s->tev[2 * sl], s->tev[2 * sl + 1]));
    if (out) out[k] = ms * 1e-3;
    ++k;
  }
  s->tev_read = s->tev_recorded;
  *count = k;
  return CO2_OK;
}

extern "C" co2_status_t co2_sharded_drain(co2_sharded_t* s, co2_aar_t* e, void* stream) {
  if (!s || !e) return fail(CO2_ERR_VALIDATION, "sharded: bad arguments");
  if (!s->has_pending) return CO2_OK;
  CO2_TRY(co2_aar_wait(e, s->pending, stream));
  s->has_pending = false;
  return CO2_OK;
}

// All-gather of the sharded P2P round (CO2_SHARD_AG = ce | fused): "fused"
// stores the x_{t+1,0} slice into every rank's params from the step kernel
// itself; "ce" lets the step write locally and the copy engines push it.
static bool shard_allgather_ce() {
  static const bool ce = [] {
    const char* v = getenv("CO2_SHARD_AG");
    return v && strcmp(v, "ce") == 0;
  }();
  return ce;
}

extern "C" co2_status_t co2_sharded_round(co2_sharded_t* s, co2_aar_t* e,
                                          const co2_hyper_t* hyper, void* stream, int32_t sync,
                                          co2_round_result_t* res) {
  CO2_TRY(co2_hyper_validate(hyper));  // outer_algorithms.cpp:115
  if (!s || !e) return fail(CO2_ERR_VALIDATION, "sharded: bad arguments");
  if (hyper->tau < 1) return fail(CO2_ERR_VALIDATION, "staleness_gap: tau must be >= 1");
  if (!hyper->ghost_consistent)
    return fail(CO2_ERR_VALIDATION, "sharded outer state requires ghost_consistent semantics");
  if (e->transport != (s->p2p ? T_P2P : T_NCCL) || e->world != s->world || e->rank != s->rank)
    return fail(CO2_ERR_VALIDATION, "sharded: engine does not match the shard layout");
  cudaStream_t st = S(stream);
  const co2_dtype_t ldt = low_dtype(s->mode);
  const size_t lb = low_bytes(s->mode);
  co2_round_result_t r{};
  r.min_gap = INFINITY;
  const int t = s->t;
  if (t == 0 && !s->started)
    return fail(CO2_ERR_VALIDATION, "sharded: snapshot_start must precede round 0");
  if (t == 0) {
    // x_{1,0} = x_{0,tau} stays worker-local: continue on the other buffer.
    CO2_CUDA(cudaMemcpyAsync(s->params[1 - s->cur], s->params[s->cur], lb * s->n_pad,
                             cudaMemcpyDeviceToDevice, st));
  }
  uint64_t launched = 0;
  if (s->p2p) {
    // bar1 (average of x_{t,1}) is first used as prev_x1 NEXT round, so it is
    // reduced asynchronously together with the one-step-stale x_{t,tau}: one
    // deterministic slice-average launch on the comm stream.
    CO2_TRY(launch_slice(e, ldt, s->params[s->cur], s->xfirst_cur(), s->xsum[t % 2],
                         s->p1sum[t % 2], s->offset, s->length, stream, &launched));
  } else {
    // bar1 of this round: the worker sum of x_{t,1} for this shard (consumed
    // as prev_x1 next round; the reference's average(firsts), :133-145/:167).
    CO2_TRY(rs_blocking(e, ldt, s->xfirst, s->p1sum[t % 2], s->shard, st));
    // The one-step-stale reduce of x_{t,tau}, scattered by shard (:120).
    const void* bufs[1] = {s->params[s->cur]};
    CO2_TRY(launch_impl(e, 1, ldt, bufs, s->xsum[t % 2], s->n_pad, stream, &launched));
  }
  if (t == 0) {
    // prev_x0 <- average(x_{0,0}) was computed by co2_sharded_snapshot_start.
    s->cur = 1 - s->cur;
    s->pending = launched;
    s->has_pending = true;
    s->t = 1;
    r.outer_applied = 0;
    if (sync) CO2_CUDA(cudaStreamSynchronize(st));
    if (res) *res = r;
    return CO2_OK;
  }
  if (!s->has_pending)
    return fail(CO2_ERR_VALIDATION, "outer round: no pending reduce to consume");
  const uint64_t prev = s->pending;
  int32_t done = 0;
  CO2_TRY(co2_aar_poll(e, prev, &done));
  CO2_TRY(co2_aar_wait(e, prev, stream));
  void* xsum = s->xsum[(t - 1) % 2];
  void* p1 = s->p1sum[(t - 1) % 2];
  char* out_params = static_cast<char*>(s->params[1 - s->cur]) + lb * s->offset;
  // Round 1: x_{1,0} = x_{0,tau} differ per worker and their average is the
  // consumed reduce itself; later rounds start from identical x_{t,0}.
  const int ghost_copies = t == 1 ? 0 : s->world;
  const int64_t cap = (int64_t)s->tev.size() / 2;
  const int64_t slot = cap ? s->tev_recorded % cap : 0;
  if (cap) CO2_CUDA(cudaEventRecord(s->tev[2 * slot], st));
  if (s->p2p) {
    // Fused step + all-gather: the x_{t+1,0} slice goes straight into every
    // rank's next params buffer over NVLink; the kernel's exit barrier makes
    // all slices visible before this stream's next work (the inner loop).
    const P2PBuffer* pb = find_p2p(e, s->params[1 - s->cur]);
    if (!pb) return fail(CO2_ERR_VALIDATION, "sharded: params not registered for P2P");
    std::vector<void*> outs(s->world);
    for (int p = 0; p < s->world; ++p) outs[p] = static_cast<char*>(pb->ptrs[p]) + lb * s->offset;
    e->shard_epoch += 1;
    if (shard_allgather_ce()) {
      // The step writes the x_{t+1,0} slice locally (the slice averages are
      // averages: divisors 1); the copy engines push it into every peer's
      // params; the exit barrier runs after the copies on this stream.
      CO2_TRY(outer_step_ghost_impl(s->mode, s->length, s->anchor, s->prev_x0, p1, 1, xsum, 1,
                                    ghost_copies, s->m, s->anchor, s->prev_x0, out_params, s->gap,
                                    hyper, s->ws, st));
      if (cap) CO2_CUDA(cudaEventRecord(s->tev[2 * slot + 1], st));  // the step kernel alone
      for (int p = 0; p < s->world; ++p)
        if (p != s->rank && s->length > 0)
          CO2_CUDA(cudaMemcpyAsync(outs[p], out_params, lb * (size_t)s->length,
                                   cudaMemcpyDeviceToDevice, st));
      CO2_TRY(p2p_barrier_launch(e->peer_signals.data(), s->world, s->rank, e->shard_epoch, st));
    } else {
      CO2_TRY(outer_step_ghost_p2p_impl(s->mode, s->length, s->anchor, s->prev_x0, p1, xsum,
                                        ghost_copies, s->m, s->anchor, s->prev_x0, outs.data(),
                                        e->peer_signals.data(), s->world, s->rank,
                                        e->shard_epoch, s->gap, hyper, s->ws, st));
      if (cap) CO2_CUDA(cudaEventRecord(s->tev[2 * slot + 1], st));
    }
  } else {
    CO2_TRY(outer_step_ghost_impl(s->mode, s->length, s->anchor, s->prev_x0, p1,
                                  reduce_divisor(e), xsum, reduce_divisor(e), ghost_copies,
                                  s->m, s->anchor, s->prev_x0, out_params, s->gap, hyper, s->ws,
                                  st));
  }
  if (cap) {
    if (!s->p2p) CO2_CUDA(cudaEventRecord(s->tev[2 * slot + 1], st));
    s->tev_recorded += 1;
  }
  CO2_TRY(diag_to_host(s->ws, s->host_diag, stream));
  // x_{t+1,0} for every worker: in-place all-gather of the updated shards.
  if (!s->p2p) CO2_TRY(ag_inplace(e, ldt, s->params[1 - s->cur], s->shard, st));
  s->xbar = xsum;
  s->cur = 1 - s->cur;
  s->pending = launched;
  s->t += 1;
  r.outer_applied = 1;
  if (sync) {
    CO2_CUDA(cudaStreamSynchronize(st));
    const co2_diag_t& d = *s->host_diag;
    r.min_gap = d.min_gap;
    r.max_outer_step = d.max_outer_step;
    r.n_clipped = d.n_clipped;
    r.n_floored = d.n_floored;
    double stall = 0.0;
    co2_status_t s2 = co2_aar_stall(e, prev, &stall, nullptr);
    r.stall_seconds = stall;
    if (res) *res = r;
    if (d.flags) return co2_diag_status(&d);
    return s2;
  }
  if (res) *res = r;
  return CO2_OK;
}

// ================================================ baseline round drivers
// SlowMo / Local-SGD (blocking reduce every round) and Overlap-Local-SGD
// (anchor correction consumed one round late), outer_algorithms.cpp:213-313,
// over the same worker state and CollectiveEngine as co2_round.
namespace {

co2_status_t check_workers(co2_worker_t* const* ws, int32_t g, co2_aar* e) {
  if (!e || !ws || g < 1) return fail(CO2_ERR_VALIDATION, "round: bad arguments");
  const int expect = e->transport == T_LOCAL ? e->workers : 1;
  if (g != expect)
    return fail(CO2_ERR_VALIDATION,
                "launch_all_reduce: contribution count %d does not match worker count %d", g,
                expect);
  for (int i = 1; i < g; ++i)
    if (ws[i]->mode != ws[0]->mode || ws[i]->n != ws[0]->n)
      return fail(CO2_ERR_VALIDATION, "round: worker dimensions differ");
  return CO2_OK;
}

// Launch the reduce of one buffer per worker; returns where the consumer
// reads it and with which divisor.
co2_status_t launch_reduce(co2_worker_t* const* ws, int32_t g, co2_aar* e,
                           const void* const* bufs, int slot, cudaStream_t st,
                           uint64_t* handle, const void** xbar, int32_t* divisor) {
  co2_worker* w0 = ws[0];
  const size_t lb = low_bytes(w0->mode) * w0->n;
  const bool local = e->transport == T_LOCAL;
  if (local && !w0->avg[0]) {
    CO2_TRY(walloc(&w0->avg[0], lb));
    CO2_TRY(walloc(&w0->avg[1], lb));
  }
  void* out = local ? w0->avg[slot] : const_cast<void*>(bufs[0]);
  CO2_TRY(co2_aar_launch(e, low_dtype(w0->mode), bufs, out, w0->n, st, handle));
  *xbar = out;
  *divisor = reduce_divisor(e);
  return CO2_OK;
}

co2_status_t finish_round(co2_worker_t* const* ws, int32_t g, cudaStream_t st, int32_t sync,
                          co2_round_result_t* r) {
  if (!sync) return CO2_OK;
  return co2_round_finish(ws, g, st, r);
}

}  // namespace

extern "C" co2_status_t co2_slowmo_round(co2_worker_t* const* ws, int32_t g, co2_aar_t* e,
                                         double alpha, double beta, void* stream, int32_t sync,
                                         co2_round_result_t* res) {
  CO2_TRY(check_round_args(ws, g, e, "slowmo_round"));
  // slowmo_round, outer_algorithms.cpp:213-240
  if (!(alpha > 0.0)) return fail(CO2_ERR_VALIDATION, "slowmo: alpha must be positive");
  if (beta < 0.0 || beta >= 1.0) return fail(CO2_ERR_VALIDATION, "slowmo: beta must lie in [0, 1)");
  CO2_TRY(check_workers(ws, g, e));
  cudaStream_t st = S(stream);
  const void* bufs[64];
  for (int i = 0; i < g; ++i) bufs[i] = ws[i]->params[ws[i]->cur];
  uint64_t h = 0;
  const void* xbar = nullptr;
  int32_t div = 1;
  CO2_TRY(launch_reduce(ws, g, e, bufs, 0, st, &h, &xbar, &div));
  int32_t done = 0;
  CO2_TRY(co2_aar_poll(e, h, &done));
  CO2_TRY(co2_aar_wait(e, h, stream));  // blocking: consumed in the same round
  for (int i = 0; i < g; ++i) {
    co2_worker* w = ws[i];
    // x_start = x_{t,0} (anchor); the new iterate is also the next anchor.
    CO2_TRY(slowmo_impl(w->mode, w->n, w->anchor, xbar, div, w->m, w->params[w->cur], w->anchor,
                        alpha, beta, w->ws, st));
    CO2_TRY(diag_to_host(w->ws, w->host_diag, stream));
    w->xbar = const_cast<void*>(xbar);
    w->t += 1;
  }
  co2_round_result_t r{};
  r.outer_applied = 1;
  CO2_TRY(finish_round(ws, g, st, sync, &r));
  if (sync) {
    double stall = 0.0;
    CO2_TRY(co2_aar_stall(e, h, &stall, nullptr));
    r.stall_seconds = stall;
  }
  if (res) *res = r;
  return CO2_OK;
}

extern "C" co2_status_t co2_local_sgd_round(co2_worker_t* const* ws, int32_t g, co2_aar_t* e,
                                            void* stream, int32_t sync,
                                            co2_round_result_t* res) {
  CO2_TRY(check_round_args(ws, g, e, "local_sgd_round"));
  // local_sgd_round, outer_algorithms.cpp:242-260
  CO2_TRY(check_workers(ws, g, e));
  cudaStream_t st = S(stream);
  const void* bufs[64];
  for (int i = 0; i < g; ++i) bufs[i] = ws[i]->params[ws[i]->cur];
  uint64_t h = 0;
  const void* xbar = nullptr;
  int32_t div = 1;
  CO2_TRY(launch_reduce(ws, g, e, bufs, 0, st, &h, &xbar, &div));
  int32_t done = 0;
  CO2_TRY(co2_aar_poll(e, h, &done));
  CO2_TRY(co2_aar_wait(e, h, stream));
  for (int i = 0; i < g; ++i) {
    co2_worker* w = ws[i];
    CO2_TRY(local_sgd_impl(w->mode, w->n, w->anchor, xbar, div, w->params[w->cur], w->anchor,
                           w->ws, st));
    CO2_TRY(diag_to_host(w->ws, w->host_diag, stream));
    w->xbar = const_cast<void*>(xbar);
    w->t += 1;
  }
  co2_round_result_t r{};
  r.outer_applied = 1;
  CO2_TRY(finish_round(ws, g, st, sync, &r));
  if (res) *res = r;
  return CO2_OK;
}

extern "C" co2_status_t co2_overlap_local_sgd_round(co2_worker_t* const* ws, int32_t g,
                                                    co2_aar_t* e, int32_t instant, void* stream,
                                                    int32_t sync, co2_round_result_t* res) {
  CO2_TRY(check_round_args(ws, g, e, "overlap_local_sgd_round"));
  // overlap_local_sgd_round, outer_algorithms.cpp:262-313.  The anchors are
  // reduced from a snapshot copy in each worker's spare params buffer, so the
  // next inner loop can keep mutating the working params.  `instant` selects
  // the reference's zero-cost-reduce behaviour (consumed in the same round,
  // :283-297); otherwise the reduce is consumed next round (:267-281).
  CO2_TRY(check_workers(ws, g, e));
  cudaStream_t st = S(stream);
  co2_worker* w0 = ws[0];
  const co2_mode_t mode = w0->mode;
  const int64_t n = w0->n;
  const size_t lb = low_bytes(mode) * n;
  bool applied = false;
  auto correct = [&](const void* xbar, int32_t div) -> co2_status_t {
    for (int i = 0; i < g; ++i) {
      co2_worker* w = ws[i];
      CO2_TRY(overlap_correction_impl(mode, n, w->params[w->cur], w->anchor, xbar, div, w->ws,
                                      st));
      CO2_TRY(diag_to_host(w->ws, w->host_diag, stream));
    }
    applied = true;
    return CO2_OK;
  };
  if (w0->has_pending) {  // :267-281
    const uint64_t prev = w0->pending;
    int32_t done = 0;
    CO2_TRY(co2_aar_poll(e, prev, &done));
    CO2_TRY(co2_aar_wait(e, prev, stream));
    const void* xbar = e->transport == T_LOCAL ? w0->avg[(w0->t + 1) % 2]
                                               : ws[0]->params[1 - ws[0]->cur];
    CO2_TRY(correct(xbar, reduce_divisor(e)));
    for (int i = 0; i < g; ++i) {
      ws[i]->has_pending = false;
      // LOCAL keeps the consumed average readable; in-place transports
      // overwrite it with the next anchor snapshot below.
      ws[i]->xbar = e->transport == T_LOCAL ? const_cast<void*>(xbar) : nullptr;
    }
  }
  // Fresh anchors (:284-288), snapshotted into the spare buffer for the reduce.
  const void* bufs[64];
  for (int i = 0; i < g; ++i) {
    co2_worker* w = ws[i];
    CO2_TRY(co2_convert(state_dtype(mode), w->anchor, low_dtype(mode), w->params[w->cur], n,
                        stream));
    CO2_TRY(copy_dev(w->params[1 - w->cur], w->params[w->cur], lb, st));
    bufs[i] = w->params[1 - w->cur];
  }
  uint64_t h = 0;
  const void* xbar = nullptr;
  int32_t div = 1;
  CO2_TRY(launch_reduce(ws, g, e, bufs, w0->t % 2, st, &h, &xbar, &div));
  if (instant) {  // :290-297
    int32_t done = 0;
    CO2_TRY(co2_aar_poll(e, h, &done));
    CO2_TRY(co2_aar_wait(e, h, stream));
    CO2_TRY(correct(xbar, div));
    for (int i = 0; i < g; ++i) ws[i]->xbar = const_cast<void*>(xbar);
  } else {
    for (int i = 0; i < g; ++i) {
      ws[i]->pending = h;
      ws[i]->has_pending = true;
    }
  }
  for (int i = 0; i < g; ++i) {
    ws[i]->t += 1;
    if (!applied) {
      ws[i]->host_diag->flags = 0;
      ws[i]->host_diag->min_gap = INFINITY;
      ws[i]->host_diag->max_outer_step = 0.0;
      ws[i]->host_diag->n_clipped = ws[i]->host_diag->n_floored = 0;
    }
  }
  co2_round_result_t r{};
  r.outer_applied = 1;  // :309 -- every overlap round counts as an outer update
  CO2_TRY(finish_round(ws, g, st, sync, &r));
  if (res) *res = r;
  return CO2_OK;
}
