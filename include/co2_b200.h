/*
 * co2_b200.h -- C ABI of the B200-native CO2 outer-step hot path.
 *
 * Drop-in boundary for the reference's C++ operator API (paths relative to
 * /root/reference/).  Each entry point names the reference interface it
 * replaces.  No exceptions and no torch/CUDA types cross this boundary: device
 * buffers are plain pointers, streams are `void*` (a cudaStream_t, NULL = the
 * legacy default stream), sizes are int64 element counts.
 *
 * Error convention (proj/include/co2sim/errors.hpp:8-20):
 *   CO2_ERR_VALIDATION (2) <-> validation_error   (CLI exit 2)
 *   CO2_ERR_NUMERIC    (3) <-> numeric_error      (CLI exit 3)
 * with co2_last_error() returning the reference's exact message text.
 * Host-checkable validation happens before any launch; numeric checks are
 * device flags read back by co2_diag_fetch / the synchronous entry points.
 *
 * Threading: every launch is asynchronous on the caller's stream.  A
 * workspace (device scratch for the deterministic block-reduction finish)
 * must not be used by two streams concurrently.  co2_last_error() is
 * thread-local.
 */
#ifndef CO2_B200_H
#define CO2_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CO2_ABI_VERSION 3  /* 2: 72-byte IPC export records (handle + offset);
                              3: HandleInfo audit fields, NCCL algorithm, xbar capture */

typedef int32_t co2_status_t;
enum {
  CO2_OK = 0,
  CO2_ERR_VALIDATION = 2, /* validation_error */
  CO2_ERR_NUMERIC = 3,    /* numeric_error */
  CO2_ERR_CUDA = 4,
  CO2_ERR_NCCL = 5
};

/* Storage/compute modes of the fused step.
 *   F64        every buffer fp64, fp64 arithmetic: bit-identical to the
 *              reference's fp64 semantics.
 *   F32        every buffer fp32, fp32 arithmetic.
 *   BF16_MIXED x_t0 / prev_x0 / momentum / anchor / gap fp32 ("state"),
 *              prev_x1 / xbar / params bf16 ("low"), fp32 arithmetic. */
typedef enum { CO2_MODE_F64 = 0, CO2_MODE_F32 = 1, CO2_MODE_BF16_MIXED = 2 } co2_mode_t;
typedef enum { CO2_DTYPE_F64 = 0, CO2_DTYPE_F32 = 1, CO2_DTYPE_BF16 = 2 } co2_dtype_t;

/* Device flag bits (OR over coordinates), mapped to the reference's error
 * precedence by co2_diag_status. */
enum {
  CO2_FLAG_GAP_NONFINITE = 1u,   /* outer_algorithms.cpp:62  numeric  */
  CO2_FLAG_GAP_BELOW_ONE = 2u,   /* outer_algorithms.cpp:81  validation */
  CO2_FLAG_M_NONFINITE = 4u,     /* outer_algorithms.cpp:88  numeric  */
  CO2_FLAG_CLIP_NONFINITE = 8u,  /* param_ops.cpp:41         numeric  */
  CO2_FLAG_X_NONFINITE = 16u,    /* outer_algorithms.cpp:106 numeric  */
  CO2_FLAG_AVG_NONFINITE = 32u,  /* param_ops.cpp:31         numeric  */
  CO2_FLAG_SLOWMO_M = 64u,       /* outer_algorithms.cpp:231 numeric  */
  CO2_FLAG_SLOWMO_X = 128u,      /* outer_algorithms.cpp:233 numeric  */
  CO2_FLAG_OVERLAP = 256u,       /* outer_algorithms.cpp:279 numeric  */
  CO2_FLAG_NORM_NONFINITE = 512u, /* global-norm clip extension numeric */
  CO2_FLAG_NONFINITE_INPUT = 1024u /* ensure_finite, param_ops.cpp:10-14 */
};

/* Co2Hyper (proj/include/co2sim/outer_algorithms.hpp:17-30) plus tau. */
typedef struct co2_hyper {
  double alpha, beta, phi, epsilon;
  int32_t tau;
  uint8_t penalty, clip, ghost_consistent, pad;
} co2_hyper_t;

/* Round diagnostics (RoundResult min_gap / max_outer_step,
 * outer_algorithms.hpp:63-69) plus decision counts and flags. */
typedef struct co2_diag {
  double min_gap;        /* +inf when n == 0 */
  double max_outer_step; /* max_j |x'_j - x_t0_j| */
  int64_t n_clipped;     /* coordinates with |m'| > phi (clip on) */
  int64_t n_floored;     /* coordinates with tau*|p1 - p0| < epsilon */
  uint32_t flags;
  uint32_t pad;
} co2_diag_t;

const char* co2_last_error(void);
int32_t co2_abi_version(void);

/* Co2Hyper::validate (proj/src/outer_algorithms.cpp:37-46). */
co2_status_t co2_hyper_validate(const co2_hyper_t* hyper);

/* ---- workspace -------------------------------------------------------- */
size_t co2_workspace_bytes(void);
/* Zero a caller-allocated device workspace (once, before first use). */
co2_status_t co2_workspace_init(void* workspace, void* stream);
/* Async copy of the last launch's diagnostics into host memory (pinned for
 * true asynchrony); valid after the stream is synchronized. */
co2_status_t co2_diag_fetch_async(const void* workspace, co2_diag_t* host_out, void* stream);
/* Synchronous: fetch, synchronize the stream, return co2_diag_status(). */
co2_status_t co2_diag_fetch(const void* workspace, co2_diag_t* host_out, void* stream);
/* Map flags to the reference's first error (precedence: staleness_gap
 * numeric, gap<1 validation, momentum numeric, clip input numeric,
 * outer_iterate numeric, average numeric). */
co2_status_t co2_diag_status(const co2_diag_t* diag);

/* ---- the fused outer step ---------------------------------------------- */
/* Replaces co2_round's per-worker body (proj/src/outer_algorithms.cpp:186-202):
 *   staleness_gap (outer_algorithms.hpp:37-38) -> delta = prev_x0 - xbar
 *   (cpp:189) -> penalized_momentum_update (hpp:43-46) -> outer_iterate
 *   (hpp:49-50) -> min_gap / max_outer_step (cpp:194-196),
 * in ONE pass over HBM.  xbar is the consumed all-reduce: the average
 * (xbar_divisor = 1) or the worker sum (xbar_divisor = G; divided once, as
 * average() does, param_ops.cpp:30).  momentum is updated in place.
 * anchor_out (state dtype) receives x_{t+1,0} and may alias prev_x0 (the
 * snapshot rotation then becomes a pointer swap); params_out (low dtype)
 * receives x_{t+1,0} and may alias xbar.  gap_out (state dtype) receives
 * Lambda (fixture / debug only).  Any of the three outputs may be NULL.
 * Asynchronous; diagnostics land in the workspace. */
co2_status_t co2_outer_step(co2_mode_t mode, int64_t n, const void* x_t0, const void* prev_x0,
                            const void* prev_x1, const void* xbar, int32_t xbar_divisor,
                            void* momentum, void* anchor_out, void* params_out, void* gap_out,
                            const co2_hyper_t* hyper, void* workspace, void* stream);

/* EXTENSION, outside the reference parity contract (the reference clips
 * coordinate-wise, param_ops.cpp:35-43; SURVEY.md 8 note 3): the outer step
 * with a GLOBAL-norm clip of the outer momentum, as the north star words it.
 * Same buffers and hyper as co2_outer_step; with hyper->clip set,
 *   c = m' * min(1, phi / ||m'||_2),  x' = x_t0 - alpha * c,
 * where ||m'||_2 is summed in fp64 over fixed chunks in a fixed order (two
 * kernels, deterministic for a given n and mode on any grid).  With clip
 * off it equals co2_outer_step bit for bit.  n_clipped counts coordinates
 * that were scaled (0 or n).  Async on `stream`; read the diagnostics with
 * co2_diag_fetch and the norm with co2_global_clip_norm_fetch. */
co2_status_t co2_outer_step_global_clip(co2_mode_t mode, int64_t n, const void* x_t0,
                                        const void* prev_x0, const void* prev_x1,
                                        const void* xbar, int32_t xbar_divisor, void* momentum,
                                        void* anchor_out, void* params_out, void* gap_out,
                                        const co2_hyper_t* hyper, void* workspace, void* stream);
/* Clip mode of a worker's co2_round step: CO2_CLIP_COORDINATE is the
 * reference (default); CO2_CLIP_GLOBAL_NORM runs co2_outer_step_global_clip
 * instead (the extension above; not with the fused P2P schedule). */
enum { CO2_CLIP_COORDINATE = 0, CO2_CLIP_GLOBAL_NORM = 1 };
/* ||m'||_2 of the last co2_outer_step_global_clip on this workspace
 * (synchronizes `stream`). */
co2_status_t co2_global_clip_norm_fetch(const void* workspace, double* norm_out, void* stream);
/* The fixed summation chunk (coordinates) that pass 1 uses for n. */
int64_t co2_global_clip_chunk(co2_mode_t mode, int64_t n);

/* Tuning knob: select the fused kernel's instantiation (elements per vector,
 * vectors in flight per thread, CTAs per SM); 0 = the measured default.
 * Also settable once per process with CO2_FUSED_VARIANT.  See
 * tools/tune_fused.py. */
co2_status_t co2_set_fused_variant(int32_t variant);
/* Tuning knob: grid size of the step kernels in waves of the idle-GPU
 * resident CTA count (1 = persistent; the default 32 oversubscribes so the
 * block scheduler balances the tail and a co-running reduce kernel does
 * not leave a late second wave), in [1, 64].  Grids stop growing where a
 * CTA would get fewer than 8 grid-stride iterations (CO2_MIN_CTA_ITERS).
 * Also CO2_GRID_WAVES. */
co2_status_t co2_set_grid_waves(int32_t waves);

/* End-to-end form of co2_outer_step over HOST buffers (the reference's own
 * calling convention: host vectors in, host vectors out).  Streams the
 * coordinates through the GPU in chunks with H2D / compute / D2H overlapped
 * on `nstreams` streams (1..4).  Pinned host buffers give full PCIe speed.
 * Synchronous; returns the diagnostics' status and fills *diag_out. */
co2_status_t co2_outer_step_host(co2_mode_t mode, int64_t n, const void* x_t0,
                                 const void* prev_x0, const void* prev_x1, const void* xbar,
                                 int32_t xbar_divisor, void* momentum, void* anchor_out,
                                 void* params_out, const co2_hyper_t* hyper, int64_t chunk,
                                 int32_t nstreams, co2_diag_t* diag_out);

/* ---- unfused reference operators (per-op parity) ------------------------ */
/* All buffers of dtype dt; asynchronous; flags in the workspace.  Scalar
 * validation (tau, epsilon, beta, alpha, phi) happens here, before launch. */
/* staleness_gap: proj/include/co2sim/outer_algorithms.hpp:37-38 */
co2_status_t co2_staleness_gap(co2_dtype_t dt, int64_t n, const void* x_t0, const void* prev_x0,
                               const void* prev_x1, int32_t tau, double epsilon, void* gap_out,
                               void* workspace, void* stream);
/* penalized_momentum_update: outer_algorithms.hpp:43-46 */
co2_status_t co2_penalized_momentum(co2_dtype_t dt, int64_t n, const void* m_prev, double beta,
                                    const void* gap, const void* delta, int32_t penalty,
                                    void* m_out, void* workspace, void* stream);
/* outer_iterate: outer_algorithms.hpp:49-50 */
co2_status_t co2_outer_iterate(co2_dtype_t dt, int64_t n, const void* x_t0, double alpha,
                               const void* m, double phi, int32_t clip, void* x_out,
                               void* workspace, void* stream);
/* clip_elementwise: proj/include/co2sim/param_ops.hpp:23-24 */
co2_status_t co2_clip_elementwise(co2_dtype_t dt, int64_t n, const void* v, double phi,
                                  void* out, void* workspace, void* stream);
/* average: proj/include/co2sim/param_ops.hpp:16-21.  contributions is a
 * HOST array of g device pointers (g <= 64), summed in ascending index
 * order and divided by g once.  F64: fp64; F32: fp32; BF16: fp32
 * accumulation, one rounding to bf16. */
/* ensure_finite (param_ops.hpp:14, param_ops.cpp:10-14): numeric error
 * "non-finite value in <what>" if any of the n values is NaN or +-inf.
 * Synchronizes `stream`. */
co2_status_t co2_ensure_finite(co2_dtype_t dt, int64_t n, const void* v, const char* what,
                               void* workspace, void* stream);
/* elementwise_abs_diff (param_ops.cpp:44-51): out = |a - b|; numeric error
 * "non-finite value in elementwise_abs_diff".  Synchronizes `stream`. */
co2_status_t co2_elementwise_abs_diff(co2_dtype_t dt, int64_t n, const void* a, const void* b,
                                      void* out, void* workspace, void* stream);
/* l2_norm (param_ops.cpp:54-60): the Euclidean norm, squares summed in fp64
 * in a fixed order (the global-norm clip's chunked order, so it is
 * deterministic for a given n and dtype; the reference's Eigen reduction
 * order differs, so it agrees to fp64 rounding, not bitwise); numeric error
 * "l2_norm: non-finite result".  Synchronizes `stream`. */
co2_status_t co2_l2_norm(co2_dtype_t dt, int64_t n, const void* v, double* norm_out,
                         void* workspace, void* stream);
co2_status_t co2_average(co2_dtype_t dt, int32_t g, const void* const* contributions, int64_t n,
                         void* out, void* workspace, void* stream);
/* Round diagnostic of Simulation::step (outer_algorithms.cpp:503-508):
 * xbar = fixed-order average of the g workers' params, per_worker[i] =
 * ||params_i - xbar||_2 (fp64 accumulation, deterministic fixed-order
 * reduction), *max_out = max_i.  Synchronous; g <= 64.  Either output may
 * be NULL. */
co2_status_t co2_divergence(co2_dtype_t dt, int32_t g, const void* const* params, int64_t n,
                            double* per_worker, double* max_out, void* workspace, void* stream);
/* a - b elementwise (the delta of outer_algorithms.cpp:189) */
co2_status_t co2_sub(co2_dtype_t dt, int64_t n, const void* a, const void* b, void* out,
                     void* stream);
/* dst[j] = convert(src[j]) (snapshot copies, InnerTrace contract
 * proj/src/inner_loop.cpp:73,96-100) */
co2_status_t co2_convert(co2_dtype_t dst_dt, void* dst, co2_dtype_t src_dt, const void* src,
                         int64_t n, void* stream);

/* ---- synthetic inputs ------------------------------------ */
/* Counter-SplitMix64 generator of RngStream (proj/include/co2sim/rng.hpp:
 * 12-54) in random-access form; fills coordinates [j0, j0+count) of one
 * worker's buffers in the mode's storage dtypes.  Any pointer may be NULL. */
co2_status_t co2_synth(co2_mode_t mode, uint64_t seed, int32_t worker, int64_t j0, int64_t count,
                       void* x_t0, void* prev_x0, void* prev_x1, void* x_end, void* momentum,
                       void* stream);
/* Inner-step stand-in x <- x - lr * g with g = scale*(2U-1) drawn from the
 * counter stream (seed, (5<<32)|worker, draw offset j + step*n).  Used by
 * the schedule benchmarks as the local compute the all-reduce overlaps. */
co2_status_t co2_synthetic_inner_step(co2_dtype_t dt, int64_t n, void* params, double lr,
                                      double scale, uint64_t seed, int32_t worker, int64_t step,
                                      int32_t repeat, void* stream);
/* The same inner step with the InnerTrace x_{t,1} snapshot (inner_loop.cpp:
 * 96-98) fused into its store: pass the worker's
 * CO2_BUF_XFIRST as snapshot_out on the first inner step of a round instead
 * of calling co2_worker_snapshot_first (saves a read+write pass). */
co2_status_t co2_synthetic_inner_step_snapshot(co2_dtype_t dt, int64_t n, void* params,
                                               double lr, double scale, uint64_t seed,
                                               int32_t worker, int64_t step, int32_t repeat,
                                               void* snapshot_out, void* stream);
/* Fill a buffer with a constant (L2 flush helper for benchmarks). */
co2_status_t co2_fill_u32(void* dst, uint32_t value, int64_t count, void* stream);

/* ---- timing model (proj/src/timing_model.cpp:27-43,107-123) ------------- */
/* ClusterSpec (proj/include/co2sim/timing_model.hpp:14-25). */
typedef struct co2_cluster {
  int32_t workers, gpus_per_node;
  double t_comp, t_outer, param_bytes, inter_bandwidth, latency;
  int32_t has_measured_override;
  double measured_override;
} co2_cluster_t;
typedef struct co2_round_timing {
  int32_t t;
  double start, stall, end;
} co2_round_timing_t;
typedef struct co2_timeline {
  int32_t workers, tau, rounds, batch_size;
  double comm_time, wall_time, total_stall, overlap_ratio_achieved, throughput;
} co2_timeline_t;
co2_status_t co2_cluster_validate(const co2_cluster_t* spec);
co2_status_t co2_allreduce_time(const co2_cluster_t* spec, double* out);
co2_status_t co2_overlap_ratio(int32_t tau, double t_comp, double t_comm, double* out);
/* simulate_timeline(AlgorithmKind::co2, ...); per_round (nullable) must hold
 * `rounds` entries. */
co2_status_t co2_simulate_timeline_co2(const co2_cluster_t* spec, int32_t tau, int32_t rounds,
                                       int32_t batch_size, co2_timeline_t* out,
                                       co2_round_timing_t* per_round);
/* simulate_timeline for every AlgorithmKind (algorithm_kind.hpp:9,
 * timing_model.cpp:76-173); co2_simulate_timeline_co2 is kind CO2_ALG_CO2. */
enum {
  CO2_ALG_CO2 = 0,
  CO2_ALG_SLOWMO = 1,
  CO2_ALG_LOCAL_SGD = 2,
  CO2_ALG_OVERLAP_LOCAL_SGD = 3,
  CO2_ALG_SYNC_SGD = 4
};
co2_status_t co2_simulate_timeline(int32_t kind, const co2_cluster_t* spec, int32_t tau,
                                   int32_t rounds, int32_t batch_size, co2_timeline_t* out,
                                   co2_round_timing_t* per_round);
/* scalability_ratio (timing_model.cpp:45-53): throughput gain over worker
 * gain. */
co2_status_t co2_scalability_ratio(double throughput_small, double throughput_large,
                                   double workers_small, double workers_large, double* out);

/* ---- one-step-stale all-reduce engine (CollectiveEngine,
 *      proj/include/co2sim/collective.hpp:54-93) ----------------------------
 * A handle is launched after the compute stream's current work (event
 * fence), runs on the engine's own high-priority comm stream, and is
 * consumed exactly once by co2_aar_wait, which makes the consumer stream
 * wait on its completion event.  At most two handles are live (the
 * reference's overlap window, collective.cpp:39-42).
 * Transports:
 *   NCCL  one rank per GPU, in place.  Default algorithm CO2_NCCL_FIXED_ORDER:
 *         grouped ncclSend/ncclRecv slice exchange, the fixed-order average
 *         kernel on this rank's slice (ascending rank order, one division:
 *         average(), param_ops.cpp:16-33), grouped send/recv all-gather --
 *         the reference's average bit for bit at any world size, with a
 *         ring all-reduce's NVLink volume; the consumer uses divisor 1.
 *         CO2_NCCL_SUM: ncclAllReduce(sum) in the storage dtype (order and
 *         per-hop rounding are NCCL's), the consumer divides by world size.
 *   LOCAL G simulated workers on one GPU; fixed-order average kernel of the
 *         G contribution buffers into `out` (bitwise the reference average).
 */
typedef struct co2_aar co2_aar_t;
#define CO2_NCCL_ID_BYTES 128
co2_status_t co2_nccl_unique_id(uint8_t id_out[CO2_NCCL_ID_BYTES]);
co2_status_t co2_aar_create_nccl(co2_aar_t** out, const uint8_t id[CO2_NCCL_ID_BYTES],
                                 int32_t rank, int32_t world, int32_t max_ctas);
co2_status_t co2_aar_create_local(co2_aar_t** out, int32_t workers);
/* NCCL engines only; not while reduces are live.  Worker-local and sharded
 * rounds pick the matching consumer divisor themselves. */
enum { CO2_NCCL_FIXED_ORDER = 0, CO2_NCCL_SUM = 1 };
co2_status_t co2_aar_set_nccl_algo(co2_aar_t* engine, int32_t algo);
/* P2P transport: a deterministic fixed-order average
 * over NVLink peer memory.  Rank r reduces slice r from every rank's buffer
 * in ascending rank order, divides by G once (average(), param_ops.cpp:16-33)
 * and stores the result into slice r of every rank's buffer, so the result
 * is bitwise the reference's average for any G and the consumer uses
 * xbar_divisor = 1.  Setup (collective, same order on every rank):
 *   1. co2_aar_create_p2p;
 *   2. export co2_aar_signal_buffer with co2_ipc_export, exchange the
 *      handles (rank-indexed, world * CO2_IPC_HANDLE_BYTES), call
 *      co2_aar_p2p_attach_signals;
 *   3. for every buffer that will be reduced (e.g. both ping-pong params of
 *      a worker): export, exchange, co2_aar_p2p_attach.
 * `ctas` bounds the SMs the reduce occupies while it overlaps compute. */
/* An exported buffer: the CUDA IPC handle of the allocation that contains
 * dev_ptr (64 bytes) followed by dev_ptr's int64 byte offset in it, so
 * sub-allocated buffers (e.g. from a caching allocator) map correctly. */
#define CO2_IPC_HANDLE_BYTES 72
co2_status_t co2_ipc_export(const void* dev_ptr, uint8_t handle_out[CO2_IPC_HANDLE_BYTES]);
co2_status_t co2_aar_create_p2p(co2_aar_t** out, int32_t rank, int32_t world, int32_t ctas);
void* co2_aar_signal_buffer(co2_aar_t* engine);
co2_status_t co2_aar_p2p_attach_signals(co2_aar_t* engine, const uint8_t* handles);
co2_status_t co2_aar_p2p_attach(co2_aar_t* engine, const void* local_buf, const uint8_t* handles);
/* Undo co2_aar_p2p_attach for `local`: waits for this engine's reduces and
 * closes the peer mappings.  Every rank detaches the buffer, then the group
 * synchronises, before any rank frees it (peers must not read freed
 * memory). */
co2_status_t co2_aar_p2p_detach(co2_aar_t* engine, const void* local);
/* P2P only: run worker-local co2_round (t >= 1) as ONE kernel that does the
 * outer step on the previously reduced average AND the fixed-order NVLink
 * average of this round's x_{t,tau} (consumed next round, so the schedule
 * stays one step stale), with cross-GPU entry / exit barriers.  Results are
 * bitwise those of the two-kernel schedule; the reduce then overlaps the
 * outer step's HBM stream instead of the inner loop. */
co2_status_t co2_aar_set_fused(co2_aar_t* engine, int32_t on);
/* P2P: adaptive reduce occupancy (no reference counterpart; a runtime
 * policy of this transport).  When on, the all-reduce's CTA count follows
 * the measured slack of the consumed reduces between 16 and the SM count:
 * more CTAs after a reduce stalled its consumer, fewer while reduces finish
 * with more than half their duration to spare (fewer SMs taken from the
 * overlapped compute).  Results are unaffected.  Also the environment
 * variable CO2_P2P_ADAPT (1: on).
 * co2_aar_ctas reports the current count. */
co2_status_t co2_aar_set_adaptive(co2_aar_t* engine, int32_t on);
int32_t co2_aar_ctas(const co2_aar_t* engine);
co2_status_t co2_aar_destroy(co2_aar_t* engine);
int32_t co2_aar_world(const co2_aar_t* engine);
/* launch_all_reduce (collective.cpp:31-58).  NCCL: bufs[0] is reduced in
 * place (sum) and out must equal bufs[0] or be NULL.  LOCAL: bufs holds
 * `workers` device pointers, out receives the average. */
co2_status_t co2_aar_launch(co2_aar_t* engine, co2_dtype_t dt, const void* const* bufs,
                            void* out, int64_t n, void* producer_stream, uint64_t* handle_out);
/* is_completed (collective.cpp:74-86): non-blocking cudaEventQuery. */
co2_status_t co2_aar_poll(co2_aar_t* engine, uint64_t handle, int32_t* done);
/* wait (collective.cpp:88-105): consumer stream waits on completion;
 * consume-once.  Stall is measured on the device (events straddling the
 * wait) and is readable with co2_aar_stall once the consumer passed it. */
co2_status_t co2_aar_wait(co2_aar_t* engine, uint64_t handle, void* consumer_stream);
co2_status_t co2_aar_stall(co2_aar_t* engine, uint64_t handle, double* stall_seconds,
                           double* comm_seconds);
/* Make `stream` wait for the reduce to finish WITHOUT consuming the handle,
 * so the caller may overwrite the contributions afterwards (the reference's
 * launch snapshots them, collective.cpp:44-50; the C++ facade's value-
 * semantics launch_all_reduce uses this). */
co2_status_t co2_aar_order_after(co2_aar_t* engine, uint64_t handle, void* stream);
co2_status_t co2_aar_live(const co2_aar_t* engine, int32_t* live);
/* info(handle) (collective.hpp:40-50,68): HandleInfo from device events.
 * Times are seconds since engine creation; completion_time is valid once
 * `completed`, stall once `consumed` and the consumer stream passed the
 * wait (else NaN).  Never blocks. */
typedef struct co2_handle_info {
  uint64_t id;
  double launch_time, completion_time, stall, comm;
  int32_t completed, consumed;
  int32_t contributions;     /* worker contributions reduced (HandleInfo::contributions) */
  int32_t polled;            /* co2_aar_poll was called at least once */
  int32_t last_poll;         /* result of the most recent poll */
  int32_t completion_logged; /* a poll (or the wait) observed completion */
} co2_handle_info_t;
co2_status_t co2_aar_info(co2_aar_t* engine, uint64_t handle, co2_handle_info_t* out);
/* total_stall() and handle_count() (collective.hpp:64-67): the stall summed
 * over consumed handles (synchronizes on their wait events) and the number
 * of handles ever launched. */
co2_status_t co2_aar_totals(co2_aar_t* engine, double* total_stall, uint64_t* handle_count);
/* Blocking all-reduce (sum) on the given stream; used by ghost-consistent
 * mode for the averaged snapshots (outer_algorithms.cpp:163-169). */
co2_status_t co2_aar_allreduce_blocking(co2_aar_t* engine, co2_dtype_t dt, void* buf, int64_t n,
                                        void* stream);
/* Event log (collective.hpp:24-29): kind 0 launch, 1 complete, 2 wait;
 * t is seconds since engine creation on the device clock. */
typedef struct co2_event {
  int32_t kind;
  int32_t pad;
  uint64_t handle;
  double t, stall;
} co2_event_t;
co2_status_t co2_aar_events(co2_aar_t* engine, co2_event_t* out, int64_t cap, int64_t* count);

/* ---- worker state + co2_round (outer_algorithms.cpp:110-211) ------------- */
/* Device-resident worker: ping-pong params, anchor x_{t,0}, x_{t,1}
 * snapshot, prev_x0, prev_x1, momentum, gap.  The inner loop mutates the
 * buffer returned by co2_worker_params(); the snapshot hooks capture the
 * InnerTrace contract (proj/include/co2sim/inner_loop.hpp:51-61). */
typedef struct co2_worker co2_worker_t;
enum {
  CO2_BUF_PARAMS = 0,  /* current working params (low dtype) */
  CO2_BUF_ANCHOR = 1,  /* x_{t,0} (state dtype) */
  CO2_BUF_XFIRST = 2,  /* x_{t,1} (low dtype) */
  CO2_BUF_PREV_X0 = 3, /* state dtype */
  CO2_BUF_PREV_X1 = 4, /* low dtype */
  CO2_BUF_MOMENTUM = 5,/* state dtype */
  CO2_BUF_GAP = 6,     /* state dtype */
  CO2_BUF_XBAR = 7,    /* last consumed all-reduce result (low dtype; NCCL: the sum) */
  CO2_BUF_PARAMS_ALT = 8, /* the other ping-pong params buffer (P2P registration) */
  CO2_BUF_XFIRST_ALT = 9  /* sharded + P2P: the other x_{t,1} snapshot buffer */
};
/* init_params: device buffer in the low dtype (or NULL for zeros). */
co2_status_t co2_worker_create(co2_worker_t** out, co2_mode_t mode, int64_t n,
                               const void* init_params, int32_t keep_gap, void* stream);
co2_status_t co2_worker_destroy(co2_worker_t* w);
void* co2_worker_buffer(co2_worker_t* w, int32_t which);
co2_status_t co2_worker_set_clip_mode(co2_worker_t* worker, int32_t clip_mode);
int32_t co2_worker_round(const co2_worker_t* w);
/* RoundResult::consumed_average (outer_algorithms.hpp:68, outer_algorithms.cpp:
 * 159) on the in-place transports: when on, every co2_round step also writes
 * the reduce it consumed (low dtype; the average, also under CO2_NCCL_SUM)
 * into a worker-owned buffer returned by co2_worker_buffer(CO2_BUF_XBAR).
 * Costs one low-dtype write per coordinate.  LOCAL always keeps it. */
co2_status_t co2_worker_keep_average(co2_worker_t* w, int32_t on);
/* Snapshot hooks: x_{t,0} <- params (call before the first inner step;
 * a no-op for t >= 1 where the outer step already wrote the anchor), and
 * x_{t,1} <- params (call after the first inner step). */
co2_status_t co2_worker_snapshot_start(co2_worker_t* w, void* stream);
co2_status_t co2_worker_snapshot_first(co2_worker_t* w, void* stream);
typedef struct co2_round_result {
  double stall_seconds; /* device-measured, 0 when not yet available */
  int32_t outer_applied;
  int32_t pad;
  double min_gap, max_outer_step;
  int64_t n_clipped, n_floored;
} co2_round_result_t;
/* co2_round over the `g` workers this process owns (g == engine workers
 * for LOCAL, g == 1 for NCCL).  Synchronous only when `sync` != 0 (then
 * diagnostics and errors are reported); otherwise the diagnostics are read
 * by co2_round_finish. */
co2_status_t co2_round(co2_worker_t* const* workers, int32_t g, co2_aar_t* engine,
                       const co2_hyper_t* hyper, void* stream, int32_t sync,
                       co2_round_result_t* result);
co2_status_t co2_round_finish(co2_worker_t* const* workers, int32_t g, void* stream,
                              co2_round_result_t* result);
/* co2_round with the inner loop on the HOST (the reference's own setting:
 * proj/include/co2sim/outer_algorithms.hpp:77-81 takes WorkerState /
 * InnerTrace in host memory, proj/include/co2sim/inner_loop.hpp:18-24).
 * The outer state (x_{t,0} anchor, the previous snapshots, momentum, the
 * reduce buffers) stays resident on the device; per round only the inner
 * loop's trace crosses PCIe: each worker's x_{t,1} (`x_first_host[i]`,
 * nullable: then the device snapshot is kept) and x_{t,tau}
 * (`x_end_host[i]`) are uploaded into the worker's buffers, the round runs
 * (reduce launch, stale wait, fused step), and the params the next inner
 * loop starts from (x_{t+1,0}; x_{0,tau} after round 0) are downloaded into
 * `x_next_host[i]`.  Host buffers hold n low-dtype values each and should be
 * pinned.  The worker's x_{0,0} anchor must be on the device before round 0
 * (co2_worker_create's init + co2_worker_snapshot_start).  Asynchronous on
 * `stream` unless `sync` != 0 (then as co2_round, after the download). */
co2_status_t co2_round_host(co2_worker_t* const* workers, int32_t g, co2_aar_t* engine,
                            const co2_hyper_t* hyper, const void* const* x_first_host,
                            const void* const* x_end_host, void* const* x_next_host,
                            void* stream, int32_t sync, co2_round_result_t* result);
/* End of a run: consume (wait on, without applying) the reduce the last
 * round launched, releasing its slot in the engine's two-handle window. */
co2_status_t co2_round_drain(co2_worker_t* const* workers, int32_t g, co2_aar_t* engine,
                             void* stream);
/* ---- baseline outer algorithms on the same kernel family (SURVEY.md 8f
 *      item 3; proj/src/outer_algorithms.cpp:213-313) ----------------------
 * Per-worker bodies (one HBM pass, reference op order, reference messages
 * "non-finite value in slowmo momentum" / "slowmo outer iterate" /
 * "overlap correction"; diag.max_outer_step as RoundResult). */
/* slowmo_round body (:228-236): m = beta*m + (x_start - xbar);
 * params = x_start - alpha*m (anchor_out, nullable, receives it too). */
co2_status_t co2_slowmo_step(co2_mode_t mode, int64_t n, const void* x_start, const void* xbar,
                             int32_t xbar_divisor, void* momentum, void* params_out,
                             void* anchor_out, double alpha, double beta, void* workspace,
                             void* stream);
/* local_sgd_round body (:251-256): params = xbar. */
co2_status_t co2_local_sgd_step(co2_mode_t mode, int64_t n, const void* x_start,
                                const void* xbar, int32_t xbar_divisor, void* params_out,
                                void* anchor_out, void* workspace, void* stream);
/* overlap_local_sgd correction (:277-280, :293-296): params -= anchor - xbar. */
co2_status_t co2_overlap_correction(co2_mode_t mode, int64_t n, void* params,
                                    const void* anchor, const void* xbar, int32_t xbar_divisor,
                                    void* workspace, void* stream);
/* Round drivers over co2_worker_t and the engine (blocking reduce for SlowMo
 * and Local-SGD; Overlap-Local-SGD consumes the anchor reduce next round
 * unless `instant`, the reference's zero-cost-reduce case). */
co2_status_t co2_slowmo_round(co2_worker_t* const* workers, int32_t g, co2_aar_t* engine,
                              double alpha, double beta, void* stream, int32_t sync,
                              co2_round_result_t* result);
co2_status_t co2_local_sgd_round(co2_worker_t* const* workers, int32_t g, co2_aar_t* engine,
                                 void* stream, int32_t sync, co2_round_result_t* result);
co2_status_t co2_overlap_local_sgd_round(co2_worker_t* const* workers, int32_t g,
                                         co2_aar_t* engine, int32_t instant, void* stream,
                                         int32_t sync, co2_round_result_t* result);

/* ---- ghost-consistent, sharded outer state (C4; outer_algorithms.cpp:
 *      126-145,161-184) ------------------------------------------------------
 * The fused step on one shard where x_t0 is the average of `ghost_copies`
 * identical anchors (ghost_copies == 0: x_t0 is the consumed average itself,
 * the round-1 case x_{1,0} = x_{0,tau}), prev_x1 is a worker SUM divided once
 * by prev_x1_divisor and xbar a worker sum divided by xbar_divisor.  bar0_out
 * (state dtype, may alias prev_x0) receives the x_t0 used, i.e. the next
 * prev_x0; anchor_out (may alias anchor_in) receives x_{t+1,0}. */
co2_status_t co2_outer_step_ghost(co2_mode_t mode, int64_t n, const void* anchor_in,
                                  const void* prev_x0, const void* prev_x1_sum,
                                  int32_t prev_x1_divisor, const void* xbar_sum,
                                  int32_t xbar_divisor, int32_t ghost_copies, void* momentum,
                                  void* anchor_out, void* bar0_out, void* params_out,
                                  void* gap_out, const co2_hyper_t* hyper, void* workspace,
                                  void* stream);
/* Sharded worker over the NCCL engine: params and the x_{t,1} snapshot are
 * replicated (low dtype, full length); x_{t,0}, prev_x0, prev_x1, momentum
 * and gap live only for this rank's contiguous shard.  Per round:
 * reduce-scatter of x_{t,tau} (async, consumed next round), reduce-scatter
 * of x_{t,1}, the ghost step on the shard, and an in-place all-gather of
 * x_{t+1,0} into the params.  Requires hyper.ghost_consistent. */
typedef struct co2_sharded co2_sharded_t;
co2_status_t co2_sharded_create(co2_sharded_t** out, co2_mode_t mode, int64_t n,
                                co2_aar_t* engine, const void* init_params, int32_t keep_gap,
                                void* stream);
co2_status_t co2_sharded_destroy(co2_sharded_t* s);
/* which: CO2_BUF_PARAMS / CO2_BUF_XFIRST (full length), CO2_BUF_ANCHOR,
 * CO2_BUF_PREV_X0, CO2_BUF_MOMENTUM, CO2_BUF_GAP (shard), CO2_BUF_PREV_X1
 * (shard, worker sum), CO2_BUF_XBAR (shard, last consumed worker sum). */
void* co2_sharded_buffer(co2_sharded_t* s, int32_t which);
/* Shard geometry: returns the shard capacity; *offset and *length give the
 * global offset and the real coordinate count of this rank's shard. */
int64_t co2_sharded_shard(const co2_sharded_t* s, int64_t* offset, int64_t* length);
/* x_{0,0} snapshot of round 0 (call before the first inner step; no-op
 * afterwards) and x_{t,1} snapshot (call after the first inner step). */
co2_status_t co2_sharded_snapshot_start(co2_sharded_t* s, void* stream);
co2_status_t co2_sharded_snapshot_first(co2_sharded_t* s, void* stream);
co2_status_t co2_sharded_round(co2_sharded_t* s, co2_aar_t* engine, const co2_hyper_t* hyper,
                               void* stream, int32_t sync, co2_round_result_t* result);
co2_status_t co2_sharded_drain(co2_sharded_t* s, co2_aar_t* engine, void* stream);
co2_status_t co2_sharded_enable_timing(co2_sharded_t* s, int32_t cap);
co2_status_t co2_sharded_step_times(co2_sharded_t* s, double* out, int32_t cap, int32_t* count);

/* Device timing of the fused outer-step launch inside co2_round: events
 * bracket the kernel on the round's stream (a ring of `cap` pairs).
 * co2_worker_step_times synchronizes on the recorded events and returns the
 * durations (seconds) since the previous call, oldest first. */
co2_status_t co2_worker_enable_timing(co2_worker_t* w, int32_t cap);
co2_status_t co2_worker_step_times(co2_worker_t* w, double* out, int32_t cap, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* CO2_B200_H */
