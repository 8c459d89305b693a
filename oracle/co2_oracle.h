/*
 * co2_oracle.h -- CPU restatement of the reference's CO2 outer-step path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or as the timed
 * CPU baseline.  The product path (paper_2401_16265_b200/) never links it.
 *
 * What it restates (all paths relative to /root/reference/):
 *   - RngStream counter SplitMix64          proj/include/co2sim/rng.hpp:12-54
 *   - ensure_finite / average / clip        proj/src/param_ops.cpp:10-43
 *   - Co2Hyper::validate                    proj/src/outer_algorithms.cpp:37-46
 *   - staleness_gap                         proj/src/outer_algorithms.cpp:48-64
 *   - penalized_momentum_update             proj/src/outer_algorithms.cpp:66-90
 *   - outer_iterate                         proj/src/outer_algorithms.cpp:92-108
 *   - co2_round per-worker body             proj/src/outer_algorithms.cpp:185-202
 *
 * Two instantiations:
 *   1. fp64 "reference semantics": the reference's unfused pass structure with
 *      a fresh heap temporary per Eigen expression (orc_worker_step_f64).  It is
 *      bit-for-bit the reference (the reference builds with -ffp-contract=off,
 *      proj/CMakeLists.txt:12-13, and every op is one IEEE op).  It is pinned by
 *      the reference's own KATs and fixtures (tests/test_oracle_golden.py).
 *   2. fused "same op order" in fp64 / fp32 / bf16-mixed (orc_outer_step): the
 *      per-element formula of SURVEY.md section 8(a), evaluated in the compute
 *      type the GPU uses.  The CUDA kernels must equal it bit for bit.
 *
 * Parity is pinned (not unpinned): the reference itself cannot be compiled in
 * this image (Eigen 3 is absent), so the restatement is checked against every
 * known-answer test and fixture the reference ships for this path.
 */
#ifndef CO2_ORACLE_H
#define CO2_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_VALIDATION = 2, ORC_NUMERIC = 3 };
enum { ORC_MODE_F64 = 0, ORC_MODE_F32 = 1, ORC_MODE_BF16_MIXED = 2 };

/* Device-flag bits, shared meaning with the product (include/co2_b200.h). */
enum {
  ORC_FLAG_GAP_NONFINITE = 1u,  /* staleness_gap ensure_finite           */
  ORC_FLAG_GAP_BELOW_ONE = 2u,  /* momentum update: gap coordinate < 1   */
  ORC_FLAG_M_NONFINITE = 4u,    /* momentum update ensure_finite         */
  ORC_FLAG_CLIP_NONFINITE = 8u, /* clip_elementwise input ensure_finite  */
  ORC_FLAG_X_NONFINITE = 16u    /* outer_iterate ensure_finite           */
};

typedef struct {
  double alpha, beta, phi, epsilon;
  int32_t tau;
  uint8_t penalty, clip, ghost_consistent, pad;
} orc_hyper;

typedef struct {
  double min_gap;        /* +inf when n == 0 */
  double max_outer_step; /* max |x' - x_t0| */
  int64_t n_clipped;     /* coordinates with |m'| > phi (clip on) */
  int64_t n_floored;     /* coordinates with tau*|p1-p0| < epsilon */
  uint32_t flags;
  uint32_t pad;
} orc_diag;

const char* orc_last_error(void);

/* ---- RngStream (rng.hpp:12-54), random-access form ------------------- */
uint64_t orc_mix(uint64_t z);
uint64_t orc_rng_key(uint64_t seed, uint64_t stream);
/* Draw number j (0-based) of the stream: mix(key + (j+1)*golden). */
uint64_t orc_rng_u64_at(uint64_t key, uint64_t j);
double orc_rng_double_at(uint64_t key, uint64_t j);
uint64_t orc_rng_below_at(uint64_t key, uint64_t j, uint64_t n);
void orc_rng_fill_u64(uint64_t seed, uint64_t stream, int64_t count, uint64_t* out);

/* ---- bf16 helpers ------------------------------------------------------ */
uint16_t orc_f32_to_bf16(float f);
float orc_bf16_to_f32(uint16_t h);

/* ---- param_ops (param_ops.cpp:10-43) --------------------------------- */
int orc_ensure_finite_f64(int64_t n, const double* v, const char* context);
int orc_average_f64(int g, const double* const* contrib, int64_t n, double* out);
int orc_clip_f64(int64_t n, const double* v, double phi, double* out);

/* ---- outer ops (outer_algorithms.cpp:37-108) -------------------------- */
int orc_hyper_validate(const orc_hyper* h);
int orc_staleness_gap_f64(int64_t n, const double* x_t0, const double* p0,
                          const double* p1, int tau, double epsilon, double* gap);
int orc_penalized_momentum_f64(int64_t n, const double* m_prev, double beta,
                               const double* gap, const double* delta,
                               int penalty, double* m);
int orc_outer_iterate_f64(int64_t n, const double* x_t0, double alpha,
                          const double* m, double phi, int clip, double* x);

/* ---- co2_round per-worker body, unfused fp64 (cpp:186-202) ------------ */
/* Allocates the reference's temporaries per call (numer, denom, gap, delta,
 * m, clip, x) and runs the reference's passes in the reference's order.
 * m_inout is replaced by m'; next receives x_{t+1,0}; gap_out (nullable)
 * receives Lambda.  threads > 1 splits the coordinates into contiguous
 * ranges, each running the same unfused sequence (used only to time the
 * reference arm on all host cores). */
int orc_worker_step_f64(int64_t n, const double* x_t0, const double* p0,
                        const double* p1, const double* avg, double* m_inout,
                        const orc_hyper* h, double* next, double* gap_out,
                        double* min_gap, double* max_step, int threads);

/* ---- fused same-op-order step (the GPU's bitwise target) -------------- */
/* mode F64: every buffer double.  F32: every buffer float.
 * BF16_MIXED: x_t0, p0, m, anchor_out float; p1, xbar, params_out bf16 bits.
 * xbar holds either the average (divisor 1) or the worker sum (divisor G,
 * divided once as in average()).  anchor_out / params_out / gap_out nullable.
 * m may alias nothing but itself; anchor_out may alias p0; params_out may
 * alias xbar. */
int orc_outer_step(int mode, int64_t n, const void* x_t0, const void* p0,
                   const void* p1, const void* xbar, int divisor, void* m,
                   void* anchor_out, void* params_out, void* gap_out,
                   const orc_hyper* h, orc_diag* diag);
/* Ghost-consistent / sharded step (outer_algorithms.cpp:161-184): x_t0 =
 * average of `ghost` identical anchors (ghost == 0: the consumed average),
 * prev_x1 = p1sum / p1_div, xbar = xsum / xdiv; bar0_out gets the x_t0 used. */
int orc_outer_step_ghost(int mode, int64_t n, const void* anchor, const void* p0,
                         const void* p1sum, int p1_div, const void* xsum, int xdiv, int ghost,
                         void* m, void* anchor_out, void* bar0_out, void* params_out,
                         void* gap_out, const orc_hyper* h, orc_diag* diag);
/* Reference error precedence over a diag's flags. */
int orc_diag_status(const orc_diag* d);

/* ---- baseline outer steps (outer_algorithms.cpp:213-313) -------------- */
/* Same storage convention as orc_outer_step (mode); xbar is the average
 * (divisor 1) or a worker sum (divisor G).  Each returns the reference's
 * status and message for its ensure_finite checks and fills diag
 * (max_outer_step and flags only). */
enum { ORC_FLAG_SLOWMO_M = 64u, ORC_FLAG_SLOWMO_X = 128u, ORC_FLAG_OVERLAP = 256u };

/* EXTENSION outside the reference parity contract (the reference clips
 * coordinate-wise, proj/src/param_ops.cpp:35-43): the global-norm clip the
 * north star words, restated in the GPU's exact summation order
 * (paper_2401_16265_b200/csrc/outer_step.cu, gclip_pass1/2):
 *   m' per coordinate as orc_outer_step; ||m'||^2 in fp64: fixed chunks of
 *   orc_gc_chunk(n, V) coordinates; within a chunk, "thread" t (0..255) sums
 *   (double)m'^2 over its V-wide vectors t, t+256, ... in order (the n % V
 *   scalar tail goes to thread 0 of the last chunk, after its vectors);
 *   a xor butterfly (16, 8, 4, 2, 1) per 32-thread warp; the 8 warps in
 *   order.  Chunk sums fold the same way (thread t: chunks t, t+256, ...).
 *   norm = sqrt; scale = (clip && norm > phi) ? phi / norm : 1 (fp64);
 *   c = (T)((double)m' * scale); x' = x_t0 - alpha * c.
 * V = 2 (fp64), 4 (fp32), 8 (bf16-mixed).  n_clipped = n when scaled. */
enum { ORC_FLAG_NORM_NONFINITE = 512u };
int64_t orc_gc_chunk(int64_t n, int V);
/* l2_norm (proj/src/param_ops.cpp:54-60) in the GPU's fixed order (the
 * global-clip chunked sum above, V by dtype: 0 fp64 -> 2, 1 fp32 -> 4,
 * 2 bf16 -> 8). */
double orc_l2_norm(int dtype, int64_t n, const void* v);
int orc_outer_step_global_clip(int mode, int64_t n, const void* x_t0, const void* p0,
                               const void* p1, const void* xbar, int divisor, void* m,
                               void* anchor, void* params, void* gap, const orc_hyper* h,
                               orc_diag* diag, double* norm_out);
/* slowmo_round body (cpp:228-236): m = beta*m + (x_start - xbar);
 * params = x_start - alpha*m. */
int orc_slowmo_step(int mode, int64_t n, const void* x_start, const void* xbar, int divisor,
                    void* m, void* params_out, double alpha, double beta, orc_diag* diag);
/* local_sgd_round body (cpp:251-256): params = xbar. */
int orc_local_sgd_step(int mode, int64_t n, const void* x_start, const void* xbar, int divisor,
                       void* params_out, orc_diag* diag);
/* overlap_local_sgd correction (cpp:277-280 / :293-296):
 * params -= anchor - xbar; diag.max_outer_step = max |params' - params|. */
int orc_overlap_correction(int mode, int64_t n, void* params, const void* anchor,
                           const void* xbar, int divisor, orc_diag* diag);

/* ---- fixed-order average in the storage type (param_ops.cpp:16-33) ---- */
int orc_average_lp(int dtype_bf16, int g, const void* const* contrib, int64_t n,
                   void* out);

/* ---- synthetic inputs ---------------------------------- */
/* buffer ids */
enum { ORC_BUF_P0 = 0, ORC_BUF_P1 = 1, ORC_BUF_XT0 = 2, ORC_BUF_XEND = 3, ORC_BUF_M = 4 };
/* Fills one worker's inputs for coordinates [j0, j0+count).  Any pointer may
 * be NULL.  Storage types follow the mode (as orc_outer_step); x_end is in the
 * params dtype. */
void orc_synth(int mode, uint64_t seed, int worker, int64_t j0, int64_t count,
               void* x_t0, void* p0, void* p1, void* x_end, void* m);

#ifdef __cplusplus
}
#endif
#endif
