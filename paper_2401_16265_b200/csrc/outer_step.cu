// Fused CO2 outer step and the unfused reference operators for sm_100a.
//
// The path is HBM-bandwidth bound (~0.5 FLOP/B): no tensor
// cores.  The fused kernel reads x_t0, prev_x0, prev_x1, xbar and m once and
// writes m', the new anchor and the params once: 32 B/param in fp32, 26 B in
// bf16-mixed, 64 B in fp64 (versus ~264 B/param in the reference's unfused
// fp64 passes, outer_algorithms.cpp:48-108).  Streams are 128-bit
// coalesced with evict-first cache hints, U independent vectors per thread
// are in flight before any arithmetic, and the grid-stride loop runs on a
// grid of up to 32 waves of the 148 SMs' resident CTAs (grid_for below), so
// the block scheduler balances the tail and any co-running reduce kernel.
//
// Bit-exactness: built with --fmad=false and IEEE division, every element op
// below is exactly one IEEE op in the reference's order, so the F64 mode is
// bitwise the reference (built -ffp-contract=off, proj/CMakeLists.txt:12-13)
// and the F32 / BF16-mixed modes are bitwise the same-op-order oracle.
//
// Diagnostics (min Lambda, max |x' - x_t0|, clip / floor counts, error
// flags) are reduced warp-shuffle -> shared memory -> per-block partials,
// and the last block to arrive (atomic ticket) folds the partials in fixed
// index order, so results are deterministic without a second launch.
#include <atomic>
#include <cuda_bf16.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "bulk.cuh"
#include "p2p_sync.cuh"

namespace co2 {
namespace {

// ------------------------------------------------------------ storage types
struct bf16s {  // bf16 storage as raw bits
  uint16_t b;
};

__device__ __forceinline__ float to_c(float v) { return v; }
__device__ __forceinline__ double to_c(double v) { return v; }
__device__ __forceinline__ float to_c(bf16s v) { return __uint_as_float(((uint32_t)v.b) << 16); }

template <typename T>
struct Store;
template <>
struct Store<double> {
  __device__ static __forceinline__ double from(double v) { return v; }
};
template <>
struct Store<float> {
  __device__ static __forceinline__ float from(float v) { return v; }
};
template <>
struct Store<bf16s> {
  __device__ static __forceinline__ bf16s from(float v) {
    // cvt.rn.bf16.f32: round-to-nearest-even, canonical NaN 0x7fff.
    __nv_bfloat16 h = __float2bfloat16_rn(v);
    return bf16s{__bfloat16_as_ushort(h)};
  }
};

// Modes: storage of state (x_t0, prev_x0, m, anchor, gap), storage of low
// (prev_x1, xbar, params) and compute type.
struct ModeF64 {
  using TS = double;
  using TL = double;
  using TC = double;
};
struct ModeF32 {
  using TS = float;
  using TL = float;
  using TC = float;
};
struct ModeBF16 {
  using TS = float;
  using TL = bf16s;
  using TC = float;
};

// ------------------------------------------------------- vector load/store
template <typename T, int N>
__device__ __forceinline__ void ld_vec(const T* __restrict__ p, T (&out)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
    uint4 r[BYTES / 16];
#pragma unroll
    for (int k = 0; k < BYTES / 16; ++k) r[k] = __ldcs(reinterpret_cast<const uint4*>(p) + k);
    memcpy(out, r, BYTES);
  } else if constexpr (BYTES == 8) {
    uint2 r = __ldcs(reinterpret_cast<const uint2*>(p));
    memcpy(out, &r, 8);
  } else if constexpr (BYTES == 4) {
    unsigned int r = __ldcs(reinterpret_cast<const unsigned int*>(p));
    memcpy(out, &r, 4);
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = p[k];
  }
}

template <typename T, int N>
__device__ __forceinline__ void st_vec(T* __restrict__ p, const T (&in)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
    uint4 r[BYTES / 16];
    memcpy(r, in, BYTES);
#pragma unroll
    for (int k = 0; k < BYTES / 16; ++k) __stcs(reinterpret_cast<uint4*>(p) + k, r[k]);
  } else if constexpr (BYTES == 8) {
    uint2 r;
    memcpy(&r, in, 8);
    __stcs(reinterpret_cast<uint2*>(p), r);
  } else if constexpr (BYTES == 4) {
    unsigned int r;
    memcpy(&r, in, 4);
    __stcs(reinterpret_cast<unsigned int*>(p), r);
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) p[k] = in[k];
  }
}

// --------------------------------------------------------- diag reduction
struct Acc {
  double min_gap = INFINITY;
  double max_step = 0.0;
  unsigned int clipped = 0, floored = 0, flags = 0;
};

// Per-thread accumulator in the compute type: min / max in fp32 are exact
// and convert to double once per thread, not once per element.
template <typename TC>
struct AccT {
  TC min_gap = (TC)INFINITY;
  TC max_step = (TC)0;
  unsigned int clipped = 0, floored = 0, flags = 0;
  __device__ Acc widen() const {
    Acc a;
    a.min_gap = (double)min_gap;
    a.max_step = (double)max_step;
    a.clipped = clipped;
    a.floored = floored;
    a.flags = flags;
    return a;
  }
};

// Order-preserving 64-bit key of a double (monotone in the value for every
// non-NaN double) and its inverse.
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
  return __longlong_as_double((long long)b);
}

// Returns true in every thread of the last block to arrive (after it wrote
// the folded diagnostics), false elsewhere.
//
// Each block folds its threads (warp shuffles, then warps in fixed order)
// and merges the block result into the workspace header with atomics: min
// Lambda and max |x' - x_t0| as atomicMax over order-preserving keys, the
// counts as 64-bit adds, the flags as OR.  Min, max, integer sums and OR are
// exact and order-independent, so the result is bitwise deterministic for
// any grid and any block completion order (per-thread and per-block values
// are never NaN: a NaN never wins the `<` / `>` folds that produce them).
// The last block (atomic ticket) publishes the diagnostics and resets the
// accumulators: an O(1) tail instead of a fold over every block's partial.
template <int NT>
__device__ bool block_finish(const Acc& a, void* ws, const P2PExit* px = nullptr) {
  // Warp level.
  double mg = a.min_gap, ms = a.max_step;
  unsigned long long cl = a.clipped, fl = a.floored;
  unsigned int fg = a.flags;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double omg = __shfl_xor_sync(0xffffffffu, mg, o);
    double oms = __shfl_xor_sync(0xffffffffu, ms, o);
    mg = omg < mg ? omg : mg;
    ms = oms > ms ? oms : ms;
    cl += __shfl_xor_sync(0xffffffffu, cl, o);
    fl += __shfl_xor_sync(0xffffffffu, fl, o);
    fg |= __shfl_xor_sync(0xffffffffu, fg, o);
  }
  constexpr int NW = NT / 32;
  __shared__ Partial sh[NW];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = Partial{mg, ms, cl, fl, fg, 0u};
  __syncthreads();
  WsHeader* hdr = ws_header(ws);
  if (threadIdx.x == 0) {
    Partial b = sh[0];
    for (int w = 1; w < NW; ++w) {  // fixed order
      b.min_gap = sh[w].min_gap < b.min_gap ? sh[w].min_gap : b.min_gap;
      b.max_step = sh[w].max_step > b.max_step ? sh[w].max_step : b.max_step;
      b.clipped += sh[w].clipped;
      b.floored += sh[w].floored;
      b.flags |= sh[w].flags;
    }
    // min as a max of inverted keys (0 = empty = +inf), max as a max of keys
    // (0 = empty; the initial max_step +0.0 has a larger key than any "empty")
    atomicMax(&hdr->acc_min_key, ~dkey(b.min_gap));
    atomicMax(&hdr->acc_max_key, dkey(b.max_step));
    if (b.clipped) atomicAdd(&hdr->acc_clipped, b.clipped);
    if (b.floored) atomicAdd(&hdr->acc_floored, b.floored);
    if (b.flags) atomicOr(&hdr->acc_flags, b.flags);
    if (px)
      __threadfence_system();  // this CTA's peer stores before the ticket
    else
      __threadfence();
    unsigned int t = atomicAdd(&hdr->ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  if (threadIdx.x == 0) {
    __threadfence();
    volatile WsHeader* vh = hdr;
    const unsigned long long kmin = vh->acc_min_key, kmax = vh->acc_max_key;
    hdr->diag.min_gap = kmin ? dkey_inv(~kmin) : (double)INFINITY;
    hdr->diag.max_outer_step = kmax ? dkey_inv(kmax) : 0.0;
    hdr->diag.n_clipped = (int64_t)vh->acc_clipped;
    hdr->diag.n_floored = (int64_t)vh->acc_floored;
    hdr->diag.flags = vh->acc_flags;
    hdr->diag.pad = 0;
    hdr->acc_min_key = 0ull;  // self-reset for the next launch on this workspace
    hdr->acc_max_key = 0ull;
    hdr->acc_clipped = 0ull;
    hdr->acc_floored = 0ull;
    hdr->acc_flags = 0u;
    hdr->ticket = 0;
    __threadfence();
    if (px) p2p_exit_barrier(*px);
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ void partial_merge(Partial& b, const Partial& q) {
  b.min_gap = q.min_gap < b.min_gap ? q.min_gap : b.min_gap;
  b.max_step = q.max_step > b.max_step ? q.max_step : b.max_step;
  b.clipped += q.clipped;
  b.floored += q.floored;
  b.flags |= q.flags;
  b.pad |= q.pad;
}

__device__ __forceinline__ Partial warp_fold(Partial b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Partial q;
    q.min_gap = __shfl_xor_sync(0xffffffffu, b.min_gap, o);
    q.max_step = __shfl_xor_sync(0xffffffffu, b.max_step, o);
    q.clipped = __shfl_xor_sync(0xffffffffu, b.clipped, o);
    q.floored = __shfl_xor_sync(0xffffffffu, b.floored, o);
    q.flags = __shfl_xor_sync(0xffffffffu, b.flags, o);
    q.pad = __shfl_xor_sync(0xffffffffu, b.pad, o);
    partial_merge(b, q);
  }
  return b;
}

// Fold one Partial per thread warp -> smem -> fixed warp order; the result
// is valid in thread 0.  Every thread must call it.
template <int NT>
__device__ Partial block_fold(const Partial& mine) {
  constexpr int NW = NT / 32;
  __shared__ Partial sh[NW];
  const Partial b = warp_fold(mine);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // sh may still be read by a previous call's thread 0
  if (lane == 0) sh[wid] = b;
  __syncthreads();
  Partial r = sh[0];
  if (threadIdx.x == 0)
    for (int w = 1; w < NW; ++w) partial_merge(r, sh[w]);
  return r;
}

// This CTA's diagnostics (valid in thread 0).
template <int NT>
__device__ Partial block_partial(const Acc& a) {
  return block_fold<NT>(Partial{a.min_gap, a.max_step, (unsigned long long)a.clipped,
                                (unsigned long long)a.floored, a.flags, 0u});
}

// Fold count partials written by other CTAs in fixed order: thread-strided,
// then block_fold.  Valid in thread 0; all threads call.
template <int NT>
__device__ Partial fold_partials(const Partial* parts, int count) {
  Partial b{INFINITY, 0.0, 0ull, 0ull, 0u, 0u};
  for (int i = threadIdx.x; i < count; i += NT) {
    const Partial* q = parts + i;
    Partial v{__ldcg(&q->min_gap), __ldcg(&q->max_step), __ldcg(&q->clipped),
              __ldcg(&q->floored), __ldcg(&q->flags), __ldcg(&q->pad)};
    partial_merge(b, v);
  }
  return block_fold<NT>(b);
}

// ---------------------------------------------------------- fused element
template <typename TC>
struct Hyp {
  TC tau, eps, beta, phi, alpha, divisor;
  int penalty, clip, divide;
};

// One coordinate of SURVEY.md 8(a) "Fused per-element semantics":
//   n0 = |x_t0 - p0|                       outer_algorithms.cpp:57
//   d  = max(|tau*(p1 - p0)|, eps)          :58-60 (std::max NaN semantics)
//   L  = n0/d + 1                           :61
//   D  = p0 - xbar                          :189
//   m' = beta*m + D/L   (or beta*m + D)     :84 / :86
//   c  = min(max(m', -phi), phi)  (or m')   param_ops.cpp:42
//   x' = x_t0 - alpha*c                     outer_algorithms.cpp:102 / :104
// Bf16-mixed (LQ): the inner loop started from the bf16 params, i.e. from
// the bf16 rounding of the fp32 anchor q0, so the first-step displacement in
// the gap's denominator is q1 - bf16(q0) (exactly 0 at a coordinate the first
// inner step did not move, as in the reference); the numerator and Delta
// use the fp32 anchors.  Identity for the fp32 / fp64 modes.
template <typename TC, bool LQ>
__device__ __forceinline__ TC start_of_inner(TC q0) {
  if constexpr (LQ) {
    return __uint_as_float(((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(q0))) << 16);
  } else {
    return q0;
  }
}

template <typename TC, bool LQ = false>
__device__ __forceinline__ void co2_elem(TC x, TC q0, TC q1, TC xb, TC& m, TC& xn, TC& lam,
                                         const Hyp<TC>& h, AccT<TC>& acc) {
  if (h.divide) xb = div_rn_nz(xb, h.divisor);  // average(): sum / G, param_ops.cpp:30
  TC n0 = fabs(x - q0);
  TC av = fabs(h.tau * (q1 - start_of_inner<TC, LQ>(q0)));
  bool floored = av < h.eps;
  TC d = floored ? h.eps : av;
  lam = div_rn(n0, d) + (TC)1;
  TC dl = q0 - xb;
  TC mn;
  if (h.penalty) {
    TC bm = h.beta * m;
    TC q = div_rn_nz(dl, lam);  // lam >= 1, +inf or NaN
    mn = bm + q;
  } else {
    TC bm = h.beta * m;
    mn = bm + dl;
  }
  TC c = mn;
  bool clipped = false;
  if (h.clip) {
    clipped = (mn < -h.phi) || (h.phi < mn);
    TC lo = (mn < -h.phi) ? -h.phi : mn;  // std::max(mn, -phi)
    c = (h.phi < lo) ? h.phi : lo;         // std::min(lo, phi)
  }
  TC ac = h.alpha * c;
  xn = x - ac;
  m = mn;
  unsigned int f = 0;
  if (!isfinite(lam)) f |= CO2_FLAG_GAP_NONFINITE;
  if (h.penalty && lam < (TC)1) f |= CO2_FLAG_GAP_BELOW_ONE;
  if (!isfinite(mn)) f |= CO2_FLAG_M_NONFINITE;
  if (!isfinite(xn)) f |= CO2_FLAG_X_NONFINITE;
  acc.flags |= f;
  acc.floored += floored;
  acc.clipped += clipped;
  // fmin / fmax: a NaN operand never wins, as in the `<` / `>` folds of the
  // block and role merges; lam >= 1 and |x' - x| >= +0 have no signed zeros.
  TC st = fabs(xn - x);
  if constexpr (std::is_same<TC, float>::value) {
    acc.min_gap = fmin(lam, acc.min_gap);
    acc.max_step = fmax(st, acc.max_step);
  } else {  // fp64: the compare-select form keeps the F64 body within 64 registers
    acc.min_gap = lam < acc.min_gap ? lam : acc.min_gap;
    acc.max_step = st > acc.max_step ? st : acc.max_step;
  }
}

struct StepArgs {
  const void* x_t0;
  const void* p0;
  const void* p1;
  const void* xbar;
  void* m;
  void* anchor;
  void* params;
  void* gap;
  int64_t n;
  double alpha, beta, phi, eps;
  int tau, divisor, penalty, clip;
  void* ws;
  // ghost-consistent / sharded extension (GHOST instantiations only)
  int p1_div;       // prev_x1 holds a worker sum: divide once by p1_div
  int ghost_g;      // x_t0 = average of ghost_g identical copies of x_t0
  int x_from_xbar;  // x_t0 = the consumed average itself (round 1)
  void* bar0_out;   // receives the x_t0 actually used (next prev_x0)
  // P2P fused all-gather (P2POUT instantiations only)
  void* out_peers[kMaxRanks];
  P2PExit exit;
  // Fused one-step-stale all-reduce (AAR > 0 instantiations; AAR = rank capacity): slice
  // [aar_lo, aar_lo + aar_len) of the rank-indexed buffers aar_bufs (x_{t,tau}
  // on every rank) is averaged in rank order and stored into every rank.
  void* aar_bufs[kMaxRanks];
  int64_t aar_lo, aar_len;
  // RoundResult::consumed_average (outer_algorithms.hpp:68): when non-null
  // the step copies the reduce it consumed (as read: a worker sum stays a
  // sum), so in-place transports keep it readable.
  void* xbar_out;
};

// One 16-byte vector of the fixed-order P2P average (param_ops.cpp:16-33):
// gather from every rank, sum in rank order, divide once, store to every rank.
template <typename TL, typename TC, int R>
__device__ __forceinline__ void aar_vector(const StepArgs& a, int64_t e) {
  constexpr int VA = 16 / (int)sizeof(TL);
  // Ranks are gathered in groups of at most 4 (ascending), so the 8-rank
  // instantiation holds 4 x 16 B of loads, not 8, beside the step's state
  // (it spilled 152 B at 3 CTAs/SM with all 8 in flight).
  constexpr int RG = R < 2 ? R : 2;
  TC acc[VA];
#pragma unroll
  for (int p0 = 0; p0 < R; p0 += RG) {
    uint4 raw[RG];
#pragma unroll
    for (int q = 0; q < RG; ++q)
      if (p0 + q < a.exit.world)
        raw[q] = __ldcg(
            reinterpret_cast<const uint4*>(static_cast<const TL*>(a.aar_bufs[p0 + q]) + e));
#pragma unroll
    for (int q = 0; q < RG; ++q)
      if (p0 + q < a.exit.world)
#pragma unroll
        for (int k = 0; k < VA; ++k) {
          const TC v = to_c(reinterpret_cast<const TL*>(&raw[q])[k]);
          acc[k] = (p0 + q == 0) ? v : acc[k] + v;  // ascending rank order
        }
  }
  uint4 out;
  const TC g = (TC)a.exit.world;
#pragma unroll
  for (int k = 0; k < VA; ++k) reinterpret_cast<TL*>(&out)[k] = Store<TL>::from(div_rn_nz(acc[k], (TC)g));
#pragma unroll
  for (int p = 0; p < R; ++p)
    if (p < a.exit.world) __stcg(reinterpret_cast<uint4*>(static_cast<TL*>(a.aar_bufs[p]) + e), out);
}

// average() of g identical copies (param_ops.cpp:26-30 with every
// contribution equal): ascending-order sum, one division.
template <typename TC>
__device__ __forceinline__ TC ghost_avg(TC v, int g) {
  TC s = v;
  for (int i = 1; i < g; ++i) s = s + v;
  return div_rn_nz(s, (TC)g);
}

// The fused step's body, shared by the launch-bounded kernel and the
// register-capped variant below.
template <class M, int V, int U, int NT, bool GHOST, bool P2POUT, int AAR>
__device__ __forceinline__ void fused_step_body(const StepArgs& a) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  Hyp<TC> h;
  h.tau = (TC)a.tau;
  h.eps = (TC)a.eps;
  h.beta = (TC)a.beta;
  h.phi = (TC)a.phi;
  h.alpha = (TC)a.alpha;
  h.divisor = (TC)a.divisor;
  h.penalty = a.penalty;
  h.clip = a.clip;
  h.divide = a.divisor > 1;
  Hyp<TC> hg = h;  // GHOST: xbar is divided before the element body
  hg.divide = 0;
  const TC p1d = (TC)a.p1_div;
  TS* B0 = static_cast<TS*>(a.bar0_out);
  TL* XO = static_cast<TL*>(a.xbar_out);
  constexpr bool LQ = !std::is_same<TS, TL>::value;  // bf16-mixed: see start_of_inner

  const TS* __restrict__ X = static_cast<const TS*>(a.x_t0);
  const TS* __restrict__ P0 = static_cast<const TS*>(a.p0);
  const TL* __restrict__ P1 = static_cast<const TL*>(a.p1);
  const TL* XB = static_cast<const TL*>(a.xbar);  // may alias params
  TS* Mm = static_cast<TS*>(a.m);
  TS* A = static_cast<TS*>(a.anchor);  // may alias prev_x0
  TL* PR = static_cast<TL*>(a.params);  // may alias xbar
  TS* G = static_cast<TS*>(a.gap);

  AccT<TC> acc;
  const int64_t nv = a.n / V;
  const int64_t stride = (int64_t)gridDim.x * NT;
  int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
  // AAR > 0: every rank's x_{t,tau} is final once all ranks arrived; the
  // all-reduce vectors are interleaved with the outer-step vectors (one per
  // world-size step vectors) so both streams share HBM and NVLink evenly.
  constexpr int VA = 16 / (int)sizeof(TL);
  const int64_t aar_nvec = AAR > 0 ? a.aar_len / VA : 0;
  bool aar_ok = true;
  if constexpr (AAR > 0) {
    __shared__ int s_go;
    if (threadIdx.x == 0) s_go = p2p_entry_barrier(a.exit);
    __syncthreads();
    aar_ok = s_go != 0;
  }
  const int gw = AAR > 0 ? a.exit.world : 1;
  auto aar_for = [&](int64_t iv) {
    if constexpr (AAR > 0) {
      if (aar_ok && iv % gw == 0 && iv / gw < aar_nvec) aar_vector<TL, TC, (AAR > 0 ? AAR : 1)>(a, a.aar_lo + (iv / gw) * VA);
    }
  };

  auto process = [&](const int64_t (&idx)[U], int cnt) {
    TS x[U][V], q0[U][V], mo[U][V];
    TL q1[U][V], xb[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < cnt) {
        const int64_t e = idx[u] * V;
        ld_vec<TS, V>(X + e, x[u]);
        ld_vec<TS, V>(P0 + e, q0[u]);
        ld_vec<TL, V>(P1 + e, q1[u]);
        ld_vec<TL, V>(XB + e, xb[u]);
        ld_vec<TS, V>(Mm + e, mo[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < cnt) {
        const int64_t e = idx[u] * V;
        TS mn[V], xs[V], gs[V], b0[V];
        TL xl[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          TC m = to_c(mo[u][v]), xn, lam;
          TC xbv = to_c(xb[u][v]);
          if (h.divide) xbv = div_rn_nz(xbv, h.divisor);  // average(): sum / G, param_ops.cpp:30
          if constexpr (GHOST) {
            TC xv = a.x_from_xbar ? xbv : ghost_avg<TC>(to_c(x[u][v]), a.ghost_g);
            TC p1v = to_c(q1[u][v]);
            if (a.p1_div > 1) p1v = div_rn_nz(p1v, p1d);
            b0[v] = (TS)xv;
            co2_elem<TC, LQ>(xv, to_c(q0[u][v]), p1v, xbv, m, xn, lam, hg, acc);
          } else {
            co2_elem<TC, LQ>(to_c(x[u][v]), to_c(q0[u][v]), to_c(q1[u][v]), xbv, m, xn, lam,
                             hg, acc);
          }
          mn[v] = (TS)m;
          xs[v] = (TS)xn;
          gs[v] = (TS)lam;
          xl[v] = Store<TL>::from(xn);
        }
        st_vec<TS, V>(Mm + e, mn);
        if (A) st_vec<TS, V>(A + e, xs);
        if (PR) st_vec<TL, V>(PR + e, xl);
        if (G) st_vec<TS, V>(G + e, gs);
        if (XO) st_vec<TL, V>(XO + e, xb[u]);  // as consumed (a sum stays a sum)
        if constexpr (GHOST) {
          if (B0) st_vec<TS, V>(B0 + e, b0);
        }
        if constexpr (P2POUT) {  // fused all-gather: x_{t+1,0} into every rank's params
          for (int p = 0; p < a.exit.world; ++p)
            st_vec<TL, V>(static_cast<TL*>(a.out_peers[p]) + e, xl);
        }
      }
    }
  };

  for (; i + (int64_t)(U - 1) * stride < nv; i += (int64_t)U * stride) {
    int64_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) idx[u] = i + (int64_t)u * stride;
    process(idx, U);
#pragma unroll
    for (int u = 0; u < U; ++u) aar_for(idx[u]);
  }
  for (; i < nv; i += stride) {
    int64_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) idx[u] = i;
    process(idx, 1);
    aar_for(i);
  }
  if constexpr (AAR > 0) {
    // all-reduce vectors not covered by the interleave, then its scalar tail
    const int64_t covered = (nv + gw - 1) / gw;
    for (int64_t ia = covered + (int64_t)blockIdx.x * NT + threadIdx.x; aar_ok && ia < aar_nvec;
         ia += stride)
      aar_vector<TL, TC, (AAR > 0 ? AAR : 1)>(a, a.aar_lo + ia * VA);
    if (aar_ok && blockIdx.x == 0) {
      for (int64_t j = a.aar_lo + aar_nvec * VA + threadIdx.x; j < a.aar_lo + a.aar_len;
           j += NT) {
        TC s0 = to_c(static_cast<const TL*>(a.aar_bufs[0])[j]);
        for (int p = 1; p < a.exit.world; ++p) s0 = s0 + to_c(static_cast<const TL*>(a.aar_bufs[p])[j]);
        const TL r = Store<TL>::from(div_rn_nz(s0, (TC)a.exit.world));
        for (int p = 0; p < a.exit.world; ++p) static_cast<TL*>(a.aar_bufs[p])[j] = r;
      }
    }
  }
  // Scalar tail (n % V coordinates).
  const int64_t t = nv * V + (int64_t)blockIdx.x * NT + threadIdx.x;
  if (V > 1 && t < a.n) {
    TC m = to_c(Mm[t]), xn, lam;
    TC xbv = to_c(XB[t]);
    if (h.divide) xbv = div_rn_nz(xbv, h.divisor);
    if constexpr (GHOST) {
      TC xv = a.x_from_xbar ? xbv : ghost_avg<TC>(to_c(X[t]), a.ghost_g);
      TC p1v = to_c(P1[t]);
      if (a.p1_div > 1) p1v = div_rn_nz(p1v, p1d);
      const TC q0 = to_c(P0[t]);  // read before bar0_out (may alias prev_x0) is written
      if (B0) B0[t] = (TS)xv;
      co2_elem<TC, LQ>(xv, q0, p1v, xbv, m, xn, lam, hg, acc);
    } else {
      co2_elem<TC, LQ>(to_c(X[t]), to_c(P0[t]), to_c(P1[t]), xbv, m, xn, lam, hg, acc);
    }
    if (XO) XO[t] = XB[t];
    Mm[t] = (TS)m;
    if (A) A[t] = (TS)xn;
    if (PR) PR[t] = Store<TL>::from(xn);
    if constexpr (P2POUT) {
      for (int p = 0; p < a.exit.world; ++p)
        static_cast<TL*>(a.out_peers[p])[t] = Store<TL>::from(xn);
    }
    if (G) G[t] = (TS)lam;
  }
  if constexpr (P2POUT || AAR > 0)
    block_finish<NT>(acc.widen(), a.ws, &a.exit);
  else
    block_finish<NT>(acc.widen(), a.ws);
}

template <class M, int V, int U, int NT, int MINB, bool GHOST = false, bool P2POUT = false,
          int AAR = 0>
__global__ void __launch_bounds__(NT, MINB) fused_step_kernel(const StepArgs a) {
  fused_step_body<M, V, U, NT, GHOST, P2POUT, AAR>(a);
}

// Register-capped worker-local step (co2_set_fused_variant 6 / 7): with at
// most REGS registers, four 256-thread CTAs leave 65536 - 1024 * REGS
// registers of the SM free, so a reduce CTA on the comm stream can be
// resident beside them instead of displacing one (the multi-GPU rounds).
template <class M, int V, int U, int REGS>
__global__ void __maxnreg__(REGS) fused_step_kernel_r(const StepArgs a) {
  fused_step_body<M, V, U, 256, false, false, 0>(a);
}

constexpr int kThreads = 256;

// Grid waves for the grid-stride kernels, in units of the resident CTAs of an
// idle GPU (1 = persistent).  Measured on B200 (profiles/r01/README.md): a
// persistent grid leaves SMs idle at the end (uneven per-CTA progress across
// the two dies' HBM) and, when a reduce kernel co-runs on the comm stream and
// holds registers on some SMs, runs a late second wave.  Oversubscribing with
// short CTAs lets the block scheduler balance: C3 N=1 0.887 -> 1.03 of the
// measured copy bandwidth, N=2 / N=4 +24% / +33%.  Default 32 waves
// (co2_set_grid_waves / CO2_GRID_WAVES to tune).
// Knobs are atomics: a setter may race launches issued from other threads.
std::atomic<int> g_waves{-1};
int grid_waves() {
  int w = g_waves.load(std::memory_order_relaxed);
  if (w < 0) {
    const char* e = getenv("CO2_GRID_WAVES");
    w = e ? atoi(e) : 32;
    if (w < 1) w = 1;
    if (w > 64) w = 64;
    int expect = -1;
    g_waves.compare_exchange_strong(expect, w, std::memory_order_relaxed);
    w = g_waves.load(std::memory_order_relaxed);
  }
  return w;
}

// Oversubscription stops where CTAs would get shorter than min_cta_iters()
// grid-stride iterations: below that the per-CTA fixed cost (diagnostic
// partial + ticket atomic, CTA launch) shows.  C2 (125M fp32, 0.72 ms) at
// 32 waves gives 6.4 iterations per CTA.  Sweep (profiles/r01/bench/
// c2_min_iters.txt): 8 -> N=1 +1.6 %, N=2 +0.9 %, N=4 +-0; 32 -> N=1 +4 %
// but N=2 -2.5 % (the co-running reduce wants the shorter CTAs).  C3 (33
// iterations at 32 waves) is unaffected.  CO2_MIN_CTA_ITERS overrides
// (0 = always the full wave count).
int min_cta_iters() {
  static const int v = [] {
    const char* e = getenv("CO2_MIN_CTA_ITERS");
    int x = e ? atoi(e) : 8;
    return x < 0 ? 0 : x;
  }();
  return v;
}

template <typename K>
int grid_for(K kernel, int64_t work_items, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t wave = (int64_t)per_sm * sm_count();
  int64_t waves = grid_waves();
  if (min_cta_iters() > 0) {
    const int64_t fit = (work_items + threads - 1) / threads / (wave * min_cta_iters());
    if (fit < waves) waves = fit < 1 ? 1 : fit;
  }
  int64_t cap = wave * waves;
  if (cap > kMaxBlocks) cap = kMaxBlocks;
  int64_t need = (work_items + threads - 1) / threads;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

template <class M, int V, int U, int MINB = 1>
void launch_variant(const StepArgs& a, cudaStream_t s) {
  auto k = fused_step_kernel<M, V, U, kThreads, MINB>;
  int grid = grid_for(k, (a.n / V + U - 1) / U, kThreads);
  k<<<grid, kThreads, 0, s>>>(a);
}

template <class M, int V, int U, int REGS>
void launch_variant_r(const StepArgs& a, cudaStream_t s) {
  auto k = fused_step_kernel_r<M, V, U, REGS>;
  int grid = grid_for(k, (a.n / V + U - 1) / U, kThreads);
  k<<<grid, kThreads, 0, s>>>(a);
}

template <class M>
co2_status_t launch_ghost_p2p(const StepArgs& a, cudaStream_t s) {
  bool vec_ok = aligned16(a.x_t0) && aligned16(a.p0) && aligned16(a.p1) && aligned16(a.xbar) &&
                aligned16(a.m) && aligned16(a.anchor) && aligned16(a.gap) &&
                aligned16(a.bar0_out);
  for (int p = 0; p < a.exit.world; ++p) vec_ok = vec_ok && aligned16(a.out_peers[p]);
  if (!vec_ok) return fail(CO2_ERR_VALIDATION, "p2p sharded step: buffers must be 16-byte aligned");
  constexpr int V = std::is_same<M, ModeF64>::value ? 2 : (std::is_same<M, ModeF32>::value ? 4 : 8);
  auto k = fused_step_kernel<M, V, 1, kThreads, 3, true, true>;
  k<<<grid_for(k, a.n / V, kThreads), kThreads, 0, s>>>(a);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

template <class M>
co2_status_t launch_ghost(const StepArgs& a, cudaStream_t s) {
  bool vec_ok = aligned16(a.x_t0) && aligned16(a.p0) && aligned16(a.p1) && aligned16(a.xbar) &&
                aligned16(a.m) && aligned16(a.anchor) && aligned16(a.params) &&
                aligned16(a.gap) && aligned16(a.bar0_out);
  if (!vec_ok) {
    auto k = fused_step_kernel<M, 1, 4, kThreads, 1, true>;
    k<<<grid_for(k, (a.n + 3) / 4, kThreads), kThreads, 0, s>>>(a);
  } else {
    constexpr int V = std::is_same<M, ModeF64>::value ? 2 : (std::is_same<M, ModeF32>::value ? 4 : 8);
    auto k = fused_step_kernel<M, V, 1, kThreads, 3, true>;
    k<<<grid_for(k, a.n / V, kThreads), kThreads, 0, s>>>(a);
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

// Tuning knob: CO2_FUSED_VARIANT selects the (elements per vector, vectors
// in flight per thread) instantiation; 0 is the measured default.
std::atomic<int> g_variant{-1};
int fused_variant() {
  int v = g_variant.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("CO2_FUSED_VARIANT");
    v = e ? atoi(e) : 0;
    if (v < 0) v = 0;
    int expect = -1;
    g_variant.compare_exchange_strong(expect, v, std::memory_order_relaxed);
    v = g_variant.load(std::memory_order_relaxed);
  }
  return v;
}

// ------------------------------------------- bulk-copy (TMA 1D) fused step
// The same per-element body as fused_step_kernel, with the five input
// streams moved by the TMA engine instead of per-thread LDGs:
//   * one producer lane per CTA claims TILE-element tiles from a global
//     counter (dynamic: a co-running reduce kernel slows some SMs, the
//     counter keeps every SM busy to the end) and issues five
//     cp.async.bulk global->shared copies per tile into a STAGES-deep ring,
//     completing on the stage's `full` mbarrier (expect_tx);
//   * NCW consumer warps wait on `full`, read 16 B per lane per stream from
//     shared memory (conflict-free: lane-contiguous), compute, store the
//     outputs with 128-bit evict-first STGs, and release the stage on its
//     `empty` mbarrier (one arrive per warp).
// Bytes in flight sit in shared memory (STAGES x 16-20 KB per CTA), so the
// kernel needs few registers and threads per SM: a reduce kernel on the comm
// stream co-resides without displacing step CTAs (the register-file limit of
// the LDG kernel at 4 x 256 x 64 registers).  Diagnostics are min / max /
// counts / OR, independent of which CTA processed which tile, so dynamic
// scheduling keeps them deterministic.  Aliasing as in fused_step_kernel
// (anchor over prev_x0, params over xbar) is safe: a tile's outputs are
// written after its inputs landed in shared memory.
// Lane-contiguous shared-memory vector read (16 / 8 B per lane).
template <typename T, int N>
__device__ __forceinline__ void ld_smem(const T* p, T (&out)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  static_assert(BYTES == 16 || BYTES == 8, "smem vector");
  if constexpr (BYTES == 16) {
    const uint4 r = *reinterpret_cast<const uint4*>(p);
    memcpy(out, &r, 16);
  } else {
    const uint2 r = *reinterpret_cast<const uint2*>(p);
    memcpy(out, &r, 8);
  }
}

template <class M, int TILE>
struct BulkStage {
  using TS = typename M::TS;
  using TL = typename M::TL;
  static constexpr int kS = TILE * (int)sizeof(TS);
  static constexpr int kL = TILE * (int)sizeof(TL);
  static constexpr int kBytes = 3 * kS + 2 * kL;  // x_t0, p0, m | p1, xbar
};

// mbarriers full[STAGES], empty[STAGES] and the tile index per stage, padded
// so every stage buffer stays 128-byte aligned.
__host__ __device__ constexpr size_t bulk_hdr_bytes(int stages) { return ((size_t)stages * 24 + 127) / 128 * 128; }

template <class M, int TILE, int STAGES, int NCW>
constexpr size_t bulk_smem_bytes() {
  return (size_t)STAGES * BulkStage<M, TILE>::kBytes + bulk_hdr_bytes(STAGES);
}

template <class M, int TILE, int STAGES, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) bulk_step_kernel(const StepArgs a) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  using SG = BulkStage<M, TILE>;
  constexpr int NT = (NCW + 1) * 32;
  constexpr int VE = 16 / (int)sizeof(TS);  // elements per lane per access
  constexpr int GROUPS = TILE / (NCW * 32 * VE);
  static_assert(TILE % (NCW * 32 * VE) == 0, "tile must split evenly over the consumer lanes");
  constexpr bool LQ = !std::is_same<TS, TL>::value;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + STAGES;
  long long* tile_of = reinterpret_cast<long long*>(empty + STAGES);
  unsigned char* ring = smem + bulk_hdr_bytes(STAGES);

  Hyp<TC> h;
  h.tau = (TC)a.tau;
  h.eps = (TC)a.eps;
  h.beta = (TC)a.beta;
  h.phi = (TC)a.phi;
  h.alpha = (TC)a.alpha;
  h.divisor = (TC)a.divisor;
  h.penalty = a.penalty;
  h.clip = a.clip;
  h.divide = a.divisor > 1;
  Hyp<TC> hg = h;
  hg.divide = 0;

  const TS* __restrict__ X = static_cast<const TS*>(a.x_t0);
  const TS* __restrict__ P0 = static_cast<const TS*>(a.p0);
  const TL* __restrict__ P1 = static_cast<const TL*>(a.p1);
  const TL* XB = static_cast<const TL*>(a.xbar);
  TS* Mm = static_cast<TS*>(a.m);
  TS* A = static_cast<TS*>(a.anchor);
  TL* PR = static_cast<TL*>(a.params);
  TS* G = static_cast<TS*>(a.gap);
  TL* XO = static_cast<TL*>(a.xbar_out);
  WsHeader* hdr = ws_header(a.ws);
  const long long ntiles = a.n / TILE;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  AccT<TC> acc;
  if (warp == NCW) {
    if (lane == 0) {  // producer
      const uint64_t pol = evict_first_policy();
      for (int it = 0;; ++it) {
        const int s = it % STAGES;
        const unsigned ph = (unsigned)(it / STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        const long long t = (long long)atomicAdd(&hdr->tile_next, 1u);
        if (t >= ntiles) {
          tile_of[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        tile_of[s] = t;
        unsigned char* st = ring + (size_t)s * SG::kBytes;
        const int64_t e = t * (int64_t)TILE;
        mbar_arrive_expect_tx(&full[s], SG::kBytes);
        bulk_g2s(st, X + e, SG::kS, &full[s], pol);
        bulk_g2s(st + SG::kS, P0 + e, SG::kS, &full[s], pol);
        bulk_g2s(st + 2 * SG::kS, Mm + e, SG::kS, &full[s], pol);
        bulk_g2s(st + 3 * SG::kS, P1 + e, SG::kL, &full[s], pol);
        bulk_g2s(st + 3 * SG::kS + SG::kL, XB + e, SG::kL, &full[s], pol);
      }
    }
  } else {  // consumers
    for (int it = 0;; ++it) {
      const int s = it % STAGES;
      const unsigned ph = (unsigned)(it / STAGES) & 1u;
      mbar_wait(&full[s], ph);
      const long long t = tile_of[s];
      if (t < 0) break;
      const unsigned char* st = ring + (size_t)s * SG::kBytes;
      const TS* sx = reinterpret_cast<const TS*>(st);
      const TS* sp0 = reinterpret_cast<const TS*>(st + SG::kS);
      const TS* sm = reinterpret_cast<const TS*>(st + 2 * SG::kS);
      const TL* sp1 = reinterpret_cast<const TL*>(st + 3 * SG::kS);
      const TL* sxb = reinterpret_cast<const TL*>(st + 3 * SG::kS + SG::kL);
#pragma unroll
      for (int g = 0; g < GROUPS; ++g) {
        const int o = (g * NCW * 32 + warp * 32 + lane) * VE;
        TS x[VE], q0[VE], mo[VE];
        TL q1[VE], xb[VE];
        ld_smem<TS, VE>(sx + o, x);
        ld_smem<TS, VE>(sp0 + o, q0);
        ld_smem<TS, VE>(sm + o, mo);
        ld_smem<TL, VE>(sp1 + o, q1);
        ld_smem<TL, VE>(sxb + o, xb);
        TS mn[VE], xs[VE], gs[VE];
        TL xl[VE];
#pragma unroll
        for (int v = 0; v < VE; ++v) {
          TC m = to_c(mo[v]), xn, lam;
          TC xbv = to_c(xb[v]);
          if (h.divide) xbv = div_rn_nz(xbv, h.divisor);  // average(): sum / G, param_ops.cpp:30
          co2_elem<TC, LQ>(to_c(x[v]), to_c(q0[v]), to_c(q1[v]), xbv, m, xn, lam, hg, acc);
          mn[v] = (TS)m;
          xs[v] = (TS)xn;
          gs[v] = (TS)lam;
          xl[v] = Store<TL>::from(xn);
        }
        const int64_t e = t * (int64_t)TILE + o;
        st_vec<TS, VE>(Mm + e, mn);
        if (A) st_vec<TS, VE>(A + e, xs);
        if (PR) st_vec<TL, VE>(PR + e, xl);
        if (G) st_vec<TS, VE>(G + e, gs);
        if (XO) st_vec<TL, VE>(XO + e, xb);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  // Tail (n % TILE coordinates): the last CTA, straight from global memory.
  if (blockIdx.x == gridDim.x - 1) {
    for (int64_t j = ntiles * (int64_t)TILE + threadIdx.x; j < a.n; j += NT) {
      TC m = to_c(Mm[j]), xn, lam;
      TC xbv = to_c(XB[j]);
      if (h.divide) xbv = div_rn_nz(xbv, h.divisor);
      co2_elem<TC, LQ>(to_c(X[j]), to_c(P0[j]), to_c(P1[j]), xbv, m, xn, lam, hg, acc);
      if (XO) XO[j] = XB[j];
      Mm[j] = (TS)m;
      if (A) A[j] = (TS)xn;
      if (PR) PR[j] = Store<TL>::from(xn);
      if (G) G[j] = (TS)lam;
    }
  }
  if (block_finish<NT>(acc.widen(), a.ws) && threadIdx.x == 0) {
    // Every producer has fetched its terminating index: reset the tile
    // counter for the next launch on this workspace (like the ticket).
    hdr->tile_next = 0u;
    __threadfence();
  }
}

template <class M, int TILE, int STAGES, int NCW>
co2_status_t launch_bulk(const StepArgs& a, cudaStream_t s) {
  auto k = bulk_step_kernel<M, TILE, STAGES, NCW>;
  constexpr size_t smem = bulk_smem_bytes<M, TILE, STAGES, NCW>();
  constexpr int NT = (NCW + 1) * 32;
  static const int per_sm = [&] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, NT, smem);
    return v < 1 ? 1 : v;
  }();
  int64_t grid = (int64_t)per_sm * sm_count();
  const int64_t tiles = a.n / TILE;
  if (grid > tiles) grid = tiles < 1 ? 1 : tiles;
  k<<<(int)grid, NT, smem, s>>>(a);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

// Bulk-copy variants (co2_set_fused_variant >= 10): (TILE, STAGES, consumer
// warps) per mode.  Stage bytes: TILE x 16 (bf16-mixed), x 20 (fp32), x 40 (fp64).
template <class M>
co2_status_t launch_bulk_variant(int v, const StepArgs& a, cudaStream_t s) {
  if constexpr (std::is_same<M, ModeBF16>::value) {
    switch (v) {
      case 11: return launch_bulk<M, 1024, 4, 4>(a, s);   // 64 KB: 3 CTA/SM
      case 12: return launch_bulk<M, 2048, 3, 8>(a, s);   // 96 KB: 2 CTA/SM
      case 13: return launch_bulk<M, 4096, 3, 8>(a, s);   // 192 KB: 1 CTA/SM
      case 14: return launch_bulk<M, 1024, 6, 8>(a, s);   // 96 KB: 2 CTA/SM
      default: return launch_bulk<M, 2048, 4, 4>(a, s);   // 128 KB: 1 CTA/SM
    }
  } else if constexpr (std::is_same<M, ModeF32>::value) {
    switch (v) {
      case 11: return launch_bulk<M, 1024, 4, 4>(a, s);   // 80 KB: 2 CTA/SM
      case 12: return launch_bulk<M, 2048, 4, 8>(a, s);   // 160 KB: 1 CTA/SM
      case 13: return launch_bulk<M, 1024, 8, 8>(a, s);   // 160 KB
      case 14: return launch_bulk<M, 512, 6, 4>(a, s);    // 60 KB: 3 CTA/SM
      default: return launch_bulk<M, 1024, 5, 4>(a, s);   // 100 KB: 2 CTA/SM
    }
  } else {
    switch (v) {
      case 11: return launch_bulk<M, 256, 6, 2>(a, s);    // 60 KB: 3 CTA/SM
      case 12: return launch_bulk<M, 1024, 4, 8>(a, s);   // 160 KB: 1 CTA/SM
      default: return launch_bulk<M, 512, 5, 4>(a, s);    // 100 KB: 2 CTA/SM
    }
  }
}

template <class M>
co2_status_t launch_fused(const StepArgs& a, cudaStream_t s) {
  bool vec_ok = aligned16(a.x_t0) && aligned16(a.p0) && aligned16(a.p1) && aligned16(a.xbar) &&
                aligned16(a.m) && aligned16(a.anchor) && aligned16(a.params) && aligned16(a.gap) &&
                aligned16(a.xbar_out);
  if (vec_ok && fused_variant() >= 10) {
    return launch_bulk_variant<M>(fused_variant(), a, s);
  }
  if (!vec_ok) {
    launch_variant<M, 1, 4>(a, s);
  } else if constexpr (std::is_same<M, ModeBF16>::value) {
    // Measured on B200 (tools/tune_fused.py, C3 1.3B): one 8-element vector
    // per thread (32 B fp32 + 16 B bf16 per stream) at >= 3 CTAs/SM beats
    // deeper per-thread unrolling, which costs occupancy.
    switch (fused_variant()) {
      case 1: launch_variant<M, 8, 2>(a, s); break;
      case 2: launch_variant<M, 4, 4>(a, s); break;
      case 3: launch_variant<M, 4, 1>(a, s); break;
      case 4: launch_variant<M, 8, 1>(a, s); break;
      case 5: launch_variant<M, 4, 2, 3>(a, s); break;
      case 6: launch_variant_r<M, 8, 1, 56>(a, s); break;
      case 7: launch_variant_r<M, 4, 1, 56>(a, s); break;
      default: launch_variant<M, 8, 1, 4>(a, s); break;
    }
  } else if constexpr (std::is_same<M, ModeF32>::value) {
    switch (fused_variant()) {
      case 1: launch_variant<M, 4, 2>(a, s); break;
      case 2: launch_variant<M, 4, 1>(a, s); break;
      case 3: launch_variant<M, 8, 1>(a, s); break;
      case 4: launch_variant<M, 8, 1, 4>(a, s); break;
      case 5: launch_variant<M, 4, 2, 4>(a, s); break;
      case 6: launch_variant_r<M, 4, 1, 56>(a, s); break;
      case 7: launch_variant_r<M, 4, 1, 48>(a, s); break;
      default: launch_variant<M, 4, 1, 4>(a, s); break;
    }
  } else {
    switch (fused_variant()) {
      case 1: launch_variant<M, 2, 2>(a, s); break;
      case 2: launch_variant<M, 2, 1>(a, s); break;
      case 3: launch_variant<M, 4, 1>(a, s); break;
      case 4: launch_variant<M, 2, 2, 3>(a, s); break;
      case 5: launch_variant<M, 2, 1, 3>(a, s); break;
      default: launch_variant<M, 2, 1, 4>(a, s); break;
    }
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

// ------------------------------------------------------ unfused operators
template <typename T>
struct Ptrs64 {
  const T* p[64];
};

enum OpKind { OP_GAP = 0, OP_MOMENTUM = 1, OP_ITERATE = 2, OP_CLIP = 3, OP_FINITE = 4,
              OP_ABSDIFF = 5 };

struct OpArgs {
  const void* a;
  const void* b;
  const void* c;
  void* out;
  int64_t n;
  double s0, s1;  // scalars (tau/eps, beta/-, alpha/phi, phi/-)
  int i0;         // penalty / clip flag
  void* ws;
};

// T storage, TC compute.
template <typename T, typename TC, int OP>
__global__ void __launch_bounds__(kThreads) op_kernel(const OpArgs a) {
  const T* A = static_cast<const T*>(a.a);
  const T* B = static_cast<const T*>(a.b);
  const T* Cc = static_cast<const T*>(a.c);
  T* O = static_cast<T*>(a.out);
  Acc acc;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < a.n;
       j += (int64_t)gridDim.x * kThreads) {
    if (OP == OP_GAP) {  // outer_algorithms.cpp:57-62
      TC tau = (TC)a.s0, eps = (TC)a.s1;
      TC x = to_c(A[j]), q0 = to_c(B[j]), q1 = to_c(Cc[j]);
      TC n0 = fabs(x - q0);
      TC av = fabs(tau * (q1 - q0));
      bool fl = av < eps;
      TC d = fl ? eps : av;
      TC lam = div_rn(n0, d) + (TC)1;
      if (!isfinite(lam)) acc.flags |= CO2_FLAG_GAP_NONFINITE;
      acc.floored += fl;
      double dl = (double)lam;
      acc.min_gap = dl < acc.min_gap ? dl : acc.min_gap;
      O[j] = Store<T>::from(lam);
    } else if (OP == OP_MOMENTUM) {  // outer_algorithms.cpp:78-88
      TC beta = (TC)a.s0;
      TC mp = to_c(A[j]), g = to_c(B[j]), dl = to_c(Cc[j]);
      TC m;
      if (a.i0) {
        if (g < (TC)1) acc.flags |= CO2_FLAG_GAP_BELOW_ONE;
        TC bm = beta * mp;
        TC q = div_rn(dl, g);  // gap: an arbitrary input array
        m = bm + q;
      } else {
        TC bm = beta * mp;
        m = bm + dl;
      }
      if (!isfinite(m)) acc.flags |= CO2_FLAG_M_NONFINITE;
      O[j] = Store<T>::from(m);
    } else if (OP == OP_ITERATE) {  // outer_algorithms.cpp:100-106
      TC alpha = (TC)a.s0, phi = (TC)a.s1;
      TC x = to_c(A[j]), m = to_c(B[j]);
      TC c = m;
      if (a.i0) {
        if (!isfinite(m)) acc.flags |= CO2_FLAG_CLIP_NONFINITE;
        acc.clipped += (m < -phi) || (phi < m);
        TC lo = (m < -phi) ? -phi : m;
        c = (phi < lo) ? phi : lo;
      }
      TC ac = alpha * c;
      TC xn = x - ac;
      if (!isfinite(xn)) acc.flags |= CO2_FLAG_X_NONFINITE;
      double st = (double)fabs(xn - x);
      acc.max_step = st > acc.max_step ? st : acc.max_step;
      O[j] = Store<T>::from(xn);
    } else if (OP == OP_CLIP) {  // param_ops.cpp:35-43
      TC phi = (TC)a.s0;
      TC v = to_c(A[j]);
      if (!isfinite(v)) acc.flags |= CO2_FLAG_CLIP_NONFINITE;
      acc.clipped += (v < -phi) || (phi < v);
      TC lo = (v < -phi) ? -phi : v;
      O[j] = Store<T>::from((phi < lo) ? phi : lo);
    } else if (OP == OP_ABSDIFF) {  // elementwise_abs_diff, param_ops.cpp:44-51
      TC r = fabs(to_c(A[j]) - to_c(B[j]));
      if (!isfinite(r)) acc.flags |= CO2_FLAG_NONFINITE_INPUT;
      O[j] = Store<T>::from(r);
    } else {  // OP_FINITE, ensure_finite (param_ops.cpp:10-14)
      if (!isfinite(to_c(A[j]))) acc.flags |= CO2_FLAG_NONFINITE_INPUT;
    }
  }
  block_finish<kThreads>(acc, a.ws);
}

template <typename T, typename TC>
__global__ void __launch_bounds__(kThreads)
    average_kernel(const Ptrs64<T> c, int g, T* out, int64_t n, void* ws) {
  // param_ops.cpp:16-33: ascending-worker sum, one division by G.
  Acc acc;
  const TC gd = (TC)g;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kThreads) {
    TC s = to_c(c.p[0][j]);
    for (int i = 1; i < g; ++i) s += to_c(c.p[i][j]);
    TC r = div_rn_nz(s, gd);
    if (!isfinite(r)) acc.flags |= CO2_FLAG_AVG_NONFINITE;
    out[j] = Store<T>::from(r);
  }
  block_finish<kThreads>(acc, ws);
}

// 16-byte-vector form of average_kernel (every contribution and the output
// 16-byte aligned): per vector the contributions are loaded four at a time
// and accumulated in ascending worker order, then divided once -- the same
// per-element op sequence as the scalar kernel, so results are identical.
template <typename T, typename TC>
__global__ void __launch_bounds__(kThreads)
    average_vec_kernel(const Ptrs64<T> c, int g, T* out, int64_t n, void* ws) {
  constexpr int V = 16 / (int)sizeof(T);
  Acc acc;
  const TC gd = (TC)g;
  const int64_t nv = n / V;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nv; i += stride) {
    const int64_t e = i * V;
    TC s[V];
    for (int i0 = 0; i0 < g; i0 += 4) {
      uint4 raw[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i0 + k < g) raw[k] = __ldcs(reinterpret_cast<const uint4*>(c.p[i0 + k] + e));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (i0 + k < g) {
          const T* v = reinterpret_cast<const T*>(&raw[k]);
#pragma unroll
          for (int q = 0; q < V; ++q) s[q] = (i0 + k == 0) ? to_c(v[q]) : s[q] + to_c(v[q]);
        }
      }
    }
    T o[V];
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const TC r = div_rn_nz(s[q], gd);
      if (!isfinite(r)) acc.flags |= CO2_FLAG_AVG_NONFINITE;
      o[q] = Store<T>::from(r);
    }
    st_vec<T, V>(out + e, o);
  }
  if (blockIdx.x == 0) {  // scalar tail
    for (int64_t j = nv * V + threadIdx.x; j < n; j += kThreads) {
      TC s = to_c(c.p[0][j]);
      for (int i = 1; i < g; ++i) s += to_c(c.p[i][j]);
      const TC r = div_rn_nz(s, gd);
      if (!isfinite(r)) acc.flags |= CO2_FLAG_AVG_NONFINITE;
      out[j] = Store<T>::from(r);
    }
  }
  block_finish<kThreads>(acc, ws);
}

template <typename T, typename TC>
__global__ void sub_kernel(const T* a, const T* b, T* o, int64_t n) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    TC r = to_c(a[j]) - to_c(b[j]);
    o[j] = Store<T>::from(r);
  }
}

template <typename TD, typename TSRC>
__global__ void convert_kernel(TD* d, const TSRC* s, int64_t n) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(TD) == 8 || sizeof(TSRC) == 8) {
      d[j] = Store<TD>::from((decltype(to_c(TD{})))to_c(s[j]));
    } else {
      d[j] = Store<TD>::from((float)to_c(s[j]));
    }
  }
}

// ------------------------------------------------------- synthetic inputs
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:45-49
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ double sym_at(uint64_t key, int64_t j) {
  // rng.hpp:17-25 in random-access form: draw j uses counter j+1.
  uint64_t u = mix64(key + (uint64_t)(j + 1) * kGolden);
  double U = (double)(u >> 11) * 0x1.0p-53;
  return 2.0 * U - 1.0;
}

template <class M>
__global__ void synth_kernel(uint64_t kp0, uint64_t kp1, uint64_t kx, uint64_t ke, uint64_t km,
                             int64_t j0, int64_t count, typename M::TS* x_t0,
                             typename M::TS* p0, typename M::TL* p1, typename M::TL* x_end,
                             typename M::TS* m) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + i;
    // round_state: double -> state dtype -> back to double.
    double p0v = (double)(TS)(0.02 * sym_at(kp0, j));
    const bool stalled = (j % 61) == 0;
    if (stalled) p0v = (double)to_c(Store<TL>::from((TC)p0v));
    if (p0) p0[i] = (TS)p0v;
    if (p1) {
      double v = stalled ? p0v : p0v - 1e-3 * sym_at(kp1, j);
      p1[i] = Store<TL>::from((TC)v);
    }
    if (x_t0) x_t0[i] = (TS)(p0v + 4e-3 * sym_at(kx, j));
    if (x_end) x_end[i] = Store<TL>::from((TC)(p0v - 4e-3 * sym_at(ke, j)));
    if (m) m[i] = (TS)(1e-2 * sym_at(km, j));
  }
}

// snap (nullable): SURVEY.md 8f item 2 -- the InnerTrace snapshot x_{t,1}
// (inner_loop.cpp:96-98) captured by the inner step's own store instead of a
// separate copy pass over the params.
template <typename T, typename TC>
__global__ void inner_step_kernel(T* x, int64_t n, double lr, double scale, uint64_t key,
                                  int64_t offset, int repeat, T* snap) {
  const TC lrc = (TC)lr, sc = (TC)scale;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    TC g = 0;
    for (int r = 0; r < repeat; ++r) g += sc * (TC)sym_at(key, offset + j + (int64_t)r * n);
    TC v = to_c(x[j]);
    TC step = lrc * g;
    const T out = Store<T>::from(v - step);
    x[j] = out;
    if (snap) snap[j] = out;
  }
}

__global__ void fill_u32_kernel(uint32_t* d, uint32_t v, int64_t n) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    d[j] = v;
}

uint64_t host_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t host_key(uint64_t seed, uint64_t stream) {  // rng.hpp:14-15
  return host_mix(host_mix(seed + kGolden) ^ stream);
}

int simple_grid(int64_t n, int threads) {
  int64_t need = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 8;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

co2_status_t check_dtype(co2_dtype_t dt) {
  if (dt != CO2_DTYPE_F64 && dt != CO2_DTYPE_F32 && dt != CO2_DTYPE_BF16)
    return fail(CO2_ERR_VALIDATION, "unknown dtype %d", (int)dt);
  return CO2_OK;
}

template <int OP>
co2_status_t launch_op(co2_dtype_t dt, const OpArgs& a, cudaStream_t s) {
  CO2_TRY(check_dtype(dt));
  if (!a.ws) return fail(CO2_ERR_VALIDATION, "null workspace");
  // operands each op reads: GAP (x_t0, prev_x0, prev_x1), MOMENTUM (m, gap,
  // delta), ITERATE (x_t0, m), CLIP (v)
  const bool need_b = OP != OP_CLIP && OP != OP_FINITE;  // ABSDIFF reads b
  const bool need_c = OP == OP_GAP || OP == OP_MOMENTUM, need_out = OP != OP_FINITE;
  if (a.n > 0 && (!a.a || (need_out && !a.out) || (need_b && !a.b) || (need_c && !a.c)))
    return fail(CO2_ERR_VALIDATION, "null buffer");
  int grid = simple_grid(a.n, kThreads);
  if (grid > kMaxBlocks) grid = kMaxBlocks;
  if (dt == CO2_DTYPE_F64)
    op_kernel<double, double, OP><<<grid, kThreads, 0, s>>>(a);
  else if (dt == CO2_DTYPE_F32)
    op_kernel<float, float, OP><<<grid, kThreads, 0, s>>>(a);
  else
    op_kernel<bf16s, float, OP><<<grid, kThreads, 0, s>>>(a);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

}  // namespace

// ===================================================================== ABI
co2_status_t outer_step_impl(co2_mode_t mode, int64_t n, const void* x_t0, const void* p0,
                             const void* p1, const void* xbar, int32_t divisor, void* m,
                             void* anchor, void* params, void* gap, const co2_hyper_t* h,
                             void* ws, cudaStream_t s, void* xbar_out) {
  StepArgs a{x_t0, p0, p1, xbar, m, anchor, params, gap, n, h->alpha, h->beta, h->phi,
             h->epsilon, h->tau, divisor, h->penalty ? 1 : 0, h->clip ? 1 : 0, ws, 1, 0, 0,
             nullptr};
  a.xbar_out = xbar_out;
  switch (mode) {
    case CO2_MODE_F64: return launch_fused<ModeF64>(a, s);
    case CO2_MODE_F32: return launch_fused<ModeF32>(a, s);
    case CO2_MODE_BF16_MIXED: return launch_fused<ModeBF16>(a, s);
  }
  return fail(CO2_ERR_VALIDATION, "outer step: unknown mode %d", (int)mode);
}

namespace {
// ---------------------------------------------- global-norm clip extension
// NOT part of the reference parity contract: the reference clips
// coordinate-wise (param_ops.cpp:35-43, SURVEY.md 8 note 3).  The north
// star's wording asks for a global-norm clip of the outer momentum; it is
// provided as a separate entry (co2_outer_step_global_clip) with its own
// restatement in the test oracle:
//   pass 1: m' as in the fused step (gap, penalty), written in place, and
//           ||m'||^2 summed in fp64 over fixed chunks (gc_chunk) -- thread t
//           sums its vectors t, t+256, ... of the chunk in order, a fixed
//           xor-butterfly per warp, warps in order; the last block folds
//           the chunk sums the same way and stores sqrt into the workspace;
//   pass 2: c = m' * min(1, phi/||m'||) (scale in fp64), x' = x_t0 - alpha*c.
// The order depends on n and the mode only, so the norm is bitwise
// reproducible across grids and GPUs.  34 B/param in bf16-mixed (pass 1
// reads 16, writes 4; pass 2 reads 8, writes 6).
__device__ __forceinline__ double warp_sum_fixed(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

template <typename TC, bool LQ>
__device__ __forceinline__ TC gc_momentum(TC x, TC q0, TC q1, TC xb, TC m, TC& lam,
                                          const Hyp<TC>& h, AccT<TC>& acc) {
  TC n0 = fabs(x - q0);
  TC av = fabs(h.tau * (q1 - start_of_inner<TC, LQ>(q0)));
  bool floored = av < h.eps;
  TC d = floored ? h.eps : av;
  lam = div_rn(n0, d) + (TC)1;
  TC dl = q0 - xb;
  TC bm = h.beta * m;
  TC mn = h.penalty ? bm + div_rn_nz(dl, lam) : bm + dl;
  unsigned int f = 0;
  if (!isfinite(lam)) f |= CO2_FLAG_GAP_NONFINITE;
  if (h.penalty && lam < (TC)1) f |= CO2_FLAG_GAP_BELOW_ONE;
  if (!isfinite(mn)) f |= CO2_FLAG_M_NONFINITE;
  acc.flags |= f;
  acc.floored += floored;
  acc.min_gap = lam < acc.min_gap ? lam : acc.min_gap;
  return mn;
}

template <typename T, int V, bool VEC>
__device__ __forceinline__ void gc_load(const T* p, T (&out)[V]) {
  if constexpr (VEC) {
    ld_vec<T, V>(p, out);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = p[v];
  }
}

template <typename T, int V, bool VEC>
__device__ __forceinline__ void gc_store(T* p, const T (&in)[V]) {
  if constexpr (VEC) {
    st_vec<T, V>(p, in);
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) p[v] = in[v];
  }
}

template <class M>
__device__ __forceinline__ Hyp<typename M::TC> make_hyp(const StepArgs& a) {
  using TC = typename M::TC;
  Hyp<TC> h;
  h.tau = (TC)a.tau;
  h.eps = (TC)a.eps;
  h.beta = (TC)a.beta;
  h.phi = (TC)a.phi;
  h.alpha = (TC)a.alpha;
  h.divisor = (TC)a.divisor;
  h.penalty = a.penalty;
  h.clip = a.clip;
  h.divide = a.divisor > 1;
  return h;
}

template <class M, int V, bool VEC>
__global__ void __launch_bounds__(kGcThreads) gclip_pass1(const StepArgs a, int64_t chunk) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  constexpr int NT = kGcThreads, NW = NT / 32;
  const Hyp<TC> h = make_hyp<M>(a);
  const TS* X = static_cast<const TS*>(a.x_t0);
  const TS* P0 = static_cast<const TS*>(a.p0);
  const TL* P1 = static_cast<const TL*>(a.p1);
  const TL* XB = static_cast<const TL*>(a.xbar);
  TS* Mm = static_cast<TS*>(a.m);
  TS* G = static_cast<TS*>(a.gap);
  TL* XO = static_cast<TL*>(a.xbar_out);
  constexpr bool LQ = !std::is_same<TS, TL>::value;
  double* cs = ws_chunks(a.ws);
  __shared__ double sh[NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  AccT<TC> acc;
  const int64_t nvE = a.n / V * V;
  const int64_t K = (a.n + chunk - 1) / chunk;
  for (int64_t c = blockIdx.x; c < K; c += gridDim.x) {
    double s = 0.0;
    const int64_t e0 = c * chunk;
    const int64_t e1 = e0 + chunk < nvE ? e0 + chunk : nvE;
    for (int64_t e = e0 + (int64_t)threadIdx.x * V; e < e1; e += (int64_t)NT * V) {
      TS x[V], q0[V], mo[V], mn[V], gs[V];
      TL q1[V], xb[V];
      gc_load<TS, V, VEC>(X + e, x);
      gc_load<TS, V, VEC>(P0 + e, q0);
      gc_load<TL, V, VEC>(P1 + e, q1);
      gc_load<TL, V, VEC>(XB + e, xb);
      gc_load<TS, V, VEC>(Mm + e, mo);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        TC lam;
        TC xbv = to_c(xb[v]);
        if (h.divide) xbv = div_rn_nz(xbv, h.divisor);
        const TC m = gc_momentum<TC, LQ>(to_c(x[v]), to_c(q0[v]), to_c(q1[v]), xbv, to_c(mo[v]),
                                         lam, h, acc);
        mn[v] = (TS)m;
        gs[v] = (TS)lam;
        const double md = (double)mn[v];
        s = s + md * md;
      }
      gc_store<TS, V, VEC>(Mm + e, mn);
      if (G) gc_store<TS, V, VEC>(G + e, gs);
      if (XO) gc_store<TL, V, VEC>(XO + e, xb);
    }
    if (threadIdx.x == 0 && c == K - 1) {  // scalar tail, in index order
      for (int64_t e = nvE; e < a.n; ++e) {
        TC lam;
        TC xbv = to_c(XB[e]);
        if (h.divide) xbv = div_rn_nz(xbv, h.divisor);
        if (XO) XO[e] = XB[e];
        const TC m =
            gc_momentum<TC, LQ>(to_c(X[e]), to_c(P0[e]), to_c(P1[e]), xbv, to_c(Mm[e]), lam, h,
                                acc);
        Mm[e] = (TS)m;
        if (G) G[e] = (TS)lam;
        const double md = (double)(TS)m;
        s = s + md * md;
      }
    }
    s = warp_sum_fixed(s);
    if (lane == 0) sh[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = sh[0];
      for (int w = 1; w < NW; ++w) t = t + sh[w];
      cs[c] = t;
    }
    __syncthreads();
  }
  if (block_finish<NT>(acc.widen(), a.ws)) {  // last block: fold the chunk sums
    double b = 0.0;
    for (int64_t i = threadIdx.x; i < K; i += NT) b = b + __ldcg(cs + i);
    b = warp_sum_fixed(b);
    __syncthreads();
    if (lane == 0) sh[wid] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = sh[0];
      for (int w = 1; w < NW; ++w) t = t + sh[w];
      const double nrm = sqrt(t);
      WsHeader* hdr = ws_header(a.ws);
      hdr->pre = hdr->diag;
      if (!isfinite(nrm)) hdr->pre.flags |= CO2_FLAG_NORM_NONFINITE;
      hdr->gnorm = nrm;
      __threadfence();
    }
  }
}

template <class M, int V, bool VEC>
__global__ void __launch_bounds__(kGcThreads) gclip_pass2(const StepArgs a) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  constexpr int NT = kGcThreads;
  const TS* X = static_cast<const TS*>(a.x_t0);
  const TS* Mm = static_cast<const TS*>(a.m);
  TS* A = static_cast<TS*>(a.anchor);
  TL* PR = static_cast<TL*>(a.params);
  const double nrm = ws_header(a.ws)->gnorm;
  const double sc = (a.clip && nrm > a.phi) ? a.phi / nrm : 1.0;
  const unsigned int scaled = sc < 1.0 ? 1u : 0u;
  const TC alpha = (TC)a.alpha;
  AccT<TC> acc;
  auto elem = [&](TC x, TC m) -> TC {
    TC c;
    if constexpr (std::is_same<TC, double>::value)
      c = m * sc;
    else
      c = (TC)((double)m * sc);
    const TC ac = alpha * c;
    const TC xn = x - ac;
    if (!isfinite(xn)) acc.flags |= CO2_FLAG_X_NONFINITE;
    acc.clipped += scaled;
    const TC st = fabs(xn - x);
    acc.max_step = st > acc.max_step ? st : acc.max_step;
    return xn;
  };
  const int64_t nv = a.n / V;
  const int64_t stride = (int64_t)gridDim.x * NT;
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < nv; i += stride) {
    const int64_t e = i * V;
    TS x[V], mo[V], xs[V];
    TL xl[V];
    gc_load<TS, V, VEC>(X + e, x);
    gc_load<TS, V, VEC>(Mm + e, mo);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const TC xn = elem(to_c(x[v]), to_c(mo[v]));
      xs[v] = (TS)xn;
      xl[v] = Store<TL>::from(xn);
    }
    if (A) gc_store<TS, V, VEC>(A + e, xs);
    if (PR) gc_store<TL, V, VEC>(PR + e, xl);
  }
  const int64_t t = nv * V + (int64_t)blockIdx.x * NT + threadIdx.x;
  if (V > 1 && t < a.n) {
    const TC xn = elem(to_c(X[t]), to_c(Mm[t]));
    if (A) A[t] = (TS)xn;
    if (PR) PR[t] = Store<TL>::from(xn);
  }
  if (block_finish<NT>(acc.widen(), a.ws) && threadIdx.x == 0) {
    // merge pass 1's gap / momentum diagnostics (stored by its last block)
    WsHeader* hdr = ws_header(a.ws);
    hdr->diag.min_gap = hdr->pre.min_gap;
    hdr->diag.n_floored = hdr->pre.n_floored;
    hdr->diag.flags |= hdr->pre.flags;
    __threadfence();
  }
}

// l2_norm (param_ops.cpp:54-60) in the global-norm clip's fixed order: fp64
// squares summed per fixed chunk (thread t: vectors t, t+256, ...; the n % V
// tail to thread 0 of the last chunk), xor butterfly per warp, warps in
// order; the last CTA folds the chunk sums the same way and stores the sqrt
// in the workspace header.  Deterministic for a given n and dtype.
template <typename T, int V>
__global__ void __launch_bounds__(kGcThreads) sumsq_kernel(const T* v, int64_t n, int64_t chunk,
                                                          void* ws) {
  constexpr int NT = kGcThreads, NW = NT / 32;
  double* cs = ws_chunks(ws);
  __shared__ double sh[NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nvE = n / V * V;
  const int64_t K = (n + chunk - 1) / chunk;
  Acc acc;
  for (int64_t c = blockIdx.x; c < K; c += gridDim.x) {
    double s = 0.0;
    const int64_t e0 = c * chunk;
    const int64_t e1 = e0 + chunk < nvE ? e0 + chunk : nvE;
    for (int64_t e = e0 + (int64_t)threadIdx.x * V; e < e1; e += (int64_t)NT * V) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const double d = (double)to_c(v[e + k]);
        s = s + d * d;
      }
    }
    if (threadIdx.x == 0 && c == K - 1)
      for (int64_t e = nvE; e < n; ++e) {
        const double d = (double)to_c(v[e]);
        s = s + d * d;
      }
    s = warp_sum_fixed(s);
    if (lane == 0) sh[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = sh[0];
      for (int w = 1; w < NW; ++w) t = t + sh[w];
      cs[c] = t;
    }
    __syncthreads();
  }
  if (block_finish<NT>(acc, ws)) {
    double b = 0.0;
    for (int64_t i = threadIdx.x; i < K; i += NT) b = b + __ldcg(cs + i);
    b = warp_sum_fixed(b);
    __syncthreads();
    if (lane == 0) sh[wid] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = sh[0];
      for (int w = 1; w < NW; ++w) t = t + sh[w];
      ws_header(ws)->gnorm = sqrt(t);
      __threadfence();
    }
  }
}

template <typename T, int V>
co2_status_t launch_sumsq(const void* v, int64_t n, void* ws, cudaStream_t s) {
  const int64_t chunk = gc_chunk(n, V);
  const int64_t K = (n + chunk - 1) / chunk;
  auto k = sumsq_kernel<T, V>;
  k<<<grid_for(k, K * kGcThreads, kGcThreads), kGcThreads, 0, s>>>(static_cast<const T*>(v), n,
                                                                    chunk, ws);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

template <class M>
co2_status_t launch_global_clip(const StepArgs& a, cudaStream_t s) {
  constexpr int V = std::is_same<M, ModeF64>::value ? 2 : (std::is_same<M, ModeF32>::value ? 4 : 8);
  const bool vec = aligned16(a.x_t0) && aligned16(a.p0) && aligned16(a.p1) &&
                   aligned16(a.xbar) && aligned16(a.m) && aligned16(a.anchor) &&
                   aligned16(a.params) && aligned16(a.gap) && aligned16(a.xbar_out);
  const int64_t chunk = gc_chunk(a.n, V);
  const int64_t K = (a.n + chunk - 1) / chunk;
  if (vec) {
    auto k1 = gclip_pass1<M, V, true>;
    k1<<<grid_for(k1, K * kGcThreads, kGcThreads), kGcThreads, 0, s>>>(a, chunk);
    auto k2 = gclip_pass2<M, V, true>;
    k2<<<grid_for(k2, a.n / V, kGcThreads), kGcThreads, 0, s>>>(a);
  } else {
    auto k1 = gclip_pass1<M, V, false>;
    k1<<<grid_for(k1, K * kGcThreads, kGcThreads), kGcThreads, 0, s>>>(a, chunk);
    auto k2 = gclip_pass2<M, V, false>;
    k2<<<grid_for(k2, a.n / V, kGcThreads), kGcThreads, 0, s>>>(a);
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}
}  // namespace

co2_status_t outer_step_global_clip_impl(co2_mode_t mode, int64_t n, const void* x_t0,
                                         const void* p0, const void* p1, const void* xbar,
                                         int32_t divisor, void* m, void* anchor, void* params,
                                         void* gap, const co2_hyper_t* h, void* ws,
                                         cudaStream_t s, void* xbar_out) {
  StepArgs a{x_t0, p0, p1, xbar, m, anchor, params, gap, n, h->alpha, h->beta, h->phi,
             h->epsilon, h->tau, divisor, h->penalty ? 1 : 0, h->clip ? 1 : 0, ws, 1, 0, 0,
             nullptr};
  a.xbar_out = xbar_out;
  switch (mode) {
    case CO2_MODE_F64: return launch_global_clip<ModeF64>(a, s);
    case CO2_MODE_F32: return launch_global_clip<ModeF32>(a, s);
    case CO2_MODE_BF16_MIXED: return launch_global_clip<ModeBF16>(a, s);
  }
  return fail(CO2_ERR_VALIDATION, "outer step: unknown mode %d", (int)mode);
}

namespace {
template <class M>
co2_status_t launch_fused_aar(const StepArgs& a, cudaStream_t s) {
  constexpr int V = std::is_same<M, ModeF64>::value ? 2 : (std::is_same<M, ModeF32>::value ? 4 : 8);
  bool ok = aligned16(a.x_t0) && aligned16(a.p0) && aligned16(a.p1) && aligned16(a.xbar) &&
            aligned16(a.m) && aligned16(a.anchor) && aligned16(a.params) && aligned16(a.gap) &&
            aligned16(a.xbar_out);
  for (int p = 0; p < a.exit.world; ++p) ok = ok && aligned16(a.aar_bufs[p]);
  if (!ok) return fail(CO2_ERR_VALIDATION, "fused all-reduce step: buffers must be 16-byte aligned");
  // Rank capacity of the instantiation: the gather registers scale with it
  // (8 x 16 B spilled at 4 CTAs/SM when one instantiation served all G).
  if (a.exit.world <= 2) {
    auto k = fused_step_kernel<M, V, 1, kThreads, 3, false, false, 2>;
    k<<<grid_for(k, a.n / V, kThreads), kThreads, 0, s>>>(a);
  } else if (a.exit.world <= 4) {
    auto k = fused_step_kernel<M, V, 1, kThreads, 3, false, false, 4>;
    k<<<grid_for(k, a.n / V, kThreads), kThreads, 0, s>>>(a);
  } else {
    auto k = fused_step_kernel<M, V, 1, kThreads, 3, false, false, 8>;
    k<<<grid_for(k, a.n / V, kThreads), kThreads, 0, s>>>(a);
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}
}  // namespace

co2_status_t outer_step_fused_aar_impl(co2_mode_t mode, int64_t n, const void* x_t0,
                                       const void* p0, const void* p1, const void* xbar_avg,
                                       void* m, void* anchor, void* params, void* gap,
                                       const co2_hyper_t* h, void* const* aar_bufs,
                                       int64_t aar_lo, int64_t aar_len, void* const* sigs,
                                       int world, int rank, uint32_t epoch, void* ws,
                                       cudaStream_t s, void* xbar_out) {
  if (world < 1 || world > kMaxRanks)
    return fail(CO2_ERR_VALIDATION, "fused all-reduce step: world must lie in [1, %d]", kMaxRanks);
  StepArgs a{x_t0, p0, p1, xbar_avg, m, anchor, params, gap, n, h->alpha, h->beta, h->phi,
             h->epsilon, h->tau, 1, h->penalty ? 1 : 0, h->clip ? 1 : 0, ws, 1, 0, 0, nullptr};
  a.xbar_out = xbar_out;
  for (int p = 0; p < world; ++p) {
    a.aar_bufs[p] = aar_bufs[p];
    a.exit.sig[p] = static_cast<Signals*>(sigs[p]);
  }
  a.exit.world = world;
  a.exit.rank = rank;
  a.exit.epoch = epoch;
  a.exit.counter = 1;
  a.aar_lo = aar_lo;
  a.aar_len = aar_len;
  switch (mode) {
    case CO2_MODE_F64: return launch_fused_aar<ModeF64>(a, s);
    case CO2_MODE_F32: return launch_fused_aar<ModeF32>(a, s);
    case CO2_MODE_BF16_MIXED: return launch_fused_aar<ModeBF16>(a, s);
  }
  return fail(CO2_ERR_VALIDATION, "outer step: unknown mode %d", (int)mode);
}

co2_status_t outer_step_ghost_p2p_impl(co2_mode_t mode, int64_t n, const void* anchor_in,
                                       const void* p0, const void* p1_avg, const void* xbar_avg,
                                       int32_t ghost_copies, void* m, void* anchor_out,
                                       void* bar0_out, void* const* out_peers,
                                       void* const* sigs, int world, int rank, uint32_t epoch,
                                       void* gap, const co2_hyper_t* h, void* ws,
                                       cudaStream_t s) {
  if (world < 1 || world > kMaxRanks)
    return fail(CO2_ERR_VALIDATION, "p2p sharded step: world must lie in [1, %d]", kMaxRanks);
  // x_t0 is loaded as the STATE dtype even when unused (x_from_xbar): never
  // alias it to the low-dtype average, which is half as long in bytes.
  StepArgs a{anchor_in ? anchor_in : p0, p0, p1_avg, xbar_avg, m, anchor_out,
             nullptr, gap, n, h->alpha, h->beta, h->phi, h->epsilon, h->tau, 1,
             h->penalty ? 1 : 0, h->clip ? 1 : 0, ws, 1, ghost_copies,
             ghost_copies == 0 ? 1 : 0, bar0_out};
  for (int p = 0; p < world; ++p) {
    a.out_peers[p] = out_peers[p];
    a.exit.sig[p] = static_cast<Signals*>(sigs[p]);
  }
  a.exit.world = world;
  a.exit.rank = rank;
  a.exit.epoch = epoch;
  switch (mode) {
    case CO2_MODE_F64: return launch_ghost_p2p<ModeF64>(a, s);
    case CO2_MODE_F32: return launch_ghost_p2p<ModeF32>(a, s);
    case CO2_MODE_BF16_MIXED: return launch_ghost_p2p<ModeBF16>(a, s);
  }
  return fail(CO2_ERR_VALIDATION, "outer step: unknown mode %d", (int)mode);
}

co2_status_t outer_step_ghost_impl(co2_mode_t mode, int64_t n, const void* anchor_in,
                                   const void* p0, const void* p1_sum, int32_t p1_div,
                                   const void* xbar_sum, int32_t divisor, int32_t ghost_copies,
                                   void* m, void* anchor_out, void* bar0_out, void* params,
                                   void* gap, const co2_hyper_t* h, void* ws, cudaStream_t s) {
  StepArgs a{anchor_in, p0, p1_sum, xbar_sum, m, anchor_out, params, gap, n, h->alpha, h->beta,
             h->phi, h->epsilon, h->tau, divisor, h->penalty ? 1 : 0, h->clip ? 1 : 0, ws,
             p1_div, ghost_copies, ghost_copies == 0 ? 1 : 0, bar0_out};
  switch (mode) {
    case CO2_MODE_F64: return launch_ghost<ModeF64>(a, s);
    case CO2_MODE_F32: return launch_ghost<ModeF32>(a, s);
    case CO2_MODE_BF16_MIXED: return launch_ghost<ModeBF16>(a, s);
  }
  return fail(CO2_ERR_VALIDATION, "outer step: unknown mode %d", (int)mode);
}

}  // namespace co2

using namespace co2;

extern "C" co2_status_t co2_set_grid_waves(int32_t waves) {
  if (waves < 1 || waves > 64) return fail(CO2_ERR_VALIDATION, "waves out of range");
  g_waves.store(waves, std::memory_order_relaxed);
  return CO2_OK;
}

extern "C" co2_status_t co2_set_fused_variant(int32_t variant) {
  if (variant < 0 || variant > 15) return fail(CO2_ERR_VALIDATION, "variant out of range");
  g_variant.store(variant, std::memory_order_relaxed);
  return CO2_OK;
}

extern "C" co2_status_t co2_staleness_gap(co2_dtype_t dt, int64_t n, const void* x_t0,
                                          const void* prev_x0, const void* prev_x1, int32_t tau,
                                          double epsilon, void* gap_out, void* ws, void* stream) {
  // outer_algorithms.cpp:50-56 (scalar validation first)
  if (tau < 1) return fail(CO2_ERR_VALIDATION, "staleness_gap: tau must be >= 1");
  if (!(epsilon > 0.0)) return fail(CO2_ERR_VALIDATION, "staleness_gap: epsilon must be positive");
  if (n < 0) return fail(CO2_ERR_VALIDATION, "staleness_gap: dimensions differ");
  OpArgs a{x_t0, prev_x0, prev_x1, gap_out, n, (double)tau, epsilon, 0, ws};
  return launch_op<OP_GAP>(dt, a, S(stream));
}

extern "C" co2_status_t co2_penalized_momentum(co2_dtype_t dt, int64_t n, const void* m_prev,
                                               double beta, const void* gap, const void* delta,
                                               int32_t penalty, void* m_out, void* ws,
                                               void* stream) {
  // outer_algorithms.cpp:70-72
  if (beta < 0.0 || beta >= 1.0)
    return fail(CO2_ERR_VALIDATION, "momentum update: beta must lie in [0, 1)");
  if (n < 0) return fail(CO2_ERR_VALIDATION, "momentum update: dimensions differ");
  OpArgs a{m_prev, gap, delta, m_out, n, beta, 0.0, penalty ? 1 : 0, ws};
  return launch_op<OP_MOMENTUM>(dt, a, S(stream));
}

extern "C" co2_status_t co2_outer_iterate(co2_dtype_t dt, int64_t n, const void* x_t0,
                                          double alpha, const void* m, double phi, int32_t clip,
                                          void* x_out, void* ws, void* stream) {
  // outer_algorithms.cpp:94-96; clip_elementwise's phi check param_ops.cpp:36-38
  if (!(alpha > 0.0)) return fail(CO2_ERR_VALIDATION, "outer_iterate: alpha must be positive");
  if (n < 0) return fail(CO2_ERR_VALIDATION, "outer_iterate: dimensions differ");
  if (clip && !(phi > 0.0))
    return fail(CO2_ERR_VALIDATION, "clip_elementwise: phi must be positive");
  OpArgs a{x_t0, m, nullptr, x_out, n, alpha, phi, clip ? 1 : 0, ws};
  return launch_op<OP_ITERATE>(dt, a, S(stream));
}

extern "C" co2_status_t co2_clip_elementwise(co2_dtype_t dt, int64_t n, const void* v, double phi,
                                             void* out, void* ws, void* stream) {
  if (!(phi > 0.0)) return fail(CO2_ERR_VALIDATION, "clip_elementwise: phi must be positive");
  OpArgs a{v, nullptr, nullptr, out, n, phi, 0.0, 0, ws};
  return launch_op<OP_CLIP>(dt, a, S(stream));
}

extern "C" co2_status_t co2_ensure_finite(co2_dtype_t dt, int64_t n, const void* v,
                                         const char* what, void* ws, void* stream) {
  // ensure_finite (param_ops.cpp:10-14): "non-finite value in " + context
  if (n < 0) return fail(CO2_ERR_VALIDATION, "ensure_finite: negative length");
  OpArgs a{v, nullptr, nullptr, nullptr, n, 0.0, 0.0, 0, ws};
  CO2_TRY(launch_op<OP_FINITE>(dt, a, S(stream)));
  co2_diag_t d;
  CO2_CUDA(cudaMemcpyAsync(&d, &ws_header(ws)->diag, sizeof d, cudaMemcpyDeviceToHost,
                           S(stream)));
  CO2_CUDA(cudaStreamSynchronize(S(stream)));
  if (d.flags & CO2_FLAG_NONFINITE_INPUT)
    return fail(CO2_ERR_NUMERIC, "non-finite value in %s", what ? what : "");
  return CO2_OK;
}

extern "C" co2_status_t co2_elementwise_abs_diff(co2_dtype_t dt, int64_t n, const void* a,
                                                 const void* b, void* out, void* ws,
                                                 void* stream) {
  if (n < 0) return fail(CO2_ERR_VALIDATION, "elementwise_abs_diff: dimensions differ");
  OpArgs oa{a, b, nullptr, out, n, 0.0, 0.0, 0, ws};
  CO2_TRY(launch_op<OP_ABSDIFF>(dt, oa, S(stream)));
  co2_diag_t d;
  CO2_CUDA(cudaMemcpyAsync(&d, &ws_header(ws)->diag, sizeof d, cudaMemcpyDeviceToHost,
                           S(stream)));
  CO2_CUDA(cudaStreamSynchronize(S(stream)));
  if (d.flags & CO2_FLAG_NONFINITE_INPUT)
    return fail(CO2_ERR_NUMERIC, "non-finite value in elementwise_abs_diff");
  return CO2_OK;
}

extern "C" co2_status_t co2_l2_norm(co2_dtype_t dt, int64_t n, const void* v, double* out,
                                   void* ws, void* stream) {
  CO2_TRY(check_dtype(dt));
  if (n < 0) return fail(CO2_ERR_VALIDATION, "l2_norm: negative length");
  if (!ws || !out || (n > 0 && !v)) return fail(CO2_ERR_VALIDATION, "null buffer");
  if (dt == CO2_DTYPE_F64)
    CO2_TRY((launch_sumsq<double, 2>(v, n, ws, S(stream))));
  else if (dt == CO2_DTYPE_F32)
    CO2_TRY((launch_sumsq<float, 4>(v, n, ws, S(stream))));
  else
    CO2_TRY((launch_sumsq<bf16s, 8>(v, n, ws, S(stream))));
  CO2_CUDA(cudaMemcpyAsync(out, &ws_header(ws)->gnorm, sizeof(double), cudaMemcpyDeviceToHost,
                           S(stream)));
  CO2_CUDA(cudaStreamSynchronize(S(stream)));
  if (!isfinite(*out)) return fail(CO2_ERR_NUMERIC, "l2_norm: non-finite result");
  return CO2_OK;
}

extern "C" co2_status_t co2_average(co2_dtype_t dt, int32_t g, const void* const* contributions,
                                    int64_t n, void* out, void* ws, void* stream) {
  if (g <= 0) return fail(CO2_ERR_VALIDATION, "average: empty contribution list");
  if (g > 64) return fail(CO2_ERR_VALIDATION, "average: at most 64 contributions");
  CO2_TRY(check_dtype(dt));
  if (!ws) return fail(CO2_ERR_VALIDATION, "null workspace");
  if (n < 0) return fail(CO2_ERR_VALIDATION, "average: contribution dimensions differ");
  if (n > 0) {
    if (!contributions || !out) return fail(CO2_ERR_VALIDATION, "null buffer");
    for (int i = 0; i < g; ++i)
      if (!contributions[i]) return fail(CO2_ERR_VALIDATION, "null buffer");
  }
  bool vec = aligned16(out);
  for (int i = 0; i < g && vec; ++i) vec = aligned16(contributions[i]);
  cudaStream_t s = S(stream);
  auto run = [&](auto tag) -> co2_status_t {
    using T = decltype(tag);
    using TC = decltype(to_c(T{}));
    Ptrs64<T> p{};
    for (int i = 0; i < g; ++i) p.p[i] = static_cast<const T*>(contributions[i]);
    if (vec) {
      auto k = average_vec_kernel<T, TC>;
      const int64_t nv = n / (16 / (int64_t)sizeof(T));
      k<<<grid_for(k, nv > 0 ? nv : 1, kThreads), kThreads, 0, s>>>(p, g, static_cast<T*>(out), n,
                                                                     ws);
    } else {
      int grid = simple_grid(n, kThreads);
      if (grid > kMaxBlocks) grid = kMaxBlocks;
      average_kernel<T, TC><<<grid, kThreads, 0, s>>>(p, g, static_cast<T*>(out), n, ws);
    }
    CO2_CUDA(cudaGetLastError());
    return CO2_OK;
  };
  if (dt == CO2_DTYPE_F64) return run(double{});
  if (dt == CO2_DTYPE_F32) return run(float{});
  return run(bf16s{});
}

extern "C" co2_status_t co2_sub(co2_dtype_t dt, int64_t n, const void* a, const void* b, void* out,
                                void* stream) {
  CO2_TRY(check_dtype(dt));
  if (n < 0) return fail(CO2_ERR_VALIDATION, "sub: negative length");
  if (n == 0) return CO2_OK;
  if (!a || !b || !out) return fail(CO2_ERR_VALIDATION, "null buffer");
  int grid = simple_grid(n, kThreads);
  cudaStream_t s = S(stream);
  if (dt == CO2_DTYPE_F64)
    sub_kernel<double, double><<<grid, kThreads, 0, s>>>(
        static_cast<const double*>(a), static_cast<const double*>(b), static_cast<double*>(out), n);
  else if (dt == CO2_DTYPE_F32)
    sub_kernel<float, float><<<grid, kThreads, 0, s>>>(
        static_cast<const float*>(a), static_cast<const float*>(b), static_cast<float*>(out), n);
  else
    sub_kernel<bf16s, float><<<grid, kThreads, 0, s>>>(
        static_cast<const bf16s*>(a), static_cast<const bf16s*>(b), static_cast<bf16s*>(out), n);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

namespace {
template <typename TD>
co2_status_t convert_from(TD* d, co2_dtype_t sdt, const void* s, int64_t n, cudaStream_t st) {
  int grid = simple_grid(n, kThreads);
  if (sdt == CO2_DTYPE_F64)
    convert_kernel<TD, double><<<grid, kThreads, 0, st>>>(d, static_cast<const double*>(s), n);
  else if (sdt == CO2_DTYPE_F32)
    convert_kernel<TD, float><<<grid, kThreads, 0, st>>>(d, static_cast<const float*>(s), n);
  else
    convert_kernel<TD, bf16s><<<grid, kThreads, 0, st>>>(d, static_cast<const bf16s*>(s), n);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}
}  // namespace

extern "C" co2_status_t co2_convert(co2_dtype_t ddt, void* dst, co2_dtype_t sdt, const void* src,
                                    int64_t n, void* stream) {
  CO2_TRY(check_dtype(ddt));
  CO2_TRY(check_dtype(sdt));
  if (n < 0) return fail(CO2_ERR_VALIDATION, "convert: negative length");
  if (n == 0) return CO2_OK;
  if (!dst || !src) return fail(CO2_ERR_VALIDATION, "null buffer");
  if (ddt == sdt) {
    size_t es = ddt == CO2_DTYPE_F64 ? 8 : (ddt == CO2_DTYPE_F32 ? 4 : 2);
    CO2_CUDA(cudaMemcpyAsync(dst, src, es * (size_t)n, cudaMemcpyDeviceToDevice, S(stream)));
    return CO2_OK;
  }
  if (ddt == CO2_DTYPE_F64) return convert_from(static_cast<double*>(dst), sdt, src, n, S(stream));
  if (ddt == CO2_DTYPE_F32) return convert_from(static_cast<float*>(dst), sdt, src, n, S(stream));
  return convert_from(static_cast<bf16s*>(dst), sdt, src, n, S(stream));
}

extern "C" co2_status_t co2_synth(co2_mode_t mode, uint64_t seed, int32_t worker, int64_t j0,
                                  int64_t count, void* x_t0, void* p0, void* p1, void* x_end,
                                  void* m, void* stream) {
  if (count < 0 || j0 < 0) return fail(CO2_ERR_VALIDATION, "synth: negative range");
  if (count == 0) return CO2_OK;
  uint64_t w = (uint64_t)(uint32_t)worker;
  // stream key = (buffer_id << 32) | worker; p0 worker-independent.
  uint64_t kp0 = host_key(seed, (0ull << 32) | 0ull), kp1 = host_key(seed, (1ull << 32) | w),
           kx = host_key(seed, (2ull << 32) | w), ke = host_key(seed, (3ull << 32) | w),
           km = host_key(seed, (4ull << 32) | w);
  int grid = simple_grid(count, kThreads);
  cudaStream_t s = S(stream);
  switch (mode) {
    case CO2_MODE_F64:
      synth_kernel<ModeF64><<<grid, kThreads, 0, s>>>(
          kp0, kp1, kx, ke, km, j0, count, (double*)x_t0, (double*)p0, (double*)p1,
          (double*)x_end, (double*)m);
      break;
    case CO2_MODE_F32:
      synth_kernel<ModeF32><<<grid, kThreads, 0, s>>>(kp0, kp1, kx, ke, km, j0, count,
                                                       (float*)x_t0, (float*)p0, (float*)p1,
                                                       (float*)x_end, (float*)m);
      break;
    case CO2_MODE_BF16_MIXED:
      synth_kernel<ModeBF16><<<grid, kThreads, 0, s>>>(kp0, kp1, kx, ke, km, j0, count,
                                                        (float*)x_t0, (float*)p0, (bf16s*)p1,
                                                        (bf16s*)x_end, (float*)m);
      break;
    default:
      return fail(CO2_ERR_VALIDATION, "synth: unknown mode %d", (int)mode);
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

extern "C" co2_status_t co2_synthetic_inner_step_snapshot(co2_dtype_t dt, int64_t n,
                                                          void* params, double lr, double scale,
                                                          uint64_t seed, int32_t worker,
                                                          int64_t step, int32_t repeat,
                                                          void* snapshot_out, void* stream) {
  CO2_TRY(check_dtype(dt));
  if (repeat < 1) repeat = 1;
  uint64_t key = host_key(seed, (5ull << 32) | (uint64_t)(uint32_t)worker);
  int64_t offset = step * n * (int64_t)repeat;
  int grid = simple_grid(n, kThreads);
  cudaStream_t s = S(stream);
  if (dt == CO2_DTYPE_F64)
    inner_step_kernel<double, double><<<grid, kThreads, 0, s>>>(
        (double*)params, n, lr, scale, key, offset, repeat, (double*)snapshot_out);
  else if (dt == CO2_DTYPE_F32)
    inner_step_kernel<float, float><<<grid, kThreads, 0, s>>>(
        (float*)params, n, lr, scale, key, offset, repeat, (float*)snapshot_out);
  else
    inner_step_kernel<bf16s, float><<<grid, kThreads, 0, s>>>(
        (bf16s*)params, n, lr, scale, key, offset, repeat, (bf16s*)snapshot_out);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

extern "C" co2_status_t co2_synthetic_inner_step(co2_dtype_t dt, int64_t n, void* params,
                                                 double lr, double scale, uint64_t seed,
                                                 int32_t worker, int64_t step, int32_t repeat,
                                                 void* stream) {
  return co2_synthetic_inner_step_snapshot(dt, n, params, lr, scale, seed, worker, step, repeat,
                                           nullptr, stream);
}

extern "C" co2_status_t co2_fill_u32(void* dst, uint32_t value, int64_t count, void* stream) {
  if (count <= 0) return CO2_OK;
  fill_u32_kernel<<<simple_grid(count, kThreads), kThreads, 0, S(stream)>>>((uint32_t*)dst, value,
                                                                             count);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

namespace co2 {
namespace {
template <typename T>
__global__ void scale_div_kernel(T* b, int64_t n, int g) {
  using TC = decltype(to_c(T{}));
  const TC gd = (TC)g;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    b[j] = Store<T>::from(div_rn_nz(to_c(b[j]), gd));
}
}  // namespace

co2_status_t scale_div_impl(co2_dtype_t dt, void* buf, int64_t n, int g, cudaStream_t s) {
  if (n <= 0) return CO2_OK;
  const int grid = simple_grid(n, kThreads);
  if (dt == CO2_DTYPE_F64)
    scale_div_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<double*>(buf), n, g);
  else if (dt == CO2_DTYPE_F32)
    scale_div_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<float*>(buf), n, g);
  else
    scale_div_kernel<bf16s><<<grid, kThreads, 0, s>>>(static_cast<bf16s*>(buf), n, g);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}
}  // namespace co2

// ------------------------------------------------ sharded-mode helpers
namespace co2 {
namespace {
// Round 0 of the sharded ghost driver: anchor <- x_{0,0} (the params shard,
// widened) and prev_x0 <- average of g identical copies of it
// (outer_algorithms.cpp:133-145 with identical starts).
template <typename TS, typename TL>
__global__ void ghost_init_kernel(const TL* params, TS* anchor, TS* prev_x0, int64_t n, int g) {
  using TC = decltype(to_c(TS{}));
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    TC v = (TC)to_c(params[j]);
    anchor[j] = (TS)v;
    prev_x0[j] = (TS)ghost_avg<TC>(v, g);
  }
}
}  // namespace

co2_status_t ghost_init_impl(co2_mode_t mode, int64_t n, const void* params, void* anchor,
                             void* prev_x0, int g, cudaStream_t s) {
  if (n <= 0) return CO2_OK;
  int grid = simple_grid(n, kThreads);
  switch (mode) {
    case CO2_MODE_F64:
      ghost_init_kernel<double, double><<<grid, kThreads, 0, s>>>(
          (const double*)params, (double*)anchor, (double*)prev_x0, n, g);
      break;
    case CO2_MODE_F32:
      ghost_init_kernel<float, float><<<grid, kThreads, 0, s>>>(
          (const float*)params, (float*)anchor, (float*)prev_x0, n, g);
      break;
    default:
      ghost_init_kernel<float, bf16s><<<grid, kThreads, 0, s>>>(
          (const bf16s*)params, (float*)anchor, (float*)prev_x0, n, g);
      break;
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}
}  // namespace co2

extern "C" co2_status_t co2_outer_step_ghost(co2_mode_t mode, int64_t n, const void* anchor_in,
                                             const void* prev_x0, const void* prev_x1_sum,
                                             int32_t p1_div, const void* xbar_sum,
                                             int32_t xbar_div, int32_t ghost_copies,
                                             void* momentum, void* anchor_out, void* bar0_out,
                                             void* params_out, void* gap_out,
                                             const co2_hyper_t* h, void* ws, void* stream) {
  CO2_TRY(co2_hyper_validate(h));
  if (h->tau < 1) return fail(CO2_ERR_VALIDATION, "staleness_gap: tau must be >= 1");
  if (n < 0 || p1_div < 1 || xbar_div < 1 || ghost_copies < 0)
    return fail(CO2_ERR_VALIDATION, "ghost step: bad sizes or divisors");
  if (!ws) return fail(CO2_ERR_VALIDATION, "null workspace");
  if (n > 0 && (!prev_x0 || !prev_x1_sum || !xbar_sum || !momentum ||
                (ghost_copies > 0 && !anchor_in)))
    return fail(CO2_ERR_VALIDATION, "outer step: null input buffer");
  return outer_step_ghost_impl(mode, n, anchor_in ? anchor_in : prev_x0, prev_x0,
                               prev_x1_sum, p1_div, xbar_sum, xbar_div, ghost_copies, momentum,
                               anchor_out, bar0_out, params_out, gap_out, h, ws, S(stream));
}

// ==================================================== baseline outer steps
// SlowMo, Local-SGD and Overlap-Local-SGD outer updates
// (proj/src/outer_algorithms.cpp:213-313) on the same kernel family: one
// HBM pass per worker, IEEE ops in the reference's order, max_outer_step and
// the reference's finiteness checks reduced into the workspace.
namespace co2 {
namespace {

enum BaseOp { B_SLOWMO = 0, B_LOCAL = 1, B_OVERLAP = 2 };

struct BaseArgs {
  const void* x;   // x_start (state)              SLOWMO, LOCAL
  const void* xb;  // consumed reduce (low)        all
  void* m;         // momentum (state, in/out)     SLOWMO
  void* params;    // params (low): out / in-out   all
  void* anchor;    // SLOWMO/LOCAL: x_{t+1,0} out (state, nullable); OVERLAP: anchor in
  int64_t n;
  double alpha, beta;
  int divisor;
  void* ws;
};

// One coordinate of the baseline updates, IEEE ops in the reference's order.
template <class M, int OP>
__device__ __forceinline__ void base_elem(typename M::TC xb, typename M::TC x, typename M::TS& m,
                                          typename M::TL& pr, typename M::TS& an,
                                          typename M::TC af, typename M::TC bf,
                                          AccT<typename M::TC>& acc) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  if (OP == B_SLOWMO) {  // outer_algorithms.cpp:229-233
    TC delta = x - xb;
    TC bm = bf * to_c(m);
    TC mn = bm + delta;
    TC am = af * mn;
    TC xn = x - am;
    if (!isfinite(mn)) acc.flags |= CO2_FLAG_SLOWMO_M;
    if (!isfinite(xn)) acc.flags |= CO2_FLAG_SLOWMO_X;
    m = (TS)mn;
    pr = Store<TL>::from(xn);
    an = (TS)xn;
    TC st = fabs(xn - x);
    acc.max_step = st > acc.max_step ? st : acc.max_step;
  } else if (OP == B_LOCAL) {  // outer_algorithms.cpp:252-255
    TC st = fabs(xb - x);
    acc.max_step = st > acc.max_step ? st : acc.max_step;
    pr = Store<TL>::from(xb);
    an = (TS)xb;
  } else {  // B_OVERLAP, outer_algorithms.cpp:278-279 (an = the anchor, read only)
    TC p = to_c(pr);
    TC d = to_c(an) - xb;
    TC pn = p - d;
    if (!isfinite(pn)) acc.flags |= CO2_FLAG_OVERLAP;
    TL stored = Store<TL>::from(pn);
    pr = stored;
    TC st = fabs(to_c(stored) - p);
    acc.max_step = st > acc.max_step ? st : acc.max_step;
  }
}

// V-element vectors per thread (128-bit state streams; V = 1 is the
// unaligned path), grid-stride over grid_for()'s oversubscribed grid, the
// n % V tail in scalar form.  Streams per op (bf16-mixed bytes / param):
// SlowMo reads x, xbar, m and writes m, params, anchor (22 B); Local-SGD
// reads x, xbar and writes params, anchor (12 B; 10 B without the anchor);
// Overlap reads params, anchor, xbar and writes params (10 B).
template <class M, int OP, int V>
__global__ void __launch_bounds__(kThreads) baseline_kernel(const BaseArgs a) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  const TC af = (TC)a.alpha, bf = (TC)a.beta, gd = (TC)a.divisor;
  const bool div = a.divisor > 1;
  AccT<TC> acc;
  const TS* X = static_cast<const TS*>(a.x);
  const TL* XB = static_cast<const TL*>(a.xb);
  TS* Mm = static_cast<TS*>(a.m);
  TL* PR = static_cast<TL*>(a.params);
  TS* A = static_cast<TS*>(a.anchor);
  const int64_t nv = a.n / V;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nv; i += stride) {
    const int64_t e = i * V;
    TL xb[V], pr[V];
    TS x[V], m[V], an[V];
    ld_vec<TL, V>(XB + e, xb);
    if (OP != B_OVERLAP) ld_vec<TS, V>(X + e, x);
    if (OP == B_SLOWMO) ld_vec<TS, V>(Mm + e, m);
    if (OP == B_OVERLAP) {
      ld_vec<TL, V>(PR + e, pr);
      ld_vec<TS, V>(A + e, an);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      TC xbv = to_c(xb[v]);
      if (div) xbv = div_rn_nz(xbv, gd);  // average(): one division, param_ops.cpp:30
      base_elem<M, OP>(xbv, OP == B_OVERLAP ? (TC)0 : to_c(x[v]), m[v], pr[v], an[v], af, bf,
                       acc);
    }
    if (OP == B_SLOWMO) st_vec<TS, V>(Mm + e, m);
    st_vec<TL, V>(PR + e, pr);
    if (OP != B_OVERLAP && A) st_vec<TS, V>(A + e, an);
  }
  for (int64_t j = nv * V + (int64_t)blockIdx.x * kThreads + threadIdx.x; V > 1 && j < a.n;
       j += stride) {
    TC xbv = to_c(XB[j]);
    if (div) xbv = div_rn_nz(xbv, gd);
    TS m = OP == B_SLOWMO ? Mm[j] : (TS)0;
    TS an = OP == B_OVERLAP ? A[j] : (TS)0;
    TL pr = OP == B_OVERLAP ? PR[j] : TL{};
    base_elem<M, OP>(xbv, OP == B_OVERLAP ? (TC)0 : to_c(X[j]), m, pr, an, af, bf, acc);
    if (OP == B_SLOWMO) Mm[j] = m;
    PR[j] = pr;
    if (OP != B_OVERLAP && A) A[j] = an;
  }
  block_finish<kThreads>(acc.widen(), a.ws);
}

template <class M, int OP>
void launch_baseline_mode(const BaseArgs& a, cudaStream_t s) {
  constexpr int V = std::is_same<M, ModeF64>::value ? 2 : (std::is_same<M, ModeF32>::value ? 4 : 8);
  const bool vec = aligned16(a.x) && aligned16(a.xb) && aligned16(a.m) && aligned16(a.params) &&
                   aligned16(a.anchor);
  if (vec) {
    auto k = baseline_kernel<M, OP, V>;
    k<<<grid_for(k, a.n / V, kThreads), kThreads, 0, s>>>(a);
  } else {
    auto k = baseline_kernel<M, OP, 1>;
    k<<<grid_for(k, a.n, kThreads), kThreads, 0, s>>>(a);
  }
}

template <int OP>
co2_status_t launch_baseline(co2_mode_t mode, const BaseArgs& a, cudaStream_t s) {
  switch (mode) {
    case CO2_MODE_F64: launch_baseline_mode<ModeF64, OP>(a, s); break;
    case CO2_MODE_F32: launch_baseline_mode<ModeF32, OP>(a, s); break;
    case CO2_MODE_BF16_MIXED: launch_baseline_mode<ModeBF16, OP>(a, s); break;
    default: return fail(CO2_ERR_VALIDATION, "baseline step: unknown mode %d", (int)mode);
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

}  // namespace

co2_status_t slowmo_impl(co2_mode_t mode, int64_t n, const void* x_start, const void* xbar,
                         int32_t divisor, void* m, void* params_out, void* anchor_out,
                         double alpha, double beta, void* ws, cudaStream_t s) {
  BaseArgs a{x_start, xbar, m, params_out, anchor_out, n, alpha, beta, divisor, ws};
  return launch_baseline<B_SLOWMO>(mode, a, s);
}
co2_status_t local_sgd_impl(co2_mode_t mode, int64_t n, const void* x_start, const void* xbar,
                            int32_t divisor, void* params_out, void* anchor_out, void* ws,
                            cudaStream_t s) {
  BaseArgs a{x_start, xbar, nullptr, params_out, anchor_out, n, 0.0, 0.0, divisor, ws};
  return launch_baseline<B_LOCAL>(mode, a, s);
}
co2_status_t overlap_correction_impl(co2_mode_t mode, int64_t n, void* params, const void* anchor,
                                     const void* xbar, int32_t divisor, void* ws,
                                     cudaStream_t s) {
  BaseArgs a{nullptr, xbar, nullptr, params, const_cast<void*>(anchor), n, 0.0, 0.0, divisor,
             ws};
  return launch_baseline<B_OVERLAP>(mode, a, s);
}

}  // namespace co2

namespace co2 {
namespace {
// ================================================ single-launch LOCAL round
// C1 (BASELINE configs[0]): G simulated workers on one GPU.  One co2_round
// (outer_algorithms.cpp:110-211, worker-local branch, t >= 1) as ONE grid:
//   * this round's launch_all_reduce of x_{t,tau} (collect_params, :120):
//     the fixed-order average of every worker's params into avg_out
//     (param_ops.cpp:16-33: ascending worker order, one division);
//   * every worker's fused outer step consuming the previous round's
//     average xbar (:186-202).
// The two halves touch disjoint buffers (the average reads params[cur] and
// writes avg[t%2]; the steps read avg[(t-1)%2] and write params[1-cur],
// m and the anchor), so one grid is exactly the two-kernel schedule.  Per
// element every op is the fused step's / average_kernel's, so results and
// per-worker diagnostics are bitwise those of the separate launches.
//
// Work split: G + 1 roles (worker w's step, then the average) of
// tiles_per_role tiles each, NT threads x TV vectors per tile, numbered
// role-major.  A persistent grid (one wave) claims tiles from a counter in
// worker 0's workspace, the next claim issued while the current tile runs,
// so CTAs stay busy to the end whatever the per-role cost (a step tile moves
// 28 B/param, an average tile 20) and whatever the HBM unevenness.  The C1
// working set (1M params x 4 workers, 142 MB) is a single short wave: the
// earlier oversubscribed grid (5 waves of CTAs that each did 1-2 vectors per
// thread, then a fold) ran at 0.58 of copy.  xbar (one buffer, read by every
// worker role) is read with default caching and stays in L2 between roles;
// every other stream is evict-first.
// Diagnostics: a CTA folds its accumulators (warp shuffles, warps in fixed
// order) whenever its claimed role changes and merges them into that role's
// order-independent atomic accumulators (block_finish's keys / counts / OR;
// the average's flags in worker 0's acc_flags2), so the result does not
// depend on which CTA ran which tile.  The last CTA (ticket) publishes every
// role into the worker's workspace header (and the average's flags and this
// launch's %globaltimer start / end into the engine's device slot of the
// handle) and resets them.  Nothing is written to mapped host memory: those
// PCIe writes and the system fence they need cost ~2.3 us at the kernel's
// end (profiles/r02/c1/), and the engine fetches the slots only on demand.
struct LocalRoundArgs {
  const void* x_t0[kMaxLocalRound];
  const void* p0[kMaxLocalRound];
  const void* p1[kMaxLocalRound];
  void* m[kMaxLocalRound];
  void* anchor[kMaxLocalRound];
  void* params[kMaxLocalRound];
  void* gap[kMaxLocalRound];
  const void* cur[kMaxLocalRound];  // x_{t,tau}: this round's contributions
  void* ws[kMaxLocalRound];
  co2_diag_t* host_diag[kMaxLocalRound];  // extra copy of each worker's diag (nullable)
  co2_diag_t* avg_diag;                   // the average's diag slot (nullable)
  const void* xbar;                       // the average consumed this round
  void* avg_out;                          // this round's average
  int g;
  int64_t n;
  double alpha, beta, phi, eps;
  int tau, penalty, clip;
  int tiles_per_role;
  int tv;        // vectors per thread per tile
  int prefetch;  // L2 bulk prefetch of the tile after next (CO2_LOCAL_ROUND_PF=1 enables)
  int pdl_early;  // signal dependents at entry rather than after the tiles
  int stages;     // bulk-copy round: ring stages that fit in shared memory
  // [start, end] %globaltimer of this launch (nullable): the engine's
  // kernel-timed handle's device slot
  unsigned long long* ts;
};

// Merge this CTA's accumulators for one role into the role's atomic
// accumulators.  Every thread calls (block-uniform role).
template <int NT>
__device__ __forceinline__ void role_merge(const Acc& a, WsHeader* hdr, bool avg) {
  const Partial b = block_partial<NT>(a);  // valid in thread 0
  if (threadIdx.x == 0) {
    if (avg) {
      if (b.flags) atomicOr(&hdr->acc_flags2, b.flags);
    } else {
      atomicMax(&hdr->acc_min_key, ~dkey(b.min_gap));
      atomicMax(&hdr->acc_max_key, dkey(b.max_step));
      if (b.clipped) atomicAdd(&hdr->acc_clipped, b.clipped);
      if (b.floored) atomicAdd(&hdr->acc_floored, b.floored);
      if (b.flags) atomicOr(&hdr->acc_flags, b.flags);
    }
  }
}

template <class M, int V, int U, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) local_round_kernel(const LocalRoundArgs a) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  constexpr bool LQ = !std::is_same<TS, TL>::value;
  const int TV = a.tv;  // vectors per thread per tile (a multiple of U)
  Hyp<TC> h;
  h.tau = (TC)a.tau;
  h.eps = (TC)a.eps;
  h.beta = (TC)a.beta;
  h.phi = (TC)a.phi;
  h.alpha = (TC)a.alpha;
  h.divisor = (TC)1;
  h.penalty = a.penalty;
  h.clip = a.clip;
  h.divide = 0;
  const int G = a.g;
  const int tpr = a.tiles_per_role;
  const int ntiles = tpr * (G + 1);
  const int64_t nv = a.n / V;
  const int64_t tail = a.n - nv * V;  // n % V coordinates, by the last tile of each role
  const TL* XB = static_cast<const TL*>(a.xbar);
  WsHeader* h0 = ws_header(a.ws[0]);
  // Programmatic dependent launch: with the launch attribute this grid is
  // scheduled while the previous kernel on the stream finishes; nothing
  // above touched memory it writes, and this waits for its completion and
  // memory flush (a no-op without the attribute).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.ts && blockIdx.x == 0 && threadIdx.x == 0) h0->t_start = (unsigned long long)global_ns();

  // Tile pipeline (thread 0): while tile i runs, the claim of tile i + 2 is
  // in flight, and at the end of tile i the streams of tile i + 2 are
  // prefetched into L2 with bulk prefetches, so tile i + 1's loads were
  // issued to HBM a whole tile earlier and hit L2.  The kernel is short
  // (~1 MB per SM) and latency-bound without it: 768 threads x 80 B in
  // flight per SM cover only ~1 us of HBM latency.
  const int64_t per_tile = (int64_t)NT * TV;
  auto prefetch = [&](int t) {  // thread 0 only
    if (t >= ntiles) return;
    const int r = t / tpr;
    const int64_t v0 = (int64_t)(t - r * tpr) * per_tile;
    int64_t cnt = nv - v0 < per_tile ? nv - v0 : per_tile;
    if (cnt <= 0) return;
    auto pf = [&](const void* base, int esz) {
      const unsigned bytes = (unsigned)((cnt * V * esz) & ~(int64_t)15);
      if (bytes) bulk_prefetch_l2(static_cast<const char*>(base) + v0 * V * esz, bytes);
    };
    if (r < G) {
      pf(a.x_t0[r], sizeof(TS));
      pf(a.p0[r], sizeof(TS));
      pf(a.p1[r], sizeof(TL));
      pf(a.m[r], sizeof(TS));
      pf(a.xbar, sizeof(TL));
    } else {
      for (int w = 0; w < G; ++w) pf(a.cur[w], sizeof(TL));
    }
  };
  // The first two tiles of CTA b are static (b and grid + b): the launch
  // does not open with 2 x grid atomics on one counter (serialised in L2,
  // microseconds at this kernel's scale); later claims are spread in time.
  const int nstatic = 2 * (int)gridDim.x;
  __shared__ int s_next[2];
  int ahead = (int)gridDim.x + (int)blockIdx.x;  // thread 0: the tile after the next one
  if (threadIdx.x == 0 && V * (int)sizeof(TL) % 16 == 0 && a.prefetch) prefetch(ahead);
  int tile = (int)blockIdx.x;
  int slot = 0;
  int role_cur = -1;
  AccT<TC> acc;

  while (tile < ntiles) {
    int claim = 0;
    if (threadIdx.x == 0 && ahead < ntiles)  // used after the tile
      claim = nstatic + (int)atomicAdd(&h0->tile_next, 1u);
    else
      claim = ntiles;
    const int role = tile / tpr;
    const int k = tile - role * tpr;
    if (role != role_cur) {
      if (role_cur >= 0) {
        role_merge<NT>(acc.widen(), ws_header(a.ws[role_cur < G ? role_cur : 0]), role_cur == G);
        acc = AccT<TC>();
      }
      role_cur = role;
    }
    const int64_t vbase = (int64_t)k * per_tile + threadIdx.x;
    const bool last_tile = k == tpr - 1;
    if (role < G) {
      const TS* X = static_cast<const TS*>(a.x_t0[role]);
      const TS* P0 = static_cast<const TS*>(a.p0[role]);
      const TL* P1 = static_cast<const TL*>(a.p1[role]);
      TS* Mm = static_cast<TS*>(a.m[role]);
      TS* A = static_cast<TS*>(a.anchor[role]);
      TL* PR = static_cast<TL*>(a.params[role]);
      TS* Gp = static_cast<TS*>(a.gap[role]);
      auto elem = [&](TS x, TS q0, TL q1, TL xb, TS& mo, TS& xs, TL& xl, TS& gs) {
        TC m = to_c(mo), xn, lam;
        co2_elem<TC, LQ>(to_c(x), to_c(q0), to_c(q1), to_c(xb), m, xn, lam, h, acc);
        mo = (TS)m;
        xs = (TS)xn;
        gs = (TS)lam;
        xl = Store<TL>::from(xn);
      };
#pragma unroll 1
      for (int j = 0; j < TV; j += U) {
        TS x[U][V], q0[U][V], mo[U][V];
        TL q1[U][V], xb[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // every load of the U vectors in flight together
          const int64_t v = vbase + (int64_t)(j + u) * NT;
          if (v < nv) {
            const int64_t e = v * V;
            ld_vec<TS, V>(X + e, x[u]);
            ld_vec<TS, V>(P0 + e, q0[u]);
            ld_vec<TL, V>(P1 + e, q1[u]);
            ld_vec<TS, V>(Mm + e, mo[u]);
            constexpr int XBYTES = V * (int)sizeof(TL);
            if constexpr (XBYTES % 16 == 0) {  // default-cached: the other roles hit it in L2
              uint4 r[XBYTES / 16];
#pragma unroll
              for (int q = 0; q < XBYTES / 16; ++q) r[q] = reinterpret_cast<const uint4*>(XB + e)[q];
              memcpy(xb[u], r, XBYTES);
            } else {
#pragma unroll
              for (int q = 0; q < V; ++q) xb[u][q] = XB[e + q];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t v = vbase + (int64_t)(j + u) * NT;
          if (v < nv) {
            const int64_t e = v * V;
            TS xs[V], gs[V];
            TL xl[V];
#pragma unroll
            for (int q = 0; q < V; ++q) elem(x[u][q], q0[u][q], q1[u][q], xb[u][q], mo[u][q], xs[q], xl[q], gs[q]);
            st_vec<TS, V>(Mm + e, mo[u]);
            if (A) st_vec<TS, V>(A + e, xs);
            st_vec<TL, V>(PR + e, xl);
            if (Gp) st_vec<TS, V>(Gp + e, gs);
          }
        }
      }
      if (V > 1 && last_tile && (int64_t)threadIdx.x < tail) {
        const int64_t e = nv * V + threadIdx.x;
        TS mo = Mm[e], xs, gs;
        TL xl;
        elem(X[e], P0[e], P1[e], XB[e], mo, xs, xl, gs);
        Mm[e] = mo;
        if (A) A[e] = xs;
        PR[e] = xl;
        if (Gp) Gp[e] = gs;
      }
    } else {
      const TC gd = (TC)G;
      TL* AO = static_cast<TL*>(a.avg_out);
      auto average = [&](int64_t e, int cnt) {
        // contributions in groups of 4 (all loads of a group in flight
        // together), summed in ascending worker order, param_ops.cpp:26-28
        TC s[V];
#pragma unroll
        for (int w0 = 0; w0 < kMaxLocalRound; w0 += 4) {
          if (w0 < G) {
            TL c[4][V];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              if (w0 + w < G) {
                const TL* C = static_cast<const TL*>(a.cur[w0 + w]);
                if (cnt == V)
                  ld_vec<TL, V>(C + e, c[w]);
                else
                  c[w][0] = C[e];
              }
            }
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              if (w0 + w < G) {
#pragma unroll
                for (int q = 0; q < V; ++q)
                  s[q] = (w0 + w == 0) ? to_c(c[w][q]) : s[q] + to_c(c[w][q]);
              }
            }
          }
        }
        TL o[V];
#pragma unroll
        for (int q = 0; q < V; ++q) {
          if (q < cnt) {
            const TC r = div_rn_nz(s[q], gd);  // one division, :30
            if (!isfinite(r)) acc.flags |= CO2_FLAG_AVG_NONFINITE;
            o[q] = Store<TL>::from(r);
          }
        }
        if (cnt == V)
          st_vec<TL, V>(AO + e, o);
        else
          AO[e] = o[0];
      };
#pragma unroll 1
      for (int j = 0; j < TV; ++j) {
        const int64_t v = vbase + (int64_t)j * NT;
        if (v < nv) average(v * V, V);
      }
      if (V > 1 && last_tile && (int64_t)threadIdx.x < tail) average(nv * V + threadIdx.x, 1);
    }
    if (threadIdx.x == 0) {
      s_next[slot ^ 1] = ahead;
      if (V * (int)sizeof(TL) % 16 == 0 && a.prefetch) prefetch(claim);
      ahead = claim;
    }
    __syncthreads();  // s_next[slot ^ 1] is visible
    tile = s_next[slot ^ 1];
    slot ^= 1;
  }
  if (role_cur >= 0)
    role_merge<NT>(acc.widen(), ws_header(a.ws[role_cur < G ? role_cur : 0]), role_cur == G);
  // This CTA's tiles are done: the next kernel on the stream (launched with
  // programmatic serialization) may start scheduling; it still waits for
  // this grid's completion before touching memory.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // Last CTA: publish and reset every role (thread r publishes role r).
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&h0->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int r = (int)threadIdx.x;
  if (r < G) {
    volatile WsHeader* vh = ws_header(a.ws[r]);
    const unsigned long long kmin = vh->acc_min_key, kmax = vh->acc_max_key;
    co2_diag_t d;
    d.min_gap = kmin ? dkey_inv(~kmin) : (double)INFINITY;
    d.max_outer_step = kmax ? dkey_inv(kmax) : 0.0;
    d.n_clipped = (int64_t)vh->acc_clipped;
    d.n_floored = (int64_t)vh->acc_floored;
    d.flags = vh->acc_flags;
    d.pad = 0;
    WsHeader* hr = ws_header(a.ws[r]);
    hr->diag = d;
    hr->acc_min_key = 0ull;
    hr->acc_max_key = 0ull;
    hr->acc_clipped = 0ull;
    hr->acc_floored = 0ull;
    hr->acc_flags = 0u;
    if (a.host_diag[r]) *a.host_diag[r] = d;
  } else if (r == G) {
    volatile WsHeader* vh = h0;
    const unsigned int f = vh->acc_flags2;
    h0->acc_flags2 = 0u;
    if (a.avg_diag) {
      co2_diag_t ad{INFINITY, 0.0, 0, 0, f, 0};
      *a.avg_diag = ad;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    h0->tile_next = 0u;  // self-reset for the next launch
    h0->ticket = 0u;
    if (a.ts) {
      a.ts[0] = *static_cast<volatile unsigned long long*>(&h0->t_start);
      a.ts[1] = (unsigned long long)global_ns();
    }
  }
}

// Programmatic dependent launch of the round kernel (CO2_LOCAL_ROUND_PDL:
// 0 off, 1 (default) dependents signalled after this CTA's tiles, 2 at
// entry): back-to-back rounds overlap one kernel's launch with the previous
// one's tail.  C1, 4 rotating jobs: 36.1-36.8 -> 33.7-34.6 us per round
// (profiles/r02/c1/r24, r25; 1 and 2 measure the same).
int local_round_pdl() {
  static const int v = [] {
    const char* e = getenv("CO2_LOCAL_ROUND_PDL");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <class M, int V, int U, int MINB>
co2_status_t launch_local_round_k(LocalRoundArgs a, cudaStream_t s) {
  auto k = local_round_kernel<M, V, U, kThreads, MINB>;
  const int TV = a.tv;
  const int64_t nv = a.n / V;
  const int64_t per_tile = (int64_t)kThreads * TV;
  int64_t tpr = (nv + per_tile - 1) / per_tile;
  if (tpr < 1) tpr = 1;  // the scalar tail (and n = 0) still gets a tile per role
  const int64_t ntiles = tpr * (a.g + 1);
  if (ntiles > (int64_t)INT32_MAX / 2)
    return fail(CO2_ERR_VALIDATION, "local round: %lld params per worker is too many",
                (long long)a.n);
  a.tiles_per_role = (int)tpr;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sm_count();  // persistent: one wave
  if (grid > ntiles) grid = ntiles;
  a.pdl_early = local_round_pdl() == 2;
  if (local_round_pdl()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CO2_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  } else {
    k<<<(int)grid, kThreads, 0, s>>>(a);
  }
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

// Vectors in flight per thread (CO2_LOCAL_ROUND_U = 1 | 2, default 1): U = 2
// needs the register budget of 2 CTAs/SM, U = 1 fits 3 (fp32).
int local_round_u() {
  static const int v = [] {
    const char* e = getenv("CO2_LOCAL_ROUND_U");
    return (e && atoi(e) == 2) ? 2 : 1;
  }();
  return v;
}

int local_round_pf() {
  static const int v = [] {
    const char* e = getenv("CO2_LOCAL_ROUND_PF");
    return (e && atoi(e) == 1) ? 1 : 0;
  }();
  return v;
}

// Vectors per thread per tile (CO2_LOCAL_ROUND_TV, even, 2..32, default 4).
int local_round_tv() {
  static const int v = [] {
    const char* e = getenv("CO2_LOCAL_ROUND_TV");
    const int x = e ? atoi(e) : 4;
    return x < 2 ? 2 : (x > 32 ? 32 : x & ~1);
  }();
  return v;
}

template <class M, int V>
co2_status_t launch_local_round(LocalRoundArgs a, cudaStream_t s) {
  a.prefetch = local_round_pf();
  a.tv = local_round_tv();
  if (local_round_u() == 1)
    return launch_local_round_k<M, V, 1, std::is_same<M, ModeF32>::value ? 3 : 2>(a, s);
  return launch_local_round_k<M, V, 2, 2>(a, s);
}

// ---------------------------------- bulk-copy (TMA 1D) single-launch LOCAL round
// The LDG round kernel above is latency-bound at C1's size: 24 warps per SM
// with one 16-byte vector per stream in flight cover ~60 KB per SM, and 40 %
// of the warps' cycles wait on loads (profiles/r02/ncu/c1_local_round_*).
// Here one producer lane per CTA claims role-major tiles (as above) and
// moves each tile's input streams with cp.async.bulk into a STAGES-deep
// shared-memory ring (up to ~190 KB in flight per SM, no registers held);
// NCW consumer warps compute from shared memory and store to global.
// Step tiles carry x_t0, p0, m (state) and p1, xbar (low); average tiles the
// G contributions.  Per element the ops are the LDG kernel's, so results and
// diagnostics are bitwise the same.  The n % TILE tail of every role is done
// by the last CTA straight from global memory.
template <class M, int TILE>
struct LrStage {
  using TS = typename M::TS;
  using TL = typename M::TL;
  static constexpr int kS = TILE * (int)sizeof(TS);
  static constexpr int kL = TILE * (int)sizeof(TL);
  static constexpr int kStep = 3 * kS + 2 * kL;
  __host__ __device__ static constexpr int bytes(int g) {
    return kStep > g * kL ? kStep : g * kL;
  }
};

// Fold one consumer warp's accumulators into a per-warp slot; consumer
// thread 0 merges the NCW slots into the role's atomic accumulators after a
// named barrier over the consumer warps only (the producer lane never joins).
template <int NCW>
__device__ __forceinline__ void lr_bulk_merge(const Acc& a, Partial* slots, WsHeader* hdr,
                                              bool avg) {
  Partial b{a.min_gap, a.max_step, (unsigned long long)a.clipped, (unsigned long long)a.floored,
            a.flags, 0u};
  b = warp_fold(b);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) slots[warp] = b;
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
  if (threadIdx.x == 0) {
    Partial r = slots[0];
    for (int w = 1; w < NCW; ++w) partial_merge(r, slots[w]);
    if (avg) {
      if (r.flags) atomicOr(&hdr->acc_flags2, r.flags);
    } else {
      atomicMax(&hdr->acc_min_key, ~dkey(r.min_gap));
      atomicMax(&hdr->acc_max_key, dkey(r.max_step));
      if (r.clipped) atomicAdd(&hdr->acc_clipped, r.clipped);
      if (r.floored) atomicAdd(&hdr->acc_floored, r.floored);
      if (r.flags) atomicOr(&hdr->acc_flags, r.flags);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");  // slots reusable
}

template <class M, int TILE, int STAGES, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) local_round_bulk_kernel(const LocalRoundArgs a) {
  using TS = typename M::TS;
  using TL = typename M::TL;
  using TC = typename M::TC;
  using SG = LrStage<M, TILE>;
  constexpr int NT = (NCW + 1) * 32;
  constexpr int VE = 16 / (int)sizeof(TS);  // elements per lane per state access
  static_assert(TILE % (NCW * 32 * VE) == 0, "tile must split evenly over the consumer lanes");
  constexpr int GROUPS = TILE / (NCW * 32 * VE);
  constexpr bool LQ = !std::is_same<TS, TL>::value;
  const int G = a.g;
  const int stage_bytes = SG::bytes(G);
  const int NS = a.stages;  // <= STAGES: as many as fit beside G contributions

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + STAGES;
  int* tile_of = reinterpret_cast<int*>(empty + STAGES);
  Partial* slots = reinterpret_cast<Partial*>(smem + 256);
  unsigned char* ring = smem + 256 + ((sizeof(Partial) * NCW + 127) / 128) * 128;

  Hyp<TC> h;
  h.tau = (TC)a.tau;
  h.eps = (TC)a.eps;
  h.beta = (TC)a.beta;
  h.phi = (TC)a.phi;
  h.alpha = (TC)a.alpha;
  h.divisor = (TC)1;
  h.penalty = a.penalty;
  h.clip = a.clip;
  h.divide = 0;
  const int tpr = a.tiles_per_role;  // full tiles per role
  const int ntiles = tpr * (G + 1);
  WsHeader* h0 = ws_header(a.ws[0]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
  if (a.ts && blockIdx.x == 0 && threadIdx.x == 0) h0->t_start = (unsigned long long)global_ns();

  AccT<TC> acc;
  if (warp == NCW) {
    if (lane == 0) {  // producer: static first tile, then claims
      const uint64_t pol = evict_first_policy();
      int t = (int)blockIdx.x;
      for (int it = 0;; ++it) {
        const int s = it % NS;
        const unsigned ph = (unsigned)(it / NS) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        if (it > 0) t = (int)gridDim.x + (int)atomicAdd(&h0->tile_next, 1u);
        if (t >= ntiles) {
          tile_of[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        tile_of[s] = t;
        const int role = t / tpr;
        const int64_t e = (int64_t)(t - role * tpr) * TILE;
        unsigned char* st = ring + (size_t)s * stage_bytes;
        if (role < G) {
          mbar_arrive_expect_tx(&full[s], SG::kStep);
          bulk_g2s(st, static_cast<const TS*>(a.x_t0[role]) + e, SG::kS, &full[s], pol);
          bulk_g2s(st + SG::kS, static_cast<const TS*>(a.p0[role]) + e, SG::kS, &full[s], pol);
          bulk_g2s(st + 2 * SG::kS, static_cast<const TS*>(a.m[role]) + e, SG::kS, &full[s], pol);
          bulk_g2s(st + 3 * SG::kS, static_cast<const TL*>(a.p1[role]) + e, SG::kL, &full[s], pol);
          bulk_g2s_nohint(st + 3 * SG::kS + SG::kL, static_cast<const TL*>(a.xbar) + e, SG::kL,
                          &full[s]);  // default priority: every worker's tiles read it
        } else {
          mbar_arrive_expect_tx(&full[s], (unsigned)(G * SG::kL));
          for (int w = 0; w < G; ++w)
            bulk_g2s(st + w * SG::kL, static_cast<const TL*>(a.cur[w]) + e, SG::kL, &full[s], pol);
        }
      }
    }
  } else {  // consumers
    int role_cur = -1;
    for (int it = 0;; ++it) {
      const int s = it % NS;
      const unsigned ph = (unsigned)(it / NS) & 1u;
      mbar_wait(&full[s], ph);
      const int t = tile_of[s];
      if (t < 0) break;
      const int role = t / tpr;
      if (role != role_cur) {
        if (role_cur >= 0) {
          lr_bulk_merge<NCW>(acc.widen(), slots, ws_header(a.ws[role_cur < G ? role_cur : 0]),
                             role_cur == G);
          acc = AccT<TC>();
        }
        role_cur = role;
      }
      const int64_t e0 = (int64_t)(t - role * tpr) * TILE;
      const unsigned char* st = ring + (size_t)s * stage_bytes;
      if (role < G) {
        const TS* sx = reinterpret_cast<const TS*>(st);
        const TS* sp0 = reinterpret_cast<const TS*>(st + SG::kS);
        const TS* sm = reinterpret_cast<const TS*>(st + 2 * SG::kS);
        const TL* sp1 = reinterpret_cast<const TL*>(st + 3 * SG::kS);
        const TL* sxb = reinterpret_cast<const TL*>(st + 3 * SG::kS + SG::kL);
        TS* Mm = static_cast<TS*>(a.m[role]);
        TS* A = static_cast<TS*>(a.anchor[role]);
        TL* PR = static_cast<TL*>(a.params[role]);
        TS* Gp = static_cast<TS*>(a.gap[role]);
#pragma unroll
        for (int g = 0; g < GROUPS; ++g) {
          const int o = (g * NCW * 32 + warp * 32 + lane) * VE;
          TS x[VE], q0[VE], mo[VE];
          TL q1[VE], xb[VE];
          ld_smem<TS, VE>(sx + o, x);
          ld_smem<TS, VE>(sp0 + o, q0);
          ld_smem<TS, VE>(sm + o, mo);
          ld_smem<TL, VE>(sp1 + o, q1);
          ld_smem<TL, VE>(sxb + o, xb);
          TS mn[VE], xs[VE], gs[VE];
          TL xl[VE];
#pragma unroll
          for (int v = 0; v < VE; ++v) {
            TC m = to_c(mo[v]), xn, lam;
            co2_elem<TC, LQ>(to_c(x[v]), to_c(q0[v]), to_c(q1[v]), to_c(xb[v]), m, xn, lam, h,
                             acc);
            mn[v] = (TS)m;
            xs[v] = (TS)xn;
            gs[v] = (TS)lam;
            xl[v] = Store<TL>::from(xn);
          }
          const int64_t e = e0 + o;
          st_vec<TS, VE>(Mm + e, mn);
          if (A) st_vec<TS, VE>(A + e, xs);
          st_vec<TL, VE>(PR + e, xl);
          if (Gp) st_vec<TS, VE>(Gp + e, gs);
        }
      } else {
        const TC gd = (TC)G;
        TL* AO = static_cast<TL*>(a.avg_out);
        constexpr int VL = 16 / (int)sizeof(TL);  // low elements per lane per access
        constexpr int GL = TILE / (NCW * 32 * VL);
        static_assert(TILE % (NCW * 32 * VL) == 0, "tile must split evenly (low dtype)");
#pragma unroll 1
        for (int g = 0; g < GL; ++g) {
          const int o = (g * NCW * 32 + warp * 32 + lane) * VL;
          TC sacc[VL];
          for (int w = 0; w < G; ++w) {  // ascending worker order, param_ops.cpp:26-28
            TL c[VL];
            ld_smem<TL, VL>(reinterpret_cast<const TL*>(st + w * SG::kL) + o, c);
#pragma unroll
            for (int q = 0; q < VL; ++q) sacc[q] = w == 0 ? to_c(c[q]) : sacc[q] + to_c(c[q]);
          }
          TL out[VL];
#pragma unroll
          for (int q = 0; q < VL; ++q) {
            const TC r = div_rn_nz(sacc[q], gd);  // one division, :30
            if (!isfinite(r)) acc.flags |= CO2_FLAG_AVG_NONFINITE;
            out[q] = Store<TL>::from(r);
          }
          st_vec<TL, VL>(AO + e0 + o, out);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (role_cur >= 0)
      lr_bulk_merge<NCW>(acc.widen(), slots, ws_header(a.ws[role_cur < G ? role_cur : 0]),
                         role_cur == G);
  }
  __syncthreads();
  // Tail: the n % TILE coordinates of every role, by the last CTA.
  const int64_t full_n = (int64_t)tpr * TILE;
  if (blockIdx.x == gridDim.x - 1 && full_n < a.n) {
    const TL* XB = static_cast<const TL*>(a.xbar);
    for (int r = 0; r <= G; ++r) {
      AccT<TC> ta;
      for (int64_t j = full_n + threadIdx.x; j < a.n; j += NT) {
        if (r < G) {
          TS* Mm = static_cast<TS*>(a.m[r]);
          TC m = to_c(Mm[j]), xn, lam;
          const TS xv = static_cast<const TS*>(a.x_t0[r])[j];
          co2_elem<TC, LQ>(to_c(xv), to_c(static_cast<const TS*>(a.p0[r])[j]),
                           to_c(static_cast<const TL*>(a.p1[r])[j]), to_c(XB[j]), m, xn, lam, h,
                           ta);
          Mm[j] = (TS)m;
          if (a.anchor[r]) static_cast<TS*>(a.anchor[r])[j] = (TS)xn;
          static_cast<TL*>(a.params[r])[j] = Store<TL>::from(xn);
          if (a.gap[r]) static_cast<TS*>(a.gap[r])[j] = (TS)lam;
        } else {
          TC sacc = to_c(static_cast<const TL*>(a.cur[0])[j]);
          for (int w = 1; w < G; ++w) sacc = sacc + to_c(static_cast<const TL*>(a.cur[w])[j]);
          const TC q = div_rn_nz(sacc, (TC)G);
          if (!isfinite(q)) ta.flags |= CO2_FLAG_AVG_NONFINITE;
          static_cast<TL*>(a.avg_out)[j] = Store<TL>::from(q);
        }
      }
      // whole-CTA merge of this role's tail
      const Partial b = block_partial<NT>(ta.widen());
      if (threadIdx.x == 0) {
        WsHeader* hr = ws_header(a.ws[r < G ? r : 0]);
        if (r == G) {
          if (b.flags) atomicOr(&hr->acc_flags2, b.flags);
        } else {
          atomicMax(&hr->acc_min_key, ~dkey(b.min_gap));
          atomicMax(&hr->acc_max_key, dkey(b.max_step));
          if (b.clipped) atomicAdd(&hr->acc_clipped, b.clipped);
          if (b.floored) atomicAdd(&hr->acc_floored, b.floored);
          if (b.flags) atomicOr(&hr->acc_flags, b.flags);
        }
      }
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // Last CTA: publish and reset every role (thread r publishes role r).
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&h0->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int r = (int)threadIdx.x;
  if (r < G) {
    volatile WsHeader* vh = ws_header(a.ws[r]);
    const unsigned long long kmin = vh->acc_min_key, kmax = vh->acc_max_key;
    co2_diag_t d;
    d.min_gap = kmin ? dkey_inv(~kmin) : (double)INFINITY;
    d.max_outer_step = kmax ? dkey_inv(kmax) : 0.0;
    d.n_clipped = (int64_t)vh->acc_clipped;
    d.n_floored = (int64_t)vh->acc_floored;
    d.flags = vh->acc_flags;
    d.pad = 0;
    WsHeader* hr = ws_header(a.ws[r]);
    hr->diag = d;
    hr->acc_min_key = 0ull;
    hr->acc_max_key = 0ull;
    hr->acc_clipped = 0ull;
    hr->acc_floored = 0ull;
    hr->acc_flags = 0u;
    if (a.host_diag[r]) *a.host_diag[r] = d;
  } else if (r == G) {
    volatile WsHeader* vh = h0;
    const unsigned int f = vh->acc_flags2;
    h0->acc_flags2 = 0u;
    if (a.avg_diag) {
      co2_diag_t ad{INFINITY, 0.0, 0, 0, f, 0};
      *a.avg_diag = ad;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    h0->tile_next = 0u;  // self-reset for the next launch
    h0->ticket = 0u;
    if (a.ts) {
      a.ts[0] = *static_cast<volatile unsigned long long*>(&h0->t_start);
      a.ts[1] = (unsigned long long)global_ns();
    }
  }
}

template <class M, int TILE, int STAGES, int NCW>
co2_status_t launch_local_round_bulk(LocalRoundArgs a, cudaStream_t s) {
  auto k = local_round_bulk_kernel<M, TILE, STAGES, NCW>;
  using SG = LrStage<M, TILE>;
  const size_t hdr = 256 + ((sizeof(Partial) * NCW + 127) / 128) * 128;
  const size_t avail = 227 * 1024 - hdr;
  int ns = (int)(avail / (size_t)SG::bytes(a.g));
  if (ns > STAGES) ns = STAGES;
  if (ns < 2)
    return fail(CO2_ERR_VALIDATION, "local round (bulk): %d workers need too much shared memory",
                a.g);
  a.stages = ns;
  const size_t smem = hdr + (size_t)ns * SG::bytes(a.g);
  constexpr int NT = (NCW + 1) * 32;
  CO2_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t tpr = a.n / TILE;
  a.tiles_per_role = (int)tpr;
  const int64_t ntiles = tpr * (a.g + 1);
  int64_t grid = (int64_t)per_sm * sm_count();
  if (grid > ntiles) grid = ntiles < 1 ? 1 : ntiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = local_round_pdl() ? 1 : 0;
  CO2_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

// CO2_LOCAL_ROUND_BULK = 1 selects the bulk-copy round kernel (vectorised
// layouts only).
int local_round_bulk() {
  static const int v = [] {
    const char* e = getenv("CO2_LOCAL_ROUND_BULK");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <class M>
co2_status_t launch_local_round_v(const LocalRoundArgs& a, bool vec, cudaStream_t s) {
  constexpr int V = std::is_same<M, ModeF64>::value ? 2 : (std::is_same<M, ModeF32>::value ? 4 : 8);
  if (vec && local_round_bulk() > 0) {
    // TILE = NCW x 32 lanes x (elements per 16-byte access of the narrower
    // dtype) x k; stage = max(3 x TILE x state + 2 x TILE x low, G x TILE x
    // low) bytes: fp32 TILE 2048 -> 40 KB, bf16-mixed 4096 -> 64 KB, fp64
    // 1024 -> 40 KB per stage at NCW = 16.
    constexpr int VM = 16 / (int)sizeof(typename M::TL);
    switch (local_round_bulk()) {  // stages: as many as fit (<= 8)
      case 2: return launch_local_round_bulk<M, 8 * 32 * VM * 2, 8, 8>(a, s);
      case 3: return launch_local_round_bulk<M, 16 * 32 * VM, 3, 16>(a, s);
      default: return launch_local_round_bulk<M, 16 * 32 * VM, 8, 16>(a, s);
    }
  }
  if (vec) return launch_local_round<M, V>(a, s);
  return launch_local_round<M, 1>(a, s);
}
}  // namespace

co2_status_t local_round_impl(co2_mode_t mode, int g, int64_t n, const void* const* x_t0,
                              const void* const* p0, const void* const* p1, void* const* m,
                              void* const* anchor, void* const* params, void* const* gap,
                              const void* const* cur, void* const* ws,
                              co2_diag_t* const* host_diag, co2_diag_t* avg_diag,
                              const void* xbar, void* avg_out, const co2_hyper_t* h,
                              unsigned long long* ts, cudaStream_t s) {
  if (g < 1 || g > kMaxLocalRound)
    return fail(CO2_ERR_VALIDATION, "local round: 1..%d workers", kMaxLocalRound);
  LocalRoundArgs a{};
  bool vec = aligned16(xbar) && aligned16(avg_out);
  for (int w = 0; w < g; ++w) {
    a.x_t0[w] = x_t0[w];
    a.p0[w] = p0[w];
    a.p1[w] = p1[w];
    a.m[w] = m[w];
    a.anchor[w] = anchor[w];
    a.params[w] = params[w];
    a.gap[w] = gap[w];
    a.cur[w] = cur[w];
    a.ws[w] = ws[w];
    a.host_diag[w] = host_diag ? host_diag[w] : nullptr;
    vec = vec && aligned16(x_t0[w]) && aligned16(p0[w]) && aligned16(p1[w]) && aligned16(m[w]) &&
          aligned16(anchor[w]) && aligned16(params[w]) && aligned16(gap[w]) && aligned16(cur[w]);
  }
  a.avg_diag = avg_diag;
  a.ts = ts;
  a.xbar = xbar;
  a.avg_out = avg_out;
  a.g = g;
  a.n = n;
  a.alpha = h->alpha;
  a.beta = h->beta;
  a.phi = h->phi;
  a.eps = h->epsilon;
  a.tau = h->tau;
  a.penalty = h->penalty ? 1 : 0;
  a.clip = h->clip ? 1 : 0;
  switch (mode) {
    case CO2_MODE_F64: return launch_local_round_v<ModeF64>(a, vec, s);
    case CO2_MODE_F32: return launch_local_round_v<ModeF32>(a, vec, s);
    case CO2_MODE_BF16_MIXED: return launch_local_round_v<ModeBF16>(a, vec, s);
  }
  return fail(CO2_ERR_VALIDATION, "local round: unknown mode %d", (int)mode);
}
}  // namespace co2

// ====================================================== divergence metric
// Simulation::step's round diagnostic (proj/src/outer_algorithms.cpp:
// 503-508): xbar = average_params() (fixed worker order, one division) and
// divergence = max_i ||x_i - xbar||_2.  Squares accumulate in fp64 per thread
// in grid-stride order, then a fixed shuffle tree, fixed warp order and
// fixed block order: deterministic for a given grid (Eigen's own reduction
// order is SIMD-shaped, so the sum is within rounding, not bitwise).
namespace co2 {
namespace {
constexpr int kDivBlocks = 256;
constexpr int kDivMaxWorkers = 64;

template <typename T, typename TC>
__global__ void __launch_bounds__(kThreads)
    divergence_kernel(const Ptrs64<T> c, int g, int64_t n, double* partials, double* out,
                      unsigned int* ticket) {
  __shared__ double sh[kThreads / 32][kDivMaxWorkers];
  __shared__ bool s_last;
  const TC gd = (TC)g;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int w0 = 0; w0 < g; w0 += 8) {  // 8 workers per pass keeps registers bounded
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * kThreads) {
      TC s = to_c(c.p[0][j]);
      for (int i = 1; i < g; ++i) s += to_c(c.p[i][j]);
      const TC xb = div_rn_nz(s, gd);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (w0 + k < g) {
          const double d = (double)to_c(c.p[w0 + k][j]) - (double)xb;  // exact widening
          acc[k] += d * d;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double v = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && w0 + k < g) sh[wid][w0 + k] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < g) {
    double b = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) b += sh[w][threadIdx.x];
    partials[(size_t)blockIdx.x * kDivMaxWorkers + threadIdx.x] = b;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < g) {
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b)
      tot += __ldcg(&partials[(size_t)b * kDivMaxWorkers + threadIdx.x]);
    out[threadIdx.x] = sqrt(tot);
  }
  if (threadIdx.x == 0) *ticket = 0;
}
}  // namespace
}  // namespace co2

extern "C" co2_status_t co2_divergence(co2_dtype_t dt, int32_t g, const void* const* params,
                                       int64_t n, double* per_worker, double* max_out, void* ws,
                                       void* stream) {
  if (g < 1 || g > kDivMaxWorkers) return fail(CO2_ERR_VALIDATION, "divergence: 1..64 workers");
  if (n < 0 || !ws) return fail(CO2_ERR_VALIDATION, "divergence: bad arguments");
  CO2_TRY(check_dtype(dt));
  if (!params) return fail(CO2_ERR_VALIDATION, "null buffer");
  for (int i = 0; i < g; ++i)
    if (n > 0 && !params[i]) return fail(CO2_ERR_VALIDATION, "null buffer");
  cudaStream_t s = S(stream);
  // Scratch inside the workspace's partials area: per-block per-worker sums,
  // then g results and a private ticket.
  char* base = reinterpret_cast<char*>(ws_partials(ws));
  double* partials = reinterpret_cast<double*>(base);
  double* out = partials + (size_t)kDivBlocks * kDivMaxWorkers;
  unsigned int* ticket = reinterpret_cast<unsigned int*>(out + kDivMaxWorkers);
  static_assert(sizeof(double) * (kDivBlocks * kDivMaxWorkers + kDivMaxWorkers) + 16 <=
                    sizeof(Partial) * kMaxBlocks,
                "divergence scratch exceeds the workspace");
  CO2_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), s));
  int grid = simple_grid(n, kThreads);
  if (grid > kDivBlocks) grid = kDivBlocks;
  if (dt == CO2_DTYPE_F64) {
    Ptrs64<double> p{};
    for (int i = 0; i < g; ++i) p.p[i] = static_cast<const double*>(params[i]);
    divergence_kernel<double, double><<<grid, kThreads, 0, s>>>(p, g, n, partials, out, ticket);
  } else if (dt == CO2_DTYPE_F32) {
    Ptrs64<float> p{};
    for (int i = 0; i < g; ++i) p.p[i] = static_cast<const float*>(params[i]);
    divergence_kernel<float, float><<<grid, kThreads, 0, s>>>(p, g, n, partials, out, ticket);
  } else {
    Ptrs64<bf16s> p{};
    for (int i = 0; i < g; ++i) p.p[i] = static_cast<const bf16s*>(params[i]);
    divergence_kernel<bf16s, float><<<grid, kThreads, 0, s>>>(p, g, n, partials, out, ticket);
  }
  CO2_CUDA(cudaGetLastError());
  double host[kDivMaxWorkers];
  CO2_CUDA(cudaMemcpyAsync(host, out, sizeof(double) * g, cudaMemcpyDeviceToHost, s));
  CO2_CUDA(cudaStreamSynchronize(s));
  double mx = 0.0;
  for (int i = 0; i < g; ++i) {
    if (per_worker) per_worker[i] = host[i];
    mx = host[i] > mx ? host[i] : mx;
  }
  if (max_out) *max_out = mx;
  return CO2_OK;
}

extern "C" co2_status_t co2_slowmo_step(co2_mode_t mode, int64_t n, const void* x_start,
                                        const void* xbar, int32_t divisor, void* momentum,
                                        void* params_out, void* anchor_out, double alpha,
                                        double beta, void* ws, void* stream) {
  // slowmo_round's checks, outer_algorithms.cpp:219-222
  if (!(alpha > 0.0)) return fail(CO2_ERR_VALIDATION, "slowmo: alpha must be positive");
  if (beta < 0.0 || beta >= 1.0) return fail(CO2_ERR_VALIDATION, "slowmo: beta must lie in [0, 1)");
  if (n < 0 || divisor < 1 || !ws) return fail(CO2_ERR_VALIDATION, "slowmo: bad arguments");
  return slowmo_impl(mode, n, x_start, xbar, divisor, momentum, params_out, anchor_out, alpha,
                     beta, ws, S(stream));
}

extern "C" co2_status_t co2_local_sgd_step(co2_mode_t mode, int64_t n, const void* x_start,
                                           const void* xbar, int32_t divisor, void* params_out,
                                           void* anchor_out, void* ws, void* stream) {
  if (n < 0 || divisor < 1 || !ws) return fail(CO2_ERR_VALIDATION, "local_sgd: bad arguments");
  return local_sgd_impl(mode, n, x_start, xbar, divisor, params_out, anchor_out, ws, S(stream));
}

extern "C" co2_status_t co2_overlap_correction(co2_mode_t mode, int64_t n, void* params,
                                               const void* anchor, const void* xbar,
                                               int32_t divisor, void* ws, void* stream) {
  if (n < 0 || divisor < 1 || !ws)
    return fail(CO2_ERR_VALIDATION, "overlap correction: bad arguments");
  return overlap_correction_impl(mode, n, params, anchor, xbar, divisor, ws, S(stream));
}
