// Deterministic fixed-order all-reduce over NVLink peer memory (SURVEY.md
// 8f item 1): the one-step-stale average of x_{t,tau} computed exactly as the
// reference's average() (proj/src/param_ops.cpp:16-33) -- contributions summed
// in ascending worker order, one division by G -- so the result is bitwise
// the oracle's for ANY worker count, which NCCL's ring/tree order is not.
//
// Rank r owns slice r of the buffer.  Each CTA grid-strides over slice r in
// 16-byte vectors: it loads the slice from every rank's buffer (peer pointers
// opened with CUDA IPC, loads over NVLink 5 / NVSwitch), accumulates in the
// compute type in rank order, divides once, and stores the rounded average
// into slice r of EVERY rank's buffer (a fused all-gather by P2P stores).
// Per GPU that moves S/G*(G-1) bytes in and out over NVLink and ~2S bytes of
// HBM (own slice read + peer reads served, own write + peer writes received)
// -- half of a ring all-reduce's HBM traffic.
//
// Cross-GPU ordering uses flag words in IPC-shared signal memory:
//   entry  : every CTA publishes ready[rank] = epoch in each peer's signal
//            area (release, system scope) and waits for all ready[p] >= epoch;
//   exit   : every CTA adds 1 to done in each peer's area after its stores
//            (release) and waits until its own done reaches epoch*G*grid.
// All spins are bounded in wall-clock time (Signals::timeout_ms, 10 s by
// default): on timeout the kernel records a flag and
// exits instead of hanging the GPU.
#include <cuda_bf16.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include "bulk.cuh"
#include "common.cuh"
#include "p2p_sync.cuh"

namespace co2 {
namespace {

struct bf16raw {
  uint16_t b;
};

__device__ __forceinline__ float ld_c(const bf16raw* p) {
  return __uint_as_float(((uint32_t)p->b) << 16);
}


struct P2PArgs {
  void* bufs[kMaxRanks];      // rank-indexed pointers to the same logical buffer
  Signals* sig[kMaxRanks];    // rank-indexed signal areas (sig[rank] is local)
  int64_t n;                  // elements in the buffer
  int64_t shard;              // elements per slice (multiple of the vector width)
  int world, rank;
  uint32_t epoch;             // 1, 2, ... (same sequence on every rank)
  uint32_t done_target;       // cumulative exit-barrier count after this launch
};

// TL storage, TC compute, V elements per 16-byte vector.  bf16 / fp32
// instantiations are capped at 64 registers per thread (min blocks 1024/NT):
// the co-running fused step fills the register file at 4 x 256 threads x 64
// registers per SM, so a reduce CTA of NT x 64 registers takes exactly NT/256
// step CTAs' worth of registers instead of rounding up to one more (the
// uncapped 256-thread bf16 kernel used 72-84 registers, i.e. two step CTAs).
// Exit of the fixed-order all-reduce, by thread 0 of every CTA: each CTA
// fences its peer stores at system scope and takes a ticket; the rank's last
// CTA alone tells every rank it is done and waits until all ranks told it
// (kernel completion then implies every slice reached every rank).  One
// signal per rank per launch, so ranks may launch different grids.
__device__ __forceinline__ void p2p_rank_exit(const P2PArgs& a, Signals* mine) {
  __threadfence_system();
  if (atomicAdd(&mine->ticket_local, 1u) != gridDim.x - 1) return;
  mine->ticket_local = 0u;  // self-reset: the next launch starts after this grid
  __threadfence_system();
  for (int p = 0; p < a.world; ++p) red_release_sys_add(&a.sig[p]->done, 1u);
  if (!spin_until(&mine->done, a.done_target, mine)) mine->error = 2;
}

template <typename TL, typename TC, int V, int R, int U, int NT>
__global__ void __launch_bounds__(NT, sizeof(TL) <= 4 ? 1024 / NT : 1)
    p2p_average_kernel(const P2PArgs a) {
  Signals* mine = a.sig[a.rank];
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    for (int p = 0; p < a.world; ++p) st_release_sys(&a.sig[p]->ready[a.rank], a.epoch);
    bool ok = true;
    for (int p = 0; p < a.world && ok; ++p) ok = spin_until(&mine->ready[p], a.epoch, mine);
    if (!ok) mine->error = 1;
    s_ok = ok;
  }
  __syncthreads();
  if (s_ok) {
    const int64_t lo = (int64_t)a.rank * a.shard;
    int64_t hi = lo + a.shard;
    if (hi > a.n) hi = a.n;
    const TC g = (TC)a.world;
    const int64_t nvec = hi > lo ? (hi - lo) / V : 0;
    const int64_t stride = (int64_t)gridDim.x * NT;
    // U vectors per thread in flight, each gathered from every rank: the
    // remote (NVLink) loads are issued back to back before any arithmetic.
    auto reduce_store = [&](const uint4 (&raw)[R], int64_t e) {
      TC acc[V];
      {
        const TL* v0 = reinterpret_cast<const TL*>(&raw[0]);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          if constexpr (sizeof(TL) == 2) acc[k] = ld_c(reinterpret_cast<const bf16raw*>(v0 + k));
          else acc[k] = (TC)v0[k];
        }
      }
#pragma unroll
      for (int p = 1; p < R; ++p) {
        if (p < a.world) {
          const TL* vp = reinterpret_cast<const TL*>(&raw[p]);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            TC x;
            if constexpr (sizeof(TL) == 2) x = ld_c(reinterpret_cast<const bf16raw*>(vp + k));
            else x = (TC)vp[k];
            acc[k] = acc[k] + x;  // ascending worker order, param_ops.cpp:26-28
          }
        }
      }
      uint4 out;
      TL* o = reinterpret_cast<TL*>(&out);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        TC r = div_rn_nz(acc[k], (TC)g);  // one division, param_ops.cpp:30
        if constexpr (sizeof(TL) == 2) {
          __nv_bfloat16 h = __float2bfloat16_rn((float)r);
          reinterpret_cast<uint16_t*>(o)[k] = __bfloat16_as_ushort(h);
        } else {
          o[k] = (TL)r;
        }
      }
#pragma unroll
      for (int p = 0; p < R; ++p)
        if (p < a.world) __stcg(reinterpret_cast<uint4*>(static_cast<TL*>(a.bufs[p]) + e), out);
    };
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    for (; i + (int64_t)(U - 1) * stride < nvec; i += (int64_t)U * stride) {
      uint4 raw[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int p = 0; p < R; ++p)
          if (p < a.world)
            raw[u][p] = __ldcg(reinterpret_cast<const uint4*>(
                static_cast<const TL*>(a.bufs[p]) + lo + (i + (int64_t)u * stride) * V));
#pragma unroll
      for (int u = 0; u < U; ++u) reduce_store(raw[u], lo + (i + (int64_t)u * stride) * V);
    }
    for (; i < nvec; i += stride) {
      uint4 raw[R];
#pragma unroll
      for (int p = 0; p < R; ++p)
        if (p < a.world)
          raw[p] = __ldcg(reinterpret_cast<const uint4*>(static_cast<const TL*>(a.bufs[p]) + lo + i * V));
      reduce_store(raw, lo + i * V);
    }
    // scalar tail of the last slice (n not a multiple of V)
    if (blockIdx.x == 0) {
      for (int64_t j = lo + nvec * V + threadIdx.x; j < hi; j += NT) {
        TC acc;
        if constexpr (sizeof(TL) == 2)
          acc = ld_c(static_cast<const bf16raw*>(a.bufs[0]) + j);
        else
          acc = (TC)__ldcg(static_cast<const TL*>(a.bufs[0]) + j);
        for (int p = 1; p < a.world; ++p) {
          TC x;
          if constexpr (sizeof(TL) == 2)
            x = ld_c(static_cast<const bf16raw*>(a.bufs[p]) + j);
          else
            x = (TC)__ldcg(static_cast<const TL*>(a.bufs[p]) + j);
          acc = acc + x;
        }
        TC r = div_rn_nz(acc, (TC)g);
        for (int p = 0; p < a.world; ++p) {
          if constexpr (sizeof(TL) == 2) {
            __nv_bfloat16 h = __float2bfloat16_rn((float)r);
            static_cast<bf16raw*>(a.bufs[p])[j].b = __bfloat16_as_ushort(h);
          } else {
            static_cast<TL*>(a.bufs[p])[j] = (TL)r;
          }
        }
      }
    }
  }
  // Exit barrier: our slice is in every peer's buffer before any rank's
  // consumer may read the result.
  __syncthreads();
  if (threadIdx.x == 0) p2p_rank_exit(a, mine);
}

// Bulk-copy variant of p2p_average_kernel (CO2_P2P_BULK=1): the same slice
// ownership, barriers and arithmetic, with the G remote loads of each tile
// issued by ONE lane as cp.async.bulk copies (TMA over NVLink) into a
// STAGES-deep shared-memory ring, so the bytes in flight sit in shared
// memory instead of registers.  NCW consumer warps sum the G copies of each
// 16-byte vector in ascending rank order, divide once, and store the result
// into every rank with 128-bit STGs.  A CTA is (NCW + 1) warps, so the reduce
// displaces far fewer registers of the co-running fused step (which fills
// the register file at 4 x 256 threads x 64 registers per SM) than the
// register-staged kernel's 256 threads x ~84 registers.
template <typename TL, typename TC, int TILE, int STAGES, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32) p2p_bulk_average_kernel(const P2PArgs a) {
  constexpr int NT = (NCW + 1) * 32;
  constexpr int V = 16 / (int)sizeof(TL);
  constexpr int CH = TILE * (int)sizeof(TL);  // bytes per rank per tile
  static_assert(TILE % (NCW * 32 * V) == 0, "tile must split over the consumer lanes");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + STAGES;
  unsigned char* ring = smem + 128;
  static_assert(STAGES * 16 <= 128, "barrier header");
  Signals* mine = a.sig[a.rank];
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int p = 0; p < a.world; ++p) st_release_sys(&a.sig[p]->ready[a.rank], a.epoch);
    bool ok = true;
    for (int p = 0; p < a.world && ok; ++p) ok = spin_until(&mine->ready[p], a.epoch, mine);
    if (!ok) mine->error = 1;
    s_ok = ok;
  }
  __syncthreads();
  const int G = a.world;
  const int64_t lo = (int64_t)a.rank * a.shard;
  int64_t hi = lo + a.shard;
  if (hi > a.n) hi = a.n;
  const int64_t len = hi > lo ? hi - lo : 0;
  const int64_t ntiles = len / TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TC g = (TC)G;
  if (s_ok) {
    if (warp == NCW) {
      if (lane == 0) {  // producer
        int it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((unsigned)(it / STAGES) & 1u) ^ 1u);
          unsigned char* st = ring + (size_t)s * CH * G;
          const int64_t e = lo + t * TILE;
          mbar_arrive_expect_tx(&full[s], (unsigned)(CH * G));
          for (int p = 0; p < G; ++p)
            bulk_g2s_nohint(st + (size_t)p * CH, static_cast<const TL*>(a.bufs[p]) + e, CH,
                            &full[s]);
        }
      }
    } else {  // consumers
      int it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (unsigned)(it / STAGES) & 1u);
        const unsigned char* st = ring + (size_t)s * CH * G;
        const int64_t e0 = lo + t * TILE;
#pragma unroll
        for (int q = 0; q < TILE / (NCW * 32 * V); ++q) {
          const int o = (q * NCW * 32 + warp * 32 + lane) * V;
          TC acc[V];
          {
            const uint4 r = *reinterpret_cast<const uint4*>(st + (size_t)o * sizeof(TL));
            const TL* v0 = reinterpret_cast<const TL*>(&r);
#pragma unroll
            for (int k = 0; k < V; ++k) {
              if constexpr (sizeof(TL) == 2) acc[k] = ld_c(reinterpret_cast<const bf16raw*>(v0 + k));
              else acc[k] = (TC)v0[k];
            }
          }
          for (int p = 1; p < G; ++p) {
            const uint4 r =
                *reinterpret_cast<const uint4*>(st + (size_t)p * CH + (size_t)o * sizeof(TL));
            const TL* vp = reinterpret_cast<const TL*>(&r);
#pragma unroll
            for (int k = 0; k < V; ++k) {
              TC x;
              if constexpr (sizeof(TL) == 2) x = ld_c(reinterpret_cast<const bf16raw*>(vp + k));
              else x = (TC)vp[k];
              acc[k] = acc[k] + x;  // ascending worker order, param_ops.cpp:26-28
            }
          }
          uint4 out;
          TL* ov = reinterpret_cast<TL*>(&out);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            TC r = div_rn_nz(acc[k], (TC)g);  // one division, param_ops.cpp:30
            if constexpr (sizeof(TL) == 2) {
              __nv_bfloat16 h = __float2bfloat16_rn((float)r);
              reinterpret_cast<uint16_t*>(ov)[k] = __bfloat16_as_ushort(h);
            } else {
              ov[k] = (TL)r;
            }
          }
          for (int p = 0; p < G; ++p)
            __stcg(reinterpret_cast<uint4*>(static_cast<TL*>(a.bufs[p]) + e0 + o), out);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    // remainder of the slice (len % TILE, vectors then scalars): CTA 0
    if (blockIdx.x == 0) {
      for (int64_t j = lo + ntiles * TILE + threadIdx.x; j < hi; j += NT) {
        TC acc;
        if constexpr (sizeof(TL) == 2)
          acc = ld_c(static_cast<const bf16raw*>(a.bufs[0]) + j);
        else
          acc = (TC)__ldcg(static_cast<const TL*>(a.bufs[0]) + j);
        for (int p = 1; p < G; ++p) {
          TC x;
          if constexpr (sizeof(TL) == 2)
            x = ld_c(static_cast<const bf16raw*>(a.bufs[p]) + j);
          else
            x = (TC)__ldcg(static_cast<const TL*>(a.bufs[p]) + j);
          acc = acc + x;
        }
        TC r = div_rn_nz(acc, (TC)g);
        for (int p = 0; p < G; ++p) {
          if constexpr (sizeof(TL) == 2) {
            __nv_bfloat16 h = __float2bfloat16_rn((float)r);
            static_cast<bf16raw*>(a.bufs[p])[j].b = __bfloat16_as_ushort(h);
          } else {
            static_cast<TL*>(a.bufs[p])[j] = (TL)r;
          }
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) p2p_rank_exit(a, mine);
}

template <typename TL, typename TC, int TILE, int STAGES, int NCW>
void launch_p2p_bulk(const P2PArgs& a, int ctas, cudaStream_t s) {
  auto k = p2p_bulk_average_kernel<TL, TC, TILE, STAGES, NCW>;
  // ring sized for the world: G chunks of TILE per stage
  const size_t smem = 128 + (size_t)STAGES * TILE * sizeof(TL) * a.world;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(128 + (size_t)STAGES * TILE * sizeof(TL) * kMaxRanks));
    attr = true;
  }
  k<<<ctas, (NCW + 1) * 32, smem, s>>>(a);
}

// Slice reduce for the sharded (ghost-consistent) layout: rank r averages
// slice r of `nb` logical buffers (x_{t,tau} and x_{t,1}) over all ranks in
// ascending rank order into local slice outputs -- a deterministic
// reduce-scatter that delivers the average itself.  Entry barrier only:
// the fused sharded step's exit barrier orders every later overwrite of the
// buffers read here (see engine.cpp, co2_sharded_round).
struct SliceArgs {
  const void* src[2][kMaxRanks];
  void* dst[2];
  int nb;
  int64_t lo, len;
  int world, rank;
  uint32_t epoch;
  Signals* sig[kMaxRanks];
};

template <typename TL, typename TC, int V, int R, int U, int NT>
__global__ void __launch_bounds__(NT) p2p_slice_average_kernel(const SliceArgs a) {
  Signals* mine = a.sig[a.rank];
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    for (int p = 0; p < a.world; ++p) st_release_sys(&a.sig[p]->ready[a.rank], a.epoch);
    bool ok = true;
    for (int p = 0; p < a.world && ok; ++p) ok = spin_until(&mine->ready[p], a.epoch, mine);
    if (!ok) mine->error = 1;
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  const TC g = (TC)a.world;
  const int64_t nvec = a.len / V;
  const int64_t stride = (int64_t)gridDim.x * NT;
  auto to_c = [](const TL* v, int k) -> TC {
    if constexpr (sizeof(TL) == 2)
      return ld_c(reinterpret_cast<const bf16raw*>(v + k));
    else
      return (TC)v[k];
  };
  auto store = [](TL* o, int k, TC r) {
    if constexpr (sizeof(TL) == 2) {
      __nv_bfloat16 h = __float2bfloat16_rn((float)r);
      reinterpret_cast<uint16_t*>(o)[k] = __bfloat16_as_ushort(h);
    } else {
      o[k] = (TL)r;
    }
  };
  for (int b = 0; b < a.nb; ++b) {
    int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
    for (; i < nvec; i += (int64_t)U * stride) {
      uint4 raw[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t iv = i + (int64_t)u * stride;
#pragma unroll
        for (int p = 0; p < R; ++p)
          if (p < a.world && iv < nvec)
            raw[u][p] = __ldcg(reinterpret_cast<const uint4*>(
                static_cast<const TL*>(a.src[b][p]) + a.lo + iv * V));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t iv = i + (int64_t)u * stride;
        if (iv >= nvec) break;
        TC acc[V];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = to_c(reinterpret_cast<const TL*>(&raw[u][0]), k);
#pragma unroll
        for (int p = 1; p < R; ++p)
          if (p < a.world)
#pragma unroll
            for (int k = 0; k < V; ++k)
              acc[k] = acc[k] + to_c(reinterpret_cast<const TL*>(&raw[u][p]), k);
        uint4 out;
#pragma unroll
        for (int k = 0; k < V; ++k) store(reinterpret_cast<TL*>(&out), k, div_rn_nz(acc[k], (TC)g));
        *reinterpret_cast<uint4*>(static_cast<TL*>(a.dst[b]) + iv * V) = out;
      }
    }
    if (blockIdx.x == 0) {  // scalar tail
      for (int64_t j = nvec * V + threadIdx.x; j < a.len; j += NT) {
        TC acc = to_c(static_cast<const TL*>(a.src[b][0]) + a.lo + j, 0);
        for (int p = 1; p < a.world; ++p)
          acc = acc + to_c(static_cast<const TL*>(a.src[b][p]) + a.lo + j, 0);
        store(static_cast<TL*>(a.dst[b]) + j, 0, div_rn_nz(acc, (TC)g));
      }
    }
  }
}

// Rank capacity R of the kernel instantiation for a world size.  The env
// CO2_P2P_RANK_CAP=4|8 forces a wider one, so the G = 8 instantiations
// (guarded loads over the unused ranks) are exercised on 2- and 4-GPU boxes
// (tests/test_gpu_multi.py); it never narrows.
int rank_cap(int world) {
  static const int forced = [] {
    const char* e = getenv("CO2_P2P_RANK_CAP");
    return e ? atoi(e) : 0;
  }();
  int cap = world <= 2 ? 2 : (world <= 4 ? 4 : 8);
  if ((forced == 4 || forced == 8) && forced > cap) cap = forced;
  return cap;
}

// Threads per CTA of the all-reduce kernel (CO2_P2P_THREADS = 128 | 256 |
// 512, default 256): its register footprint decides how many fused-step
// CTAs still fit on the SMs it occupies (the step uses the whole register
// file at 4 CTAs/SM).  C3 sweep, 3 interleaved passes on one box
// (profiles/r01/bench/p2p_threads_sweep.txt): 256 threads beat 512 by
// +1.2 % at N=2 (96 CTAs) and +4 % at N=4 (64 CTAs).
int p2p_threads() {
  static const int v = [] {
    const char* e = getenv("CO2_P2P_THREADS");
    const int x = e ? atoi(e) : 256;
    return (x == 128 || x == 512) ? x : 256;
  }();
  return v;
}

// Bulk-copy all-reduce kernel (CO2_P2P_BULK = consumer warps per CTA, 2 or
// 4; 0 / unset = the register-staged kernel).
int p2p_bulk() {
  static const int v = [] {
    const char* e = getenv("CO2_P2P_BULK");
    const int x = e ? atoi(e) : 0;
    return x <= 0 ? 0 : (x >= 4 ? 4 : 2);
  }();
  return v;
}

// Threads per CTA of the sharded slice reduce (CO2_P2P_SLICE_THREADS = 256
// | 512, default 512).  At equal total threads 256 and 512 measure the same
// (profiles/r01/bench/c4_slice_threads.txt); the slice reduce is NVLink-bound.
int p2p_slice_threads() {
  static const int v = [] {
    const char* e = getenv("CO2_P2P_SLICE_THREADS");
    return (e && atoi(e) == 256) ? 256 : 512;
  }();
  return v;
}

}  // namespace

co2_status_t p2p_slice_average_launch(co2_dtype_t dt, int nb, const void* const* src0,
                                      const void* const* src1, void* dst0, void* dst1,
                                      void* const* sigs, int world, int rank, int64_t lo,
                                      int64_t len, uint32_t epoch, int ctas, cudaStream_t s) {
  if (world < 1 || world > kMaxRanks)
    return fail(CO2_ERR_VALIDATION, "p2p: world must lie in [1, %d]", kMaxRanks);
  SliceArgs a{};
  for (int p = 0; p < world; ++p) {
    a.src[0][p] = src0[p];
    a.src[1][p] = nb > 1 ? src1[p] : nullptr;
    a.sig[p] = static_cast<Signals*>(sigs[p]);
  }
  a.dst[0] = dst0;
  a.dst[1] = dst1;
  a.nb = nb;
  a.lo = lo;
  a.len = len;
  a.world = world;
  a.rank = rank;
  a.epoch = epoch;
  // Entry barrier only (a flag per rank, not a CTA count), so CTAs need not
  // be co-resident and the grid may exceed one wave.
  // Default: at G = 2 one CTA per SM (the shard step is half the chip's
  // HBM work and competes with more), from G = 4 on 4 per SM (more remote
  // loads in flight win) -- C4 sweep in profiles/r01/bench/c4_ctas_sweep.txt.
  if (ctas < 1) ctas = (world <= 2 ? 1 : 4) * sm_count();
  if (ctas > 8 * sm_count()) ctas = 8 * sm_count();
  const int cap = rank_cap(world);
  const int nt = p2p_slice_threads();
#define CO2_SLICE_NT(TL, TC, V, R, U)                                                     \
  if (nt == 256)                                                                         \
    p2p_slice_average_kernel<TL, TC, V, R, U, 256><<<ctas, 256, 0, s>>>(a);              \
  else                                                                                   \
    p2p_slice_average_kernel<TL, TC, V, R, U, 512><<<ctas, 512, 0, s>>>(a);
#define CO2_SLICE_LAUNCH(TL, TC, V)                                                       \
  if (cap == 2) {                                                                        \
    CO2_SLICE_NT(TL, TC, V, 2, 4)                                                         \
  } else if (cap == 4) {                                                                 \
    CO2_SLICE_NT(TL, TC, V, 4, 2)                                                         \
  } else {                                                                               \
    CO2_SLICE_NT(TL, TC, V, 8, 1)                                                         \
  }
  switch (dt) {
    case CO2_DTYPE_F64: CO2_SLICE_LAUNCH(double, double, 2) break;
    case CO2_DTYPE_F32: CO2_SLICE_LAUNCH(float, float, 4) break;
    default: CO2_SLICE_LAUNCH(bf16raw, float, 8) break;
  }
#undef CO2_SLICE_LAUNCH
#undef CO2_SLICE_NT
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

co2_status_t p2p_average_launch(co2_dtype_t dt, void* const* bufs, void* const* sigs, int world,
                                int rank, int64_t n, uint32_t epoch, uint32_t* done_total,
                                int ctas, cudaStream_t s) {
  if (world < 1 || world > kMaxRanks)
    return fail(CO2_ERR_VALIDATION, "p2p: world must lie in [1, %d]", kMaxRanks);
  P2PArgs a{};
  for (int p = 0; p < world; ++p) {
    a.bufs[p] = bufs[p];
    a.sig[p] = static_cast<Signals*>(sigs[p]);
  }
  a.n = n;
  a.world = world;
  a.rank = rank;
  a.epoch = epoch;
  const int V = dt == CO2_DTYPE_F64 ? 2 : (dt == CO2_DTYPE_F32 ? 4 : 8);
  int64_t per = (n + world - 1) / world;
  per = (per + V - 1) / V * V;
  a.shard = per;
  if (ctas < 1) ctas = 1;
  if (ctas > sm_count()) ctas = sm_count();  // every CTA spins at the entry barrier
  *done_total += (uint32_t)world;  // one exit signal per rank per launch; wraps, compared wrap-safe
  a.done_target = *done_total;
  // R = rank capacity of the instantiation, U = vectors in flight per thread
  // (fewer ranks -> more vectors, keeping ~R*U*16 B of loads per thread).
  if (p2p_bulk() > 0) {
    // 4 KB per rank per tile, 4 stages; consumer warps from CO2_P2P_BULK
    const int ncw = p2p_bulk();
    switch (dt) {
      case CO2_DTYPE_F64:
        if (ncw >= 4) launch_p2p_bulk<double, double, 512, 4, 4>(a, ctas, s);
        else launch_p2p_bulk<double, double, 512, 4, 2>(a, ctas, s);
        break;
      case CO2_DTYPE_F32:
        if (ncw >= 4) launch_p2p_bulk<float, float, 1024, 4, 4>(a, ctas, s);
        else launch_p2p_bulk<float, float, 1024, 4, 2>(a, ctas, s);
        break;
      default:
        if (ncw >= 4) launch_p2p_bulk<bf16raw, float, 2048, 4, 4>(a, ctas, s);
        else launch_p2p_bulk<bf16raw, float, 2048, 4, 2>(a, ctas, s);
        break;
    }
    CO2_CUDA(cudaGetLastError());
    return CO2_OK;
  }
  const int cap = rank_cap(world);
  const int nt = p2p_threads();
#define CO2_P2P_NT(TL, TC, V, R, U)                                                      \
  if (nt == 128)                                                                        \
    p2p_average_kernel<TL, TC, V, R, U, 128><<<ctas, 128, 0, s>>>(a);                   \
  else if (nt == 256)                                                                   \
    p2p_average_kernel<TL, TC, V, R, U, 256><<<ctas, 256, 0, s>>>(a);                   \
  else                                                                                  \
    p2p_average_kernel<TL, TC, V, R, U, 512><<<ctas, 512, 0, s>>>(a);
#define CO2_P2P_LAUNCH(TL, TC, V)                                                        \
  if (cap == 2) {                                                                       \
    CO2_P2P_NT(TL, TC, V, 2, 4)                                                          \
  } else if (cap == 4) {                                                                \
    CO2_P2P_NT(TL, TC, V, 4, 2)                                                          \
  } else {                                                                              \
    CO2_P2P_NT(TL, TC, V, 8, 1)                                                          \
  }
  switch (dt) {
    case CO2_DTYPE_F64: CO2_P2P_LAUNCH(double, double, 2) break;
    case CO2_DTYPE_F32: CO2_P2P_LAUNCH(float, float, 4) break;
    default: CO2_P2P_LAUNCH(bf16raw, float, 8) break;
  }
#undef CO2_P2P_LAUNCH
#undef CO2_P2P_NT
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

namespace {
// One thread: the sharded step's exit barrier on its own, after an
// all-gather the copy engines did (cudaMemcpyAsync into the peers' params,
// ordered before this kernel on the stream).
__global__ void p2p_barrier_kernel(const P2PExit x) { p2p_exit_barrier(x); }
}  // namespace

co2_status_t p2p_barrier_launch(void* const* sigs, int world, int rank, uint32_t epoch,
                                cudaStream_t s) {
  if (world < 1 || world > kMaxRanks)
    return fail(CO2_ERR_VALIDATION, "p2p: world must lie in [1, %d]", kMaxRanks);
  P2PExit x{};
  for (int p = 0; p < world; ++p) x.sig[p] = static_cast<Signals*>(sigs[p]);
  x.world = world;
  x.rank = rank;
  x.epoch = epoch;
  x.counter = 0;  // done2, as the fused sharded step's exit barrier
  p2p_barrier_kernel<<<1, 1, 0, s>>>(x);
  CO2_CUDA(cudaGetLastError());
  return CO2_OK;
}

size_t p2p_signal_bytes() { return sizeof(Signals); }
size_t p2p_signal_timeout_offset() { return offsetof(Signals, timeout_ms); }
size_t p2p_signal_error_offset() { return offsetof(Signals, error); }

}  // namespace co2
