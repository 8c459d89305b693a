// Cross-GPU flag primitives for kernels that exchange data over NVLink peer
// memory (CUDA IPC mappings).  Every spin is bounded so a missing peer turns
// into a recorded error instead of a hung GPU.
#pragma once

#include <stdint.h>

namespace co2 {

constexpr int kMaxRanks = 8;

// Per-rank signal area (256 B, IPC-exported):
//   ready[r]  written by rank r at the start of a slice-reduce launch
//   done      counts finished all-reduce CTAs (fixed-order P2P average)
//   error     1/2/3/4/5: a bounded spin timed out
//   done2     counts ranks that finished the fused sharded step's stores
//   ready2[r] / done3: entry / exit of the fused all-reduce + outer step
//   timeout_ms  the spin budget of this rank's barriers (0 = 10 s); set by
//               the host from CO2_P2P_TIMEOUT_MS when the engine is created
//   ticket_local  used by this rank only: counts its CTAs finishing an
//               all-reduce so the last one alone signals the peers
struct Signals {
  uint32_t ready[kMaxRanks];
  uint32_t done;
  uint32_t error;
  uint32_t done2;
  uint32_t ready2[kMaxRanks];
  uint32_t done3;
  uint32_t timeout_ms;
  uint32_t ticket_local;  // this rank's CTAs finishing an all-reduce (local, self-reset)
  uint32_t pad[42];
};
static_assert(sizeof(Signals) == 256, "signal area layout");

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wall-clock bounded (globaltimer, independent of the SM clock): the
// budget is the owning rank's timeout_ms (default 10 s).
__device__ inline bool spin_until(const uint32_t* p, uint32_t target, const Signals* mine) {
  const uint32_t ms = *reinterpret_cast<const volatile uint32_t*>(&mine->timeout_ms);
  const uint64_t budget = (uint64_t)(ms ? ms : 10000u) * 1000000ull;
  const uint64_t t0 = global_ns();
  // wrap-safe: counters and epochs are uint32 sequences that may wrap
  while ((int32_t)(ld_acquire_sys(p) - target) < 0) {
    if (global_ns() - t0 > budget) return false;
    __nanosleep(64);
  }
  return true;
}

// Exit barrier of the fused sharded step: the kernel's last CTA (after every
// CTA fenced its peer stores at system scope) tells every rank it is done
// and waits until all ranks told it.
struct P2PExit {
  Signals* sig[kMaxRanks];  // rank-indexed signal areas
  int world, rank;
  uint32_t epoch;           // 1, 2, ... per fused launch, same on every rank
  int counter;              // 0: done2 (sharded step), 1: done3 (fused all-reduce step)
};

__device__ inline void p2p_exit_barrier(const P2PExit& x) {
  __threadfence_system();
  for (int p = 0; p < x.world; ++p)
    red_release_sys_add(x.counter ? &x.sig[p]->done3 : &x.sig[p]->done2, 1u);
  const uint32_t* mine = x.counter ? &x.sig[x.rank]->done3 : &x.sig[x.rank]->done2;
  if (!spin_until(mine, x.epoch * (uint32_t)x.world, x.sig[x.rank]))
    x.sig[x.rank]->error = x.counter ? 5 : 3;
}

// Entry barrier of the fused all-reduce + outer step: every CTA publishes
// this rank's arrival and waits for all ranks (their x_{t,tau} is final).
__device__ inline bool p2p_entry_barrier(const P2PExit& x) {
  for (int p = 0; p < x.world; ++p) st_release_sys(&x.sig[p]->ready2[x.rank], x.epoch);
  for (int p = 0; p < x.world; ++p)
    if (!spin_until(&x.sig[x.rank]->ready2[p], x.epoch, x.sig[x.rank])) {
      x.sig[x.rank]->error = 4;
      return false;
    }
  return true;
}

}  // namespace co2
