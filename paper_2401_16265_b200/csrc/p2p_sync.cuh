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
struct Signals {
  uint32_t ready[kMaxRanks];
  uint32_t done;
  uint32_t error;
  uint32_t done2;
  uint32_t ready2[kMaxRanks];
  uint32_t done3;
  uint32_t pad[44];
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

// ~2 s at 1.9 GHz.
constexpr long long kSpinBudget = 4000000000LL;

__device__ inline bool spin_until(const uint32_t* p, uint32_t target) {
  long long t0 = clock64();
  while (ld_acquire_sys(p) < target) {
    if (clock64() - t0 > kSpinBudget) return false;
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
  if (!spin_until(mine, x.epoch * (uint32_t)x.world)) x.sig[x.rank]->error = x.counter ? 5 : 3;
}

// Entry barrier of the fused all-reduce + outer step: every CTA publishes
// this rank's arrival and waits for all ranks (their x_{t,tau} is final).
__device__ inline bool p2p_entry_barrier(const P2PExit& x) {
  for (int p = 0; p < x.world; ++p) st_release_sys(&x.sig[p]->ready2[x.rank], x.epoch);
  for (int p = 0; p < x.world; ++p)
    if (!spin_until(&x.sig[x.rank]->ready2[p], x.epoch)) {
      x.sig[x.rank]->error = 4;
      return false;
    }
  return true;
}

}  // namespace co2
