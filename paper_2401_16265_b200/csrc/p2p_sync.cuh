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
//   error     1/2/3: a bounded spin timed out
//   done2     counts ranks that finished the fused sharded step's stores
struct Signals {
  uint32_t ready[kMaxRanks];
  uint32_t done;
  uint32_t error;
  uint32_t done2;
  uint32_t pad[53];
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
};

__device__ inline void p2p_exit_barrier(const P2PExit& x) {
  __threadfence_system();
  for (int p = 0; p < x.world; ++p) red_release_sys_add(&x.sig[p]->done2, 1u);
  if (!spin_until(&x.sig[x.rank]->done2, x.epoch * (uint32_t)x.world))
    x.sig[x.rank]->error = 3;
}

}  // namespace co2
