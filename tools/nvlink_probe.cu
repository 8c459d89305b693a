// NVLink peer-bandwidth probe for this pool's B200 boxes (one process, every
// visible GPU, cudaDeviceEnablePeerAccess).  It measures the denominators the
// multi-GPU bench lines need instead of taking a figure from a guide:
//
//   ce_uni      copy engines, GPU0 -> GPU1 (cudaMemcpyPeerAsync)
//   ce_bidir    copy engines, GPU0 <-> GPU1 at once (per-direction GB/s)
//   sm_load     GPU0 kernel: 16-byte loads from GPU1's memory, stores local
//   sm_store    GPU0 kernel: local loads, 16-byte stores into GPU1's memory
//   sm_*_bidir  the same kernel on both GPUs at once, each toward the other
//   sm_load_all2all  (>= 3 GPUs) every GPU loads a share from every peer
//   step_mix    a step-like stream on every GPU: 64 B of local HBM traffic
//               per 16-byte unit plus 1/16 of that stored to each peer (the
//               sharded step's fused all-gather), vs the local part alone
//
// Build: make nvlink_probe   Run: build/nvlink_probe [GB per buffer, default 4]
// Prints one JSON line per measurement.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,                 \
              cudaGetErrorString(e_));                                          \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void copy16(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    __stcg(dst + i, __ldcg(src + i));
}

// Step-like mix: per 16-byte unit, 3 local loads and 1 local store (64 B of
// HBM traffic), and every 4th unit also stored to each of `peers` peers
// (remote bytes = 1/16 of the local ones, the sharded step's ratio:
// 2 B/param per peer beside ~30 B/param local).
__global__ void step_mix(const uint4* __restrict__ a, const uint4* __restrict__ b,
                         const uint4* __restrict__ c, uint4* __restrict__ o,
                         uint4* const* __restrict__ remote, int peers, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = __ldcs(a + i), y = __ldcs(b + i), z = __ldcs(c + i);
    uint4 r;
    r.x = x.x ^ y.x ^ z.x;
    r.y = x.y ^ y.y ^ z.y;
    r.z = x.z ^ y.z ^ z.z;
    r.w = x.w ^ y.w ^ z.w;
    __stcs(o + i, r);
    if ((i & 3) == 0)  // 16 B per 4 units: 1/16 of the local traffic, as the sharded step
      for (int p = 0; p < peers; ++p) __stcs(remote[p] + (i >> 2), r);
  }
}

// The same stream pulling its remote share with loads instead of pushing
// it with stores (what a pull-based all-gather would do).
__global__ void step_mix_pull(const uint4* __restrict__ a, const uint4* __restrict__ b,
                              const uint4* __restrict__ c, uint4* __restrict__ o,
                              const uint4* const* __restrict__ remote, int peers, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint4 x = __ldcs(a + i), y = __ldcs(b + i), z = __ldcs(c + i);
    uint4 r;
    r.x = x.x ^ y.x ^ z.x;
    r.y = x.y ^ y.y ^ z.y;
    r.z = x.z ^ y.z ^ z.z;
    r.w = x.w ^ y.w ^ z.w;
    if ((i & 3) == 0)
      for (int p = 0; p < peers; ++p) {
        const uint4 q = __ldcg(remote[p] + (i >> 2));
        r.x ^= q.x;
        r.y ^= q.y;
        r.z ^= q.z;
        r.w ^= q.w;
      }
    __stcs(o + i, r);
  }
}

struct Dev {
  int id;
  cudaStream_t s;
  cudaEvent_t e0, e1;
};

static double now_ms(Dev& d) {
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, d.e0, d.e1));
  return ms;
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 4.0;
  const size_t bytes = (size_t)(gb * 1e9) / 16 * 16;
  const size_t n16 = bytes / 16;
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) {
    printf("{\"probe\": \"nvlink\", \"error\": \"needs >= 2 GPUs\"}\n");
    return 0;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<Dev> dv(ng);
  std::vector<char*> src(ng), dst(ng), c3(ng), recv(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    dv[g].id = g;
    CK(cudaStreamCreateWithFlags(&dv[g].s, cudaStreamNonBlocking));
    CK(cudaEventCreate(&dv[g].e0));
    CK(cudaEventCreate(&dv[g].e1));
    for (int p = 0; p < ng; ++p)
      if (p != g) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, g, p));
        if (ok) cudaDeviceEnablePeerAccess(p, 0);
        cudaGetLastError();
      }
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&dst[g], bytes));
    CK(cudaMalloc(&c3[g], bytes));
    CK(cudaMalloc(&recv[g], bytes));  // remote stores land here (one region per peer slot)
    CK(cudaMemset(src[g], 1, bytes));
    CK(cudaMemset(dst[g], 0, bytes));
    CK(cudaMemset(c3[g], 2, bytes));
  }
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  const int grid = sms * 4, nt = 256;
  auto run = [&](const char* name, std::vector<int> gpus, auto body, double bytes_per_gpu,
                 int reps = 5) {
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
      for (int g : gpus) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g : gpus) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(dv[g].e0, dv[g].s));
      }
      for (int g : gpus) {
        CK(cudaSetDevice(g));
        body(g);
      }
      for (int g : gpus) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(dv[g].e1, dv[g].s));
      }
      double worst = 0;
      for (int g : gpus) {
        CK(cudaEventSynchronize(dv[g].e1));
        double ms = now_ms(dv[g]);
        worst = ms > worst ? ms : worst;
      }
      best = worst < best ? worst : best;
    }
    printf("{\"probe\": \"%s\", \"gpus\": %d, \"bytes_per_gpu\": %.0f, \"ms\": %.4f, "
           "\"GBps_per_gpu\": %.1f}\n",
           name, (int)gpus.size(), bytes_per_gpu, best, bytes_per_gpu / best / 1e6);
    fflush(stdout);
  };
  // copy engines
  run("ce_uni", {0}, [&](int g) { CK(cudaMemcpyPeerAsync(dst[1], 1, src[0], 0, bytes, dv[g].s)); },
      (double)bytes);
  run("ce_bidir", {0, 1},
      [&](int g) { CK(cudaMemcpyPeerAsync(dst[1 - g], 1 - g, src[g], g, bytes, dv[g].s)); },
      (double)bytes);
  // SM-driven
  run("sm_load", {0}, [&](int g) {
        copy16<<<grid, nt, 0, dv[g].s>>>((const uint4*)src[1], (uint4*)dst[0], n16);
      },
      (double)bytes);
  run("sm_store", {0}, [&](int g) {
        copy16<<<grid, nt, 0, dv[g].s>>>((const uint4*)src[0], (uint4*)dst[1], n16);
      },
      (double)bytes);
  run("sm_load_bidir", {0, 1}, [&](int g) {
        copy16<<<grid, nt, 0, dv[g].s>>>((const uint4*)src[1 - g], (uint4*)dst[g], n16);
      },
      (double)bytes);
  run("sm_store_bidir", {0, 1}, [&](int g) {
        copy16<<<grid, nt, 0, dv[g].s>>>((const uint4*)src[g], (uint4*)dst[1 - g], n16);
      },
      (double)bytes);
  if (ng >= 3) {
    // every GPU loads a 1/(ng-1) share from each peer at once (all-to-all in)
    std::vector<int> all;
    for (int g = 0; g < ng; ++g) all.push_back(g);
    const size_t share = n16 / (ng - 1);
    run("sm_load_all2all", all, [&](int g) {
          int k = 0;
          for (int p = 0; p < ng; ++p)
            if (p != g) {
              copy16<<<grid / (ng - 1), nt, 0, dv[g].s>>>((const uint4*)src[p] + k * share,
                                                           (uint4*)dst[g] + k * share, share);
              ++k;
            }
        },
        (double)share * 16 * (ng - 1));
  }
  // step-like local streaming alone, then with the fused all-gather stores
  // to every peer (each GPU's recv buffer holds the peers' slots)
  std::vector<std::vector<uint4*>> rem(ng);
  std::vector<uint4**> rem_d(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < ng; ++p)
      if (p != g) rem[g].push_back((uint4*)recv[p] + (size_t)g * (n16 / ng / 4 + 1));
    CK(cudaMalloc(&rem_d[g], sizeof(uint4*) * 8));
    CK(cudaMemcpy(rem_d[g], rem[g].data(), sizeof(uint4*) * rem[g].size(),
                  cudaMemcpyHostToDevice));
  }
  std::vector<int> all;
  for (int g = 0; g < ng; ++g) all.push_back(g);
  const size_t nmix = n16 / ng;  // keep the remote slots inside recv
  run("step_mix_local", all, [&](int g) {
        step_mix<<<grid * 8, nt, 0, dv[g].s>>>((const uint4*)src[g], (const uint4*)c3[g],
                                              (const uint4*)dst[g], (uint4*)dst[g], rem_d[g], 0,
                                              nmix);
      },
      (double)nmix * 16 * 4);
  run("step_mix_allgather", all, [&](int g) {
        step_mix<<<grid * 8, nt, 0, dv[g].s>>>((const uint4*)src[g], (const uint4*)c3[g],
                                              (const uint4*)dst[g], (uint4*)dst[g], rem_d[g],
                                              ng - 1, nmix);
      },
      (double)nmix * 16 * 4);
  run("step_mix_pull", all, [&](int g) {
        step_mix_pull<<<grid * 8, nt, 0, dv[g].s>>>((const uint4*)src[g], (const uint4*)c3[g],
                                                   (const uint4*)dst[g], (uint4*)dst[g],
                                                   (const uint4* const*)rem_d[g], ng - 1, nmix);
      },
      (double)nmix * 16 * 4);
  printf("{\"probe\": \"step_mix_note\", \"remote_bytes_per_gpu_out\": %.0f}\n",
         (double)nmix * 4 * (ng - 1));
  return 0;
}
