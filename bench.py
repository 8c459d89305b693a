#!/usr/bin/env python
"""CO2 outer-step benchmark (BASELINE.json metric: outer-step params/s,
% of the HBM roofline, exposed all-reduce %, at 1/2/4/8 B200).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
  torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)
  python bench.py --impl reference ...                   (reference CPU arm)

A step is one co2_round of the hot path on every rank (the reference's
co2_round, proj/src/outer_algorithms.cpp:110-211): launch the one-step-stale
all-reduce of x_{t,tau} (in-place NCCL sum on the engine's comm stream,
event-fenced), wait on the previous round's reduce, and run the fused
outer-step kernel over this rank's full parameter buffer.  Inputs are
synthetic, resident in HBM, and larger than L2 (126 MB), so
no L2 flush is needed between steps.  `value` is whole-job params/s
(N * n * K / max-over-ranks device time); `e2e` is the same metric through
the host-buffer C ABI entry (co2_outer_step_host: pinned H2D, kernel, D2H
inside the timed region).  The reference arm times the oracle's fp64
restatement of the reference's unfused per-worker body on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c3": {"workload": "C3: 1.3B-param bf16 params + fp32 anchor/outer momentum, one CO2 "
                       "worker per B200, tau=12 (BASELINE.json configs[2])",
           "mode": 2, "n": 1_300_000_000, "tau": 12, "bytes_per_param": 26,
           "storage": "bf16 params/x_{t-1,1}/xbar + fp32 x_{t,0}/x_{t-1,0}/momentum"},
    "c2": {"workload": "C2: 125M-param fp32 flat buffer, tau=12 (BASELINE.json configs[1])",
           "mode": 1, "n": 125_000_000, "tau": 12, "bytes_per_param": 32,
           "storage": "fp32"},
    "c4": {"workload": "C4: 7B-param bf16 params, ghost-consistent outer state (fp32 x_{t,0}, "
                       "prev_x0, momentum) sharded across the GPUs (BASELINE.json configs[3]); "
                       "needs >= 2 GPUs",
           "mode": 2, "n": 7_000_000_000, "tau": 12, "bytes_per_param": 30, "sharded": True,
           "storage": "bf16 params/x_{t,1} (replicated) + fp32 shard state"},
    "c1": {"workload": "C1: 1M-param fp32 flat vector, 4 simulated CO2 workers on one GPU, "
                       "tau=4 (BASELINE.json configs[0], the reference's CPU fixture scale)",
           "mode": 1, "n": 1 << 20, "tau": 4, "bytes_per_param": 32, "local_workers": 4,
           "storage": "fp32"},
    "c3f64": {"workload": "C3 in the reference's own precision: 1.3B-param fp64 params and state "
                          "(the F64 mode, bitwise the reference's fp64 outer step), one CO2 worker "
                          "per B200, tau=12 (secondary line; the headline C3 is bf16-mixed)",
              "mode": 0, "n": 1_300_000_000, "tau": 12, "bytes_per_param": 64,
              "storage": "fp64 everywhere", "e2e_default": False},
    "c4shard": {"workload": "C4 shard on one GPU: 7B/8 = 875M-param bf16-mixed shard, "
                            "worker-local step",
                "mode": 2, "n": 875_000_000, "tau": 12, "bytes_per_param": 26,
                "storage": "bf16 params + fp32 state"},
}
HYPER = dict(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ncu --set full captures of each config's dominant kernel (committed under
# profiles/r02/ncu/; each ran the same bench.py config, see its README).
NCU_CAPTURES = {
    "c3": os.path.join("profiles", "r02", "ncu", "c3_fused_step_raw.csv"),
    "c2": os.path.join("profiles", "r02", "ncu", "c2_fused_step_raw.csv"),
    "c1": os.path.join("profiles", "r02", "ncu", "c1_local_round_raw.csv"),
}
# NVLink denominator: B200_PROFILING.md's measured peer copy, GB/s per direction
NVLINK_PEER_GBS = 770.0


def ncu_traffic(cfg, n_gpus: int = 1):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed capture of this config's kernel (one GPU), else None."""
    path = NCU_CAPTURES.get(cfg.get("name", ""))
    if path is None or n_gpus != 1:
        return None, None
    try:
        import csv
        with open(os.path.join(ROOT, path)) as f:
            rows = list(csv.reader(f))
        hdr, units, vals = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(name)
            tot += float(vals[i]) * scale[units[i]]
        return tot, path
    except Exception:
        return None, None


class ClockSampler:
    """NVML sampling of SM clocks and clock-event reasons during the timed
    region (the recipe's clocks line)."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
             "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, torch, dev: int, period: float = 0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period, self._stop = period, threading.Event()
        try:
            self.nv, self.h = nvml_handle(torch, dev)
            nv = self.nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.NAMES.items():
                    if r & getattr(nv, attr):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def nvml_handle(torch, dev: int):
    """NVML handle of CUDA device `dev`, matched by PCI bus id (NVML and
    CUDA enumerate devices in different orders in general)."""
    import pynvml as nv
    nv.nvmlInit()
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        return nv, nv.nvmlDeviceGetHandleByPciBusId(bus)
    except Exception:
        return nv, nv.nvmlDeviceGetHandleByIndex(dev)


def bind_gpu_local_cpus(torch, dev: int):
    """Pins this rank to the CPU cores NVML reports as local to its GPU, so
    the pinned host buffers of the e2e leg are first-touched on the GPU's
    NUMA node and its copies do not cross the socket interconnect.
    CO2_BENCH_NUMA=0 disables it. Returns the core count, or None."""
    if os.environ.get("CO2_BENCH_NUMA", "1") == "0":
        return None
    try:
        nv, h = nvml_handle(torch, dev)
        nv.nvmlDeviceSetCpuAffinity(h)
        return len(os.sched_getaffinity(0))
    except Exception:
        return None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_info() -> dict:
    """nproc / affinity / CPU model / RAM of the host the CPU arms ran on."""
    info = {"nproc": os.cpu_count(), "affinity_cores": host_cores()}
    try:
        with open("/proc/cpuinfo") as f:
            info["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in f
                                      if ln.startswith("model name")), None)
        with open("/proc/meminfo") as f:
            kb = next(int(ln.split()[1]) for ln in f if ln.startswith("MemTotal"))
        info["mem_gb"] = round(kb / 1e6, 1)
    except Exception:
        pass
    return info


# ----------------------------------------------------------------- CPU arms
def cpu_sample_inputs(cfg, n_sample: int):
    """fp64 upcast of the same synthetic inputs (first n_sample coordinates)."""
    from oracle import oracle as O
    x, p0, p1, xe, m = O.synth(cfg["mode"], n_sample)
    return [O.to_f64(a) for a in (x, p0, p1, xe, m)]


def time_cpu_step(cfg, n_sample: int, threads: int, steps: int, warmup: int):
    """Times the oracle's fp64 restatement of co2_round's per-worker body
    (outer_algorithms.cpp:186-202, the reference's unfused passes and fresh
    temporaries) on n_sample coordinates."""
    from oracle import oracle as O
    x, p0, p1, xe, m = cpu_sample_inputs(cfg, n_sample)
    h = O.hyper(tau=cfg["tau"], **HYPER)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.worker_step_f64(x, p0, p1, xe, m, h, threads=threads, want_gap=False)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return n_sample / statistics.mean(times), statistics.mean(times)


def time_cpu_average(n_sample: int, workers: int = 4, reps: int = 3) -> dict:
    """The reference's CPU all-reduce arithmetic, average()
    (proj/src/param_ops.cpp:16-33), fp64 and single-threaded as the
    reference runs it, over `workers` contributions of n_sample."""
    from oracle import oracle as O
    cs = [O.to_f64(O.synth(2, n_sample, worker=w)[3]) for w in range(workers)]
    O.average(cs)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.average(cs)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return {"value": n_sample / t, "unit": "params/s", "workers": workers, "cores": 1,
            "sample": f"{n_sample} coordinates x {workers} fp64 contributions"}


def time_cpu_fused_bound(cfg, n_sample: int, threads: int, reps: int = 3) -> dict:
    """NOT the reference: the fused same-order step (oracle orc_outer_step,
    the GPU's storage types) on every host core over contiguous ranges -- a
    best-case CPU bound for the same work."""
    import concurrent.futures as cf
    from oracle import oracle as O
    mode = cfg["mode"]
    x, p0, p1, xe, m = O.synth(mode, n_sample)
    h = O.hyper(tau=cfg["tau"], **HYPER)
    bounds = [n_sample * i // threads for i in range(threads + 1)]

    def part(i):
        lo, hi = bounds[i], bounds[i + 1]
        O.outer_step(mode, x[lo:hi], p0[lo:hi], p1[lo:hi], xe[lo:hi], m[lo:hi], h)

    ts = []
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(part, range(threads)))
        for _ in range(reps):
            t0 = time.perf_counter()
            list(ex.map(part, range(threads)))
            ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return {"value": n_sample / t, "unit": "params/s", "cores": threads,
            "kind": "fused same-order C loop, storage dtypes of the config (not the reference)",
            "sample": f"{n_sample} coordinates"}


def run_reference_arm(args, cfg, rank: int):
    """The reference's CPU path on this host: the fp64 restatement of
    co2_round's per-worker body with the reference's unfused passes and fresh
    temporaries, on ONE thread -- the reference is single-threaded (Eigen
    cwise ops, no OpenMP or threads).
    The same passes split over every host core are reported separately as
    `cpu_parallel_bound` (not the reference)."""
    if rank != 0:
        return 0
    cores = host_cores()
    n_sample = args.ref_sample
    value, t = time_cpu_step(cfg, n_sample, 1, max(args.steps, 1), max(args.warmup, 0))
    pv, pt = time_cpu_step(cfg, n_sample, cores, 3, 1)
    line = {
        "impl": "reference", "metric": "CO2 outer-step params/s", "value": value,
        "unit": "params/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n_params_per_worker": cfg["n"],
                   "tau": cfg["tau"], "sample_params": n_sample},
        "cpu_baseline": {"value": value, "unit": "params/s", "cores": 1, "kind": "port",
                         "sample": f"{n_sample} coordinates of the {cfg['n']}-param workload, "
                                   "fp64 upcast, reference unfused passes and fresh "
                                   "temporaries, 1 thread (the reference is single-threaded)"},
        "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "Reference (C++20/Eigen) is not buildable here (Eigen absent); this arm times "
                "oracle/co2_oracle.c, a bit-exact restatement pinned by the reference's fixtures.",
        "cpu_aar": time_cpu_average(min(n_sample, 1 << 24)),
        "cpu_parallel_bound": {"value": pv, "unit": "params/s", "cores": cores,
                               "ms_per_step": pt * 1e3,
                               "kind": "NOT the reference: the same unfused fp64 passes split "
                                       f"over {cores} host threads (coordinate ranges)"},
        "cpu_fused_bound": time_cpu_fused_bound(cfg, n_sample, cores),
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU arm
def run_local_workers(args, cfg) -> int:
    """C1: G simulated workers on one GPU through the LOCAL engine.  Every
    co2_round (t >= 1) is ONE kernel (local_round_kernel): this round's
    fixed-order average of the G contributions plus the G fused outer steps
    on the previous average.

    One round's working set (142 MB) is about the L2 size (126 MB), so the
    timed rounds rotate over S = 4 independent simulated jobs (each G
    workers + its own LOCAL engine): consecutive rounds touch disjoint
    buffers, and a job's inputs were last touched S - 1 rounds (426 MB of
    traffic) earlier, so they stream from HBM -- the "inputs larger than L2"
    rule without a flush between rounds.  K rounds run back to back between
    one pair of CUDA events (whole-job throughput).  Two side passes, outside
    that region: the kernel duration on CUDA events around each launch (the
    roofline), and the older protocol (L2 flushed before every round, events
    around each round) for comparison."""
    import torch

    from paper_2401_16265_b200 import co2
    mode, n, tau, g = cfg["mode"], cfg["n"], cfg["tau"], cfg["local_workers"]
    hyper = co2.Co2Hyper(**HYPER)
    S = 4
    jobs = []
    for _ in range(S):
        eng = co2.CollectiveEngine(g, transport="local")
        ws = [co2.Worker(mode, n, co2.synth_params(mode, n, worker=i), keep_gap=False)
              for i in range(g)]
        for w in ws:
            w.snapshot_start()
            w.snapshot_first()
        co2.co2_round(ws, eng, hyper, tau)  # round 0
        jobs.append((eng, ws))
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        for eng, ws in jobs:
            co2.co2_round(ws, eng, hyper, tau, sync=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = []
    hc0 = [eng.handle_count() for eng, _ in jobs]  # one reduce handle per round
    with ClockSampler(torch, torch.cuda.current_device()) as clk:
        e0.record(stream)
        for k in range(args.steps):
            eng, ws = jobs[k % S]
            h0 = time.perf_counter()
            co2.co2_round(ws, eng, hyper, tau, sync=False)
            host.append(time.perf_counter() - h0)
        e1.record(stream)
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    hspan = list(zip(hc0, [eng.handle_count() for eng, _ in jobs]))
    # Side pass 1: the kernel's duration on CUDA events around each launch
    # (the worker's step-timing events, on the launching stream; they add a
    # timing record before and after every kernel, so this pass is not the
    # throughput pass above).
    for eng, ws in jobs:
        ws[0].enable_timing(args.steps + 8)
    for k in range(args.steps):
        eng, ws = jobs[k % S]
        co2.co2_round(ws, eng, hyper, tau, sync=False)
    torch.cuda.synchronize()
    kt = [x for eng, ws in jobs for x in ws[0].step_times()]
    k_mean = statistics.mean(kt) if kt else None
    # in-kernel span (CTA 0's start to the last CTA's end, %globaltimer) of
    # the throughput pass's rounds, from the engines' kernel-timed handles
    span = [eng.info(h)["comm"] for (eng, _), (a0, a1) in zip(jobs, hspan)
            for h in range(a0, a1)]
    # Side pass 2: the round-1 protocol -- L2 flushed (256 MB write, then a
    # 256 MB read, leaving clean lines) before every round, events around it.
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush_w, flush_r = flush[:256 << 20], flush[256 << 20:].view(torch.int32)
    eng, ws = jobs[0]
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 20))]
    for f0, f1 in fev:
        flush_w.zero_()
        flush_r.max()
        f0.record(stream)
        co2.co2_round(ws, eng, hyper, tau, sync=False)
        f1.record(stream)
    torch.cuda.synchronize()
    flushed_us = statistics.median(f0.elapsed_time(f1) * 1e3 for f0, f1 in fev)
    r = co2.L.RoundResult()
    arr = (co2.C.c_void_p * g)(*[w.handle.value for w in ws])
    co2.check(co2.lib().co2_round_finish(arr, g, stream.cuda_stream, co2.C.byref(r)))
    value = g * n * args.steps / t
    sb, lb = (8, 8) if mode == 0 else ((4, 4) if mode == 1 else (4, 2))
    # per coordinate and round: G steps (x_t0, p0, m state + p1 low read;
    # m, anchor state + params low written) + the consumed xbar once + the
    # launched average (G contributions read, one written)
    bytes_round = n * (g * (3 * sb + lb + 2 * sb + lb) + lb + g * lb + lb)
    peak, peak_kind = peaks()
    achieved = bytes_round / k_mean / 1e9 if k_mean else None
    line = {
        "metric": "CO2 outer-step params/s", "value": value, "unit": "params/s", "n_gpus": 1,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {0: "f64", 1: "f32", 2: "bf16-mixed"}[mode],
        "compute_dtype": "f64" if mode == 0 else "f32",
        "data": "synthetic (counter-SplitMix64 uniforms, SURVEY.md 8d)",
        "config": {"workload": cfg["workload"], "n_params_per_worker": n, "workers": g,
                   "tau": tau, "hyper": HYPER,
                   "l2": f"inputs larger than L2: rounds rotate over {S} independent simulated "
                         f"jobs, so each round's inputs were last touched {S - 1} rounds "
                         f"({(S - 1) * bytes_round / 1e6:.0f} MB of traffic) earlier; no flush",
                   "timing": "K rounds back to back between one pair of CUDA events",
                   "step": f"co2_round over {g} simulated workers: ONE kernel = fixed-order "
                           f"average of x_t,tau + {g} fused outer steps on the stale average"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None,
                     "traffic": ncu_traffic(cfg)[0], "traffic_source": ncu_traffic(cfg)[1],
                     "traffic_note": "ncu replays the kernel on cold caches: the round's "
                                     "writes mostly stay dirty in L2 and reach DRAM later",
                     "algorithmic_bytes": bytes_round, "peak_kind": peak_kind,
                     "kernel": "local_round_kernel", "kernel_ms": k_mean * 1e3 if k_mean else None,
                     "kernel_timing": "CUDA events around each launch on the launching stream "
                                      "(separate pass)",
                     "bytes_per_param": bytes_round / (g * n)},
        "kernel_span_us": 1e6 * statistics.median(span) if span else None,
        "l2_flushed_round_us": flushed_us,
        "e2e": None, "cpu_baseline": None,
        "gpu_launches": args.steps, "clocks": clk.summary(),
        "host_us_per_round": 1e6 * statistics.median(host),
        "diag": {"min_gap": r.min_gap, "max_outer_step": r.max_outer_step},
    }
    print(json.dumps(line), flush=True)
    for eng, ws in jobs:
        for w in ws:
            w.close()
        eng.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 26,
                    help="coordinates in the 1-core CPU baseline sample (~10 s of CPU work)")
    ap.add_argument("--ref-sample", type=int, default=1 << 24,
                    help="coordinates per reference-arm step (1 thread, ~0.6 s per step)")
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--schedule", default="split", choices=["split", "fused"],
                    help="P2P worker-local rounds: 'split' = reduce kernel on the comm stream "
                         "overlapping the step kernel; 'fused' = one kernel does both")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "p2p"],
                    help="collective transport at N > 1; auto = the measured faster one, "
                         "the fixed-order P2P kernels (worker-local and sharded C4)")
    ap.add_argument("--nparams", type=int, default=0, help="override the config's parameter count")
    ap.add_argument("--clip", default="coordinate", choices=["coordinate", "global"],
                    help="coordinate = the reference's clip (every headline number); global = "
                         "the global-norm clip EXTENSION (two passes, outside the parity "
                         "contract; worker-local split schedule only)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    cfg["name"] = args.config
    if args.nparams > 0:
        cfg["name"] = None  # no committed capture of that size
        cfg["n"] = args.nparams
        cfg["workload"] += f" [n overridden to {args.nparams}]"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank)
    if cfg.get("local_workers"):
        if world > 1:
            raise SystemExit("--config c1 runs simulated workers on one GPU")
        import torch
        torch.cuda.set_device(local)
        return run_local_workers(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2401_16265_b200 import co2

    torch.cuda.set_device(local)
    numa_cores = bind_gpu_local_cpus(torch, local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mode, n, tau, bpp = cfg["mode"], cfg["n"], cfg["tau"], cfg["bytes_per_param"]
    gclip = args.clip == "global"
    if gclip:
        if cfg.get("sharded") or args.schedule == "fused":
            raise SystemExit("--clip global: worker-local configs, split schedule only")
        # pass 1 reads x_t0, p0, p1, xbar, m and writes m'; pass 2 reads m', x_t0
        # and writes anchor, params
        bpp = {0: 80, 1: 40, 2: 34}[mode]
    hyper = co2.Co2Hyper(**HYPER)
    stream = torch.cuda.current_stream()

    # --- engine: NCCL unique id broadcast over torch.distributed (plumbing)
    if world > 1:
        obj = [co2.CollectiveEngine.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    else:
        uid = bytes(128)
    transport = args.transport
    if transport == "auto":
        transport = "p2p"
    if world == 1:
        transport = "nccl"  # one rank: no collective, the engine's reduce is a no-op
    transport_note = None
    eng = None
    if transport == "p2p":
        try:
            eng = co2.CollectiveEngine(world, transport="p2p", rank=rank, max_ctas=args.max_ctas)
        except Exception as exc:  # IPC unavailable: report it and use NCCL instead
            transport_note = f"p2p setup failed ({exc}); NCCL used"
            transport = "nccl"
        ok = torch.tensor([1 if eng is not None else 0], device="cuda")
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0 and eng is not None:
            eng.close()
            eng, transport = None, "nccl"
            transport_note = transport_note or "p2p setup failed on a peer; NCCL used"
    if eng is None:
        eng = co2.CollectiveEngine(world, transport="nccl", rank=rank, nccl_id=uid,
                                   max_ctas=args.max_ctas)

    # --- worker state resident in HBM, synthetic inputs
    from paper_2401_16265_b200 import _lib as L
    sharded = cfg.get("sharded", False)
    if sharded:
        hyper = co2.Co2Hyper(ghost_consistent=True, **HYPER)
        init = co2.synth_params(mode, n, worker=0)  # identical x_{0,0} on every worker
        w = co2.ShardedWorker(mode, n, eng, init, keep_gap=False)
        del init
        w.snapshot_start()
        w.snapshot_first()
        w.round(eng, hyper, tau)  # round 0: snapshots, launches the first reduce-scatter
        co2.check(co2.lib().co2_synth(mode, 7, rank, w.offset, w.length, None,
                                      w.buffer(L.BUF_PREV_X0).data_ptr(), None, None,
                                      w.buffer(L.BUF_MOMENTUM).data_ptr(), stream.cuda_stream))
        units = n  # every coordinate of the replicated params is updated per step

        def one_round():
            w.round(eng, hyper, tau, sync=False)
    else:
        init = co2.synth_params(mode, n, worker=rank)  # x_{0,tau}: the params the reduce sums
        w = co2.Worker(mode, n, init, keep_gap=False)
        del init
        if gclip:
            w.set_clip_mode("global")
        if transport == "p2p":
            eng.register_worker(w)
            if args.schedule == "fused":
                eng.set_fused(True)
        w.snapshot_start()
        w.snapshot_first()
        co2.co2_round([w], eng, hyper, tau)  # round 0: snapshots, launches the first reduce
        co2.check(co2.lib().co2_synth(mode, 7, rank, 0, n, w.buffer(L.BUF_ANCHOR).data_ptr(),
                                      w.buffer(L.BUF_PREV_X0).data_ptr(),
                                      w.buffer(L.BUF_PREV_X1).data_ptr(), None,
                                      w.buffer(L.BUF_MOMENTUM).data_ptr(), stream.cuda_stream))
        units = world * n  # one full replica per worker

        def one_round():
            co2.co2_round([w], eng, hyper, tau, sync=False)
    torch.cuda.synchronize()
    w.enable_timing(max(args.steps, 1) + max(args.warmup, 0) + 8)

    for _ in range(args.warmup):
        one_round()
    torch.cuda.synchronize()
    w.step_times()  # drop warm-up launches
    n_events_before = len(eng.events()) if world > 1 else 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_round = []
    with ClockSampler(torch, torch.cuda.current_device()) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            h0 = time.perf_counter()
            one_round()
            host_round.append(time.perf_counter() - h0)
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed = e0.elapsed_time(e1) * 1e-3
    # per-rank diagnostics: device time and the host's enqueue time per round
    per_rank = [elapsed, statistics.median(host_round), max(host_round)]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank)
    else:
        gathered = [per_rank]
    kt = w.step_times()
    r = co2.L.RoundResult()
    if sharded:
        r = w.round(eng, hyper, tau, sync=True)  # one checked round: diagnostics + flags
    else:
        arr = (co2.C.c_void_p * 1)(w.handle.value)
        co2.check(co2.lib().co2_round_finish(arr, 1, stream.cuda_stream, co2.C.byref(r)))

    # exposed communication (reference definition: 100 * sum(stall) / sum(waited comm))
    comm = None
    if world > 1:
        ev = eng.events()[n_events_before:]
        launches = {e["handle_id"]: e["t_sim"] for e in ev if e["event"] == "launch"}
        completes = {e["handle_id"]: e["t_sim"] for e in ev if e["event"] == "complete"}
        waits = [e for e in ev if e["event"] == "wait"]
        stall = sum(e["stall"] for e in waits)
        waited = sum(completes[e["handle_id"]] - launches[e["handle_id"]] for e in waits
                     if e["handle_id"] in launches and e["handle_id"] in completes)
        comm = {"exposed_pct": 100.0 * stall / waited if waited > 0 else 0.0,
                "stall_ms_per_step": 1e3 * stall / max(len(waits), 1),
                "allreduce_ms": 1e3 * waited / max(len(waits), 1),
                "stall_share_of_step_pct": 100.0 * stall / max(len(waits), 1) /
                (elapsed / args.steps) if elapsed > 0 else None,
                "allreduce_bytes": n * (2 if mode == 2 else 4 if mode == 1 else 8),
                "note": "no inner-loop compute in this step: the reduce overlaps only the "
                        "outer step itself (tau*t_comp = 0 worst case); see "
                        "tools/overlap_sweep.py for the tau sweep"}

    t_tensor = torch.tensor([elapsed, statistics.mean(kt) if kt else 0.0], device="cuda",
                            dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    t_max, k_max = t_tensor.tolist()
    value = units * args.steps / t_max
    peak, peak_kind = peaks()
    per_rank = w.length if sharded else n  # coordinates one fused launch processes
    achieved = bpp * per_rank / k_max / 1e9 if k_max else None
    # Whole-step bounds at N > 1. NVLink bytes into one
    # rank per round: the fixed-order all-reduce reads (G-1)/G of the replica
    # from peers and receives (G-1)/G of it back; the sharded round reads two
    # remote slices (x_{t,tau}, x_{t,1}) and receives the all-gather.
    link, step_hbm = None, None
    if world > 1:
        low_bytes = {0: 8, 1: 4, 2: 2}[mode] * n
        link_in = (3 if sharded else 2) * (world - 1) / world * low_bytes
        link_gbs = link_in / (t_max / args.steps) / 1e9
        link = {"bound": "nvlink", "bytes_in_per_rank": link_in, "achieved": link_gbs,
                "peak": NVLINK_PEER_GBS, "unit": "GB/s", "frac": link_gbs / NVLINK_PEER_GBS,
                "peak_kind": "measured peer copy per direction (B200_PROFILING.md)"}
        if not sharded:
            # the all-reduce reads and writes the replica once in HBM beside the step
            bpp_step = bpp + 2 * low_bytes / n
            hbm_gbs = bpp_step * n / (t_max / args.steps) / 1e9
            step_hbm = {"bytes_per_param": bpp_step, "achieved": hbm_gbs, "peak": peak,
                        "unit": "GB/s", "frac": hbm_gbs / peak}

    # --- e2e through the host-facing entries (pinned H2D + round + D2H timed)
    e2e = e2e_full = None
    if not args.no_e2e and cfg.get("e2e_default", True) and not sharded and not gclip:  # the host entry is the reference clip
        e2e = run_e2e_round(co2, torch, w, eng, mode, n, tau, hyper, args, world, rank, dist)
        e2e["numa_bound_cores"] = numa_cores  # None: not bound (CO2_BENCH_NUMA=0 / no NVML)
        e2e_full = run_e2e(co2, torch, mode, n, tau, hyper, args, world, rank, dist)

    # --- CPU baseline (rank 0, N=1 only): single-core reference restatement
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        v, t = time_cpu_step(cfg, args.cpu_sample, 1, 3, 1)
        cpu = {"value": v, "unit": "params/s", "cores": 1, "kind": "port", "host": host_info(),
               "sample": f"{args.cpu_sample} coordinates of the same synthetic inputs (fp64 "
                         "upcast), reference unfused passes + fresh temporaries, 1 thread, "
                         f"{t:.2f} s per step"}

    if rank == 0:
        line = {
            "metric": "CO2 outer-step params/s", "value": value, "unit": "params/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": {0: "f64", 1: "f32", 2: "bf16-mixed"}[mode],
            "compute_dtype": "f64" if mode == 0 else "f32",
            "data": "synthetic (counter-SplitMix64 uniforms, SURVEY.md 8d)",
            "config": {"workload": cfg["workload"],
                       "n_params_per_gpu": per_rank, "n_params_total": units, "tau": tau,
                       "storage": cfg["storage"], "hyper": HYPER,
                       "parallelism": (f"dp{world} ghost-consistent, outer state sharded ("
                                       + ("async fixed-order P2P slice averages + fused "
                                          "NVLink all-gather)" if transport == "p2p" else
                                          "NCCL reduce-scatter + all-gather)")) if sharded else
                       (f"dp{world} (one CO2 worker per GPU, "
                        + ("fixed-order NVLink P2P all-reduce)" if transport == "p2p"
                           else "NCCL all-reduce)")),
                       "transport": transport, "transport_note": transport_note,
                       "clip": args.clip + (" (extension, outside the parity contract)"
                                            if gclip else " (reference)"),
                       "schedule": (args.schedule if transport == "p2p" and not sharded
                                    else "split"),
                       "l2": "inputs larger than L2 (no flush needed)",
                       "step": (("sharded co2_round: async P2P slice average of x_{t,tau} and "
                                 "x_{t,1} + stale wait + ONE kernel: ghost step on the shard "
                                 "storing x_{t+1,0} into every rank's params over NVLink")
                                if transport == "p2p" else
                                ("sharded co2_round: RS(x_{t,1}) + async RS(x_{t,tau}) + stale "
                                 "wait + fused ghost step on the shard + AG(x_{t+1,0})"))
                       if sharded else "co2_round: AAR launch + stale wait + fused outer step"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "traffic": None if gclip else ncu_traffic(cfg, world)[0],
                         "traffic_unit": "bytes per launch",
                         "traffic_source": None if gclip else ncu_traffic(cfg, world)[1],
                         "algorithmic_bytes": bpp * per_rank, "peak_kind": peak_kind,
                         "kernel": ("gclip_pass1 + gclip_pass2 (global-norm clip extension)"
                                    if gclip else
                                    ("fused_step_kernel<ModeBF16%s>" % (", GHOST" if sharded
                                                                         else ""))
                                    if mode == 2 else "fused_step_kernel"),
                         "kernel_ms": k_max * 1e3,
                         "bytes_per_param": bpp},
            "link": link, "step_hbm": step_hbm,
            "e2e": e2e, "e2e_full_state": e2e_full, "cpu_baseline": cpu, "comm": comm,
            "ranks": {"elapsed_ms_per_step": [1e3 * g[0] / args.steps for g in gathered],
                      "host_enqueue_ms_per_round_median": [1e3 * g[1] for g in gathered],
                      "host_enqueue_ms_per_round_max": [1e3 * g[2] for g in gathered]},
            # our kernels per step per rank: the fused step (two passes for the
            # global-norm clip) and its diagnostics readback; the P2P reduce
            # (or slice reduce) and its error-word readback when it runs as its
            # own launch; the fixed-order NCCL all-reduce's ascending-rank sum
            # kernel and its diagnostics readback (one more sum kernel for the
            # sharded round's blocking x_{t,1} reduce-scatter).  NCCL's own
            # kernels are not ours.
            "gpu_launches": world * args.steps * (
                (2 if gclip else 1) + 1 +
                (2 if world > 1 and transport == "p2p" and
                 (sharded or args.schedule == "split") else 0) +
                ((3 if sharded else 2) if world > 1 and transport == "nccl" else 0)),
            "clocks": clk.summary(),
            "diag": {"min_gap": r.min_gap, "max_outer_step": r.max_outer_step,
                     "n_clipped": r.n_clipped, "n_floored": r.n_floored},
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e_round(co2, torch, w, eng, mode, n, tau, hyper, args, world, rank, dist):
    """The metric through co2_round_host, the drop-in for the reference's
    co2_round with the inner loop on the host: every step uploads this
    step's inputs -- the inner loop's trace x_{t,1} and x_{t,tau} -- from
    pinned host memory, runs the round on the device-resident outer state
    (reduce launch, stale wait, fused step) and reads its result -- the next
    inner loop's start x_{t+1,0} -- back to pinned host memory."""
    lo = co2.LOW_TORCH[mode]
    h_first = co2.synth_params(mode, n, worker=rank).cpu().pin_memory()
    h_end = co2.synth_params(mode, n, worker=rank + 64).cpu().pin_memory()
    h_next = torch.empty(n, dtype=lo, pin_memory=True)
    torch.cuda.synchronize()
    times = []
    for i in range(args.e2e_steps + 1):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        co2.co2_round_host([w], eng, hyper, tau, [h_end], [h_next], x_first=[h_first],
                           sync=False)
        torch.cuda.current_stream().synchronize()  # the result is on the host
        dt = time.perf_counter() - t0
        if i > 0:
            times.append(dt)
    # the same copies with no round: two uploads, then the download (the
    # round's data dependence orders them the same way)
    d = [torch.empty(n, dtype=lo, device="cuda") for _ in range(2)]
    copy_times = []
    for i in range(4):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d[0].copy_(h_first, non_blocking=True)
        d[1].copy_(h_end, non_blocking=True)
        h_next.copy_(d[1], non_blocking=True)
        torch.cuda.synchronize()
        if i > 0:
            copy_times.append(time.perf_counter() - t0)
    del d
    torch.cuda.empty_cache()
    t = torch.tensor([statistics.mean(times), statistics.mean(copy_times)], dtype=torch.float64,
                     device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_e2e, t_copy = t.tolist()
    lb = 8 if mode == 0 else (4 if mode == 1 else 2)
    return {"value": world * n / t_e2e, "unit": "params/s",
            "h2d_bytes_per_step": 2 * n * lb, "d2h_bytes_per_step": n * lb,
            "ms_per_step": 1e3 * t_e2e,
            "pcie_copy_only_ms": 1e3 * t_copy, "pcie_frac": t_copy / t_e2e,
            "api": "co2_round_host (the reference's co2_round with the inner loop on the host: "
                   "x_{t,1}, x_{t,tau} uploaded, x_{t+1,0} downloaded, outer state resident)"}


def run_e2e(co2, torch, mode, n, tau, hyper, args, world, rank, dist):
    """The outer step alone through co2_outer_step_host, with the WHOLE
    outer state host-resident: every step copies x_t0, p0, p1, xbar and m
    host->device from pinned memory and reads m, the anchor and the params
    back (reported as e2e_full_state)."""
    st = co2.STATE_TORCH[mode]
    lo = co2.LOW_TORCH[mode]
    x, p0, p1, xe, m = co2.synth(mode, n, worker=rank)
    hx = torch.empty(n, dtype=st, pin_memory=True)
    hp0 = torch.empty(n, dtype=st, pin_memory=True)
    hm = torch.empty(n, dtype=st, pin_memory=True)
    hp1 = torch.empty(n, dtype=lo, pin_memory=True)
    hxe = torch.empty(n, dtype=lo, pin_memory=True)
    hparams = torch.empty(n, dtype=lo, pin_memory=True)
    for h, d in ((hx, x), (hp0, p0), (hm, m), (hp1, p1), (hxe, xe)):
        h.copy_(d)
    del x, p0, p1, xe, m
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    times = []
    for i in range(args.e2e_steps + 1):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        # anchor_out aliases prev_x0 (the rotation layout), momentum in place
        co2.outer_step_host(mode, hx, hp0, hp1, hxe, hm, hyper, tau, anchor_out=hp0,
                            params_out=hparams, chunk=1 << 25, nstreams=3)
        dt = time.perf_counter() - t0
        if i > 0:
            times.append(dt)
    # PCIe ceiling: the same bytes copied with no kernel, H2D and D2H on two
    # streams at once (what the pipeline overlaps), into separate scratch.
    ins = (hx, hp0, hm, hp1, hxe)
    outs = (hm, hp0, hparams)  # momentum, anchor, params come back
    d_in = [torch.empty_like(h, device="cuda") for h in ins]
    d_out = [torch.empty_like(h, device="cuda") for h in outs]
    h_out = [torch.empty(h.shape, dtype=h.dtype, pin_memory=True) for h in outs]
    sa, sb_ = torch.cuda.Stream(), torch.cuda.Stream()
    copy_times = []
    for i in range(4):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(sa):
            for d, h in zip(d_in, ins):
                d.copy_(h, non_blocking=True)
        with torch.cuda.stream(sb_):
            for h, d in zip(h_out, d_out):
                h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        if i > 0:
            copy_times.append(time.perf_counter() - t0)
    del d_in, d_out, h_out
    torch.cuda.empty_cache()
    t = torch.tensor([statistics.mean(times), statistics.mean(copy_times)], dtype=torch.float64,
                     device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_e2e, t_copy = t.tolist()
    sb = 8 if mode == 0 else 4
    lb = 8 if mode == 0 else (4 if mode == 1 else 2)
    return {"value": world * n / t_e2e, "unit": "params/s",
            "h2d_bytes_per_step": n * (3 * sb + 2 * lb), "d2h_bytes_per_step": n * (2 * sb + lb),
            "ms_per_step": 1e3 * t_e2e,
            "pcie_copy_only_ms": 1e3 * t_copy, "pcie_frac": t_copy / t_e2e,
            "api": "co2_outer_step_host (pinned host buffers, 3 streams, 32M-coordinate chunks)"}


if __name__ == "__main__":
    sys.exit(main())
