"""Where the C1 round's time goes between the bracketing CUDA events and the
local_round_kernel itself (bench.py --config c1 reports both):

  python tools/c1_gap.py

Variants (one JSON line each; medians over --steps rounds):
  flush      the bench loop: L2 flush, e0, co2_round, e1
  noflush    rounds back to back, e0 / e1 around each
  events     L2 flush, e0, the round's event records and stream wait with no
             kernel, e1 (the GPU-side cost of the bookkeeping alone)
  torchevents L2 flush, e0, e1 (nothing between)
  timing4    L2 flush, e0, four timing event records, e1
  notiming4  L2 flush, e0, four cudaEventDisableTiming records, e1
  wait4      L2 flush, e0, one non-timing record and four stream waits on it, e1
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--workers", type=int, default=4)
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2
    mode, n, g, tau = 1, a.n, a.workers, 4
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    eng = co2.CollectiveEngine(g, transport="local")
    ws = [co2.Worker(mode, n, co2.synth_params(mode, n, worker=i), keep_gap=False)
          for i in range(g)]
    for w in ws:
        w.snapshot_start()
        w.snapshot_first()
    co2.co2_round(ws, eng, hyper, tau)
    for _ in range(5):
        co2.co2_round(ws, eng, hyper, tau, sync=False)
    ws[0].enable_timing(4 * a.steps + 8)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush_w, flush_r = flush[:256 << 20], flush[256 << 20:].view(torch.int32)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    done = torch.cuda.Event()
    nts = [torch.cuda.Event() for _ in range(8)]

    def run(kind):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(a.steps)]
        host = []
        ws[0].step_times()  # drain: step_times returns launches since the last call
        for e0, e1 in ev:
            if kind != "noflush":
                flush_w.zero_()
                flush_r.max()
            e0.record(stream)
            h0 = time.perf_counter()
            if kind in ("flush", "noflush"):
                co2.co2_round(ws, eng, hyper, tau, sync=False)
            elif kind == "events":
                for k in range(3):
                    evs[k].record(stream)
                done.record(stream)
                stream.wait_event(done)
                for k in range(3, 6):
                    evs[k].record(stream)
            elif kind == "timing4":
                for k in range(4):
                    evs[k].record(stream)
            elif kind == "notiming4":
                for k in range(4):
                    nts[k].record(stream)
            elif kind == "wait4":
                done.record(stream)
                for k in range(4):
                    stream.wait_event(done)
            host.append(time.perf_counter() - h0)
            e1.record(stream)
        torch.cuda.synchronize()
        t = [e0.elapsed_time(e1) * 1e3 for e0, e1 in ev]
        kt = ws[0].step_times()
        return {"variant": kind, "event_us_median": statistics.median(t),
                "event_us_min": min(t),
                "kernel_us_median": statistics.median(kt) * 1e6 if kt else None,
                "host_us_median": statistics.median(host) * 1e6}

    for kind in ("flush", "noflush", "events", "torchevents", "timing4", "notiming4", "wait4",
                 "flush"):
        print(json.dumps(run(kind)), flush=True)


if __name__ == "__main__":
    main()
