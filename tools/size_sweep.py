"""Fused-step time against buffer size, beside a torch copy of the same byte
count, to split a launch's time into a fixed cost and a per-byte rate:

  python tools/size_sweep.py [--mode 1] [--sizes 31250000,62500000,125000000,250000000,500000000]
                             [--iters 30] [--reps 3]

Every (size) point times K back-to-back fused steps (CUDA events per launch,
median per rep) and K back-to-back copies of bytes_per_param*n/2 bytes read
+ written (so both move the same traffic).  Reps are interleaved across the
sizes so slow drifts (clocks, power) cancel.  One JSON line per size.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BPP = {0: 64, 1: 32, 2: 26}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--sizes", default="31250000,62500000,125000000,250000000,500000000")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--inplace", type=int, default=1,
                    help="1: anchor/params written over p0/xbar (the bench's rotation "
                         "reuses two buffer sets; here one)")
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2

    mode = a.mode
    sizes = [int(s) for s in a.sizes.split(",")]
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    ws = co2.Workspace()
    bufs = {}
    for n in sizes:
        bufs[n] = co2.synth(mode, n)
        nb = BPP[mode] * n // 2
        src = torch.empty(nb, dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        bufs[n] = (bufs[n], src, dst)
    res = {n: {"step": [], "copy": []} for n in sizes}

    def step(n):
        (x, p0, p1, xe, m), _, _ = bufs[n]
        co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                       workspace=ws, check_flags=False)

    def copy(n):
        _, src, dst = bufs[n]
        dst.copy_(src)

    for rep in range(a.reps):
        for n in sizes:
            for kind, fn in (("step", step), ("copy", copy)):
                for _ in range(3):
                    fn(n)
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(a.iters)]
                for e0, e1 in evs:
                    e0.record()
                    fn(n)
                    e1.record()
                torch.cuda.synchronize()
                res[n][kind].append(statistics.median(e0.elapsed_time(e1) for e0, e1 in evs))
    for n in sizes:
        st, cp = min(res[n]["step"]), min(res[n]["copy"])
        b = BPP[mode] * n
        print(json.dumps({"mode": mode, "n": n, "bytes": b,
                          "step_ms_reps": [round(v, 4) for v in res[n]["step"]],
                          "copy_ms_reps": [round(v, 4) for v in res[n]["copy"]],
                          "step_GBps": b / st / 1e6, "copy_GBps": b / cp / 1e6,
                          "step_over_copy": cp / st}), flush=True)


if __name__ == "__main__":
    main()
