"""Host-buffer entry (co2_outer_step_host) pipeline tuning: chunk size and
stream count, C3 bf16-mixed with pinned buffers.

  python tools/e2e_tune.py [--n 1300000000]
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
    ap.add_argument("--n", type=int, default=1_300_000_000)
    ap.add_argument("--mode", type=int, default=2)
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2
    mode, n = a.mode, a.n
    st, lo = co2.STATE_TORCH[mode], co2.LOW_TORCH[mode]
    x, p0, p1, xe, m = co2.synth(mode, n)
    hs = []
    for d, dt in ((x, st), (p0, st), (m, st), (p1, lo), (xe, lo)):
        h = torch.empty(n, dtype=dt, pin_memory=True)
        h.copy_(d)
        hs.append(h)
    del x, p0, p1, xe, m
    torch.cuda.empty_cache()
    hx, hp0, hm, hp1, hxe = hs
    params = torch.empty(n, dtype=lo, pin_memory=True)
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    for chunk in (1 << 23, 1 << 24, 1 << 25, 1 << 26):
        for ns in (2, 3, 4):
            times = []
            for i in range(3):
                t0 = time.perf_counter()
                co2.outer_step_host(mode, hx, hp0, hp1, hxe, hm, hyper, 12, anchor_out=hp0,
                                    params_out=params, chunk=chunk, nstreams=ns)
                if i:
                    times.append(time.perf_counter() - t0)
            t = statistics.mean(times)
            print(json.dumps({"chunk": chunk, "nstreams": ns, "ms": t * 1e3,
                              "params_per_s": n / t,
                              "GBps_pcie": (16 + 10) * n / t / 1e9}), flush=True)


if __name__ == "__main__":
    main()
