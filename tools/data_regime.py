"""Per-launch fused-step time as the in-place iteration evolves the data
(the tune tools and the round bench feed each step's outputs back as the
next step's inputs), beside the same launch on freshly synthesised inputs,
plus value statistics of the evolved buffers:

  python tools/data_regime.py [--mode 1] [--n 125000000] [--steps 300]

Prints one JSON line per sampled launch index and one summary line.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stats(torch, t):
    f = t.float()
    tiny = torch.finfo(torch.float32).tiny
    a = f.abs()
    return {"zero": float((a == 0).float().mean()),
            "subnormal": float(((a > 0) & (a < tiny)).float().mean()),
            "lt_1e-30": float(((a > 0) & (a < 1e-30)).float().mean()),
            "absmax": float(a.max()), "nonfinite": float((~torch.isfinite(f)).float().mean())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--n", type=int, default=125_000_000)
    ap.add_argument("--steps", type=int, default=300)
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2

    mode, n = a.mode, a.n
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    ws = co2.Workspace()
    bufs = co2.synth(mode, n)
    pristine = [b.clone() for b in bufs]
    x, p0, p1, xe, m = bufs

    def launch():
        co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                       workspace=ws, check_flags=False)

    def fresh():
        for b, p in zip(bufs, pristine):
            b.copy_(p)

    def timed():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        return e0, e1

    # fresh inputs every launch (restore outside the events)
    fr = []
    for _ in range(20):
        fresh()
        fr.append(timed())
    torch.cuda.synchronize()
    fresh_ms = [e0.elapsed_time(e1) for e0, e1 in fr]
    # in-place evolution from fresh inputs
    fresh()
    ev = [timed() for _ in range(a.steps)]
    torch.cuda.synchronize()
    ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    marks = sorted({0, 1, 2, 3, 5, 10, 20, 40, 80, 120, 160, 200, 250, a.steps - 1})
    for k in marks:
        if k < len(ms):
            w = ms[k:k + 5]
            print(json.dumps({"launch": k, "ms": round(ms[k], 4),
                              "ms_next5_median": round(statistics.median(w), 4)}), flush=True)
    print(json.dumps({"mode": mode, "n": n, "fresh_ms_median": statistics.median(fresh_ms),
                      "evolved_ms_median_last50": statistics.median(ms[-50:]),
                      "evolved_stats": {"m": stats(torch, m), "p0_minus_xbar":
                                        stats(torch, p0.float() - xe.float()),
                                        "x_minus_p0": stats(torch, x.float() - p0.float())},
                      "fresh_stats": {"m": stats(torch, pristine[4]), "p0_minus_xbar":
                                      stats(torch, pristine[1].float() - pristine[3].float())}}),
          flush=True)


if __name__ == "__main__":
    main()
