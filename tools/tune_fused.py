"""Interleaved timing of every fused-step instantiation (co2_set_fused_variant)
in one process on one GPU: R repetitions x every variant x K back-to-back
launches (the bench's steady state), CUDA events per launch, median per
(rep, variant).  Interleaving cancels slow drifts (clocks, power cap).

  python tools/tune_fused.py [--mode 2] [--n 1300000000] [--iters 40] [--reps 3]
                             [--waves 32] [--variants 0,1,...]

--waves takes a comma list; every (variant, waves) pair is one interleaved
configuration.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BPP = {0: 64, 1: 32, 2: 26}
NAMES = {
    2: {0: "(8,1) 4 CTA/SM", 1: "(8,2)", 2: "(4,4)", 3: "(4,1)", 4: "(8,1)", 5: "(4,2) 3 CTA/SM",
        6: "(8,1) <= 56 regs", 7: "(4,1) <= 56 regs",
        10: "bulk 2048x4 st, 4 cw", 11: "bulk 1024x4, 4 cw", 12: "bulk 2048x3, 8 cw",
        13: "bulk 4096x3, 8 cw", 14: "bulk 1024x6, 8 cw"},
    1: {0: "(4,1) 4 CTA/SM", 1: "(4,2)", 2: "(4,1)", 3: "(8,1)", 4: "(8,1) 4 CTA/SM",
        5: "(4,2) 4 CTA/SM", 6: "(4,1) <= 56 regs", 7: "(4,1) <= 48 regs",
        10: "bulk 1024x5, 4 cw", 11: "bulk 1024x4, 4 cw", 12: "bulk 2048x4, 8 cw",
        13: "bulk 1024x8, 8 cw", 14: "bulk 512x6, 4 cw"},
    0: {0: "(2,1) 4 CTA/SM", 1: "(2,2)", 2: "(2,1)", 3: "(4,1)", 4: "(2,2) 3 CTA/SM",
        5: "(2,1) 3 CTA/SM",
        10: "bulk 512x5, 4 cw", 11: "bulk 256x6, 2 cw", 12: "bulk 1024x4, 8 cw"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--n", type=int, default=1_300_000_000)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--waves", default="32")
    ap.add_argument("--variants", default="")
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2

    mode, n = a.mode, a.n
    x, p0, p1, xe, m = co2.synth(mode, n)
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    ws = co2.Workspace()
    vs = [int(v) for v in a.variants.split(",")] if a.variants else sorted(NAMES[mode])
    variants = [(v, int(w)) for v in vs for w in a.waves.split(",")]
    res = {v: [] for v in variants}
    for rep in range(a.reps):
        for v in variants:
            co2.check(co2.lib().co2_set_fused_variant(v[0]))
            co2.check(co2.lib().co2_set_grid_waves(v[1]))
            for _ in range(3):
                co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                               workspace=ws, check_flags=False)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(a.iters)]
            for e0, e1 in evs:
                e0.record()
                co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                               workspace=ws, check_flags=False)
                e1.record()
            torch.cuda.synchronize()
            res[v].append(statistics.median(e0.elapsed_time(e1) for e0, e1 in evs) * 1e-3)
    for v in variants:
        t = min(res[v])
        print(json.dumps({"mode": mode, "n": n, "variant": v[0], "waves": v[1],
                          "shape": NAMES[mode].get(v[0], "?"),
                          "median_ms_per_rep": [round(x * 1e3, 4) for x in res[v]],
                          "GBps_best_rep": BPP[mode] * n / t / 1e9,
                          "GBps_median_rep": BPP[mode] * n / statistics.median(res[v]) / 1e9}),
              flush=True)


if __name__ == "__main__":
    main()
