"""Time every fused-step instantiation (CO2_FUSED_VARIANT) on a config with
CUDA events; one subprocess per variant (the knob is read once per process).

  python tools/tune_fused.py [--mode 2] [--n 1300000000] [--iters 30]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(mode, n, iters):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2401_16265_b200 import co2
    x, p0, p1, xe, m = co2.synth(mode, n)
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    ws = co2.Workspace()
    for _ in range(3):
        co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                       workspace=ws, check_flags=False)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(iters)]
    for a, b in evs:
        a.record()
        co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                       workspace=ws, check_flags=False)
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e-3 for a, b in evs)
    bpp = {0: 64, 1: 32, 2: 26}[mode]
    return {"median_ms": ts[len(ts) // 2] * 1e3, "min_ms": ts[0] * 1e3,
            "GBps_median": bpp * n / ts[len(ts) // 2] / 1e9, "GBps_best": bpp * n / ts[0] / 1e9}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--n", type=int, default=1_300_000_000)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--variants", default="0,1,2,3,4")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(one(a.mode, a.n, a.iters)))
        sys.exit(0)
    for v in a.variants.split(","):
        env = dict(os.environ, CO2_FUSED_VARIANT=v)
        r = subprocess.run([sys.executable, __file__, "--child", "--mode", str(a.mode), "--n",
                            str(a.n), "--iters", str(a.iters)], env=env, capture_output=True,
                           text=True)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-500:]
        print(f"mode={a.mode} n={a.n} variant={v}: {line}", flush=True)
