"""Global-norm clip EXTENSION throughput next to the reference-semantics
fused step, C3 layout (1.3B bf16-mixed) on one GPU: CUDA-event time per
call, algorithmic GB/s (34 B/param for the two passes, 26 for the fused
step) and the fraction of MEASURED_PEAKS.json's copy bandwidth.

  python tools/gclip_bench.py [--n 1300000000] [--mode 2] [--iters 20]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BPP_FUSED = {0: 64, 1: 32, 2: 26}
BPP_GCLIP = {0: 80, 1: 40, 2: 34}  # pass 1: reads x,p0,p1,xbar,m + writes m'; pass 2: m',x -> anchor,params


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_300_000_000)
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    mode, n = a.mode, a.n
    x, p0, p1, xe, m = co2.synth(mode, n)
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    ws = co2.Workspace()
    lib = co2.lib()
    st = torch.cuda.current_stream().cuda_stream

    def fused():
        co2.check(lib.co2_outer_step(mode, n, x.data_ptr(), p0.data_ptr(), p1.data_ptr(),
                                     xe.data_ptr(), 1, m.data_ptr(), p0.data_ptr(),
                                     xe.data_ptr(), None, C.byref(h.c(12)), ws.ptr, st))

    def gclip():
        co2.check(lib.co2_outer_step_global_clip(mode, n, x.data_ptr(), p0.data_ptr(),
                                                 p1.data_ptr(), xe.data_ptr(), 1, m.data_ptr(),
                                                 p0.data_ptr(), xe.data_ptr(), None,
                                                 C.byref(h.c(12)), ws.ptr, st))

    out = {}
    for name, fn, bpp in (("fused_coordinate_clip", fused, BPP_FUSED[mode]),
                          ("global_norm_clip", gclip, BPP_GCLIP[mode])):
        for _ in range(3):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.iters)]
        for e0, e1 in evs:
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        t = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs) * 1e-3
        out[name] = {"ms": t * 1e3, "params_per_s": n / t, "bytes_per_param": bpp,
                     "GBps": bpp * n / t / 1e9, "frac_of_measured_copy": bpp * n / t / 1e9 / peak}
    print(json.dumps({"mode": mode, "n": n, **out}), flush=True)


if __name__ == "__main__":
    main()
