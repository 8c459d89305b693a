"""Throughput of the baseline outer steps (SlowMo,
Local-SGD, Overlap-Local-SGD; proj/src/outer_algorithms.cpp:213-313) next to
the CO2 fused step, on one GPU, through the C ABI per-worker entries.

  python tools/baseline_bench.py [--mode 2] [--n 1300000000] [--iters 20]

One JSON line per kernel: ms per launch (median of CUDA-event-timed
back-to-back launches after 3 warm-ups; buffers larger than L2), the
algorithmic bytes per parameter of that update, GB/s and the fraction of the
measured copy bandwidth (MEASURED_PEAKS.json)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--n", type=int, default=1_300_000_000)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_2401_16265_b200 import co2

    mode, n = a.mode, a.n
    sb = 8 if mode == co2.MODE_F64 else 4
    lb = {co2.MODE_F64: 8, co2.MODE_F32: 4, co2.MODE_BF16_MIXED: 2}[mode]
    x, p0, p1, xe, m = co2.synth(mode, n)
    ws = co2.Workspace()
    st = torch.cuda.current_stream().cuda_stream
    L = co2.lib()
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    pk, pk_kind = peak()

    def co2_step():
        co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=p0, params_out=xe,
                       workspace=ws, check_flags=False)

    kernels = {
        # reads x_t0, p0, m (state) + p1, xbar (low); writes m, anchor (state) + params (low)
        "co2_fused_step": (co2_step, 5 * sb + 3 * lb),
        # reads x_start, m (state) + xbar (low); writes m, anchor (state) + params (low)
        "slowmo_step": (lambda: co2.check(L.co2_slowmo_step(
            mode, n, x.data_ptr(), xe.data_ptr(), 1, m.data_ptr(), p1.data_ptr(),
            p0.data_ptr(), 0.5, 0.5, ws.ptr, st)), 4 * sb + 2 * lb),
        # reads x_start (state) + xbar (low); writes anchor (state) + params (low)
        "local_sgd_step": (lambda: co2.check(L.co2_local_sgd_step(
            mode, n, x.data_ptr(), xe.data_ptr(), 1, p1.data_ptr(), p0.data_ptr(), ws.ptr,
            st)), 2 * sb + 2 * lb),
        # reads params, xbar (low) + anchor (state); writes params (low)
        "overlap_correction": (lambda: co2.check(L.co2_overlap_correction(
            mode, n, p1.data_ptr(), x.data_ptr(), xe.data_ptr(), 1, ws.ptr, st)), sb + 3 * lb),
    }
    for name, (fn, bpp) in kernels.items():
        for _ in range(3):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.iters)]
        for e0, e1 in evs:
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
        gbs = bpp * n / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": name, "mode": mode, "n": n, "ms": round(ms, 4),
                          "bytes_per_param": bpp, "params_per_s": n / (ms * 1e-3),
                          "GBps": round(gbs, 1), "peak": pk, "peak_kind": pk_kind,
                          "frac": round(gbs / pk, 4)}), flush=True)


if __name__ == "__main__":
    main()
