"""Debug helper: sharded (world 1) vs worker-local rounds, report mismatches."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_16265_b200 import _lib as L  # noqa: E402
from paper_2401_16265_b200 import co2  # noqa: E402


def to_np(t):
    return t.detach().cpu().numpy().copy()


mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n, tau = 200_003, 3
eng_s = co2.CollectiveEngine(1, transport="nccl", rank=0, nccl_id=bytes(128))
eng_w = co2.CollectiveEngine(1, transport="nccl", rank=0, nccl_id=bytes(128))
init = co2.synth(mode, n)[3]
sw = co2.ShardedWorker(mode, n, eng_s, init)
w = co2.Worker(mode, n, init)
hs = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, ghost_consistent=True)
hw = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
for t in range(3):
    w.snapshot_start()
    sw.snapshot_start()
    for k in range(tau):
        co2.synthetic_inner_step(sw.params, lr=1e-3, step=t * tau + k)
        co2.synthetic_inner_step(w.params, lr=1e-3, step=t * tau + k)
        if k == 0:
            sw.snapshot_first()
            w.snapshot_first()
    torch.cuda.synchronize()
    for name, a, b in [("params_before", sw.params, w.params),
                       ("xfirst", sw.buffer(L.BUF_XFIRST), w.buffer(L.BUF_XFIRST)),
                       ("anchor", sw.buffer(L.BUF_ANCHOR), w.buffer(L.BUF_ANCHOR)),
                       ("prev_x0", sw.buffer(L.BUF_PREV_X0), w.buffer(L.BUF_PREV_X0))]:
        if t == 0 and name == "prev_x0":
            continue
        A, B = to_np(a), to_np(b)
        bad = np.nonzero(A != B)[0]
        print(t, name, "bad", bad.size, bad[:5], A[bad[:3]] if bad.size else "", B[bad[:3]] if bad.size else "")
    sw.round(eng_s, hs, tau)
    co2.co2_round([w], eng_w, hw, tau)
    for name, a, b in [("params", sw.params, w.params),
                       ("m", sw.buffer(L.BUF_MOMENTUM), w.buffer(L.BUF_MOMENTUM)),
                       ("anchor", sw.buffer(L.BUF_ANCHOR), w.buffer(L.BUF_ANCHOR))]:
        A, B = to_np(a), to_np(b)
        bad = np.nonzero(A != B)[0]
        print(t, name, "bad", bad.size, bad[:5], A[bad[:3]] if bad.size else "", B[bad[:3]] if bad.size else "")
