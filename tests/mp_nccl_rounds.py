"""Multi-rank co2_round over the NCCL transport (launched by
tests/test_gpu_multi.py under torchrun; one process per GPU).

Each rank is one CO2 worker.  Rounds run the synthetic inner-step kernel,
then co2_round (in-place NCCL sum of x_{t,tau} on the engine's comm stream,
divided by G in the consumer step).  Rank 0 gathers every rank's trace and
replays the round on the CPU oracle; for G = 2 the NCCL sum is order-free,
so the comparison is bitwise.  Prints one JSON line on rank 0.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2401_16265_b200 import _lib as L  # noqa: E402
from paper_2401_16265_b200 import co2  # noqa: E402
from paper_2401_16265_b200.dist import broadcast_nccl_id, env_rank  # noqa: E402


def to_np(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def gather(arr: np.ndarray, world: int):
    out = [None] * world
    dist.all_gather_object(out, arr)
    return out


def main():
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    mode = int(os.environ.get("CO2_TEST_MODE", "1"))
    n, tau, rounds = 1 << 20, 4, 4
    transport = os.environ.get("CO2_TEST_TRANSPORT", "nccl")
    if transport in ("p2p", "p2pfused"):
        eng = co2.CollectiveEngine(world, transport="p2p", rank=rank)
        if transport == "p2pfused":
            eng.set_fused(True)
    else:
        uid = broadcast_nccl_id(co2.CollectiveEngine.unique_id, rank, world)
        eng = co2.CollectiveEngine(world, transport="nccl", rank=rank, nccl_id=uid)
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    init = co2.synth(mode, n, worker=rank)[3]
    w = co2.Worker(mode, n, init)
    if transport in ("p2p", "p2pfused"):
        eng.register_worker(w)
    ok, worst = True, None
    if rank == 0:
        from oracle import oracle as O
        from test_gpu_rounds import OracleRoundLP
        orr = OracleRoundLP(mode, world, O.hyper(alpha=1.0, beta=0.7, phi=5e-3,
                                                  epsilon=1e-12, tau=tau))
    for t in range(rounds):
        w.snapshot_start()
        for k in range(tau):
            co2.synthetic_inner_step(w.params, lr=1e-3, worker=rank, step=t * tau + k)
            if k == 0:
                w.snapshot_first()
        torch.cuda.synchronize()
        trace = (to_np(w.buffer(L.BUF_ANCHOR)), to_np(w.buffer(L.BUF_XFIRST)), to_np(w.params))
        r = co2.co2_round([w], eng, hyper, tau)
        after = (to_np(w.params), to_np(w.buffer(L.BUF_MOMENTUM)))
        traces = gather(trace, world)
        afters = gather(after, world)
        if rank == 0:
            ref = orr.round([tr[2] for tr in traces], traces, np.zeros(n, np.float32))
            for i in range(world):
                if afters[i][0].tobytes() != ref[i].tobytes():
                    ok, worst = False, (t, i, "params")
                if t >= 1 and afters[i][1].tobytes() != orr.m[i].tobytes():
                    ok, worst = False, (t, i, "momentum")
        if t >= 1:
            assert r.outer_applied == 1
    stalls = []
    for e in eng.events():
        if e["event"] == "wait":
            stalls.append(e["stall"])
    if rank == 0:
        print(json.dumps({"ok": ok, "first_mismatch": worst, "world": world, "mode": mode,
                          "transport": transport, "waits": len(stalls)}), flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
