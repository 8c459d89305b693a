"""Multi-rank co2_round over the NCCL and P2P transports (launched by
tests/test_gpu_multi.py under torchrun; one process per GPU).

Each rank is one CO2 worker.  Rounds run the synthetic inner-step kernel,
then co2_round.  Rank 0 gathers every rank's trace and replays the round on
the CPU oracle:
  * fixed-order transports ("nccl" = NCCL's default slice-exchange algorithm,
    "p2p", "p2pfused"): bitwise, every round, params, momentum AND the
    consumed average (RoundResult::consumed_average, kept by the step);
  * "ncclsum" (ncclAllReduce(sum) in the storage dtype, /G in the step):
    NCCL's order and per-hop rounding make x-bar differ from average() by
    at most delta_j = G * u * max_i |x_i[j]| (u = 2^-8 bf16, 2^-23 fp32:
    G-1 rounded hops plus the final rounding, with a factor 2 of headroom);
    the step is 1-Lipschitz in x-bar (|Delta/Lambda| <= |Delta|, clip is a
    clamp), so momentum and x' differ by at most delta_j (+ 2^-20 relative
    fp32 rounding), the bf16 params additionally by one bf16 ulp (2u|x'|: the
    two sides round independently and may straddle a rounding boundary).  The
    oracle's momentum is re-synchronised to the GPU's every round so the
    bound is per round, not accumulated.
Prints one JSON line on rank 0.
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
    n, tau, rounds = int(os.environ.get("CO2_TEST_N", 1 << 20)), 4, 4
    transport = os.environ.get("CO2_TEST_TRANSPORT", "nccl")
    if transport in ("p2p", "p2pfused"):
        # CO2_TEST_RANK_CTAS: a different reduce grid on every rank (the exit
        # barrier counts ranks, not CTAs)
        ctas = 8 + 24 * rank if os.environ.get("CO2_TEST_RANK_CTAS") else 0
        eng = co2.CollectiveEngine(world, transport="p2p", rank=rank, max_ctas=ctas)
        if transport == "p2pfused":
            eng.set_fused(True)
    else:
        uid = broadcast_nccl_id(co2.CollectiveEngine.unique_id, rank, world)
        eng = co2.CollectiveEngine(world, transport="nccl", rank=rank, nccl_id=uid,
                                   nccl_algo="sum" if transport == "ncclsum" else "fixed")
    exact = transport != "ncclsum"
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    init = co2.synth(mode, n, worker=rank)[3]
    w = co2.Worker(mode, n, init)
    w.keep_average()
    if transport in ("p2p", "p2pfused"):
        eng.register_worker(w)
    ok, worst, max_ratio = True, None, 0.0
    from oracle import oracle as O
    if rank == 0:
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
        xbar = to_np(w.buffer(L.BUF_XBAR)) if t >= 1 else None
        after = (to_np(w.params), to_np(w.buffer(L.BUF_MOMENTUM)), xbar)
        traces = gather(trace, world)
        afters = gather(after, world)
        if rank == 0:
            consumed = orr.pending  # the average the oracle consumes this round
            ends = [tr[2] for tr in traces]
            bf = mode == O.MODE_BF16_MIXED
            u = 2.0 ** -8 if bf else 2.0 ** -23
            if t >= 1 and not exact:
                # the consumed average reduces the PREVIOUS round's x_{t,tau}
                delta = world * u * prev_xmax
                prev_m = [mm.copy() for mm in orr.m]
            prev_xmax = np.max(np.stack([np.abs(O.to_f64(e)) for e in ends]), axis=0)
            ref = orr.round(ends, traces, np.zeros(n, np.float32))
            for i in range(world):
                if exact:
                    if afters[i][0].tobytes() != ref[i].tobytes():
                        ok, worst = False, (t, i, "params")
                    if t >= 1 and afters[i][1].tobytes() != orr.m[i].tobytes():
                        ok, worst = False, (t, i, "momentum")
                    if t >= 1 and afters[i][2].tobytes() != consumed.tobytes():
                        ok, worst = False, (t, i, "consumed_average")
                elif t >= 1:
                    gm, om = O.to_f64(afters[i][1]), O.to_f64(orr.m[i])
                    sm = 2 * np.abs(0.7 * O.to_f64(prev_m[i])) + np.abs(om)  # >= |bm|+|D/L|
                    bm = delta + 2.0 ** -20 * sm
                    gp, op = O.to_f64(afters[i][0]), O.to_f64(ref[i])
                    # two independently rounded bf16 values straddling a rounding boundary
                    # differ by up to one bf16 ulp <= 2^-7 |x'| = 2u |x'|
                    bp = delta + 2.0 ** -20 * (np.abs(op) + sm) + (2 * u * np.abs(op) if bf else 0)
                    ga, oa = O.to_f64(afters[i][2]), O.to_f64(consumed)
                    ba = delta
                    for name, d, b in (("momentum", np.abs(gm - om), bm),
                                       ("params", np.abs(gp - op), bp),
                                       ("consumed_average", np.abs(ga - oa), ba)):
                        ratio = float(np.max(d / np.maximum(b, 1e-300)))
                        max_ratio = max(max_ratio, ratio)
                        if ratio > 1.0:
                            ok, worst = False, (t, i, name, ratio)
                    orr.m[i] = afters[i][1].copy()  # per-round bound: re-synchronise
        if t >= 1:
            assert r.outer_applied == 1
    stalls = []
    for e in eng.events():
        if e["event"] == "wait":
            stalls.append(e["stall"])
    if rank == 0:
        print(json.dumps({"ok": ok, "first_mismatch": worst, "world": world, "mode": mode,
                          "transport": transport, "waits": len(stalls),
                          "max_bound_ratio": max_ratio}), flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
