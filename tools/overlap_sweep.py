"""C5: tau sweep of the one-step-stale schedule against a fixed-duration
synthetic local-compute kernel; reports exposed all-reduce time per tau next
to the analytic simulate_timeline prediction (proj/src/timing_model.cpp:
76-123,167-173).

  torchrun --nproc-per-node N tools/overlap_sweep.py [--mode 1] [--n 125000000]

Calibration (the knee): in the reference's CO2 timeline a round is
tau * t_comp of inner compute, the launch of the reduce, the stall on the
previous reduce, then t_outer of outer step -- so the reduce launched in
round t overlaps round t's outer step AND round t+1's tau inner steps, and
stalls by max(0, t_comm - t_outer - tau * t_comp).  The sweep measures
t_comm (the reduce alone) and t_outer (the outer step alone), then sizes the
synthetic inner step -- the HBM-streaming x <- x - lr * g kernel over the
first k coordinates, k calibrated -- to t_comp = (t_comm - t_outer) / knee,
so the predicted stall is positive for tau < knee and zero from the knee on.
If t_comm <= t_outer the outer step alone hides the reduce and no knee
exists; the sweep says so.

--inner selects the stand-in for the inner step: `hbm` (default) the
HBM-streaming update above -- the worst case for sharing HBM with the
reduce; `gemm` a bf16 tensor-core GEMM on resident operands (cuBLAS through
torch.matmul, square m x m, m calibrated to t_comp) plus the x_{t,1}
snapshot copy after the first step -- the compute-bound shape of a real
model's inner step.

exposed% = 100 * sum(stall) / sum(waited comm), the reference definition
(1 - overlap_ratio_achieved).  stall = device time the compute stream waited
on the reduce (events straddling the wait); comm = device duration of the
reduce on the comm stream.  interference = mean round time with the
all-reduce minus the same schedule with a world-1 (no-op) engine; it is also
reported as a share of the round and next to the reduce's HBM floor (the
bytes a fixed-order reduce must move through this GPU's HBM: 2 x the buffer,
read and written once, at the measured copy bandwidth).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--n", type=int, default=125_000_000)
    ap.add_argument("--taus", default="1,2,3,4,6,8,12,16,24,32")
    ap.add_argument("--rounds", type=int, default=8)
    ap.add_argument("--knee", type=float, default=4.0, help="tau at which tau*t_comp = t_comm")
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ncclsum", "p2p"])
    ap.add_argument("--inner", default="hbm", choices=["hbm", "gemm"])
    ap.add_argument("--out", default="")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2401_16265_b200 import _lib as L
    from paper_2401_16265_b200 import co2
    from paper_2401_16265_b200.dist import broadcast_nccl_id, env_rank, max_over_ranks

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    uid = broadcast_nccl_id(co2.CollectiveEngine.unique_id, rank, world)
    p2p = a.transport == "p2p" and world > 1
    if p2p:
        eng = co2.CollectiveEngine(world, transport="p2p", rank=rank, max_ctas=a.max_ctas)
    else:
        eng = co2.CollectiveEngine(world, transport="nccl", rank=rank, nccl_id=uid,
                                   max_ctas=a.max_ctas,
                                   nccl_algo="sum" if a.transport == "ncclsum" else "fixed")
    solo = co2.CollectiveEngine(1, transport="nccl", rank=0, nccl_id=bytes(128))
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    stream = torch.cuda.current_stream()
    lo = co2.LOW_TORCH[a.mode]

    # t_comm: the reduce alone (scratch buffer, same size and dtype)
    scratch = torch.zeros(a.n, dtype=lo, device="cuda")
    if p2p:
        eng.register(scratch.data_ptr())
    comms = []
    for i in range(6):
        h = eng.launch_all_reduce([scratch], scratch)
        eng.wait(h)
        torch.cuda.synchronize()
        if i >= 2:
            comms.append(eng.stall(h)[1])
    t_comm = max_over_ranks([statistics.median(comms)], device="cpu")[0] if world > 1 else 0.0
    if p2p:
        eng.deregister(scratch.data_ptr())
    del scratch

    w = co2.Worker(a.mode, a.n, co2.synth(a.mode, a.n, worker=rank)[3], keep_gap=False)

    # t_outer: the outer step alone (no-op engine), steady state
    def outer_alone():
        w2 = co2.Worker(a.mode, a.n, w.params, keep_gap=False)
        w2.snapshot_start()
        w2.snapshot_first()
        co2.co2_round([w2], solo, hyper, 1)
        w2.enable_timing(16)
        for _ in range(6):
            co2.co2_round([w2], solo, hyper, 1, sync=False)
        torch.cuda.synchronize()
        kt = w2.step_times()[2:]
        co2.co2_round_drain([w2], solo)
        w2.close()
        return statistics.median(kt)

    t_outer0 = outer_alone()
    t_outer0 = max_over_ranks([t_outer0], device="cpu")[0] if world > 1 else t_outer0

    gemm_ops = {}

    def gemm_operands(m):
        if m not in gemm_ops:
            g = torch.Generator(device="cuda").manual_seed(rank)
            gemm_ops.clear()
            gemm_ops[m] = (torch.randn(m, m, device="cuda", dtype=torch.bfloat16, generator=g),
                           torch.randn(m, m, device="cuda", dtype=torch.bfloat16, generator=g),
                           torch.empty(m, m, device="cuda", dtype=torch.bfloat16))
        return gemm_ops[m]

    def inner_step(k, params, step, snapshot_out=None):
        if a.inner == "hbm":
            co2.synthetic_inner_step(params[:k], lr=1e-6, worker=rank, step=step,
                                     snapshot_out=snapshot_out[:k] if snapshot_out is not None
                                     else None)
        else:  # k is the GEMM size m
            x, y, out = gemm_operands(k)
            torch.matmul(x, y, out=out)
            if snapshot_out is not None:
                snapshot_out.copy_(params)

    def time_inner(k, iters=6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        inner_step(k, w.params, 0)
        e0.record(stream)
        for i in range(iters):
            inner_step(k, w.params, i)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / iters

    # fixed-duration inner step: the first k coordinates, k calibrated so that
    # tau * t_comp + t_outer = t_comm at tau = knee
    knee_exists = t_comm > t_outer0
    target = (t_comm - t_outer0) / a.knee if knee_exists else t_comm / a.knee
    if a.inner == "hbm":
        k = a.n
        t_full = time_inner(k)
        for _ in range(4):
            k = max(1 << 16, min(a.n, int(k * target / max(time_inner(k), 1e-9))) // 256 * 256)
    else:  # GEMM time ~ m^3
        k = 4096
        t_full = time_inner(k)
        for _ in range(4):
            k = max(256, int(k * (target / max(time_inner(k), 1e-9)) ** (1.0 / 3.0)) // 128 * 128)
    t_comp = time_inner(k)
    k, t_comp = (max_over_ranks([k, t_comp], device="cpu") if world > 1 else (k, t_comp))
    k = int(k)
    hbm_gbs = 6452.8
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_gbs = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    low_bytes = {0: 8, 1: 4, 2: 2}[a.mode]
    hbm_floor = 2.0 * low_bytes * a.n / (hbm_gbs * 1e9)

    def run(engine, tau):
        w2 = co2.Worker(a.mode, a.n, w.params, keep_gap=False)
        if p2p and engine is eng:
            engine.register_worker(w2)
        w2.enable_timing(4 * a.rounds)
        n_ev0 = len(engine.events())
        # Rounds run back to back with no host synchronisation: a device-wide
        # synchronize between rounds would drain the comm stream and hide the
        # one-step-stale reduce's stall.  Round walls are compute-stream events.
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.rounds + 1)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for t in range(a.rounds):
            evs[t].record(stream)
            w2.snapshot_start()
            if t == 0:
                w2.snapshot_first()
            for j in range(tau):
                # the first step's store also writes the x_{t,1} snapshot of
                # the coordinates it moves (the others did not move); the
                # GEMM stand-in copies the snapshot after its first step
                inner_step(k, w2.params, t * tau + j,
                           snapshot_out=w2.buffer(L.BUF_XFIRST) if j == 0 and t > 0 else None)
            co2.co2_round([w2], engine, hyper, tau, sync=False)
        evs[a.rounds].record(stream)
        co2.co2_round_drain([w2], engine)
        torch.cuda.synchronize()
        walls = [evs[t].elapsed_time(evs[t + 1]) * 1e-3 for t in range(a.rounds)]
        kt = w2.step_times()
        ev = engine.events()[n_ev0:]
        launches = {e["handle_id"]: e["t_sim"] for e in ev if e["event"] == "launch"}
        completes = {e["handle_id"]: e["t_sim"] for e in ev if e["event"] == "complete"}
        # drop the first (warm-up) wait and the final drain
        waits = [e for e in ev if e["event"] == "wait"][1:-1]
        stall = sum(e["stall"] for e in waits)
        waited = sum(completes[e["handle_id"]] - launches[e["handle_id"]] for e in waits)
        if p2p and engine is eng:
            engine.deregister_worker(w2)
        w2.close()
        return statistics.mean(walls[2:]), stall, waited, len(waits), \
            (statistics.mean(kt) if kt else 0.0)

    rows = []
    for tau in [int(x) for x in a.taus.split(",")]:
        wall, stall, waited, nw, t_outer = run(eng, tau)
        wall0, _, _, _, _ = run(solo, tau)
        wall, stall, waited, wall0, t_outer = max_over_ranks(
            [wall, stall, waited, wall0, t_outer], device="cpu") if world > 1 else \
            (wall, stall, waited, wall0, t_outer)
        pred = co2.simulate_timeline_co2(
            co2.ClusterSpec(workers=world, t_comp=t_comp, t_outer=t_outer,
                            measured_override=t_comm), tau, a.rounds)
        # the measurement drops round 1's wait (its reduce overlapped no outer
        # step, :184-188); score the model on the same rounds
        pst = [p[2] for p in pred.per_round[2:]]
        pred_exposed = 100.0 * sum(pst) / (t_comm * len(pst)) if t_comm and pst else 0.0
        row = {"tau": tau, "world": world, "n": a.n, "mode": a.mode,
               "transport": "p2p" if p2p else a.transport, "inner": a.inner,
               "t_comm_ms": 1e3 * t_comm, "t_comp_ms": 1e3 * t_comp, "t_outer_ms": 1e3 * t_outer,
               "t_outer_alone_ms": 1e3 * t_outer0, "knee_exists": knee_exists,
               "knee_tau": a.knee, "inner_coords": k, "inner_full_ms": 1e3 * t_full,
               "exposed_pct": 100.0 * stall / waited if waited else 0.0,
               "stall_ms_per_round": 1e3 * stall / max(nw, 1),
               "comm_ms_measured": 1e3 * waited / max(nw, 1),
               "round_ms": 1e3 * wall, "round_ms_no_allreduce": 1e3 * wall0,
               "interference_ms": 1e3 * (wall - wall0),
               "interference_pct_of_round": 100.0 * (wall - wall0) / wall if wall else 0.0,
               "interference_pct_of_comm": 100.0 * (wall - wall0) / t_comm if t_comm else 0.0,
               "reduce_hbm_floor_ms": 1e3 * hbm_floor,
               "stall_pct_of_round": 100.0 * stall / max(nw, 1) / wall if wall else 0.0,
               "predicted_exposed_pct": pred_exposed,
               "predicted_exposed_pct_all_rounds": 100.0 * (1.0 - pred.overlap_ratio_achieved),
               "predicted_overlap": co2.overlap_ratio(tau, t_comp, t_comm) if t_comm else 1.0}
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
    if rank == 0 and a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    eng.close()
    solo.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
