"""Sharded ghost-consistent rounds over NCCL (C4 layout), launched by
tests/test_gpu_multi.py under torchrun.  Rank 0 gathers each round's traces
and replays ghost-consistent co2_round (outer_algorithms.cpp:126-145,161-184)
on the CPU oracle.  The fixed-order transports (P2P, and NCCL's default
slice-exchange algorithm) deliver the reference's average() and are bitwise
at any G; NCCL's sum algorithm ("ncclsum") is order-free only for G = 2.
Prints one JSON line on rank 0."""
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


def storage_sum(arrs, mode):
    """What NCCL's sum produces for G = 2 in the storage dtype."""
    from oracle import oracle as O
    if mode == O.MODE_BF16_MIXED:
        s = O.bf16_bits_to_f32(arrs[0])
        for a in arrs[1:]:
            s = O.f32_to_bf16_bits(s + O.bf16_bits_to_f32(a))
            s = O.bf16_bits_to_f32(s)
        return O.f32_to_bf16_bits(s)
    s = arrs[0].copy()
    for a in arrs[1:]:
        s = s + a
    return s


def main():
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    mode = int(os.environ.get("CO2_TEST_MODE", "1"))
    n, tau, rounds = 300_007, 3, 5
    transport = os.environ.get("CO2_TEST_TRANSPORT", "nccl")
    if transport == "p2p":
        eng = co2.CollectiveEngine(world, transport="p2p", rank=rank)
        div = 1  # the P2P slice reduce delivers the fixed-order average
    else:
        uid = broadcast_nccl_id(co2.CollectiveEngine.unique_id, rank, world)
        algo = "sum" if transport == "ncclsum" else "fixed"
        eng = co2.CollectiveEngine(world, transport="nccl", rank=rank, nccl_id=uid,
                                   nccl_algo=algo)
        div = world if algo == "sum" else 1  # the sum algorithm delivers the worker sum
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, ghost_consistent=True)
    init = co2.synth(mode, n, worker=0)[3]  # identical x_{0,0} on every worker
    sw = co2.ShardedWorker(mode, n, eng, init)
    ok, mismatch = True, None
    if rank == 0:
        from oracle import oracle as O
        oh = O.hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, tau=tau)
        st = np.float64 if mode == 0 else np.float32
        m = np.zeros(n, st)
        anchor = prev_x0 = p1sum = xsum = None
    for t in range(rounds):
        sw.snapshot_start()
        for k in range(tau):
            co2.synthetic_inner_step(sw.params, lr=1e-3, worker=rank, step=t * tau + k)
            if k == 0:
                sw.snapshot_first()
        torch.cuda.synchronize()
        x_start = to_np(sw.params)  # only used at t == 0 (identical init)
        first = to_np(sw.buffer(L.BUF_XFIRST))
        end = to_np(sw.params)
        r = sw.round(eng, hyper, tau)
        params_after = to_np(sw.params)
        shard = (sw.offset, sw.length, to_np(sw.buffer(L.BUF_MOMENTUM)))
        firsts, ends, afters, shards = ([None] * world for _ in range(4))
        dist.all_gather_object(firsts, first)
        dist.all_gather_object(ends, end)
        dist.all_gather_object(afters, params_after)
        dist.all_gather_object(shards, shard)
        if rank == 0:
            if t == 0:
                x00 = to_np(init)
                x00s = O.to_f64(x00).astype(st) if mode != 0 else x00
                anchor = x00s
                prev_x0 = O.outer_step_ghost(mode, x00s, x00s, firsts[0], 1, ends[0], 1, world,
                                             np.zeros(n, st), oh).bar0
                expect = ends  # worker-local x_{1,0} = x_{0,tau}
            else:
                res = O.outer_step_ghost(mode, anchor, prev_x0, p1sum, div, xsum, div,
                                         0 if t == 1 else world, m, oh)
                assert res.status == 0, res.message
                anchor, prev_x0, m = res.anchor, res.bar0, res.m
                expect = [res.params] * world
                for off, ln, mm in shards:
                    if mm[:ln].tobytes() != m[off:off + ln].tobytes() and ok:
                        bad = np.nonzero(mm[:ln] != m[off:off + ln])[0]
                        ok, mismatch = False, (t, "momentum", off, int(bad.size), int(bad[0]),
                                               float(mm[bad[0]]), float(m[off + bad[0]]))
            for i in range(world):
                if afters[i][:n].tobytes() != expect[i].tobytes() and ok:
                    bad = np.nonzero(afters[i][:n] != expect[i])[0]
                    ok, mismatch = False, (t, "params", i, int(bad.size), int(bad[0]),
                                           float(afters[i][bad[0]]), float(expect[i][bad[0]]))
            if transport != "ncclsum":  # fixed-order averages (param_ops.cpp:16-33)
                if mode == O.MODE_F64:
                    p1sum, xsum = O.average(firsts), O.average(ends)
                else:
                    bf = mode == O.MODE_BF16_MIXED
                    p1sum, xsum = O.average_lp(firsts, bf), O.average_lp(ends, bf)
            else:
                p1sum = storage_sum(firsts, mode)
                xsum = storage_sum(ends, mode)
        if t >= 1:
            assert r.outer_applied == 1
    if rank == 0:
        print(json.dumps({"ok": ok, "first_mismatch": mismatch, "world": world, "mode": mode,
                          "transport": transport}),
              flush=True)
    sw.drain(eng)
    torch.cuda.synchronize()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
