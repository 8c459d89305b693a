"""P2P engine buffer lifecycle across ranks (launched by
tests/test_gpu_multi.py under torchrun): register -> reduce -> deregister ->
free -> register a NEW buffer -> reduce, several cycles; every reduce must be
bitwise the oracle's fixed-order average, and unknown / twice-detached
buffers must raise.  Then fused worker-local and sharded P2P rounds run
asynchronously and their buffers are detached and freed with no host
synchronize in between (detach waits for every stream).  Prints one JSON line on rank 0."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2401_16265_b200 import co2  # noqa: E402
from paper_2401_16265_b200.dist import env_rank  # noqa: E402


def main():
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    eng = co2.CollectiveEngine(world, transport="p2p", rank=rank)
    ok = True
    for cycle in range(4):
        n = 100_003 + 7919 * cycle
        bufs = [co2.synth(co2.MODE_BF16_MIXED, n, worker=w)[3] for w in range(world)]
        mine = bufs[rank].clone()
        eng.register(mine.data_ptr())
        h = eng.launch_all_reduce([mine], mine)
        eng.wait(h)
        torch.cuda.synchronize()
        ref = O.average_lp([O.synth(co2.MODE_BF16_MIXED, n, worker=w)[3] for w in range(world)],
                           True)
        got = mine.view(torch.int16).cpu().numpy().view(np.uint16)
        good = got.tobytes() == ref.tobytes()
        if not good:
            bad = np.nonzero(got != ref)[0]
            print(f"rank {rank} cycle {cycle}: {bad.size} mismatches, first {bad[:5]}",
                  flush=True)
        ok = ok and good
        eng.deregister(mine.data_ptr())
        del mine, bufs
        torch.cuda.empty_cache()
    # Kernels on the CALLER's stream also use the peer mappings: the fused
    # all-reduce + step (worker-local) and the sharded step's NVLink
    # all-gather.  Deregister right after asynchronous rounds, with no
    # host-side synchronize: detach must wait for them before unmapping.
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    for cycle in range(2):
        n = 1 << 22
        w = co2.Worker(co2.MODE_BF16_MIXED, n, co2.synth(2, n, worker=rank)[3])
        eng.register_worker(w)
        eng.set_fused(True)
        for t in range(4):
            w.snapshot_start()
            co2.synthetic_inner_step(w.params, lr=1e-3, worker=rank, step=t)
            w.snapshot_first()
            co2.co2_round([w], eng, hyper, 2, sync=False)
        eng.set_fused(False)
        eng.deregister_worker(w)  # no synchronize before it
        w.close()
        ghost = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12,
                             ghost_consistent=True)
        sw = co2.ShardedWorker(co2.MODE_BF16_MIXED, n, eng,
                               co2.synth(2, n, worker=0)[3])
        for t in range(3):
            sw.snapshot_start()
            co2.synthetic_inner_step(sw.params, lr=1e-3, worker=rank, step=t)
            sw.snapshot_first()
            sw.round(eng, ghost, 2, sync=False)
        sw.drain(eng)
        for which in (co2.L.BUF_PARAMS, co2.L.BUF_PARAMS_ALT, co2.L.BUF_XFIRST,
                      co2.L.BUF_XFIRST_ALT):
            eng.deregister(co2.lib().co2_sharded_buffer(sw.handle, which))
        sw.close()
        torch.cuda.empty_cache()
    torch.cuda.synchronize()  # surfaces any fault from the unmapped peers
    try:
        eng.deregister(12345)
        ok = False
    except co2.ValidationError as e:
        if "not registered" not in str(e):
            print(f"rank {rank}: unexpected message {e}", flush=True)
            ok = False
    eng.close()
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if rank == 0:
        print(json.dumps({"ok": all(flags), "world": world}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
