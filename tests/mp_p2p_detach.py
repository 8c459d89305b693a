"""P2P engine buffer lifecycle across ranks (launched by
tests/test_gpu_multi.py under torchrun): register -> reduce -> deregister ->
free -> register a NEW buffer -> reduce, several cycles; every reduce must be
bitwise the oracle's fixed-order average, and unknown / twice-detached
buffers must raise.  Prints one JSON line on rank 0."""
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
