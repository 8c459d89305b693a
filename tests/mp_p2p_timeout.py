"""A P2P all-reduce whose peer never arrives must fail with a bounded,
reported timeout instead of hanging the GPU (launched by
tests/test_gpu_multi.py under torchrun with CO2_P2P_TIMEOUT_MS=300): rank 1
registers its buffer but never launches; rank 0's reduce times out, the
stall query reports the barrier error, and the GPU stays usable."""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2401_16265_b200 import co2  # noqa: E402
from paper_2401_16265_b200.dist import env_rank  # noqa: E402


def main():
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    eng = co2.CollectiveEngine(world, transport="p2p", rank=rank)
    buf = torch.ones(1 << 20, dtype=torch.float32, device="cuda")
    eng.register(buf.data_ptr())
    res = {"rank": rank}
    if rank == 0:
        t0 = time.perf_counter()
        h = eng.launch_all_reduce([buf], buf)
        eng.wait(h)
        torch.cuda.synchronize()
        res["seconds"] = time.perf_counter() - t0
        try:
            eng.stall(h)
            res["error"] = None
        except RuntimeError as e:
            res["error"] = str(e)
        # the device is still healthy
        x = torch.arange(10, device="cuda", dtype=torch.float32).sum().item()
        res["healthy"] = x == 45.0
    dist.barrier()
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        print(json.dumps(out[0]), flush=True)
    dist.destroy_process_group()
    os._exit(0)  # skip engine teardown: rank 1's signal epoch never advanced


if __name__ == "__main__":
    main()
