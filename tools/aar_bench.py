"""All-reduce microbenchmark of the CollectiveEngine transports, alone on the
GPUs (no overlapping compute): NCCL in-place sum vs the fixed-order NVLink P2P
average, reported as device time and NCCL-style bus bandwidth.

  torchrun --nproc-per-node N tools/aar_bench.py [--n 1300000000 --dtype bf16]
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
    ap.add_argument("--n", type=int, default=1_300_000_000)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32", "f64"])
    ap.add_argument("--ctas", default="16,32,64,128,148")
    ap.add_argument("--iters", type=int, default=8)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2401_16265_b200 import co2
    from paper_2401_16265_b200.dist import broadcast_nccl_id, env_rank, max_over_ranks

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[a.dtype]
    buf = torch.ones(a.n, dtype=dt, device="cuda")
    nbytes = buf.numel() * buf.element_size()

    def run(eng):
        times = []
        for i in range(a.iters + 2):
            h = eng.launch_all_reduce([buf], buf)
            eng.wait(h)
            torch.cuda.synchronize()
            if i >= 2:
                times.append(eng.stall(h)[1])
        t = max_over_ranks([statistics.median(times)], device="cpu")[0]
        return t, nbytes / t / 1e9, nbytes / t / 1e9 * 2 * (world - 1) / world

    rows = []
    uid = broadcast_nccl_id(co2.CollectiveEngine.unique_id, rank, world)
    eng = co2.CollectiveEngine(world, transport="nccl", rank=rank, nccl_id=uid)
    t, alg, bus = run(eng)
    rows.append({"transport": "nccl", "ctas": None, "ms": t * 1e3, "algbw_GBps": alg,
                 "busbw_GBps": bus})
    eng.close()
    for c in [int(x) for x in a.ctas.split(",")]:
        eng = co2.CollectiveEngine(world, transport="p2p", rank=rank, max_ctas=c)
        eng.register(buf.data_ptr())
        t, alg, bus = run(eng)
        rows.append({"transport": "p2p", "ctas": c, "ms": t * 1e3, "algbw_GBps": alg,
                     "busbw_GBps": bus})
        eng.close()
        dist.barrier()
    if rank == 0:
        for r in rows:
            print(json.dumps(dict(r, world=world, bytes=nbytes, dtype=a.dtype)), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
