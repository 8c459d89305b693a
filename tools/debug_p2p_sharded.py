"""Debug: sharded P2P rounds at a given size (torchrun, 2+ ranks).

  torchrun --nproc-per-node 2 tools/debug_p2p_sharded.py N [rounds] [only_slice]
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_16265_b200 import co2  # noqa: E402
from paper_2401_16265_b200.dist import env_rank  # noqa: E402

n = int(sys.argv[1])
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rank, world, local = env_rank()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
eng = co2.CollectiveEngine(world, transport="p2p", rank=rank)
h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, ghost_consistent=True)
init = co2.synth_params(2, n, worker=0)
w = co2.ShardedWorker(2, n, eng, init, keep_gap=False)
del init
print(rank, "created shard", w.offset, w.length, w.shard, flush=True)
for t in range(rounds):
    w.snapshot_start()
    w.snapshot_first()
    torch.cuda.synchronize()
    try:
        r = w.round(eng, h, 12, sync=True)
        print(rank, "round", t, "ok", r.outer_applied, r.min_gap, r.max_outer_step, flush=True)
    except Exception as exc:
        print(rank, "round", t, "FAILED", exc, flush=True)
        break
dist.barrier()
