"""World-size-2 host logic on CPU (gloo): NCCL-id bootstrap, max-over-ranks
timing, shard ranges of the sharded outer state."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2401_16265_b200.dist import shard_range


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2401_16265_b200 import co2
    from paper_2401_16265_b200.dist import broadcast_nccl_id, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = broadcast_nccl_id(co2.CollectiveEngine.unique_id, rank, world)
    t = max_over_ranks([0.5 + rank, 2.0 - rank])
    dist.barrier()
    q.put((rank, uid, t))
    dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, id0, t0), (r1, id1, t1) = res
    assert id0 == id1 and len(id0) == 128 and any(id0)
    assert t0 == t1 == [1.5, 2.0]


@pytest.mark.parametrize("n,world", [(7_000_000_000, 8), (1_000_003, 4), (13, 2), (0, 2),
                                     (1_300_000_000, 3)])
def test_shard_ranges_cover_and_align(n, world):
    ranges = [shard_range(n, r, world) for r in range(world)]
    assert sum(c for _, c in ranges) == n
    pos = 0
    for s, c in ranges:
        assert s == pos or c == 0
        assert s % 8 == 0 or c == 0
        pos = s + c if c else pos
    assert pos == n
