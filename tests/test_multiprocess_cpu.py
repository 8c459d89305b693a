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


def _sharded_worker(rank, world, port, mode, q):
    """One rank of the sharded ghost-consistent decomposition (what
    co2_sharded_round does on the GPU, here on the oracle): fixed-order slice
    averages of x_{t,tau} and x_{t,1}, the ghost step on the owned shard,
    and an all-gather of x_{t+1,0}."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2401_16265_b200.dist import shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 100_003
    h = O.hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, tau=12)
    anchor, p0, p1, _, m = O.synth(mode, n, worker=0)  # shared outer state
    x_tau = O.synth(mode, n, worker=1 + rank)[3]         # this rank's contributions
    x_one = O.synth(mode, n, worker=11 + rank)[3]
    lo, cnt = shard_range(n, rank, world)
    sl = slice(lo, lo + cnt)

    def gather(a):
        out = [None] * world
        dist.all_gather_object(out, a)
        return out

    bf = mode == O.MODE_BF16_MIXED
    xs = O.average_lp([c[sl] for c in gather(x_tau)], bf) if cnt else x_tau[:0]
    x1 = O.average_lp([c[sl] for c in gather(x_one)], bf) if cnt else x_one[:0]
    r = O.outer_step_ghost(mode, anchor[sl], p0[sl], x1, 1, xs, 1, world, m[sl], h)
    params = np.concatenate(gather(r.params))
    mom = np.concatenate(gather(r.m))
    anc = np.concatenate(gather(r.anchor))
    # the unsharded ghost round on every coordinate, same inputs
    xs_f = O.average_lp(gather(x_tau), bf)
    x1_f = O.average_lp(gather(x_one), bf)
    f = O.outer_step_ghost(mode, anchor, p0, x1_f, 1, xs_f, 1, world, m, h)
    ok = (params.tobytes() == f.params.tobytes() and mom.tobytes() == f.m.tobytes() and
          anc.tobytes() == f.anchor.tobytes() and r.status == 0 and f.status == 0)
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [1, 2])
def test_gloo_world2_sharded_decomposition(mode):
    """The C4 sharded layout's decomposition (slice averages in rank order,
    ghost step per shard, all-gather) reproduces the unsharded ghost round
    bit for bit, across two gloo ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_sharded_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
