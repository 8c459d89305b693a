"""NCCL transport across real GPUs (needs >= 2 visible B200s; skipped on a
single-GPU box).  Spawns tests/mp_nccl_rounds.py under torchrun."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("transport,world,n", [("nccl", 2, 1 << 20), ("nccl", 4, 1 << 20),
                                               ("nccl", 4, 1_000_003), ("p2p", 2, 1 << 20),
                                               ("p2p", 4, 1 << 20), ("p2pfused", 2, 1 << 20),
                                               ("p2pfused", 4, 1 << 20), ("p2pbulk", 2, 1 << 20),
                                               ("p2pbulk", 4, 1_000_003), ("p2pgrids", 2, 1 << 20),
                                               ("p2pgrids", 4, 1_000_003)])
def test_multi_rank_rounds_bitwise(mode, transport, world, n):
    """Worker-local co2_round across ranks, bitwise against the oracle --
    params, momentum and the consumed average -- for every fixed-order
    transport (NCCL's default slice-exchange algorithm, P2P, fused P2P): the
    reference's average() (param_ops.cpp:16-33) at any G.  NCCL: n = 2^20
    splits into equal slices (ncclAlltoAll + in-place ncclAllGather), the
    ragged n into short last slices (grouped ncclSend / ncclRecv)."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, CO2_TEST_MODE=str(mode), CO2_TEST_TRANSPORT=transport,
               CO2_TEST_N=str(n))
    if transport == "p2pbulk":  # the TMA bulk-copy all-reduce kernel
        env.update(CO2_P2P_BULK="2", CO2_TEST_TRANSPORT="p2p")
    if transport == "p2pgrids":  # a different reduce grid per rank, adaptive occupancy on
        env.update(CO2_TEST_RANK_CTAS="1", CO2_P2P_ADAPT="1", CO2_TEST_TRANSPORT="p2p")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_nccl_rounds.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["ok"], res
    # two-kernel schedule: one wait per consumed reduce (rounds 1..3); fused:
    # only the round-0 reduce is a separate handle
    assert res["waits"] == (1 if transport == "p2pfused" else 3)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_rounds_nccl_sum_within_bound(mode, world):
    """NCCL's sum algorithm (ncclAllReduce(sum) in the storage dtype, /G in
    the step): x-bar, momentum and params within the stated per-round bound
    of the reference (tests/mp_nccl_rounds.py docstring: delta = G*u*max|x|,
    u = 2^-8 bf16 / 2^-23 fp32)."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, CO2_TEST_MODE=str(mode), CO2_TEST_TRANSPORT="ncclsum")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_nccl_rounds.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["ok"], res
    assert res["max_bound_ratio"] <= 1.0


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("transport,world", [("nccl", 2), ("nccl", 4), ("ncclsum", 2),
                                             ("p2p", 2), ("p2p", 4)])
def test_sharded_ghost_bitwise(mode, transport, world):
    """Sharded ghost-consistent rounds (C4 layout) against the oracle,
    bitwise: NCCL's fixed-order slice exchange + all-gather at G = 2 and 4,
    NCCL's reduce-scatter sum at G = 2 (order-free there), and the fused P2P
    step (slice average + ghost step + NVLink all-gather) at G = 2 and 4."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, CO2_TEST_MODE=str(mode), CO2_TEST_TRANSPORT=transport)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_nccl_sharded.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["ok"], res


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("script", ["mp_nccl_rounds.py", "mp_nccl_sharded.py"])
@pytest.mark.parametrize("world", [2, 4])
def test_p2p_rank_cap8_bitwise(script, world):
    """The G = 8 instantiations of the P2P reduce kernels (what an 8-GPU run
    launches), forced at G = 2 and 4 through CO2_P2P_RANK_CAP=8: the guarded
    loads over absent ranks must leave the fixed-order average bitwise."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, CO2_TEST_MODE="2", CO2_TEST_TRANSPORT="p2p", CO2_P2P_RANK_CAP="8")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    assert json.loads(line)["ok"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_p2p_register_deregister_cycles():
    """P2P buffers can be detached and freed, and new ones attached, with
    every reduce still bitwise the fixed-order average."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_p2p_detach.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    assert json.loads(line)["ok"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_p2p_missing_peer_times_out():
    """A peer that never joins the reduce: the barrier gives up after
    CO2_P2P_TIMEOUT_MS, the error is reported, and the GPU stays usable."""
    env = dict(os.environ, CO2_P2P_TIMEOUT_MS="300")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_p2p_timeout.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["error"] and "timed out" in res["error"], res
    assert res["healthy"] and res["seconds"] < 5.0, res
