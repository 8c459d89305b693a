"""Round-level behaviour of the CPU oracle's co2_round / baseline rounds,
mirroring the reference's own round tests (proj/tests/test_outer_algorithms.cpp
178-464) on the acceptance problem of proj/tests/acceptance.cpp:178-243.
The GPU round driver is checked bitwise against this oracle in
tests/test_gpu_rounds.py; these tests pin the oracle's round semantics."""
import numpy as np
import pytest

from oracle import oracle as O
from simdrive import OracleBaselineRound, OracleRound, inner_loop


class H:
    def __init__(self, **kw):
        self.alpha, self.beta, self.phi, self.epsilon = 0.4, 0.5, 1.0, 1e-12
        self.penalty, self.clip, self.ghost_consistent = True, True, False
        self.__dict__.update(kw)


def run(golden, rounds, hyper, workers=2, lr=None):
    k = golden["delayed_momentum"]
    feats, targs = np.array(k["features"], float), np.array(k["targets"], float)
    shards = k["shards"] if workers == 2 else [list(range(len(k["targets"])))]
    lr = k["lr"] if lr is None else lr
    tau = k["tau"]
    x = [np.array(k["init"], float) for _ in range(workers)]
    orr = OracleRound(workers, 2, hyper, tau)
    hist = []
    for _ in range(rounds):
        traces = [inner_loop(feats, targs, shards[i], x[i], lr, tau) for i in range(workers)]
        ends = [tr[2] for tr in traces]
        out, consumed, min_gap, max_step = orr.round(ends, traces)
        hist.append({"ends": ends, "out": out, "consumed": consumed, "min_gap": min_gap,
                     "max_step": max_step, "starts": [tr[0] for tr in traces],
                     "gap": [g.copy() for g in orr.gap]})
        x = [o.copy() for o in out]
    return hist


def test_round_zero_only_snapshots(golden):
    """test_outer_algorithms.cpp:178-200"""
    h = run(golden, 2, H())
    assert h[0]["consumed"] is None and h[0]["min_gap"] == float("inf")
    for i in range(2):
        assert h[0]["out"][i].tobytes() == h[0]["ends"][i].tobytes()
    assert h[1]["consumed"] is not None


def test_consumed_average_is_one_round_stale(golden):
    """test_outer_algorithms.cpp:202-224"""
    h = run(golden, 6, H())
    for t in range(1, 6):
        assert h[t]["consumed"].tobytes() == O.average(h[t - 1]["ends"]).tobytes()


def test_clipping_bounds_every_outer_displacement(golden):
    """test_outer_algorithms.cpp:329-350: |x' - x_t0| <= alpha * phi."""
    hyper = H(phi=1e-3)
    h = run(golden, 12, hyper)
    for t in range(1, 12):
        assert h[t]["max_step"] <= hyper.alpha * hyper.phi * (1 + 1e-15)
        for i in range(2):
            d = np.abs(h[t]["out"][i] - h[t]["starts"][i])
            assert np.all(d <= hyper.alpha * hyper.phi * (1 + 1e-15))


def test_gap_stays_at_least_one(golden):
    """test_outer_algorithms.cpp:313-327"""
    h = run(golden, 20, H())
    for t in range(1, 20):
        assert h[t]["min_gap"] >= 1.0
        assert all(np.all(g >= 1.0) for g in h[t]["gap"])


def test_ghost_consistent_keeps_workers_identical(golden):
    """test_outer_algorithms.cpp:352-370 (and :372-383 for worker-local)."""
    hg = run(golden, 8, H(ghost_consistent=True))
    for t in range(1, 8):
        assert hg[t]["out"][0].tobytes() == hg[t]["out"][1].tobytes()
    hl = run(golden, 8, H())
    assert any(hl[t]["out"][0].tobytes() != hl[t]["out"][1].tobytes() for t in range(1, 8))


def test_single_worker_degenerates_to_serial_inner_loop(golden):
    """test_outer_algorithms.cpp:286-311: with one worker, the average is the
    worker itself; penalty and clip off and beta = 0, alpha = 1 reduce the
    round to x' = x_t0 - (x_{t-1,0} - x_{t-1,tau})."""
    h = run(golden, 5, H(beta=0.0, alpha=1.0, penalty=False, clip=False), workers=1)
    for t in range(1, 5):
        prev_start, prev_end = h[t - 1]["starts"][0], h[t - 1]["ends"][0]
        expect = h[t]["starts"][0] - 1.0 * (0.0 * 0.0 + (prev_start - prev_end))
        assert np.allclose(h[t]["out"][0], expect, rtol=0, atol=1e-15)


@pytest.mark.parametrize("kind", ["slowmo", "overlap_local_sgd"])
def test_baselines_reduce_to_local_averaging(golden, kind):
    """test_outer_algorithms.cpp:226-266: SlowMo with alpha = 1, beta = 0 and
    zero-delay (instant) anchor correction both equal local averaging."""
    k = golden["delayed_momentum"]
    feats, targs = np.array(k["features"], float), np.array(k["targets"], float)
    x = [np.array(k["init"], float) for _ in range(2)]
    y = [v.copy() for v in x]
    base = OracleBaselineRound(kind, 2, 2, alpha=1.0, beta=0.0, instant=True)
    local = OracleBaselineRound("local_sgd", 2, 2)
    for _ in range(6):
        tx = [inner_loop(feats, targs, k["shards"][i], x[i], k["lr"], k["tau"]) for i in range(2)]
        ty = [inner_loop(feats, targs, k["shards"][i], y[i], k["lr"], k["tau"]) for i in range(2)]
        x, _ = base.round([t[2] for t in tx], tx)
        y, _ = local.round([t[2] for t in ty], ty)
        for i in range(2):
            assert np.allclose(x[i], y[i], rtol=0, atol=1e-15), kind
