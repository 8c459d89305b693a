"""Test-side restatement of the reference's Simulation loop for the quadratic
fixtures (TEST INFRASTRUCTURE).

  Simulation::step             proj/src/outer_algorithms.cpp:422-512
  run_inner_loop (full shard)  proj/src/inner_loop.cpp:64-103
  accumulate / sample_loss     proj/src/problems.cpp:60-69,102-126

The inner loop is host fp64 (out of scope for the GPU path).  The outer
round is pluggable: `OracleRound` runs the CPU oracle (oracle/), while the
GPU tests plug in the product's co2_round over device workers.
"""
from __future__ import annotations

import numpy as np


def shard_gradient(features: np.ndarray, targets: np.ndarray, rows, x: np.ndarray) -> np.ndarray:
    """accumulate() for the quadratic problem, rows in the given order."""
    g = np.zeros_like(x)
    for r in rows:
        f = features[r]
        dot = f[0] * x[0]
        for c in range(1, x.size):  # Eigen redux: sequential left-to-right
            dot = dot + f[c] * x[c]
        res = dot - targets[r]
        g = g + res * f
    return g / float(len(rows))


def inner_loop(features, targets, rows, x: np.ndarray, lr: float, tau: int):
    """run_inner_loop with full-shard batches (no RNG, problems.cpp:312-315).
    Returns (x_start, x_first, x_end)."""
    x_start = x.copy()
    x_first = None
    for k in range(tau):
        g = shard_gradient(features, targets, rows, x)
        x = x - lr * g
        if k == 0:
            x_first = x.copy()
    return x_start, x_first, x


class OracleBaselineRound:
    """slowmo_round / local_sgd_round / overlap_local_sgd_round
    (proj/src/outer_algorithms.cpp:213-313) on the CPU oracle, fp64."""

    def __init__(self, kind: str, workers: int, n: int, alpha=1.0, beta=0.0,
                 instant: bool = False):
        from oracle import oracle as O
        self.O, self.kind, self.g = O, kind, workers
        self.alpha, self.beta, self.instant = alpha, beta, instant
        self.m = [np.zeros(n) for _ in range(workers)]
        self.anchor = [None] * workers
        self.pending = None

    def round(self, params, traces):
        O = self.O
        if self.kind == "slowmo":
            avg = O.average(params)
            out = []
            for i in range(self.g):
                m, p, _, code, msg = O.slowmo_step(O.MODE_F64, traces[i][0], avg, self.m[i],
                                                   self.alpha, self.beta)
                assert code == 0, msg
                self.m[i] = m
                out.append(p)
            return out, avg
        if self.kind == "local_sgd":
            avg = O.average(params)
            return [avg.copy() for _ in range(self.g)], avg
        # overlap_local_sgd
        params = [p.copy() for p in params]
        consumed = None
        if self.pending is not None:
            consumed = self.pending
            for i in range(self.g):
                params[i], _, code, msg = O.overlap_correction(O.MODE_F64, params[i],
                                                               self.anchor[i], consumed)
                assert code == 0, msg
            self.pending = None
        self.anchor = [p.copy() for p in params]
        avg = O.average(self.anchor)
        if self.instant:
            consumed = avg
            for i in range(self.g):
                params[i], _, code, msg = O.overlap_correction(O.MODE_F64, params[i],
                                                               self.anchor[i], avg)
                assert code == 0, msg
        else:
            self.pending = avg
        return params, consumed


class OracleRound:
    """co2_round (proj/src/outer_algorithms.cpp:110-211) on the CPU oracle."""

    def __init__(self, workers: int, n: int, hyper, tau: int):
        from oracle import oracle as O
        self.O = O
        self.g, self.n, self.h, self.tau = workers, n, hyper, tau
        self.t = 0
        self.m = [np.zeros(n) for _ in range(workers)]
        self.gap = [np.ones(n) for _ in range(workers)]
        self.prev_x0 = [None] * workers
        self.prev_x1 = [None] * workers
        self.pending = None

    def round(self, params, traces):
        """params: list of x_{t,tau}; traces: list of (x_start, x_first, x_end).
        Returns (new params, consumed average or None, min_gap, max_step)."""
        O, h = self.O, self.h
        launched = O.average(params)  # eager simulated average, collective.cpp:50-51
        if self.t == 0:
            if h.ghost_consistent:
                b0 = O.average([tr[0] for tr in traces])
                b1 = O.average([tr[1] for tr in traces])
                self.prev_x0 = [b0.copy() for _ in range(self.g)]
                self.prev_x1 = [b1.copy() for _ in range(self.g)]
            else:
                self.prev_x0 = [tr[0].copy() for tr in traces]
                self.prev_x1 = [tr[1].copy() for tr in traces]
            self.pending = launched
            self.t = 1
            return [p.copy() for p in params], None, float("inf"), 0.0
        avg = self.pending
        hc = O.hyper(alpha=h.alpha, beta=h.beta, phi=h.phi, epsilon=h.epsilon, tau=self.tau,
                     penalty=h.penalty, clip=h.clip)
        out, min_gap, max_step = [], float("inf"), 0.0
        if h.ghost_consistent:
            b0 = O.average([tr[0] for tr in traces])
            b1 = O.average([tr[1] for tr in traces])
            r = O.worker_step_f64(b0, self.prev_x0[0], self.prev_x1[0], avg, self.m[0], hc)
            for i in range(self.g):
                self.m[i], self.gap[i] = r.m.copy(), r.gap.copy()
                self.prev_x0[i], self.prev_x1[i] = b0.copy(), b1.copy()
                out.append(r.next.copy())
            min_gap, max_step = r.min_gap, r.max_outer_step
        else:
            for i in range(self.g):
                x0, x1 = traces[i][0], traces[i][1]
                r = O.worker_step_f64(x0, self.prev_x0[i], self.prev_x1[i], avg, self.m[i], hc)
                min_gap = min(min_gap, r.min_gap)
                max_step = max(max_step, r.max_outer_step)
                self.m[i], self.gap[i] = r.m, r.gap
                self.prev_x0[i], self.prev_x1[i] = x0.copy(), x1.copy()
                out.append(r.next)
        self.pending = launched
        self.t += 1
        return out, avg, min_gap, max_step
