"""The reference's acceptance criteria 4 and 8 (proj/tests/acceptance.cpp)
through the product co2_round on the GPU (LOCAL engine, simulated workers,
F64 = the reference's precision).  The inner loop is the synthetic
x <- x - gamma * g stand-in (the reference's problems are out of scope,
SURVEY.md 8); both criteria are properties of the outer update that hold for
any inner gradients."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2401_16265_b200 import _lib as L
from paper_2401_16265_b200 import co2

pytestmark = pytest.mark.gpu


def synthetic_grad_sum(n, worker, t, tau, scale=1.0):
    """Sum over the round's tau inner steps of the synthetic gradients the
    inner-step kernel drew (co2_synthetic_inner_step: stream (5 << 32) |
    worker, draw j of global step s at counter s*n + j), in fp64."""
    s = np.zeros(n)
    for k in range(tau):
        step = t * tau + k
        s = s + scale * O.rng_sym_array(7, (5 << 32) | worker, step * n, n)
    return s


def to_np(t):
    return t.detach().cpu().numpy().copy()


def test_acceptance_criterion4_telescoping_identity():
    """acceptance.cpp:118-163: with penalty and clip off and a constant inner
    rate gamma, ybar_t = xbar_t0 + beta/(1-beta) (xbar_t0 - xbar_{t-1,0})
    telescopes, ybar_{t+1} - ybar_t = -(alpha gamma / (1 - beta)) S_{t-1},
    S_t the worker-averaged sum of round-t inner gradients; residual <= 1e-10
    for t >= 2.  alpha .8, beta .6, gamma .05, 4 workers, tau 3, 50 rounds."""
    alpha, beta, gamma = 0.8, 0.6, 0.05
    G, tau, rounds, n = 4, 3, 50, 4099
    hyper = co2.Co2Hyper(alpha=alpha, beta=beta, phi=1.0, epsilon=1e-12, penalty=False,
                         clip=False)
    eng = co2.CollectiveEngine(G, transport="local")
    ws = [co2.Worker(co2.MODE_F64, n, co2.synth(co2.MODE_F64, n, worker=i)[3])
          for i in range(G)]
    xbar0, grad_sum = [], []
    for t in range(rounds):
        starts = []
        for i, w in enumerate(ws):
            w.snapshot_start()
            torch.cuda.synchronize()
            starts.append(to_np(w.buffer(L.BUF_ANCHOR)))  # x_{t,0}
            for k in range(tau):
                co2.synthetic_inner_step(w.params, lr=gamma, worker=i, step=t * tau + k)
                if k == 0:
                    w.snapshot_first()
        co2.co2_round(ws, eng, hyper, tau)
        s = starts[0].copy()
        for x in starts[1:]:
            s = s + x
        xbar0.append(s / G)
        gs = synthetic_grad_sum(n, 0, t, tau)
        for i in range(1, G):
            gs = gs + synthetic_grad_sum(n, i, t, tau)
        grad_sum.append(gs / G)

    def ybar(t):
        return xbar0[t] + (beta / (1.0 - beta)) * (xbar0[t] - xbar0[t - 1])

    coeff = alpha * gamma / (1.0 - beta)
    worst = 0.0
    for t in range(2, rounds - 1):
        resid = ybar(t + 1) - ybar(t) + coeff * grad_sum[t - 1]
        worst = max(worst, float(np.max(np.abs(resid))))
    assert worst <= 1e-10, worst
    for w in ws:
        w.close()
    eng.close()


@pytest.mark.parametrize("alpha,beta,phi", [(0.5, 0.5, 1.0), (2.0, 0.9, 0.02)])
@pytest.mark.parametrize("het", [0.0, 1.0])
@pytest.mark.parametrize("batch", [1, 4])
@pytest.mark.parametrize("scale", [1.0, 50.0])
def test_acceptance_criterion8_invariant_matrix(alpha, beta, phi, het, batch, scale):
    """acceptance.cpp:521-573: on every applied round min_gap is finite and
    >= 1 and max_outer_step <= alpha * phi * (1 + 1e-15), over the (alpha,
    beta, phi) matrix x worker heterogeneity x batch regime.  Synthetic
    stand-ins: heterogeneity scales worker i's gradients by (1 + het * i),
    the batch regime is the number of draws summed per step (repeat), and two
    gradient scales cover the unclipped and the clip-saturated regimes.
    4 workers, tau 3, 40 rounds, F64.  The reference's quadratic keeps
    |x| = O(1), where the rounding of x' = x - alpha*c is inside its 1e-15
    slack; the synthetic random walk drifts to |x| >> 1, so the bound adds
    that rounding explicitly: 2^-52 * max|x'| (one rounding of x' plus one
    of |x' - x|, each at most half an ulp of |x'|)."""
    G, tau, rounds, n = 4, 3, 40, 8191
    hyper = co2.Co2Hyper(alpha=alpha, beta=beta, phi=phi, epsilon=1e-12)
    eng = co2.CollectiveEngine(G, transport="local")
    ws = [co2.Worker(co2.MODE_F64, n, co2.synth(co2.MODE_F64, n, worker=i)[3])
          for i in range(G)]
    bound = alpha * phi * (1.0 + 1e-15)
    checked = clipped_rounds = 0
    for t in range(rounds):
        for i, w in enumerate(ws):
            w.snapshot_start()
            for k in range(tau):
                co2.synthetic_inner_step(w.params, lr=0.05, scale=scale * (1.0 + het * i) / batch,
                                         worker=i, step=t * tau + k, repeat=batch)
                if k == 0:
                    w.snapshot_first()
        r = co2.co2_round(ws, eng, hyper, tau)
        if not r.outer_applied:
            continue
        checked += 1
        assert np.isfinite(r.min_gap) and r.min_gap >= 1.0, (t, r.min_gap)
        xmax = max(float(w.params.abs().max()) for w in ws)
        assert r.max_outer_step <= bound + 2.0 ** -52 * xmax, (t, r.max_outer_step, bound, xmax)
        if xmax <= 1.0:  # the reference's O(1) regime: its bound as written
            assert r.max_outer_step <= bound, (t, r.max_outer_step, bound)
        clipped_rounds += r.n_clipped > 0
    assert checked == rounds - 1
    if scale == 50.0:  # the saturated regime really exercises the clip bound
        assert clipped_rounds == checked
    for w in ws:
        w.close()
    eng.close()
