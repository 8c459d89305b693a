"""GPU parity of the sm_100a kernels against the CPU oracle (bitwise).

All calls go through the C ABI (libco2b200.so).  The oracle (oracle/) is the
checker only.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import oracle as O
from paper_2401_16265_b200 import _lib as L
from paper_2401_16265_b200 import co2

pytestmark = pytest.mark.gpu

MODES = [co2.MODE_F64, co2.MODE_F32, co2.MODE_BF16_MIXED]
COMBOS = [(True, True), (True, False), (False, True), (False, False)]


def to_np(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def to_dev(a: np.ndarray, dtype=None) -> torch.Tensor:
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(a.copy()).cuda()


def same(a: np.ndarray, b: np.ndarray) -> bool:
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def hyper(tau=4, penalty=True, clip=True, phi=5e-3):
    return co2.Co2Hyper(alpha=1.0, beta=0.7, phi=phi, epsilon=1e-12, penalty=penalty, clip=clip)


def ohyper(tau=4, penalty=True, clip=True, phi=5e-3):
    return O.hyper(alpha=1.0, beta=0.7, phi=phi, epsilon=1e-12, tau=tau, penalty=penalty,
                   clip=clip)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("j0", [0, 12345])
def test_synth_generator_bitwise(mode, j0):
    n = 100003
    for worker in (0, 3):
        gpu = co2.synth(mode, n, worker=worker, j0=j0)
        torch.cuda.synchronize()
        cpu = O.synth(mode, n, worker=worker, j0=j0)
        for g, c in zip(gpu, cpu):
            assert same(to_np(g), c)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("penalty,clip", COMBOS)
@pytest.mark.parametrize("n", [1, 7, 1000003])
def test_fused_step_bitwise(mode, penalty, clip, n):
    x, p0, p1, xe, m = co2.synth(mode, n)
    ox, op0, op1, oxe, om = O.synth(mode, n)
    ref = O.outer_step(mode, ox, op0, op1, oxe, om, ohyper(4, penalty, clip))
    assert ref.status == 0
    anchor = torch.empty_like(x)
    params = torch.empty_like(xe)
    gap = torch.empty_like(x)
    d = co2.outer_step(mode, x, p0, p1, xe, m, hyper(4, penalty, clip), 4, anchor_out=anchor,
                       params_out=params, gap_out=gap)
    assert same(to_np(m), ref.m)
    assert same(to_np(anchor), ref.anchor)
    assert same(to_np(params), ref.params)
    assert same(to_np(gap), ref.gap)
    assert d.min_gap == ref.diag.min_gap
    assert d.max_outer_step == ref.diag.max_outer_step
    assert d.n_clipped == ref.diag.n_clipped and d.n_floored == ref.diag.n_floored
    assert d.flags == 0
    if mode == co2.MODE_F64:  # and bit-for-bit the reference's unfused fp64 passes
        r64 = O.worker_step_f64(ox, op0, op1, oxe, om, ohyper(4, penalty, clip))
        assert same(to_np(m), r64.m) and same(to_np(params), r64.next)
        assert d.min_gap == r64.min_gap and d.max_outer_step == r64.max_outer_step


@pytest.mark.parametrize("mode", MODES)
def test_fused_divisor_sum(mode):
    """xbar as a G-worker sum divided once in the kernel (average(), param_ops.cpp:30)."""
    n, G = 65537, 3
    x, p0, p1, _, m = co2.synth(mode, n)
    ox, op0, op1, _, om = O.synth(mode, n)
    s = O.synth(mode, n, worker=0)[3]
    for w in (1, 2):
        e = O.synth(mode, n, worker=w)[3]
        if mode == O.MODE_BF16_MIXED:
            s = O.f32_to_bf16_bits(O.bf16_bits_to_f32(s) + O.bf16_bits_to_f32(e))
        else:
            s = s + e
    ref = O.outer_step(mode, ox, op0, op1, s, om, ohyper(), divisor=G)
    params = torch.empty(n, dtype=co2.LOW_TORCH[mode], device="cuda")
    co2.outer_step(mode, x, p0, p1, to_dev(s), m, hyper(), 4, divisor=G, params_out=params)
    assert same(to_np(m), ref.m) and same(to_np(params), ref.params)


@pytest.mark.parametrize("mode", MODES)
def test_fused_in_place_aliasing(mode):
    """anchor_out aliasing prev_x0 and params_out aliasing xbar (the round
    driver's layout) give the same bits as separate outputs."""
    n = 333333
    x, p0, p1, xe, m = co2.synth(mode, n)
    a2, b2 = torch.empty_like(p0), torch.empty_like(xe)
    m2 = m.clone()
    co2.outer_step(mode, x, p0, p1, xe, m2, hyper(), 4, anchor_out=a2, params_out=b2)
    co2.outer_step(mode, x, p0, p1, xe, m, hyper(), 4, anchor_out=p0, params_out=xe)
    assert same(to_np(m), to_np(m2)) and same(to_np(p0), to_np(a2))
    assert same(to_np(xe), to_np(b2))


@pytest.mark.parametrize("mode", MODES)
def test_fused_unaligned_views(mode):
    """Sub-views that break 16-byte alignment take the scalar-vector path
    and still match bit for bit."""
    n = 10001
    x, p0, p1, xe, m = co2.synth(mode, n + 1)
    ox, op0, op1, oxe, om = O.synth(mode, n + 1)
    ref = O.outer_step(mode, ox[1:], op0[1:], op1[1:], oxe[1:], om[1:], ohyper())
    mv = m[1:]
    params = torch.empty(n + 1, dtype=xe.dtype, device="cuda")[1:]
    d = co2.outer_step(mode, x[1:], p0[1:], p1[1:], xe[1:], mv, hyper(), 4, params_out=params)
    assert same(to_np(mv), ref.m) and same(to_np(params), ref.params)
    assert d.n_clipped == ref.diag.n_clipped


def test_fused_errors_follow_reference_precedence():
    n = 4096
    mode = co2.MODE_F32
    x, p0, p1, xe, m = co2.synth(mode, n)
    bad = x.clone()
    bad[1000] = float("nan")
    with pytest.raises(co2.NumericError, match="non-finite value in staleness_gap"):
        co2.outer_step(mode, bad, p0, p1, xe, m.clone(), hyper(), 4)
    mm = m.clone()
    mm[7] = float("inf")
    with pytest.raises(co2.NumericError, match="non-finite value in momentum update"):
        co2.outer_step(mode, x, p0, p1, xe, mm, hyper(), 4)
    # both: staleness_gap wins (it is checked first in the reference)
    with pytest.raises(co2.NumericError, match="staleness_gap"):
        co2.outer_step(mode, bad, p0, p1, xe, mm.clone(), hyper(), 4)
    # p1 = +inf: Lambda = finite/inf + 1 = 1, no error (reference std::max semantics)
    pp = p1.clone()
    pp[3] = float("inf")
    gap = torch.empty_like(x)
    co2.outer_step(mode, x, p0, pp, xe, m.clone(), hyper(), 4, gap_out=gap)
    assert gap[3].item() == 1.0
    pp[3] = float("nan")
    with pytest.raises(co2.NumericError, match="staleness_gap"):
        co2.outer_step(mode, x, p0, pp, xe, m.clone(), hyper(), 4)
    with pytest.raises(co2.ValidationError, match="hyper: phi must be positive"):
        co2.outer_step(mode, x, p0, p1, xe, m.clone(), co2.Co2Hyper(phi=0.0), 4)


def special_inputs(mode: int, n: int, seed: int):
    """Edge-value inputs in the mode's storage dtypes: p1 == p0 (gap hits
    the epsilon floor), x == p0 (gap exactly 1), signed zeros, subnormals,
    near-overflow magnitudes, momentum exactly at +-phi, xbar far enough off
    to clip."""
    rng = np.random.default_rng(seed)
    st = np.float64 if mode == co2.MODE_F64 else np.float32
    tiny = 1e-310 if mode == co2.MODE_F64 else 1e-39
    big = 1e300 if mode == co2.MODE_F64 else 1e37
    u = lambda s: rng.uniform(-1.0, 1.0, n) * s  # noqa: E731
    p0 = u(0.02)
    x, p1, xb, m = p0 + u(4e-3), p0 - u(1e-3), p0 - u(4e-3), u(1e-2)
    cat = np.arange(n) % 9
    p1 = np.where(cat == 1, p0, p1)
    x = np.where(cat == 2, p0, x)
    z = cat == 3
    x, p0, p1, xb, m = (np.where(z, -0.0, a) for a in (x, p0, p1, xb, m))
    s = cat == 4
    p0 = np.where(s, u(tiny), p0)
    x, p1, xb, m = (np.where(s, p0 + u(tiny), a) for a in (x, p1, xb, m))
    b = cat == 5
    p0 = np.where(b, u(big), p0)
    x = np.where(b, p0 * (1 + u(1e-3)), x)
    p1 = np.where(b, p0 * (1 - u(1e-3)), p1)
    xb = np.where(b, p0 * (1 + u(1e-3)), xb)
    m = np.where(cat == 6, np.where(u(1.0) > 0, 5e-3, -5e-3), m)
    xb = np.where(cat == 7, p0 - u(10.0), xb)
    x = np.where(cat == 8, -x, x)
    x, p0, m = (a.astype(st) for a in (x, p0, m))
    if mode == co2.MODE_BF16_MIXED:
        p1, xb = O.f32_to_bf16_bits(p1.astype(np.float32)), O.f32_to_bf16_bits(xb.astype(np.float32))
    else:
        p1, xb = p1.astype(st), xb.astype(st)
    return x, p0, p1, xb, m


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("penalty,clip", [(True, True), (False, False)])
def test_fused_special_values_bitwise(mode, seed, penalty, clip):
    """Signed zeros, subnormals (no flush: -ftz=false), near-overflow values,
    the epsilon floor and exact clip boundaries: same bits and the same
    status as the oracle, odd length for the scalar tail."""
    n = 9 * 1111 + 5
    ox, op0, op1, oxe, om = special_inputs(mode, n, seed)
    ref = O.outer_step(mode, ox, op0, op1, oxe, om, ohyper(12, penalty, clip))
    x, p0, p1, xe, m = (to_dev(a) for a in (ox, op0, op1, oxe, om))
    anchor, params, gap = torch.empty_like(x), torch.empty_like(xe), torch.empty_like(x)
    h = hyper(12, penalty, clip)
    if ref.status != 0:
        with pytest.raises((co2.NumericError, co2.ValidationError)) as ei:
            co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=anchor, params_out=params,
                           gap_out=gap)
        assert ref.message in str(ei.value)
        return
    d = co2.outer_step(mode, x, p0, p1, xe, m, h, 12, anchor_out=anchor, params_out=params,
                       gap_out=gap)
    assert same(to_np(m), ref.m) and same(to_np(anchor), ref.anchor)
    assert same(to_np(params), ref.params) and same(to_np(gap), ref.gap)
    assert (d.min_gap, d.max_outer_step, d.n_clipped, d.n_floored) == (
        ref.diag.min_gap, ref.diag.max_outer_step, ref.diag.n_clipped, ref.diag.n_floored)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("eps", [1e-12, 1e-40, 1e-46, 1e-310])
def test_gap_zero_dividend_edges(mode, eps):
    """The divisions' zero-dividend path (div_rn, div_rn_nz): n0 = 0
    against a denominator at the epsilon floor -- normal, subnormal or
    rounded to zero in the compute type (0/0: NaN, the staleness_gap error)
    -- or +inf (p1 = inf: 0/inf = 0, gap 1); delta = 0 against the gap.
    Same bits and the same status as the oracle."""
    n = 4 * 257
    st_dt = np.float64 if mode == co2.MODE_F64 else np.float32
    rng = np.random.default_rng(11)
    p0 = rng.uniform(-0.02, 0.02, n).astype(st_dt)
    x = p0.copy()                                    # n0 = 0 everywhere
    p1 = p0.astype(np.float64).copy()
    p1[1::4] = np.inf                                # av = inf
    p1[2::4] += 1e-3                                 # ordinary denominators
    xb = p0.astype(np.float64).copy()                # delta = 0 ...
    xb[3::4] -= 1e-3                                 # ... except here
    m = rng.uniform(-1e-2, 1e-2, n).astype(st_dt)
    if mode == co2.MODE_BF16_MIXED:
        p1, xb = O.f32_to_bf16_bits(p1.astype(np.float32)), O.f32_to_bf16_bits(xb.astype(np.float32))
        x = p0 = O.bf16_bits_to_f32(O.f32_to_bf16_bits(p0)).astype(np.float32)
    else:
        p1, xb = p1.astype(st_dt), xb.astype(st_dt)
    oh = O.hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=eps, tau=4)
    ref = O.outer_step(mode, x, p0, p1, xb, m, oh)
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=eps)
    dx, dp0, dp1, dxb, dm = (to_dev(a) for a in (x, p0, p1, xb, m))
    anchor, params, gap = torch.empty_like(dx), torch.empty_like(dxb), torch.empty_like(dx)
    if ref.status != 0:
        with pytest.raises((co2.NumericError, co2.ValidationError)) as ei:
            co2.outer_step(mode, dx, dp0, dp1, dxb, dm, h, 4, anchor_out=anchor,
                           params_out=params, gap_out=gap)
        assert str(ei.value) == ref.message
        return
    d = co2.outer_step(mode, dx, dp0, dp1, dxb, dm, h, 4, anchor_out=anchor, params_out=params,
                       gap_out=gap)
    assert same(to_np(dm), ref.m) and same(to_np(anchor), ref.anchor)
    assert same(to_np(params), ref.params) and same(to_np(gap), ref.gap)
    assert (d.min_gap, d.max_outer_step, d.n_clipped, d.n_floored) == (
        ref.diag.min_gap, ref.diag.max_outer_step, ref.diag.n_clipped, ref.diag.n_floored)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("where", ["momentum", "iterate"])
def test_fused_overflow_status_matches_oracle(mode, where):
    """An overflow to inf inside the step raises the same error as the
    oracle (the reference's checks, outer_algorithms.cpp:57-61,84-86)."""
    n = 4099
    ox, op0, op1, oxe, om = special_inputs(mode, n, 5)
    top = np.finfo(ox.dtype).max
    j = 2 * 9 + 1  # an ordinary coordinate; x = p0 = p1 makes its gap exactly 1
    if where == "momentum":  # m' = 0.7*top + (0.45 + 0.45)*top overflows
        ox[j] = op0[j] = 0.45 * top
        om[j], xb = top, -0.45 * top
    else:  # m' = -0.7*top is finite, x' = 0.5*top + 0.7*top is not
        ox[j] = op0[j] = 0.5 * top
        om[j], xb = -top, 0.5 * top
    if mode == co2.MODE_BF16_MIXED:
        op1[j] = O.f32_to_bf16_bits(np.array([op0[j]], np.float32))[0]
        oxe[j] = O.f32_to_bf16_bits(np.array([xb], np.float32))[0]
        if where != "momentum":  # keep delta = p0 - xbar exactly 0 in bf16 mode
            ox[j] = op0[j] = O.bf16_bits_to_f32(np.array([oxe[j]], np.uint16))[0]
    else:
        op1[j], oxe[j] = op0[j], xb
    ref = O.outer_step(mode, ox, op0, op1, oxe, om, ohyper(12, True, False))
    assert ref.status == O.NUMERIC, ref.message
    x, p0, p1, xe, m = (to_dev(a) for a in (ox, op0, op1, oxe, om))
    with pytest.raises(co2.NumericError) as ei:
        co2.outer_step(mode, x, p0, p1, xe, m, hyper(12, True, False), 12)
    assert ref.message in str(ei.value)


def test_fused_empty_and_determinism():
    mode = co2.MODE_F32
    e = torch.empty(0, device="cuda")
    d = co2.outer_step(mode, e, e, e, e, e.clone(), hyper(), 4)
    assert d.min_gap == float("inf") and d.max_outer_step == 0.0 and d.n_clipped == 0
    x, p0, p1, xe, m = co2.synth(mode, 2_000_000)
    outs = []
    for _ in range(3):
        mm = m.clone()
        d = co2.outer_step(mode, x, p0, p1, xe, mm, hyper(), 4)
        outs.append((mm.clone(), d.min_gap, d.max_outer_step, d.n_clipped, d.n_floored))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and o[1:] == outs[0][1:]


# ---------------------------------------------------------- unfused ops
@pytest.mark.parametrize("dt", [torch.float64])
def test_unfused_ops_vs_oracle(dt):
    n = 50021
    ox, op0, op1, oxe, om = O.synth(O.MODE_F64, n)
    x, p0, p1, xe, m = (to_dev(a) for a in (ox, op0, op1, oxe, om))
    gap = co2.staleness_gap(x, p0, p1, 4, 1e-12)
    assert same(to_np(gap), O.staleness_gap(ox, op0, op1, 4, 1e-12))
    delta_np = op0 - oxe
    delta = to_dev(delta_np)
    mm = co2.penalized_momentum_update(m, 0.7, gap, delta, True)
    ref_m = O.penalized_momentum_update(om, 0.7, to_np(gap), delta_np, True)
    assert same(to_np(mm), ref_m)
    xn = co2.outer_iterate(x, 1.0, mm, 5e-3, True)
    assert same(to_np(xn), O.outer_iterate(ox, 1.0, ref_m, 5e-3, True))
    xr = co2.outer_iterate(x, 1.0, mm, 5e-3, False)
    assert same(to_np(xr), O.outer_iterate(ox, 1.0, ref_m, 5e-3, False))
    c = co2.clip_elementwise(mm, 5e-3)
    assert same(to_np(c), O.clip_elementwise(ref_m, 5e-3))


def test_unfused_kats_and_errors(golden):
    k = golden["momentum"]
    t = lambda v: torch.tensor(v, dtype=torch.float64, device="cuda")  # noqa: E731
    assert co2.penalized_momentum_update(t(k["m_prev"]), k["beta"], t(k["gap"]), t(k["delta"]),
                                         True).tolist() == k["expected_penalty"]
    with pytest.raises(co2.ValidationError, match="gap coordinate below 1"):
        co2.penalized_momentum_update(t(k["m_prev"]), k["beta"], t(k["bad_gap"]), t(k["delta"]),
                                      True)
    for g in golden["staleness_gap"]:
        got = co2.staleness_gap(t(g["x_t0"]), t(g["prev_x0"]), t(g["prev_x1"]), g["tau"],
                                g["epsilon"]).cpu().numpy()
        ref = O.staleness_gap(np.array(g["x_t0"]), np.array(g["prev_x0"]), np.array(g["prev_x1"]),
                              g["tau"], g["epsilon"])
        assert same(got, ref)
    oi = golden["outer_iterate"]
    assert co2.outer_iterate(t(oi["x"]), oi["alpha"], t(oi["m"]), oi["phi"],
                             True).tolist() == oi["expected_clip"]
    with pytest.raises(co2.NumericError, match="clip_elementwise input"):
        co2.clip_elementwise(t([float("nan")]), 1.0)
    with pytest.raises(co2.NumericError, match="clip_elementwise input"):
        co2.outer_iterate(t([1.0]), 1.0, t([float("inf")]), 1.0, True)
    with pytest.raises(co2.NumericError, match="outer_iterate"):
        co2.outer_iterate(t([1.0]), 1.0, t([float("inf")]), 1.0, False)


def test_ensure_finite_names_the_context():
    """ensure_finite (param_ops.cpp:10-14; test_param_ops.cpp:162-170)."""
    for dt in (torch.float64, torch.float32, torch.bfloat16):
        ok = torch.linspace(-1, 1, 1001, device="cuda").to(dt)
        co2.ensure_finite(ok, "outer momentum")
        for bad in (float("nan"), float("inf"), float("-inf")):
            v = ok.clone()
            v[777] = bad
            with pytest.raises(co2.NumericError, match="^non-finite value in outer momentum$"):
                co2.ensure_finite(v, "outer momentum")
    co2.ensure_finite(torch.empty(0, device="cuda"), "empty")


@pytest.mark.parametrize("dt", [torch.float64, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("n", [0, 1, 7, 100_003, 3_000_001])
def test_l2_norm_bitwise_fixed_order(dt, n):
    """l2_norm (param_ops.cpp:54-60) in the fixed chunked order: bitwise the
    oracle's restatement for every dtype and size."""
    v = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(n)).to(dt)
    got = co2.l2_norm(v)
    assert got == O.l2_norm(to_np(v))


def test_abs_diff_and_l2_norm_kats_and_errors():
    """elementwise_abs_diff / l2_norm KATs (test_param_ops.cpp:147-160)."""
    t = lambda v: torch.tensor(v, dtype=torch.float64, device="cuda")  # noqa: E731
    assert co2.elementwise_abs_diff(t([1.0, -2.0, 3.5]), t([2.5, -2.0, -1.0])).tolist() == \
        [1.5, 0.0, 4.5]
    with pytest.raises(co2.ValidationError, match="elementwise_abs_diff: dimensions differ"):
        co2.elementwise_abs_diff(t([1.0, -2.0, 3.5]), t([1.0]))
    with pytest.raises(co2.NumericError, match="non-finite value in elementwise_abs_diff"):
        co2.elementwise_abs_diff(t([float("inf")]), t([1.0]))
    assert co2.l2_norm(t([3.0, 4.0])) == 5.0 and co2.l2_norm(t([0.0, 0.0, 0.0])) == 0.0
    with pytest.raises(co2.NumericError, match="l2_norm: non-finite result"):
        co2.l2_norm(t([1e300, 1e300]))
    a = torch.randn(100_001, device="cuda", dtype=torch.float32)
    b = torch.randn(100_001, device="cuda", dtype=torch.float32)
    assert torch.equal(co2.elementwise_abs_diff(a, b), (a - b).abs())


def test_average_golden_and_fixed_order(golden):
    ins = [torch.tensor(v, dtype=torch.float64, device="cuda") for v in golden["average"]["inputs"]]
    assert co2.average(ins).tolist() == golden["average"]["expected"]
    with pytest.raises(co2.NumericError, match="non-finite value in average"):
        co2.average([torch.tensor([1.0, float("inf")], dtype=torch.float64, device="cuda"),
                     torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda")])
    n = 100001
    for mode in (O.MODE_F32, O.MODE_BF16_MIXED):
        ends = [O.synth(mode, n, worker=w)[3] for w in range(5)]
        got = co2.average([to_dev(e) for e in ends])
        assert same(to_np(got), O.average_lp(ends, mode == O.MODE_BF16_MIXED))


def test_host_e2e_entry_equals_device_path():
    """co2_outer_step_host (pinned host buffers, chunked multi-stream
    pipeline) returns the same bits and diagnostics as the device entry."""
    for mode in MODES:
        n = 1_000_003
        ox, op0, op1, oxe, om = O.synth(mode, n)
        ref = O.outer_step(mode, ox, op0, op1, oxe, om, ohyper())

        def pin(a):
            t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a.copy())
            return t.pin_memory()

        hx, hp0, hp1, hxe, hm = (pin(a) for a in (ox, op0, op1, oxe, om))
        anchor = torch.empty_like(hx).pin_memory()
        params = torch.empty_like(hxe).pin_memory()
        d = co2.outer_step_host(mode, hx, hp0, hp1, hxe, hm, hyper(), 4, anchor_out=anchor,
                                params_out=params, chunk=100_000, nstreams=3)

        def back(t, like):
            a = t.numpy()
            return a.view(np.uint16) if like.dtype == np.uint16 else a

        assert same(back(hm, om), ref.m)
        assert same(back(anchor, ox), ref.anchor)
        assert same(back(params, oxe), ref.params)
        assert d.n_clipped == ref.diag.n_clipped and d.min_gap == ref.diag.min_gap
        assert d.max_outer_step == ref.diag.max_outer_step


def test_cpp_round_driver_binary():
    """A C++ co2_round loop over the plain C ABI (tests/cpp/round_example.cpp)."""
    exe = os.path.join(ROOT, "build", "round_example")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "round_example"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ROUNDS OK" in r.stdout


def test_cpp_round_host_binary():
    """The CPU-inner-loop drop-in in C++ (tests/cpp/round_host_example.cpp):
    co2_round_host with the inner loop in plain C++ on the host, bitwise
    equal to uploading the same traces by hand and calling co2_round."""
    exe = os.path.join(ROOT, "build", "round_host_example")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "round_host_example"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "HOST ROUNDS OK" in r.stdout


def test_cpp_co2sim_round_facade_replays_fixture():
    """The reference-shaped round API (include/co2sim_b200.hpp: co2sim::
    co2_round over WorkerState / OuterState / InnerTrace / CollectiveEngine /
    Clock, outer_algorithms.hpp:77-81) replays proj/fixtures/co2_dim1.json at
    tolerance 0, plus the engine audit and the ghost branch."""
    exe = os.path.join(ROOT, "build", "co2sim_round_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "co2sim_round_test"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "co2sim round facade: all passed" in r.stdout


def test_cpp_facade_binary():
    exe = os.path.join(ROOT, "build", "facade_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "facade_test"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FACADE OK" in r.stdout


def test_host_entry_concurrent_threads():
    """Two host threads driving co2_outer_step_host at once (ctypes drops the
    GIL): the per-device staging pool serialises them and both results stay
    bitwise the oracle's."""
    import threading
    mode = co2.MODE_BF16_MIXED
    n = 300_007
    jobs = []
    for w in (0, 1):
        ox, op0, op1, oxe, om = O.synth(mode, n, worker=w)
        ref = O.outer_step(mode, ox, op0, op1, oxe, om, ohyper())
        pin = lambda a: torch.from_numpy(  # noqa: E731
            a.view(np.int16) if a.dtype == np.uint16 else a.copy()).pin_memory()
        hs = [pin(a) for a in (ox, op0, op1, oxe, om)]
        jobs.append((hs, torch.empty_like(hs[0]).pin_memory(),
                     torch.empty_like(hs[3]).pin_memory(), ref))
    errs = []

    def run(job):
        (hx, hp0, hp1, hxe, hm), anchor, params, _ = job
        try:
            for _ in range(3):
                co2.outer_step_host(mode, hx, hp0, hp1, hxe, hm.clone().pin_memory(), hyper(), 4,
                                    anchor_out=anchor, params_out=params, chunk=50_000,
                                    nstreams=2)
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(j,)) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for (_, _, _, _, _), anchor, params, ref in jobs:
        assert same(anchor.numpy(), ref.anchor)
        assert same(params.numpy().view(np.uint16), ref.params)


# ------------------------------------------- global-norm clip (extension)
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [0, 1, 7, 1000003, 3_000_001])
@pytest.mark.parametrize("clip", [True, False])
def test_global_clip_bitwise(mode, n, clip):
    """EXTENSION outside the reference parity contract: the two-pass
    global-norm clip against its oracle restatement (same fixed summation
    order), bitwise -- m', anchor, params, gap, norm and diagnostics."""
    x, p0, p1, xe, m = co2.synth(mode, n)
    o = O.synth(mode, n)
    ref, rnorm = O.outer_step_global_clip(mode, *o, ohyper(12, True, clip))
    assert ref.status == 0
    anchor, params, gap = torch.empty_like(x), torch.empty_like(xe), torch.empty_like(x)
    d, norm = co2.outer_step_global_clip(mode, x, p0, p1, xe, m, hyper(12, True, clip), 12,
                                         anchor_out=anchor, params_out=params, gap_out=gap)
    assert norm == rnorm or (n == 0 and norm == 0.0)
    assert same(to_np(m), ref.m) and same(to_np(anchor), ref.anchor)
    assert same(to_np(params), ref.params) and same(to_np(gap), ref.gap)
    assert (d.min_gap, d.max_outer_step, d.n_clipped, d.n_floored, d.flags) == (
        ref.diag.min_gap, ref.diag.max_outer_step, ref.diag.n_clipped, ref.diag.n_floored, 0)
    if not clip:  # and then it is the reference-order fused step itself
        x2, p02, p12, xe2, m2 = co2.synth(mode, n)
        params2 = torch.empty_like(xe2)
        co2.outer_step(mode, x2, p02, p12, xe2, m2, hyper(12, True, False), 12,
                       params_out=params2)
        assert same(to_np(params2), to_np(params)) and same(to_np(m2), to_np(m))


def test_global_clip_grid_independent_and_unaligned():
    """The norm's bits depend on n and the mode only: 1-wave and 32-wave
    grids and the unaligned (scalar-load) path agree."""
    mode, n = co2.MODE_BF16_MIXED, 2_000_003
    res = []
    try:
        for waves in (1, 32):
            co2.check(L.lib().co2_set_grid_waves(waves))
            x, p0, p1, xe, m = co2.synth(mode, n)
            params = torch.empty_like(xe)
            _, norm = co2.outer_step_global_clip(mode, x, p0, p1, xe, m, hyper(12), 12,
                                                 params_out=params)
            res.append((norm, to_np(params), to_np(m)))
    finally:
        co2.check(L.lib().co2_set_grid_waves(32))
    x, p0, p1, xe, m = co2.synth(mode, n + 1)
    params = torch.empty(n + 1, dtype=xe.dtype, device="cuda")[1:]
    mv = m[1:]
    _, norm_u = co2.outer_step_global_clip(mode, x[1:], p0[1:], p1[1:], xe[1:], mv, hyper(12),
                                           12, params_out=params)
    ox, op0, op1, oxe, om = O.synth(mode, n + 1)
    ref, rnorm = O.outer_step_global_clip(mode, ox[1:], op0[1:], op1[1:], oxe[1:], om[1:],
                                          ohyper(12))
    assert res[0][0] == res[1][0]
    assert same(res[0][1], res[1][1]) and same(res[0][2], res[1][2])
    assert norm_u == rnorm and same(to_np(params), ref.params) and same(to_np(mv), ref.m)


def test_global_clip_errors():
    mode, n = co2.MODE_F64, 4099
    x, p0, p1, xe, m = co2.synth(mode, n)
    m.fill_(1e200)  # m' finite, ||m'||^2 overflows
    with pytest.raises(co2.NumericError, match="non-finite value in global clip norm"):
        co2.outer_step_global_clip(mode, x, p0, p1, xe, m, hyper(12), 12)
    x, p0, p1, xe, m = co2.synth(mode, n)
    m[5] = float("inf")
    with pytest.raises(co2.NumericError, match="non-finite value in momentum update"):
        co2.outer_step_global_clip(mode, x, p0, p1, xe, m, hyper(12), 12)
    with pytest.raises(co2.ValidationError, match="hyper: phi must be positive"):
        co2.outer_step_global_clip(mode, x, p0, p1, xe, m, co2.Co2Hyper(phi=0.0), 12)


@pytest.mark.parametrize("mode", MODES)
def test_fused_step_property_vs_oracle(mode):
    """hypothesis: arbitrary finite inputs in the mode's storage type (any
    magnitudes, signed zeros, subnormals, epsilon floor, clip boundaries) and
    any hyper -- the GPU step equals the oracle bit for bit, or raises the
    oracle's exact error."""
    from hypothesis import given, settings
    from hypothesis import strategies as st
    big = 1e150 if mode == co2.MODE_F64 else float(np.float32(1e30))
    w = 64 if mode == co2.MODE_F64 else 32
    fin = st.floats(allow_nan=False, allow_infinity=False, width=w, min_value=-big, max_value=big)

    @settings(max_examples=150, deadline=None, derandomize=True)
    @given(vals=st.lists(st.tuples(fin, fin, fin, fin, fin), min_size=1, max_size=40),
           alpha=st.floats(1e-3, 4.0), beta=st.floats(0.0, 0.999), phi=st.floats(1e-9, 1e3),
           eps=st.sampled_from([1e-12, 1e-30, 1.0, 1e-40, 1e-46, 1e-310]),
           tau=st.integers(1, 64),
           penalty=st.booleans(), clip=st.booleans())
    def check(vals, alpha, beta, phi, eps, tau, penalty, clip):
        st_dt = np.float64 if mode == co2.MODE_F64 else np.float32
        x, p0, p1, xb, m = (np.array(c, dtype=st_dt) for c in zip(*vals))
        if mode == co2.MODE_BF16_MIXED:
            p1, xb = O.f32_to_bf16_bits(p1), O.f32_to_bf16_bits(xb)
        oh = O.hyper(alpha=alpha, beta=beta, phi=phi, epsilon=eps, tau=tau, penalty=penalty,
                     clip=clip)
        ref = O.outer_step(mode, x, p0, p1, xb, m, oh)
        h = co2.Co2Hyper(alpha=alpha, beta=beta, phi=phi, epsilon=eps, penalty=penalty,
                         clip=clip)
        dx, dp0, dp1, dxb, dm = (to_dev(a) for a in (x, p0, p1, xb, m))
        anchor, params, gap = torch.empty_like(dx), torch.empty_like(dxb), torch.empty_like(dx)
        if ref.status != 0:
            with pytest.raises((co2.NumericError, co2.ValidationError)) as ei:
                co2.outer_step(mode, dx, dp0, dp1, dxb, dm, h, tau, anchor_out=anchor,
                               params_out=params, gap_out=gap)
            assert str(ei.value) == ref.message
            return
        d = co2.outer_step(mode, dx, dp0, dp1, dxb, dm, h, tau, anchor_out=anchor,
                           params_out=params, gap_out=gap)
        assert same(to_np(dm), ref.m) and same(to_np(anchor), ref.anchor)
        assert same(to_np(params), ref.params) and same(to_np(gap), ref.gap)
        assert (d.min_gap, d.max_outer_step, d.n_clipped, d.n_floored) == (
            ref.diag.min_gap, ref.diag.max_outer_step, ref.diag.n_clipped, ref.diag.n_floored)

    check()


BULK_VARIANTS = [10, 11, 12, 13, 14]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("variant", BULK_VARIANTS)
@pytest.mark.parametrize("n", [1, 4095, 8192, 1000003])
def test_bulk_copy_step_bitwise(mode, variant, n):
    """The TMA bulk-copy step (co2_set_fused_variant >= 10: cp.async.bulk into
    a shared-memory ring, dynamic tile claiming) gives the oracle's bits, with
    the in-place aliasing of the round driver, a worker-sum divisor and the
    gap output, and back-to-back launches on one workspace (tile counter
    self-reset)."""
    G = 2
    try:
        co2.check(L.lib().co2_set_fused_variant(variant))
        ws = co2.Workspace()
        for penalty, clip in COMBOS[:2]:
            x, p0, p1, _, m = co2.synth(mode, n)
            ox, op0, op1, _, om = O.synth(mode, n)
            s = O.synth(mode, n, worker=0)[3]
            e = O.synth(mode, n, worker=1)[3]
            if mode == O.MODE_BF16_MIXED:
                s = O.f32_to_bf16_bits(O.bf16_bits_to_f32(s) + O.bf16_bits_to_f32(e))
            else:
                s = s + e
            ref = O.outer_step(mode, ox, op0, op1, s, om, ohyper(4, penalty, clip), divisor=G)
            xe = to_dev(s)
            gap = torch.empty_like(x)
            d = co2.outer_step(mode, x, p0, p1, xe, m, hyper(4, penalty, clip), 4, divisor=G,
                               anchor_out=p0, params_out=xe, gap_out=gap, workspace=ws)
            assert same(to_np(m), ref.m) and same(to_np(p0), ref.anchor)
            assert same(to_np(xe), ref.params) and same(to_np(gap), ref.gap)
            assert (d.min_gap, d.max_outer_step, d.n_clipped, d.n_floored, d.flags) == (
                ref.diag.min_gap, ref.diag.max_outer_step, ref.diag.n_clipped,
                ref.diag.n_floored, 0)
    finally:
        co2.check(L.lib().co2_set_fused_variant(0))


@pytest.mark.parametrize("variant", [10, 12])
def test_bulk_copy_step_flags(variant):
    """Non-finite inputs raise the same flags through the bulk-copy kernel."""
    mode, n = co2.MODE_F32, 50000
    try:
        co2.check(L.lib().co2_set_fused_variant(variant))
        x, p0, p1, xe, m = co2.synth(mode, n)
        x[31337] = float("nan")
        with pytest.raises(co2.NumericError, match="staleness_gap"):
            co2.outer_step(mode, x, p0, p1, xe, m, hyper(), 4)
    finally:
        co2.check(L.lib().co2_set_fused_variant(0))
