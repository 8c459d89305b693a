"""Global-norm clip EXTENSION (outside the reference parity contract; the
reference clips coordinate-wise, proj/src/param_ops.cpp:35-43): the CPU
restatement's own properties.  GPU parity is in test_gpu_parity.py."""
import numpy as np
import pytest

from oracle import oracle as O

H = dict(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, tau=12)


@pytest.mark.parametrize("mode", [O.MODE_F64, O.MODE_F32, O.MODE_BF16_MIXED])
@pytest.mark.parametrize("n", [0, 1, 7, 100003, 1_500_001])
def test_norm_and_clip_off_identity(mode, n):
    a = O.synth(mode, n)
    r, norm = O.outer_step_global_clip(mode, *a, O.hyper(**H))
    assert r.status == 0
    ref = float(np.sqrt(np.sum(r.m.astype(np.float64) ** 2)))
    assert norm == pytest.approx(ref, rel=1e-14, abs=0.0)
    # clip off: bit-for-bit the reference-order fused step without clip
    h2 = O.hyper(clip=False, **H)
    r2, _ = O.outer_step_global_clip(mode, *a, h2)
    r3 = O.outer_step(mode, *a, h2)
    for f in ("m", "anchor", "params", "gap"):
        assert getattr(r2, f).tobytes() == getattr(r3, f).tobytes()
    # m' itself never depends on the clip
    assert r.m.tobytes() == r3.m.tobytes()


def test_f64_scaling_semantics():
    n = 50_001
    a = O.synth(O.MODE_F64, n)
    r, norm = O.outer_step_global_clip(O.MODE_F64, *a, O.hyper(**H))
    assert norm > H["phi"] and r.diag.n_clipped == n
    sc = H["phi"] / norm
    x = a[0]
    expect = x - H["alpha"] * (r.m * sc)
    assert expect.tobytes() == r.params.tobytes() == r.anchor.tobytes()
    # the clipped update has global norm phi (up to rounding)
    assert float(np.linalg.norm(r.m * sc)) == pytest.approx(H["phi"], rel=1e-12)


def test_below_threshold_is_untouched():
    n = 1000
    a = O.synth(O.MODE_F32, n)
    h = O.hyper(alpha=1.0, beta=0.7, phi=1e9, epsilon=1e-12, tau=12)
    r, norm = O.outer_step_global_clip(O.MODE_F32, *a, h)
    assert norm < 1e9 and r.diag.n_clipped == 0
    r3 = O.outer_step(O.MODE_F32, *a, O.hyper(alpha=1.0, beta=0.7, phi=1e9, epsilon=1e-12,
                                              tau=12, clip=False))
    assert r.params.tobytes() == r3.params.tobytes()


def test_norm_overflow_and_precedence():
    n = 64
    x, p0, p1, xb, m = (np.asarray(v).copy() for v in O.synth(O.MODE_F64, n))
    m[:] = 1e200  # beta*m finite, m'^2 overflows
    r, norm = O.outer_step_global_clip(O.MODE_F64, x, p0, p1, xb, m, O.hyper(**H))
    assert not np.isfinite(norm)
    assert r.status == O.NUMERIC and r.message == "non-finite value in global clip norm"
    m[3] = np.inf  # a non-finite momentum is reported first (reference order)
    r, _ = O.outer_step_global_clip(O.MODE_F64, x, p0, p1, xb, m, O.hyper(**H))
    assert r.message == "non-finite value in momentum update"


def test_chunking_is_grid_independent_and_bounded():
    for v in (2, 4, 8):
        for n in (0, 1, 10**6, 1_300_000_000, 7_000_000_000):
            c = O.gc_chunk(n, v)
            assert c % (v * 256) == 0 and c >= v * 256 * 16
            assert (n + c - 1) // c <= 32768


def test_product_chunk_formula_matches_oracle():
    """The library's summation chunk (pure host arithmetic, no GPU call)
    equals the oracle restatement's, so both sum in the same order."""
    from paper_2401_16265_b200 import _lib as L
    lib = L.lib()
    for mode, v in ((0, 2), (1, 4), (2, 8)):
        for n in (0, 1, 7, 8191, 100003, 3_000_001, 1_300_000_000, 7_000_000_000):
            assert lib.co2_global_clip_chunk(mode, n) == O.gc_chunk(n, v)


def test_global_clip_property():
    """hypothesis: for arbitrary finite fp64 inputs the global-clip oracle's
    m' equals the reference-order step's, its norm is the fp64 norm of m'
    to rounding, and the update is x_t0 - alpha * m' * min(1, phi/norm)."""
    from hypothesis import given, settings
    from hypothesis import strategies as st
    fin = st.floats(allow_nan=False, allow_infinity=False, width=64, min_value=-1e100,
                    max_value=1e100)

    @settings(max_examples=200, deadline=None, derandomize=True)
    @given(vals=st.lists(st.tuples(fin, fin, fin, fin, fin), min_size=1, max_size=3000),
           alpha=st.floats(1e-3, 4.0), beta=st.floats(0.0, 0.999), phi=st.floats(1e-9, 1e3))
    def check(vals, alpha, beta, phi):
        x, p0, p1, xb, m = (np.array(c, dtype=np.float64) for c in zip(*vals))
        h = O.hyper(alpha=alpha, beta=beta, phi=phi, epsilon=1e-12, tau=4)
        r, norm = O.outer_step_global_clip(O.MODE_F64, x, p0, p1, xb, m, h)
        ref = O.outer_step(O.MODE_F64, x, p0, p1, xb, m,
                           O.hyper(alpha=alpha, beta=beta, phi=phi, epsilon=1e-12, tau=4,
                                   clip=False))
        if ref.status != 0 or r.status != 0:
            return  # overflow / non-finite paths are covered by the error tests
        assert r.m.tobytes() == ref.m.tobytes()
        exact = float(np.sqrt(np.sum(r.m * r.m)))
        assert norm == pytest.approx(exact, rel=1e-13, abs=0.0)
        sc = phi / norm if norm > phi else 1.0
        assert r.params.tobytes() == (x - alpha * (r.m * sc)).tobytes()

    check()
