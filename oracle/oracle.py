"""ctypes/numpy front end of the CPU oracle (oracle/libco2oracle.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, by __graft_entry__.smoke() as
the checker, and by bench.py's cpu_baseline / --impl reference legs.  The
product package never imports this module.

Every function names the reference file:line it restates (paths relative to
/root/reference/); see co2_oracle.h for the full map.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libco2oracle.so")

MODE_F64, MODE_F32, MODE_BF16_MIXED = 0, 1, 2
OK, VALIDATION, NUMERIC = 0, 2, 3
FLAG_GAP_NONFINITE, FLAG_GAP_BELOW_ONE, FLAG_M_NONFINITE = 1, 2, 4
FLAG_CLIP_NONFINITE, FLAG_X_NONFINITE = 8, 16


class ValidationError(RuntimeError):
    """Mirrors co2sim::validation_error (proj/include/co2sim/errors.hpp:8-13)."""


class NumericError(RuntimeError):
    """Mirrors co2sim::numeric_error (proj/include/co2sim/errors.hpp:15-20)."""


class Hyper(C.Structure):
    """Co2Hyper (proj/include/co2sim/outer_algorithms.hpp:17-30) + tau."""

    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("phi", C.c_double),
                ("epsilon", C.c_double), ("tau", C.c_int32), ("penalty", C.c_uint8),
                ("clip", C.c_uint8), ("ghost_consistent", C.c_uint8), ("pad", C.c_uint8)]


def hyper(alpha=1.0, beta=0.7, phi=1.0, epsilon=1e-12, tau=1, penalty=True, clip=True,
          ghost_consistent=False) -> Hyper:
    return Hyper(alpha, beta, phi, epsilon, tau, int(penalty), int(clip), int(ghost_consistent), 0)


class Diag(C.Structure):
    _fields_ = [("min_gap", C.c_double), ("max_outer_step", C.c_double),
                ("n_clipped", C.c_int64), ("n_floored", C.c_int64),
                ("flags", C.c_uint32), ("pad", C.c_uint32)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_rng_key.restype = C.c_uint64
        L.orc_rng_key.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_rng_u64_at.restype = C.c_uint64
        L.orc_rng_u64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_rng_double_at.restype = C.c_double
        L.orc_rng_double_at.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_rng_below_at.restype = C.c_uint64
        L.orc_rng_below_at.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_rng_fill_u64.argtypes = [C.c_uint64, C.c_uint64, I64, P]
        L.orc_f32_to_bf16.restype = C.c_uint16
        L.orc_f32_to_bf16.argtypes = [C.c_float]
        L.orc_average_f64.argtypes = [I, P, I64, P]
        L.orc_clip_f64.argtypes = [I64, P, D, P]
        L.orc_hyper_validate.argtypes = [C.POINTER(Hyper)]
        L.orc_staleness_gap_f64.argtypes = [I64, P, P, P, I, D, P]
        L.orc_penalized_momentum_f64.argtypes = [I64, P, D, P, P, I, P]
        L.orc_outer_iterate_f64.argtypes = [I64, P, D, P, D, I, P]
        L.orc_worker_step_f64.argtypes = [I64, P, P, P, P, P, C.POINTER(Hyper), P, P,
                                          C.POINTER(C.c_double), C.POINTER(C.c_double), I]
        L.orc_outer_step.argtypes = [I, I64, P, P, P, P, I, P, P, P, P, C.POINTER(Hyper),
                                     C.POINTER(Diag)]
        L.orc_outer_step_global_clip.argtypes = [I, I64, P, P, P, P, I, P, P, P, P,
                                                 C.POINTER(Hyper), C.POINTER(Diag),
                                                 C.POINTER(C.c_double)]
        L.orc_gc_chunk.argtypes = [I64, I]
        L.orc_l2_norm.argtypes = [I, I64, P]
        L.orc_l2_norm.restype = D
        L.orc_gc_chunk.restype = I64
        L.orc_diag_status.argtypes = [C.POINTER(Diag)]
        L.orc_average_lp.argtypes = [I, I, P, I64, P]
        L.orc_synth.argtypes = [I, C.c_uint64, I, I64, I64, P, P, P, P, P]
        _lib = L
    return _lib


def _raise(code: int) -> None:
    if code == OK:
        return
    msg = lib().orc_last_error().decode()
    if code == VALIDATION:
        raise ValidationError(msg)
    if code == NUMERIC:
        raise NumericError(msg)
    raise RuntimeError(f"oracle status {code}: {msg}")


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ RNG
class RngStream:
    """RngStream (proj/include/co2sim/rng.hpp:12-54)."""

    def __init__(self, seed: int, stream: int):
        self.key = lib().orc_rng_key(seed, stream)
        self.counter = 0

    def next_u64(self) -> int:
        v = lib().orc_rng_u64_at(self.key, self.counter)
        self.counter += 1
        return v

    def next_double(self) -> float:
        v = lib().orc_rng_double_at(self.key, self.counter)
        self.counter += 1
        return v

    def next_below(self, n: int) -> int:
        v = lib().orc_rng_below_at(self.key, self.counter, n)
        self.counter += 1
        return v


# ------------------------------------------------------------ bf16
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (NaN -> 0x7fff)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = 0x7FFF
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------ param ops
def average(contributions) -> np.ndarray:
    """average (proj/src/param_ops.cpp:16-33), fp64."""
    if len(contributions) == 0:
        raise ValidationError("average: empty contribution list")
    cs = [_f64(c) for c in contributions]
    n = cs[0].size
    if any(c.size != n for c in cs):
        raise ValidationError("average: contribution dimensions differ")
    ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
    out = np.empty(n, np.float64)
    _raise(lib().orc_average_f64(len(cs), ptrs, n, _p(out)))
    return out


def average_lp(contributions, bf16: bool) -> np.ndarray:
    """average() in fp32 arithmetic stored in the params dtype."""
    dt = np.uint16 if bf16 else np.float32
    cs = [np.ascontiguousarray(c, dtype=dt) for c in contributions]
    ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
    out = np.empty(cs[0].size, dt)
    _raise(lib().orc_average_lp(int(bf16), len(cs), ptrs, cs[0].size, _p(out)))
    return out


def clip_elementwise(v, phi: float) -> np.ndarray:
    """clip_elementwise (proj/src/param_ops.cpp:35-43)."""
    v = _f64(v)
    out = np.empty_like(v)
    _raise(lib().orc_clip_f64(v.size, _p(v), phi, _p(out)))
    return out


# ------------------------------------------------------------ outer ops
def validate(h: Hyper) -> None:
    """Co2Hyper::validate (proj/src/outer_algorithms.cpp:37-46)."""
    _raise(lib().orc_hyper_validate(C.byref(h)))


def staleness_gap(x_t0, prev_x0, prev_x1, tau: int, epsilon: float) -> np.ndarray:
    """staleness_gap (proj/src/outer_algorithms.cpp:48-64)."""
    a, b, c = _f64(x_t0), _f64(prev_x0), _f64(prev_x1)
    if tau < 1:
        raise ValidationError("staleness_gap: tau must be >= 1")
    if not epsilon > 0.0:
        raise ValidationError("staleness_gap: epsilon must be positive")
    if a.size != b.size or b.size != c.size:
        raise ValidationError("staleness_gap: dimensions differ")
    out = np.empty_like(a)
    _raise(lib().orc_staleness_gap_f64(a.size, _p(a), _p(b), _p(c), tau, epsilon, _p(out)))
    return out


def penalized_momentum_update(m_prev, beta: float, gap, delta, penalty: bool) -> np.ndarray:
    """penalized_momentum_update (proj/src/outer_algorithms.cpp:66-90)."""
    m, g, d = _f64(m_prev), _f64(gap), _f64(delta)
    if beta < 0.0 or beta >= 1.0:
        raise ValidationError("momentum update: beta must lie in [0, 1)")
    if m.size != d.size:
        raise ValidationError("momentum update: dimensions differ")
    if penalty and g.size != d.size:
        raise ValidationError("momentum update: gap dimension differs")
    out = np.empty_like(m)
    _raise(lib().orc_penalized_momentum_f64(m.size, _p(m), beta, _p(g), _p(d), int(penalty),
                                            _p(out)))
    return out


def outer_iterate(x_t0, alpha: float, m, phi: float, clip: bool) -> np.ndarray:
    """outer_iterate (proj/src/outer_algorithms.cpp:92-108)."""
    x, mm = _f64(x_t0), _f64(m)
    if not alpha > 0.0:
        raise ValidationError("outer_iterate: alpha must be positive")
    if x.size != mm.size:
        raise ValidationError("outer_iterate: dimensions differ")
    out = np.empty_like(x)
    _raise(lib().orc_outer_iterate_f64(x.size, _p(x), alpha, _p(mm), phi, int(clip), _p(out)))
    return out


@dataclass
class StepResult:
    m: np.ndarray
    next: np.ndarray
    gap: np.ndarray | None
    min_gap: float
    max_outer_step: float


def worker_step_f64(x_t0, prev_x0, prev_x1, avg, m, h: Hyper, threads: int = 1,
                    want_gap: bool = True) -> StepResult:
    """co2_round's per-worker body (proj/src/outer_algorithms.cpp:186-196),
    unfused fp64 with the reference's temporaries."""
    x, p0, p1, a = _f64(x_t0), _f64(prev_x0), _f64(prev_x1), _f64(avg)
    mm = _f64(m).copy()
    nxt = np.empty_like(x)
    gap = np.empty_like(x) if want_gap else None
    mg, ms = C.c_double(), C.c_double()
    _raise(lib().orc_worker_step_f64(x.size, _p(x), _p(p0), _p(p1), _p(a), _p(mm), C.byref(h),
                                     _p(nxt), _p(gap), C.byref(mg), C.byref(ms), threads))
    return StepResult(mm, nxt, gap, mg.value, ms.value)


@dataclass
class FusedResult:
    m: np.ndarray
    anchor: np.ndarray
    params: np.ndarray
    gap: np.ndarray
    diag: Diag
    status: int
    message: str


def outer_step(mode: int, x_t0, p0, p1, xbar, m, h: Hyper, divisor: int = 1) -> FusedResult:
    """Fused same-op-order step in the GPU's compute type.
    Inputs must already be in the mode's storage dtypes (bf16 as uint16
    bits).  Never raises on flags; returns status + message instead."""
    st = np.float64 if mode == MODE_F64 else np.float32
    lo = np.float64 if mode == MODE_F64 else (np.uint16 if mode == MODE_BF16_MIXED else np.float32)
    x = np.ascontiguousarray(x_t0, st)
    q0 = np.ascontiguousarray(p0, st)
    q1 = np.ascontiguousarray(p1, lo)
    xb = np.ascontiguousarray(xbar, lo)
    mm = np.array(m, dtype=st, copy=True)
    n = x.size
    anchor = np.empty(n, st)
    params = np.empty(n, lo)
    gap = np.empty(n, st)
    d = Diag()
    code = lib().orc_outer_step(mode, n, _p(x), _p(q0), _p(q1), _p(xb), divisor, _p(mm),
                                _p(anchor), _p(params), _p(gap), C.byref(h), C.byref(d))
    msg = lib().orc_last_error().decode() if code else ""
    if code not in (OK, VALIDATION, NUMERIC):
        raise RuntimeError(msg)
    return FusedResult(mm, anchor, params, gap, d, code, msg)


def outer_step_global_clip(mode: int, x_t0, p0, p1, xbar, m, h: Hyper, divisor: int = 1):
    """EXTENSION outside the reference parity contract: the global-norm clip
    in the GPU's fixed summation order (orc_outer_step_global_clip).
    Returns (FusedResult, norm)."""
    st = np.float64 if mode == MODE_F64 else np.float32
    lo = np.float64 if mode == MODE_F64 else (np.uint16 if mode == MODE_BF16_MIXED else np.float32)
    x = np.ascontiguousarray(x_t0, st)
    q0 = np.ascontiguousarray(p0, st)
    q1 = np.ascontiguousarray(p1, lo)
    xb = np.ascontiguousarray(xbar, lo)
    mm = np.array(m, dtype=st, copy=True)
    n = x.size
    anchor, params, gap = np.empty(n, st), np.empty(n, lo), np.empty(n, st)
    d = Diag()
    norm = C.c_double()
    code = lib().orc_outer_step_global_clip(mode, n, _p(x), _p(q0), _p(q1), _p(xb), divisor,
                                            _p(mm), _p(anchor), _p(params), _p(gap), C.byref(h),
                                            C.byref(d), C.byref(norm))
    msg = lib().orc_last_error().decode() if code else ""
    if code not in (OK, VALIDATION, NUMERIC):
        raise RuntimeError(msg)
    return FusedResult(mm, anchor, params, gap, d, code, msg), norm.value


def l2_norm(v: np.ndarray) -> float:
    """l2_norm (proj/src/param_ops.cpp:54-60) in the GPU's fixed order; bf16
    inputs as uint16 bit patterns."""
    dt = {np.dtype(np.float64): 0, np.dtype(np.float32): 1, np.dtype(np.uint16): 2}[v.dtype]
    a = np.ascontiguousarray(v)
    return lib().orc_l2_norm(dt, a.size, _p(a))


def gc_chunk(n: int, v: int) -> int:
    return lib().orc_gc_chunk(n, v)


def outer_step_ghost(mode: int, anchor, p0, p1sum, p1_div: int, xsum, xdiv: int, ghost: int, m,
                     h: Hyper) -> FusedResult:
    """Ghost-consistent / sharded step (outer_algorithms.cpp:161-184); the
    FusedResult's `anchor` field holds x_{t+1,0} and `gap` the Lambda; the
    x_t0 used (next prev_x0) is returned as result.bar0."""
    lib().orc_outer_step_ghost.argtypes = [C.c_int, C.c_int64] + [C.c_void_p] * 3 + \
        [C.c_int, C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 5 + \
        [C.POINTER(Hyper), C.POINTER(Diag)]
    st = np.float64 if mode == MODE_F64 else np.float32
    lo = np.float64 if mode == MODE_F64 else (np.uint16 if mode == MODE_BF16_MIXED else np.float32)
    an = np.ascontiguousarray(anchor, st)
    q0 = np.ascontiguousarray(p0, st)
    q1 = np.ascontiguousarray(p1sum, lo)
    xs = np.ascontiguousarray(xsum, lo)
    mm = np.array(m, dtype=st, copy=True)
    n = q0.size
    a_out, b0, gap = np.empty(n, st), np.empty(n, st), np.empty(n, st)
    params = np.empty(n, lo)
    d = Diag()
    code = lib().orc_outer_step_ghost(mode, n, _p(an), _p(q0), _p(q1), p1_div, _p(xs), xdiv, ghost,
                                      _p(mm), _p(a_out), _p(b0), _p(params), _p(gap), C.byref(h),
                                      C.byref(d))
    msg = lib().orc_last_error().decode() if code else ""
    r = FusedResult(mm, a_out, params, gap, d, code, msg)
    r.bar0 = b0
    return r


def _dts(mode):
    st = np.float64 if mode == MODE_F64 else np.float32
    lo = np.float64 if mode == MODE_F64 else (np.uint16 if mode == MODE_BF16_MIXED else np.float32)
    return st, lo


def slowmo_step(mode: int, x_start, xbar, m, alpha: float, beta: float, divisor: int = 1):
    """slowmo_round per-worker body (proj/src/outer_algorithms.cpp:228-236).
    Returns (m', params, diag, status, message)."""
    st, lo = _dts(mode)
    L = lib()
    L.orc_slowmo_step.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int,
                                  C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                  C.POINTER(Diag)]
    x = np.ascontiguousarray(x_start, st)
    xb = np.ascontiguousarray(xbar, lo)
    mm = np.array(m, dtype=st, copy=True)
    out = np.empty(x.size, lo)
    d = Diag()
    code = L.orc_slowmo_step(mode, x.size, _p(x), _p(xb), divisor, _p(mm), _p(out), alpha, beta,
                             C.byref(d))
    return mm, out, d, code, (L.orc_last_error().decode() if code else "")


def local_sgd_step(mode: int, x_start, xbar, divisor: int = 1):
    """local_sgd_round per-worker body (proj/src/outer_algorithms.cpp:251-256)."""
    st, lo = _dts(mode)
    L = lib()
    L.orc_local_sgd_step.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int,
                                     C.c_void_p, C.POINTER(Diag)]
    x = np.ascontiguousarray(x_start, st)
    xb = np.ascontiguousarray(xbar, lo)
    out = np.empty(x.size, lo)
    d = Diag()
    code = L.orc_local_sgd_step(mode, x.size, _p(x), _p(xb), divisor, _p(out), C.byref(d))
    return out, d, code


def overlap_correction(mode: int, params, anchor, xbar, divisor: int = 1):
    """overlap_local_sgd correction (proj/src/outer_algorithms.cpp:277-280)."""
    st, lo = _dts(mode)
    L = lib()
    L.orc_overlap_correction.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int, C.POINTER(Diag)]
    p = np.array(params, dtype=lo, copy=True)
    a = np.ascontiguousarray(anchor, st)
    xb = np.ascontiguousarray(xbar, lo)
    d = Diag()
    code = L.orc_overlap_correction(mode, p.size, _p(p), _p(a), _p(xb), divisor, C.byref(d))
    return p, d, code, (L.orc_last_error().decode() if code else "")


def synth(mode: int, n: int, seed: int = 7, worker: int = 0, j0: int = 0):
    """Synthetic inputs of SURVEY.md 8(d): returns (x_t0, p0, p1, x_end, m)."""
    st = np.float64 if mode == MODE_F64 else np.float32
    lo = np.float64 if mode == MODE_F64 else (np.uint16 if mode == MODE_BF16_MIXED else np.float32)
    x, p0, m = np.empty(n, st), np.empty(n, st), np.empty(n, st)
    p1, xe = np.empty(n, lo), np.empty(n, lo)
    lib().orc_synth(mode, seed, worker, j0, n, _p(x), _p(p0), _p(p1), _p(xe), _p(m))
    return x, p0, p1, xe, m


def to_f64(a: np.ndarray) -> np.ndarray:
    """Widen a storage buffer (bf16 bits as uint16) to fp64 exactly."""
    if a.dtype == np.uint16:
        return bf16_bits_to_f32(a).astype(np.float64)
    return a.astype(np.float64)


def rng_u64_array(seed: int, stream: int, j0: int, n: int) -> np.ndarray:
    """Vectorized RngStream draws j0..j0+n-1 (rng.hpp:12-54), numpy uint64."""
    with np.errstate(over="ignore"):
        key = np.uint64(lib().orc_rng_key(seed, stream))
        g = np.uint64(0x9E3779B97F4A7C15)
        z = key + (np.arange(j0, j0 + n, dtype=np.uint64) + np.uint64(1)) * g
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rng_sym_array(seed: int, stream: int, j0: int, n: int) -> np.ndarray:
    """2U-1 in double for draws j0..j0+n-1."""
    u = (rng_u64_array(seed, stream, j0, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return 2.0 * u - 1.0
