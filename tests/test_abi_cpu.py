"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/co2_b200.h declares, validates like the reference, and its host-side
timing model reproduces the reference's KATs."""
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2401_16265_b200 import _lib as L
from paper_2401_16265_b200 import co2


def header_symbols():
    with open(os.path.join(ROOT, "include", "co2_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(co2_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (co2_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(syms) == set(L.SIGNATURES), set(syms) ^ set(L.SIGNATURES)
    lib = L.lib()
    for s in syms:
        assert hasattr(lib, s)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out


def test_hyper_validation_messages():
    """Co2Hyper::validate messages (proj/src/outer_algorithms.cpp:37-46)."""
    co2.Co2Hyper().validate()
    for kw, msg in [({"alpha": 0.0}, "hyper: alpha must be positive"),
                    ({"beta": 1.0}, "hyper: beta must lie in [0, 1)"),
                    ({"beta": -0.1}, "hyper: beta must lie in [0, 1)"),
                    ({"phi": 0.0}, "hyper: phi must be positive"),
                    ({"epsilon": 0.0}, "hyper: epsilon must be positive")]:
        with pytest.raises(co2.ValidationError) as e:
            co2.Co2Hyper(**kw).validate()
        assert str(e.value) == msg


def test_outer_step_validates_before_launch():
    """Host-checkable validation happens before any device work."""
    import ctypes as C
    h = co2.Co2Hyper(alpha=-1.0).c(4)
    st = L.lib().co2_outer_step(L.MODE_F32, 0, None, None, None, None, 1, None, None, None, None,
                                C.byref(h), None, None)
    assert st == L.ERR_VALIDATION
    assert L.lib().co2_last_error().decode() == "hyper: alpha must be positive"
    h = co2.Co2Hyper().c(0)
    st = L.lib().co2_outer_step(L.MODE_F32, 0, None, None, None, None, 1, None, None, None, None,
                                C.byref(h), None, None)
    assert st == L.ERR_VALIDATION
    assert L.lib().co2_last_error().decode() == "staleness_gap: tau must be >= 1"


def test_null_buffers_are_rejected_before_launch():
    """Null device buffers with n > 0 are a validation error at the ABI, not
    an illegal address on the GPU (checked before any device work)."""
    import ctypes as C
    lib = L.lib()
    fake = C.c_void_p(0x1000)  # never dereferenced: validation fails first
    h = co2.Co2Hyper().c(4)
    cases = [
        lambda: lib.co2_outer_step(L.MODE_F32, 8, None, fake, fake, fake, 1, fake, None, None,
                                   None, C.byref(h), fake, None),
        lambda: lib.co2_outer_step_global_clip(L.MODE_F32, 8, fake, fake, None, fake, 1, fake,
                                               None, None, None, C.byref(h), fake, None),
        lambda: lib.co2_staleness_gap(L.DTYPE_F64, 8, fake, None, fake, 4, 1e-12, fake, fake,
                                      None),
        lambda: lib.co2_penalized_momentum(L.DTYPE_F64, 8, fake, 0.5, fake, None, 1, fake, fake,
                                           None),
        lambda: lib.co2_outer_iterate(L.DTYPE_F64, 8, fake, 1.0, None, 1.0, 1, fake, fake, None),
        lambda: lib.co2_clip_elementwise(L.DTYPE_F64, 8, None, 1.0, fake, fake, None),
        lambda: lib.co2_sub(L.DTYPE_F64, 8, fake, None, fake, None),
        lambda: lib.co2_convert(L.DTYPE_F32, None, L.DTYPE_F64, fake, 8, None),
        lambda: lib.co2_aar_create_local(None, 2),
        lambda: lib.co2_aar_create_p2p(None, 0, 2, 0),
    ]
    for f in cases:
        assert f() == L.ERR_VALIDATION
        assert "null" in lib.co2_last_error().decode()
    # round drivers: a null engine / worker array / worker is rejected up front
    arr = (C.c_void_p * 2)(None, None)
    res = L.RoundResult()
    for f in (lambda: lib.co2_round(arr, 2, None, C.byref(h), None, 1, C.byref(res)),
              lambda: lib.co2_local_sgd_round(arr, 2, fake, None, 1, C.byref(res)),
              lambda: lib.co2_slowmo_round(arr, 2, fake, 1.0, 0.5, None, 1, C.byref(res)),
              lambda: lib.co2_round_finish(arr, 2, None, C.byref(res))):
        assert f() == L.ERR_VALIDATION
        msg = lib.co2_last_error().decode()
        assert "bad arguments" in msg or "null worker" in msg, msg


def test_allreduce_time_ring_formula(golden):
    """proj/tests/test_timing_model.cpp:23-47"""
    k = golden["allreduce_time"]
    s = co2.ClusterSpec(workers=k["workers"], latency=k["latency"], param_bytes=k["param_bytes"],
                        inter_bandwidth=k["bandwidth"])
    assert co2.allreduce_time(s) == pytest.approx(k["expected"], rel=1e-15)
    s.workers = 2
    assert co2.allreduce_time(s) == pytest.approx(k["expected_w2"], rel=1e-15)
    s = co2.ClusterSpec(workers=8, latency=1.0, param_bytes=1e12, measured_override=0.25)
    assert co2.allreduce_time(s) == 0.25
    s.workers = 1
    assert co2.allreduce_time(s) == 0.0


def test_cluster_validation():
    """proj/tests/test_timing_model.cpp:49-62"""
    for kw in [{"workers": 0}, {"latency": -1.0}, {"inter_bandwidth": 0.0},
               {"measured_override": -0.5}]:
        with pytest.raises(co2.ValidationError):
            co2.ClusterSpec(**({"workers": 2} | kw)).validate()


def test_overlap_ratio():
    """proj/tests/test_timing_model.cpp:64-71"""
    assert co2.overlap_ratio(2, 0.25, 1.0) == 0.5
    assert co2.overlap_ratio(8, 0.25, 1.0) == 1.0
    assert co2.overlap_ratio(1, 0.0, 1.0) == 0.0
    assert co2.overlap_ratio(1, 0.5, 0.0) == 1.0
    with pytest.raises(co2.ValidationError):
        co2.overlap_ratio(0, 0.1, 1.0)
    with pytest.raises(co2.ValidationError):
        co2.overlap_ratio(1, -0.1, 1.0)


def test_overlap_table_acceptance(golden):
    """proj/tests/acceptance.cpp:60-75: paper's overlap table within 0.5pp."""
    k = golden["overlap_table"]
    for tau, exp in zip(k["taus"], k["expected_pct"]):
        assert abs(100.0 * co2.overlap_ratio(tau, k["t_comp"], k["t_comm"]) - exp) <= k["tol_pp"]


def test_co2_timeline_hand_traces(golden):
    """proj/tests/test_timing_model.cpp:79-116"""
    for k in golden["timeline"]:
        spec = co2.ClusterSpec(workers=k["workers"], t_comp=k["t_comp"], t_outer=k["t_outer"],
                               measured_override=k["comm"])
        r = co2.simulate_timeline_co2(spec, k["tau"], k["rounds"])
        assert r.wall_time == k["wall_time"]
        if "total_stall" in k:
            assert r.total_stall == k["total_stall"]
        if "overlap" in k:
            assert r.overlap_ratio_achieved == pytest.approx(k["overlap"])
        if "per_round" in k:
            assert [list(p[1:]) for p in r.per_round] == k["per_round"]
        if "throughput" in k:
            assert r.throughput == k["throughput"]
    with pytest.raises(co2.ValidationError):
        co2.simulate_timeline_co2(co2.ClusterSpec(workers=2, measured_override=1.0), 0, 3)
    with pytest.raises(co2.ValidationError):
        co2.simulate_timeline_co2(co2.ClusterSpec(workers=2, measured_override=1.0), 2, 0)


def test_timeline_every_algorithm_kind(golden):
    """simulate_timeline's slowmo / local_sgd / overlap_local_sgd / sync_sgd
    branches against the reference's hand traces
    (proj/tests/test_timing_model.cpp:118-162), and scalability_ratio."""
    for k in golden["timeline_kinds"]:
        spec = co2.ClusterSpec(workers=k["workers"], t_comp=k["t_comp"], t_outer=k["t_outer"],
                               measured_override=k["comm"])
        r = co2.simulate_timeline(k["kind"], spec, k["tau"], k["rounds"])
        assert r.wall_time == pytest.approx(k["wall_time"]) and r.total_stall == k["total_stall"]
        assert r.overlap_ratio_achieved == pytest.approx(k["overlap"])
        if "throughput" in k:
            assert r.throughput == pytest.approx(k["throughput"])
    spec = co2.ClusterSpec(workers=4, t_comp=1.0, t_outer=0.0, measured_override=1.0)
    r1 = co2.simulate_timeline("local_sgd", spec, 2, 3, 1)
    r8 = co2.simulate_timeline("local_sgd", spec, 2, 3, 8)
    assert r8.throughput == pytest.approx(8.0 * r1.throughput)
    # the co2 kind through the general entry equals the co2-only entry
    s2 = co2.ClusterSpec(workers=2, t_comp=1.0, t_outer=0.5, measured_override=3.0)
    assert co2.simulate_timeline("co2", s2, 2, 3) == co2.simulate_timeline_co2(s2, 2, 3)
    for a, b, c, d, e in golden["scalability_ratio"]["cases"]:
        assert co2.scalability_ratio(a, b, c, d) == e
    with pytest.raises(co2.ValidationError, match="scalability_ratio: non-positive input"):
        co2.scalability_ratio(0.0, 1.0, 1.0, 2.0)
    with pytest.raises(co2.ValidationError, match="unknown algorithm"):
        co2.simulate_timeline("diloco", s2, 2, 3)
    # to_json (test_timing_model.cpp:164-175)
    j = co2.simulate_timeline("co2", s2, 2, 3).to_json()
    assert j["algorithm"] == "co2" and j["workers"] == 2 and j["tau"] == 2
    assert j["wall_time"] == 8.0 and j["total_stall"] == 1.0
    assert len(j["per_round"]) == 3 and j["per_round"][1]["stall"] == 1.0


def test_overlap_flatness_acceptance():
    """proj/tests/acceptance.cpp:88-116 (co2 half): with tau*t_comp >= t_comm
    the one-round-stale pattern has zero stall and flat throughput."""
    fast = co2.simulate_timeline_co2(co2.ClusterSpec(workers=16, t_comp=0.109,
                                                     measured_override=0.109), 12, 50)
    slow = co2.simulate_timeline_co2(co2.ClusterSpec(workers=16, t_comp=0.109,
                                                     measured_override=1.09), 12, 50)
    assert fast.total_stall == 0.0 and slow.total_stall == 0.0
    assert abs(fast.throughput - slow.throughput) / fast.throughput < 1e-3


def test_facade_header_compiles():
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I" + os.path.join(ROOT, "include"),
                        "-I/usr/local/cuda/include",
                        os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_product_does_not_reference_oracle():
    """The product path never links or imports the oracle (test infra only)."""
    pkg = os.path.join(ROOT, "paper_2401_16265_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    src = f.read()
                for needle in ("import oracle", "from oracle", "co2_oracle.h", "libco2oracle",
                               "orc_"):
                    assert needle not in src, (fn, needle)
    out = subprocess.run(["ldd", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out


def test_timeline_invariants_property():
    """hypothesis over simulate_timeline (timing_model.cpp:76-173): for every
    algorithm the wall time covers the compute, stalls never exceed the
    reduce, co2's stall is the uncovered remainder of the previous reduce,
    and the achieved overlap lies in [0, 1]."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    pos = st.floats(0.0, 100.0, allow_nan=False)

    @settings(max_examples=300, deadline=None, derandomize=True)
    @given(kind=st.sampled_from(sorted(co2.ALGORITHMS)), workers=st.integers(1, 64),
           t_comp=pos, comm=pos, t_outer=pos, tau=st.integers(1, 48), rounds=st.integers(1, 12),
           batch=st.integers(1, 16))
    def check(kind, workers, t_comp, comm, t_outer, tau, rounds, batch):
        spec = co2.ClusterSpec(workers=workers, t_comp=t_comp, t_outer=t_outer,
                               measured_override=comm)
        r = co2.simulate_timeline(kind, spec, tau, rounds, batch)
        c = r.comm_time
        assert len(r.per_round) == rounds
        assert r.wall_time >= rounds * tau * t_comp * (1 - 1e-12)
        assert 0.0 <= r.overlap_ratio_achieved <= 1.0
        prev_end = 0.0
        for t, start, stall, end in r.per_round:
            assert start == prev_end and end >= start and stall >= 0.0
            assert stall <= (tau if kind == "sync_sgd" else 1) * c * (1 + 1e-12)
            prev_end = end
        assert r.wall_time == prev_end
        if kind == "co2":
            assert r.per_round[0][2] == 0.0  # round 0 never stalls
            if tau * t_comp >= c:  # the local steps alone hide the reduce
                assert r.total_stall <= 1e-9 * max(r.wall_time, 1.0)
        if kind in ("slowmo", "local_sgd"):
            assert r.total_stall == pytest.approx(rounds * c)

    check()


def test_header_constants_match_the_python_binding():
    """Every CO2_* constant of include/co2_b200.h (status codes, modes,
    dtypes, flags, buffers, algorithms, clip modes, record sizes, ABI
    version) has the same value in the ctypes binding."""
    import re
    text = open(os.path.join(ROOT, "include", "co2_b200.h")).read()
    consts = {m.group(1): int(m.group(2))
              for m in re.finditer(r"\b(CO2_[A-Z0-9_]+)\s*=\s*(\d+)u?\b", text)}
    consts.update({m.group(1): int(m.group(2))
                   for m in re.finditer(r"#define\s+(CO2_[A-Z0-9_]+)\s+(\d+)", text)})
    assert len(consts) > 40
    for name, value in consts.items():
        py = name[len("CO2_"):]
        if name in ("CO2_OK",):
            py = "OK"
        assert hasattr(L, py), f"{name} missing from _lib.py"
        assert getattr(L, py) == value, (name, getattr(L, py), value)
    assert L.lib().co2_abi_version() == consts["CO2_ABI_VERSION"]
