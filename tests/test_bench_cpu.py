"""bench.py contract pieces that run without a GPU: the reference arm's
JSON line (single process and rank != 0 under a launcher) and the helpers
the GPU arm uses for its roofline denominators."""
import json
import os
import subprocess
import sys

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _run(env_extra=None, *args):
    env = dict(os.environ, **(env_extra or {}))
    return subprocess.run([sys.executable, BENCH, "--impl", "reference", *args],
                          capture_output=True, text=True, timeout=300, env=env)


def test_reference_arm_line():
    r = _run(None, "--steps", "2", "--warmup", "1", "--ref-sample", "8192")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "params/s" and d["higher_is_better"]
    assert d["metric"] == "CO2 outer-step params/s" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    # the reference is single-threaded: the arm runs on 1 thread
    assert cb["kind"] in ("port", "reference") and cb["cores"] == 1 and cb["value"] == d["value"]
    assert d["cpu_parallel_bound"]["value"] > 0 and "NOT the reference" in d["cpu_parallel_bound"]["kind"]
    assert d["e2e"] == {"value": d["value"], "unit": "params/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C3")
    # the CPU AAR timed separately, a labelled best-case CPU
    # bound, and the host the numbers came from
    assert d["cpu_aar"]["value"] > 0 and d["cpu_aar"]["cores"] == 1
    assert d["cpu_fused_bound"]["value"] > 0 and "not the reference" in d["cpu_fused_bound"]["kind"]
    assert d["host"]["nproc"] >= 1


def test_reference_arm_non_zero_rank_is_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--steps", "1", "--warmup",
             "0", "--ref-sample", "4096")
    assert r.returncode == 0 and not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_roofline_denominators():
    sys.path.insert(0, ROOT)
    import bench
    peak, kind = bench.peaks()
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        assert kind == "measured" and peak > 1000
    # the committed ncu captures give the DRAM traffic of the default C3 and
    # C2 launches (26 / 32 algorithmic B/param); none for other sizes or N > 1
    t, src = bench.ncu_traffic(dict(bench.CONFIGS["c3"], name="c3"))
    assert t is not None and abs(t / 1.3e9 - 26.0) < 0.5 and src.endswith(".csv")
    t, _ = bench.ncu_traffic(dict(bench.CONFIGS["c2"], name="c2"))
    assert t is not None and abs(t / 125e6 - 32.0) < 1.0
    assert bench.ncu_traffic(dict(bench.CONFIGS["c3"], name="c3"), 2) == (None, None)
    assert bench.ncu_traffic(dict(bench.CONFIGS["c3"], name=None)) == (None, None)
    assert bench.NVLINK_PEER_GBS == 770.0
