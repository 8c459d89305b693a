"""Generate tests/golden/*.json from the reference's own fixtures and KATs.

Run in the build container (it reads /root/reference, which does not exist on
the GPU box):  python tests/golden/make_golden.py

Every transcribed literal is checked against the cited reference source text
(the script asserts that the literal appears in that file), so a typo here
fails loudly instead of silently pinning the oracle to a wrong value.
"""
from __future__ import annotations

import json
import os

REF = "/root/reference/proj"
HERE = os.path.dirname(os.path.abspath(__file__))


def src(path: str) -> str:
    with open(os.path.join(REF, path)) as f:
        return f.read()


def must_contain(path: str, *literals: str) -> None:
    text = src(path)
    for lit in literals:
        assert lit in text, f"{lit!r} not found in {path}"


def main() -> None:
    # ---- fixture co2_dim1 (replayed bitwise, proj/src/harness.cpp:336-500)
    for name in ("co2_dim1", "slowmo_dim1", "local_sgd_dim1", "overlap_dim1"):
        fx = json.loads(src(f"fixtures/{name}.json"))
        fx["_source"] = f"proj/fixtures/{name}.json (reference fixture, tolerance 0)"
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(fx, f, indent=1)

    kats: dict = {}

    # ---- RNG (proj/tests/test_rng.cpp:11-40)
    must_contain("tests/test_rng.cpp", "0xf33dc6bd55ffa86bull", "0xe1332a7db412c5a9ull",
                 "0xe6af094f768935b3ull", "0x0fdf2d08f5c29727ull", "0x57c324c96eea3787ull",
                 "0x45a3c0ce45dacd67ull", "0x112329151d0eae7aull", "0x0eea3b932b216798ull",
                 "0x04ed0f79d3881c5cull", "0xcedef41df9e91f8full", "0.950161381935685",
                 "0.8796869809048742", "0.9011083430291691", "{9, 8, 9, 0, 7, 1, 2, 6}")
    must_contain("include/co2sim/rng.hpp", "kShardStream = 0x0001000000000001ull")
    kats["rng"] = {
        "_source": "proj/tests/test_rng.cpp:11-40",
        "u64": [
            {"seed": 7, "stream": 0, "values": ["0xf33dc6bd55ffa86b", "0xe1332a7db412c5a9",
                                                "0xe6af094f768935b3", "0x0fdf2d08f5c29727"]},
            {"seed": 7, "stream": 1, "values": ["0x57c324c96eea3787", "0x45a3c0ce45dacd67",
                                                "0x112329151d0eae7a", "0x0eea3b932b216798"]},
            {"seed": 42, "stream": "0x0001000000000001",
             "values": ["0x04ed0f79d3881c5c", "0xcedef41df9e91f8f"]},
        ],
        "double": {"seed": 7, "stream": 0,
                   "values": [0.950161381935685, 0.8796869809048742, 0.9011083430291691]},
        "below10": {"seed": 7, "stream": 0, "values": [9, 8, 9, 0, 7, 1, 2, 6]},
    }

    # ---- average golden vector (proj/tests/test_param_ops.cpp:30-52)
    avg_in = [
        [0.5442868880568308, 1.8113273945956503, 0.19139323188558377, 1.6248311340530925,
         0.40218505048593167, 0.04286966237077339],
        [0.6314264412370334, 1.9654648029382469, 0.3630702349745145, -1.6270775115457816,
         1.0069351598601868, 0.9299044643529717],
        [1.234339331698358, -1.746282902040115, 1.2644511896284585, -0.7586432236672516,
         -1.2602236517597354, -0.861636910493905],
        [-0.4532469812019473, -1.6901608867535085, -1.676126903631042, 1.4676310219404995,
         -0.02718374543101465, -1.0251692135856851],
        [1.247027127420412, 0.8302750132245422, -1.4892671475422357, 1.808391263414844,
         1.8002180507247614, -1.8361414984061626],
    ]
    avg_out = [0.6407665614421374, 0.2341246843929632, -0.2692958789369442, 0.5030265368390806,
               0.38438617277602594, -0.5500346991524016]
    must_contain("tests/test_param_ops.cpp", *[repr(v) for row in avg_in for v in row],
                 *[repr(v) for v in avg_out])
    kats["average"] = {"_source": "proj/tests/test_param_ops.cpp:30-52", "inputs": avg_in,
                       "expected": avg_out}

    # ---- outer-op KATs (proj/tests/test_outer_algorithms.cpp:85-150)
    must_contain("tests/test_outer_algorithms.cpp", "vec({1.6, 0.3})", "vec({1.0, 0.2})",
                 "vec({1.2, 0.3})", "0.6 / 0.4 + 1.0", "0.1 / 0.2 + 1.0",
                 "staleness_gap(x_t0, prev_x0, prev_x1, 4, 0.5)", "1.0 / 0.5 + 1.0",
                 "vec({1.0, -2.0})", "vec({2.0, 1.0})", "vec({0.5, 0.3})",
                 "0.5 * 1.0 + 0.5 / 2.0", "0.5 * -2.0 + 0.3", "raw(1) == -0.7",
                 "vec({0.5, 1.0})", "vec({1.0, -1.0, 0.0})", "vec({4.0, -0.25, -9.0})",
                 "outer_iterate(x, 0.5, m, 1.0, true)", "next(2) == 0.5", "raw(0) == -1.0",
                 "raw(2) == 4.5")
    kats["staleness_gap"] = [
        {"_source": "proj/tests/test_outer_algorithms.cpp:85-94", "x_t0": [1.6, 0.3],
         "prev_x0": [1.0, 0.2], "prev_x1": [1.2, 0.3], "tau": 2, "epsilon": 1e-12,
         "expected": [0.6 / 0.4 + 1.0, 0.1 / 0.2 + 1.0], "rel_tol": 1e-15},
        {"_source": "proj/tests/test_outer_algorithms.cpp:96-103", "x_t0": [2.0, 1.0],
         "prev_x0": [1.0, 1.0], "prev_x1": [1.0, 1.0], "tau": 4, "epsilon": 0.5,
         "expected": [1.0 / 0.5 + 1.0, 1.0], "rel_tol": 0.0},
    ]
    kats["momentum"] = {
        "_source": "proj/tests/test_outer_algorithms.cpp:122-137",
        "m_prev": [1.0, -2.0], "gap": [2.0, 1.0], "delta": [0.5, 0.3], "beta": 0.5,
        "expected_penalty": [0.5 * 1.0 + 0.5 / 2.0, 0.5 * -2.0 + 0.3],
        "expected_raw": [1.0, -0.7], "bad_gap": [0.5, 1.0],
    }
    kats["outer_iterate"] = {
        "_source": "proj/tests/test_outer_algorithms.cpp:139-150",
        "x": [1.0, -1.0, 0.0], "m": [4.0, -0.25, -9.0], "alpha": 0.5, "phi": 1.0,
        "expected_clip": [1.0 - 0.5 * 1.0, -1.0 + 0.5 * 0.25, 0.5],
        "expected_raw_0": -1.0, "expected_raw_2": 4.5,
    }
    must_contain("tests/test_param_ops.cpp", "vec({-3.0, -0.5, 0.0, 0.25, 7.0})",
                 "clip_elementwise(v, 0.5)")
    kats["clip"] = {"_source": "proj/tests/test_param_ops.cpp:113-120",
                    "v": [-3.0, -0.5, 0.0, 0.25, 7.0], "phi": 0.5,
                    "expected": [-0.5, -0.5, 0.0, 0.25, 0.5]}

    # ---- timing model (proj/tests/test_timing_model.cpp:79-116, acceptance.cpp:60-116)
    must_contain("tests/test_timing_model.cpp", "spec_with(2, 1.0, 3.0, 0.5), 2, 3",
                 "r.per_round[1].end == 5.5", "r.per_round[2].end == 8.0",
                 "doctest::Approx(1.0 - 1.0 / 6.0)", "r.throughput == 1.5",
                 "spec_with(2, 1.0, 3.0, 0.0), 4, 5", "r.wall_time == 20.0",
                 "spec_with(2, 1.0, 0.0, 100.0), 2, 1", "Approx(1.506)")
    kats["timeline"] = [
        {"_source": "proj/tests/test_timing_model.cpp:79-100", "workers": 2, "t_comp": 1.0,
         "comm": 3.0, "t_outer": 0.5, "tau": 2, "rounds": 3,
         "per_round": [[0.0, 0.0, 2.0], [2.0, 1.0, 5.5], [5.5, 0.0, 8.0]],
         "wall_time": 8.0, "total_stall": 1.0, "overlap": 1.0 - 1.0 / 6.0, "throughput": 1.5},
        {"_source": "proj/tests/test_timing_model.cpp:102-110", "workers": 2, "t_comp": 1.0,
         "comm": 3.0, "t_outer": 0.0, "tau": 4, "rounds": 5, "wall_time": 20.0,
         "total_stall": 0.0, "overlap": 1.0},
        {"_source": "proj/tests/test_timing_model.cpp:112-116", "workers": 2, "t_comp": 1.0,
         "comm": 0.0, "t_outer": 100.0, "tau": 2, "rounds": 1, "wall_time": 2.0},
    ]
    # the other AlgorithmKind branches (proj/tests/test_timing_model.cpp:118-162)
    must_contain("tests/test_timing_model.cpp",
                 "doctest::Approx(3 * (2.0 + 3.0 + 0.5))", "r.total_stall == 9.0",
                 "AlgorithmKind::overlap_local_sgd,\n                                       "
                 "spec_with(2, 1.0, 3.0, 0.0), 2, 3", "doctest::Approx(2.0 / 3.0)",
                 "spec_with(2, 1.0, 0.0, 0.0), 2, 4", "doctest::Approx(3 * 2 * (1.0 + 3.0))",
                 "r.total_stall == 18.0", "doctest::Approx(12.0 / 24.0)",
                 "spec_with(4, 1.0, 1.0, 0.0), 2, 3, 8", "doctest::Approx(8.0 * r1.throughput)",
                 "scalability_ratio(100.0, 200.0, 2.0, 4.0) == 1.0",
                 "scalability_ratio(100.0, 150.0, 1.0, 2.0) == 0.75")
    kats["timeline_kinds"] = [
        {"_source": "proj/tests/test_timing_model.cpp:118-126", "kind": k, "workers": 2,
         "t_comp": 1.0, "comm": 3.0, "t_outer": 0.5, "tau": 2, "rounds": 3,
         "wall_time": 3 * (2.0 + 3.0 + 0.5), "total_stall": 9.0, "overlap": 0.0}
        for k in ("slowmo", "local_sgd")] + [
        {"_source": "proj/tests/test_timing_model.cpp:128-137", "kind": "overlap_local_sgd",
         "workers": 2, "t_comp": 1.0, "comm": 3.0, "t_outer": 0.0, "tau": 2, "rounds": 3,
         "wall_time": 8.0, "total_stall": 2.0, "overlap": 2.0 / 3.0},
        {"_source": "proj/tests/test_timing_model.cpp:139-145", "kind": "overlap_local_sgd",
         "workers": 2, "t_comp": 1.0, "comm": 0.0, "t_outer": 0.0, "tau": 2, "rounds": 4,
         "wall_time": 8.0, "total_stall": 0.0, "overlap": 1.0},
        {"_source": "proj/tests/test_timing_model.cpp:147-154", "kind": "sync_sgd",
         "workers": 2, "t_comp": 1.0, "comm": 3.0, "t_outer": 0.0, "tau": 2, "rounds": 3,
         "wall_time": 3 * 2 * (1.0 + 3.0), "total_stall": 18.0, "overlap": 0.0,
         "throughput": 12.0 / 24.0},
    ]
    kats["scalability_ratio"] = {"_source": "proj/tests/test_timing_model.cpp:73-77",
                                 "cases": [[100.0, 200.0, 2.0, 4.0, 1.0],
                                           [100.0, 150.0, 1.0, 2.0, 0.75]]}
    kats["allreduce_time"] = {"_source": "proj/tests/test_timing_model.cpp:23-34",
                              "workers": 4, "latency": 0.001, "param_bytes": 1e9,
                              "bandwidth": 1e9, "expected": 1.506,
                              "expected_w2": 2.0 * 0.001 + 1.0}
    must_contain("tests/acceptance.cpp", "{1, 3, 6, 12, 24, 48}",
                 "{6.52, 20.39, 41.81, 83.28, 100.0, 100.0}", "overlap_ratio(taus[i], 0.109, 1.566)")
    kats["overlap_table"] = {"_source": "proj/tests/acceptance.cpp:60-75",
                             "taus": [1, 3, 6, 12, 24, 48], "t_comp": 0.109, "t_comm": 1.566,
                             "expected_pct": [6.52, 20.39, 41.81, 83.28, 100.0, 100.0],
                             "tol_pp": 0.5}

    # ---- delayed-momentum equivalence (proj/tests/acceptance.cpp:178-243)
    must_contain("tests/acceptance.cpp", "f << 1, 0, 0, 1, 1, 1, 1, -1;", "tg << 1, 2, 0, 3;",
                 "alpha = 0.4, beta = 0.5, lr = 0.1", "tau = 3, rounds = 100",
                 "init << 0.5, -0.25;")
    kats["delayed_momentum"] = {
        "_source": "proj/tests/acceptance.cpp:178-243",
        "features": [[1, 0], [0, 1], [1, 1], [1, -1]], "targets": [1, 2, 0, 3],
        "shards": [[0, 1], [2, 3]], "init": [0.5, -0.25], "alpha": 0.4, "beta": 0.5,
        "lr": 0.1, "tau": 3, "rounds": 100,
    }
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats, f, indent=1)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
