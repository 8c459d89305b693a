"""co2_round + CollectiveEngine on the GPU against the reference's fixtures and
the oracle (bitwise).  Inner loops run on the host (fixtures) or as the
synthetic inner-step kernel; the outer rounds run through the C ABI."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2401_16265_b200 import _lib as L
from paper_2401_16265_b200 import co2
from simdrive import OracleRound, inner_loop, shard_gradient

pytestmark = pytest.mark.gpu


def to_np(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def run_fixture_rounds(fx, ghost=False, check_expect=True):
    feats = np.array(fx["features"], dtype=np.float64)
    targs = np.array(fx["targets"], dtype=np.float64)
    shards, hd, tau = fx["shards"], fx["hyper"], fx["tau"]
    lr = fx["schedule"]["base_lr"]
    g, n = len(shards), len(fx["init"])
    hyper = co2.Co2Hyper(alpha=hd["alpha"], beta=hd["beta"], phi=hd["phi"],
                         epsilon=hd["epsilon"], penalty=hd["penalty"], clip=hd["clip"],
                         ghost_consistent=ghost)
    eng = co2.CollectiveEngine(g, transport="local")
    init = torch.tensor(fx["init"], dtype=torch.float64, device="cuda")
    ws = [co2.Worker(co2.MODE_F64, n, init) for _ in range(g)]
    rounds = []
    for t in range(fx["rounds"]):
        traces = []
        for w in ws:
            w.snapshot_start()
            x = w.params.cpu().numpy()
            xs, xf, xe = inner_loop(feats, targs, shards[len(traces)], x, lr, tau)
            w.params.copy_(torch.from_numpy(xf))
            w.snapshot_first()
            w.params.copy_(torch.from_numpy(xe))
            traces.append((xs, xf, xe))
        r = co2.co2_round(ws, eng, hyper, tau)
        rounds.append({
            "traces": traces,
            "result": (r.outer_applied, r.min_gap, r.max_outer_step),
            "xbar": None if t == 0 else ws[0].buffer(L.BUF_XBAR).cpu().numpy(),
            "params": [w.params.cpu().numpy() for w in ws],
            "m": [w.buffer(L.BUF_MOMENTUM).cpu().numpy() for w in ws],
            "gap": [w.buffer(L.BUF_GAP).cpu().numpy() for w in ws],
        })
    return rounds, ws, eng


def test_fixture_co2_dim1_on_gpu(fixture_co2_dim1):
    """proj/fixtures/co2_dim1.json at tolerance 0 through the product path."""
    fx = fixture_co2_dim1
    rounds, _, _ = run_fixture_rounds(fx)
    for t, er in enumerate(fx["expect"]["rounds"]):
        got = rounds[t]
        if "consumed_average" in er:
            assert got["xbar"].tolist() == er["consumed_average"]
        for i, ew in enumerate(er["workers"]):
            assert got["traces"][i][1].tolist() == ew["x_first"]
            assert got["traces"][i][2].tolist() == ew["x_end"]
            assert got["params"][i].tolist() == ew["params_after"]
            if "momentum_after" in ew:
                assert got["m"][i].tolist() == ew["momentum_after"]
                assert got["gap"][i].tolist() == ew["gap_after"]
    fin = fx["expect"]
    assert [p.tolist() for p in rounds[-1]["params"]] == fin["final_params"]
    assert [m.tolist() for m in rounds[-1]["m"]] == fin["final_momentum"]
    assert rounds[0]["result"][0] == 0 and rounds[1]["result"][0] == 1
    assert rounds[1]["result"][1] == 1.875  # min_gap (RoundResult)


def test_delayed_momentum_recurrence_on_gpu(golden):
    """proj/tests/acceptance.cpp:178-243 through co2_round (penalty/clip off):
    bitwise against an independently coded delayed-momentum recurrence."""
    k = golden["delayed_momentum"]
    fx = {"features": k["features"], "targets": k["targets"], "shards": k["shards"],
          "hyper": {"alpha": k["alpha"], "beta": k["beta"], "phi": 1.0, "epsilon": 1e-12,
                    "penalty": False, "clip": False},
          "tau": k["tau"], "schedule": {"base_lr": k["lr"]}, "init": k["init"],
          "rounds": k["rounds"]}
    rounds, _, _ = run_fixture_rounds(fx)
    feats, targs = np.array(k["features"], float), np.array(k["targets"], float)
    x = [np.array(k["init"], float) for _ in range(2)]
    m = [np.zeros(2), np.zeros(2)]
    prev0 = avg_prev = None
    for t in range(k["rounds"]):
        starts = [xi.copy() for xi in x]
        for i in range(2):
            for _ in range(k["tau"]):
                x[i] = x[i] - k["lr"] * shard_gradient(feats, targs, k["shards"][i], x[i])
        avg_t = O.average(x)
        if t == 0:
            prev0, avg_prev = starts, avg_t
        else:
            for i in range(2):
                m[i] = k["beta"] * m[i] + (prev0[i] - avg_prev)
                x[i] = starts[i] - k["alpha"] * m[i]
                prev0[i] = starts[i]
            avg_prev = avg_t
        for i in range(2):
            assert rounds[t]["params"][i].tobytes() == x[i].tobytes(), (t, i)


def test_ghost_consistent_rounds_match_oracle(fixture_co2_dim1):
    """Ghost-consistent branch (outer_algorithms.cpp:161-184): identical
    workers, bitwise equal to the oracle's ghost round."""
    fx = dict(fixture_co2_dim1)
    fx["rounds"] = 6
    rounds, _, _ = run_fixture_rounds(fx, ghost=True)

    class H:
        pass

    h = H()
    hd = fx["hyper"]
    h.alpha, h.beta, h.phi, h.epsilon = hd["alpha"], hd["beta"], hd["phi"], hd["epsilon"]
    h.penalty, h.clip, h.ghost_consistent = hd["penalty"], hd["clip"], True
    orr = OracleRound(2, 1, h, fx["tau"])
    for t, rd in enumerate(rounds):
        traces = rd["traces"]
        params, _, _, _ = orr.round([tr[2] for tr in traces], traces)
        for i in range(2):
            assert rd["params"][i].tobytes() == params[i].tobytes()
            assert rd["m"][i].tobytes() == orr.m[i].tobytes()
        if t >= 1:
            assert rd["params"][0].tobytes() == rd["params"][1].tobytes()


class OracleRoundLP:
    """co2_round in the fp32 / bf16-mixed storage layout on the oracle."""

    def __init__(self, mode, g, hyper):
        self.mode, self.g, self.h = mode, g, hyper
        self.t, self.m, self.p0, self.p1, self.pending = 0, None, None, None, None

    def round(self, params, traces, m0):
        launched = O.average_lp(params, self.mode == O.MODE_BF16_MIXED)
        if self.t == 0:
            self.p0 = [tr[0] for tr in traces]
            self.p1 = [tr[1] for tr in traces]
            self.m = [m0.copy() for _ in range(self.g)]
            self.pending, self.t = launched, 1
            return [p.copy() for p in params]
        out = []
        for i in range(self.g):
            r = O.outer_step(self.mode, traces[i][0], self.p0[i], self.p1[i], self.pending,
                             self.m[i], self.h)
            assert r.status == 0
            self.m[i] = r.m
            self.p0[i], self.p1[i] = traces[i][0], traces[i][1]
            out.append(r.params)
        self.pending, self.t = launched, self.t + 1
        return out


@pytest.mark.parametrize("mode", [co2.MODE_F32, co2.MODE_BF16_MIXED])
def test_c1_simulated_workers_bitwise(mode):
    """Config C1: 1M params, 4 simulated workers, tau=4, synthetic deltas;
    4 rounds of the product co2_round vs the oracle, bitwise every round."""
    n, G, tau = 1 << 20, 4, 4
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    oh = O.hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, tau=tau)
    eng = co2.CollectiveEngine(G, transport="local")
    ws = []
    for w in range(G):
        init = co2.synth(mode, n, worker=w)[3]  # x_end-style draws as x_{0,0}
        ws.append(co2.Worker(mode, n, init))
    orr = OracleRoundLP(mode, G, oh)
    m0 = np.zeros(n, np.float32)
    for t in range(4):
        traces = []
        for i, w in enumerate(ws):
            w.snapshot_start()
            for k in range(tau):
                # odd rounds: the x_{t,1} snapshot fused into the first inner
                # step's store (8f item 2); even rounds: the separate copy
                fuse = k == 0 and t % 2 == 1
                co2.synthetic_inner_step(w.params, lr=1e-3, scale=1.0, worker=i,
                                         step=t * tau + k,
                                         snapshot_out=w.buffer(L.BUF_XFIRST) if fuse else None)
                if k == 0 and not fuse:
                    w.snapshot_first()
            traces.append((to_np(w.buffer(L.BUF_ANCHOR)), to_np(w.buffer(L.BUF_XFIRST)),
                           to_np(w.params)))
        params_before = [tr[2] for tr in traces]
        r = co2.co2_round(ws, eng, hyper, tau)
        ref = orr.round(params_before, traces, m0)
        for i, w in enumerate(ws):
            assert to_np(w.params).tobytes() == ref[i].tobytes(), (t, i)
            if t >= 1:
                assert to_np(w.buffer(L.BUF_MOMENTUM)).tobytes() == orr.m[i].tobytes()
        if t >= 1:
            assert r.outer_applied == 1 and r.min_gap >= 1.0
            assert r.max_outer_step <= np.float32(5e-3) * (1 + 1e-6)


@pytest.mark.parametrize("mode", [co2.MODE_F32, co2.MODE_BF16_MIXED])
@pytest.mark.parametrize("g", [1, 3, 8])
@pytest.mark.parametrize("n", [1, 7, 1029, 263171])
def test_local_round_kernel_shapes_bitwise(mode, g, n):
    """The single-launch LOCAL round (persistent grid, role-major tiles, the
    scalar tail in each role's last tile, atomic per-role diagnostics) at
    ragged sizes and 1..8 workers: params, momentum and the round's
    min_gap / max_outer_step bitwise against the oracle, three rounds."""
    tau = 3
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    oh = O.hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, tau=tau)
    eng = co2.CollectiveEngine(g, transport="local")
    ws = [co2.Worker(mode, n, co2.synth(mode, n, worker=w)[3]) for w in range(g)]
    orr = OracleRoundLP(mode, g, oh)
    m0 = np.zeros(n, np.float32)
    for t in range(4):
        traces = []
        for i, w in enumerate(ws):
            w.snapshot_start()
            for k in range(tau):
                co2.synthetic_inner_step(w.params, lr=1e-3, scale=1.0, worker=i,
                                         step=t * tau + k)
                if k == 0:
                    w.snapshot_first()
            traces.append((to_np(w.buffer(L.BUF_ANCHOR)), to_np(w.buffer(L.BUF_XFIRST)),
                           to_np(w.params)))
        params_before = [tr[2] for tr in traces]
        r = co2.co2_round(ws, eng, hyper, tau)
        if t >= 1:  # the oracle's per-worker diagnostics, folded as RoundResult does
            diags = [O.outer_step(mode, traces[i][0], orr.p0[i], orr.p1[i], orr.pending,
                                  orr.m[i], oh).diag for i in range(g)]
        ref = orr.round(params_before, traces, m0)
        for i, w in enumerate(ws):
            assert to_np(w.params).tobytes() == ref[i].tobytes(), (t, i)
            if t >= 1:
                assert to_np(w.buffer(L.BUF_MOMENTUM)).tobytes() == orr.m[i].tobytes(), (t, i)
        if t >= 1:
            assert r.min_gap == min(d.min_gap for d in diags)
            assert r.max_outer_step == max(d.max_outer_step for d in diags)
            assert r.n_clipped == sum(d.n_clipped for d in diags)
            assert r.n_floored == sum(d.n_floored for d in diags)


def test_engine_semantics():
    """CollectiveEngine contract (proj/tests/test_collective.cpp:43-207)."""
    eng = co2.CollectiveEngine(2, transport="local")
    a = torch.tensor([1.0, -2.0], dtype=torch.float64, device="cuda")
    b = torch.tensor([3.0, 6.0], dtype=torch.float64, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    h0 = eng.launch_all_reduce([a, b], out)
    h1 = eng.launch_all_reduce([a, b], out)
    assert eng.live_handles() == 2
    with pytest.raises(co2.ValidationError, match="overlap window exceeded"):
        eng.launch_all_reduce([a, b], out)
    torch.cuda.synchronize()
    assert eng.is_completed(h0)
    eng.wait(h0)
    assert eng.live_handles() == 1
    with pytest.raises(co2.ValidationError, match="wait: handle already consumed"):
        eng.wait(h0)
    with pytest.raises(co2.ValidationError, match="is_completed: handle already consumed"):
        eng.is_completed(h0)
    with pytest.raises(co2.ValidationError, match="unknown reduce handle"):
        eng.is_completed(99)
    with pytest.raises(co2.ValidationError, match="contribution count 3"):
        eng.launch_all_reduce([a, b, a], out)
    eng.wait(h1)
    torch.cuda.synchronize()
    assert out.tolist() == O.average([np.array([1.0, -2.0]), np.array([3.0, 6.0])]).tolist()
    stall, comm = eng.stall(h1)
    assert stall >= 0.0 and comm >= 0.0
    ev = eng.events()
    kinds = [e["event"] for e in ev if e["handle_id"] == 0]
    assert kinds == ["launch", "complete", "wait"]
    assert ev[0]["t_sim"] <= ev[1]["t_sim"] <= ev[2]["t_sim"]
    # info / total_stall / handle_count (collective.hpp:64-68)
    i0 = eng.info(h0)
    assert i0["id"] == h0 and i0["completed"] and i0["consumed"]
    assert i0["launch_time"] <= i0["completion_time"] and i0["stall"] >= 0.0
    assert eng.handle_count() == 2
    assert eng.total_stall() == pytest.approx(i0["stall"] + eng.info(h1)["stall"])
    h2 = eng.launch_all_reduce([a, b], out)
    i2 = eng.info(h2)
    assert not i2["consumed"] and np.isnan(i2["stall"])
    with pytest.raises(co2.ValidationError, match="unknown reduce handle"):
        eng.info(99)
    eng.wait(h2)
    torch.cuda.synchronize()
    assert eng.info(h2)["consumed"] and eng.handle_count() == 3
    assert eng.reduce_time() > 0.0


def test_single_launch_round_handles():
    """Kernel-timed handles of the single-launch LOCAL round: the kernel
    stamps its own start / end, completion is a non-timing event, and the
    previous round's reduce is consumed in stream order (stall 0, its wait
    at the next launch).  300 rounds also recycle the 256-slot handle ring
    (the device slots are fetched before their events are reused)."""
    g, n, rounds = 3, 4099, 300
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    eng = co2.CollectiveEngine(g, transport="local")
    ws = [co2.Worker(co2.MODE_F32, n, co2.synth_params(co2.MODE_F32, n, worker=i))
          for i in range(g)]
    for w in ws:
        w.snapshot_start()
        w.snapshot_first()
    for _ in range(rounds):
        co2.co2_round(ws, eng, hyper, 2, sync=False)
    r = co2.L.RoundResult()
    arr = (co2.C.c_void_p * g)(*[w.handle.value for w in ws])
    co2.check(co2.lib().co2_round_finish(arr, g, torch.cuda.current_stream().cuda_stream,
                                         co2.C.byref(r)))
    assert r.min_gap >= 1.0 and 0.0 <= r.max_outer_step <= 5e-3 * (1 + 1e-6)
    assert eng.handle_count() == rounds
    ev = eng.events()
    by = {}
    for e in ev:
        by.setdefault(e["handle_id"], {})[e["event"]] = e
    for h in range(1, rounds - 1):  # launched by a single-launch round, consumed in order
        i = eng.info(h)
        assert i["completed"] and i["consumed"] and i["comm"] > 0.0
        assert 0.0 <= i["launch_time"] <= i["completion_time"]
        assert i["stall"] == 0.0
        assert by[h]["wait"]["stall"] == 0.0
        assert by[h]["wait"]["t_sim"] == by[h + 1]["launch"]["t_sim"]  # stream order
        assert by[h]["complete"]["t_sim"] <= by[h + 1]["launch"]["t_sim"] + 1e-5
    last = eng.info(rounds - 1)
    assert not last["consumed"] and last["completed"] and np.isnan(last["stall"])
    assert "wait" not in by[rounds - 1]
    assert eng.total_stall() >= 0.0 and eng.reduce_time() > 0.0
    co2.co2_round_drain(ws, eng)
    torch.cuda.synchronize()
    assert eng.info(rounds - 1)["consumed"]


@pytest.mark.parametrize("mode", [co2.MODE_F32, co2.MODE_BF16_MIXED])
def test_round_host_matches_device_round(mode):
    """co2_round_host (inner loop on the host, outer state resident) equals
    uploading the same traces by hand and calling co2_round, bitwise, and
    hands back the next inner loop's start."""
    g, n, tau, rounds = 2, 10007, 3, 5
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    lo = co2.LOW_TORCH[mode]
    ea, eb = co2.CollectiveEngine(g, transport="local"), co2.CollectiveEngine(g, transport="local")
    wa = [co2.Worker(mode, n, co2.synth_params(mode, n, worker=i)) for i in range(g)]
    wb = [co2.Worker(mode, n, co2.synth_params(mode, n, worker=i)) for i in range(g)]
    for w in wa + wb:
        w.snapshot_start()
    gen = torch.Generator().manual_seed(5)
    for t in range(rounds):
        first = [(torch.rand(n, generator=gen) * 0.02 - 0.01).to(lo).pin_memory()
                 for _ in range(g)]
        end = [(torch.rand(n, generator=gen) * 0.02 - 0.01).to(lo).pin_memory()
               for _ in range(g)]
        for i, w in enumerate(wa):
            if t % 2 == 0:  # odd rounds: x_first omitted, the device snapshot stays
                w.buffer(L.BUF_XFIRST).copy_(first[i])
            w.params.copy_(end[i])
        co2.co2_round(wa, ea, hyper, tau)
        nxt = [torch.empty(n, dtype=lo).pin_memory() for _ in range(g)]
        rb = co2.co2_round_host(wb, eb, hyper, tau, end, nxt,
                                x_first=first if t % 2 == 0 else None, sync=True)
        for i in range(g):
            assert to_np(wa[i].params).tobytes() == to_np(nxt[i]).tobytes(), (t, i)
            assert to_np(wa[i].buffer(L.BUF_MOMENTUM)).tobytes() == \
                to_np(wb[i].buffer(L.BUF_MOMENTUM)).tobytes(), (t, i)
        if t >= 1:
            assert rb.outer_applied == 1 and rb.min_gap >= 1.0


def test_round_rejects_bad_hyper_and_counts():
    eng = co2.CollectiveEngine(2, transport="local")
    ws = [co2.Worker(co2.MODE_F32, 16) for _ in range(2)]
    with pytest.raises(co2.ValidationError, match="hyper: beta"):
        co2.co2_round(ws, eng, co2.Co2Hyper(beta=1.5), 2)
    with pytest.raises(co2.ValidationError, match="contribution count"):
        co2.co2_round(ws[:1], eng, co2.Co2Hyper(), 2)


@pytest.mark.parametrize("mode", [co2.MODE_F64, co2.MODE_F32, co2.MODE_BF16_MIXED])
@pytest.mark.parametrize("ghost", [0, 1, 2, 3, 4, 8])
def test_ghost_step_bitwise(mode, ghost):
    """The sharded/ghost fused step vs the oracle (outer_algorithms.cpp:161-184)."""
    n, G = 70001, max(ghost, 2)
    x, p0, p1, xe, m = co2.synth(mode, n)
    ox, op0, op1, oxe, om = O.synth(mode, n)
    oh = O.hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, tau=6)
    ref = O.outer_step_ghost(mode, ox, op0, op1, G, oxe, G, ghost, om, oh)
    assert ref.status == 0
    h = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    a_out, b0, params = torch.empty_like(x), torch.empty_like(x), torch.empty_like(xe)
    co2.check(co2.lib().co2_outer_step_ghost(
        mode, n, x.data_ptr(), p0.data_ptr(), p1.data_ptr(), G, xe.data_ptr(), G, ghost,
        m.data_ptr(), a_out.data_ptr(), b0.data_ptr(), params.data_ptr(), None,
        co2.C.byref(h.c(6)), co2._ws().ptr, torch.cuda.current_stream().cuda_stream))
    d = co2._ws().fetch()
    assert to_np(m).tobytes() == ref.m.tobytes()
    assert to_np(a_out).tobytes() == ref.anchor.tobytes()
    assert to_np(b0).tobytes() == ref.bar0.tobytes()
    assert to_np(params).tobytes() == ref.params.tobytes()
    assert d.n_clipped == ref.diag.n_clipped and d.min_gap == ref.diag.min_gap


@pytest.mark.parametrize("mode", [co2.MODE_F64, co2.MODE_F32])
def test_sharded_world1_equals_worker_local(mode):
    """With one rank, ghost-consistent sharded rounds reduce to worker-local
    co2_round (average of one worker is the identity): bitwise."""
    n, tau = 200_003, 3
    eng_s = co2.CollectiveEngine(1, transport="nccl", rank=0, nccl_id=bytes(128))
    eng_w = co2.CollectiveEngine(1, transport="nccl", rank=0, nccl_id=bytes(128))
    init = co2.synth(mode, n)[3]
    sw = co2.ShardedWorker(mode, n, eng_s, init)
    w = co2.Worker(mode, n, init)
    hs = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12, ghost_consistent=True)
    hw = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    assert sw.length == n and sw.offset == 0
    for t in range(5):
        w.snapshot_start()
        sw.snapshot_start()
        for k in range(tau):
            co2.synthetic_inner_step(sw.params, lr=1e-3, step=t * tau + k)
            co2.synthetic_inner_step(w.params, lr=1e-3, step=t * tau + k)
            if k == 0:
                sw.snapshot_first()
                w.snapshot_first()
        rs = sw.round(eng_s, hs, tau)
        rw = co2.co2_round([w], eng_w, hw, tau)
        assert to_np(sw.params).tobytes() == to_np(w.params).tobytes(), t
        if t >= 1:
            assert to_np(sw.buffer(L.BUF_MOMENTUM)).tobytes() == \
                to_np(w.buffer(L.BUF_MOMENTUM)).tobytes()
            assert rs.min_gap == rw.min_gap and rs.max_outer_step == rw.max_outer_step
    with pytest.raises(co2.ValidationError, match="ghost_consistent"):
        sw.round(eng_s, hw, tau)
    sw.drain(eng_s)
    co2.co2_round_drain([w], eng_w)


# --------------------------------------------- round diagnostics (8f-4)
def test_divergence_metric_and_event_log(tmp_path, fixture_co2_dim1):
    """Simulation::step's divergence (outer_algorithms.cpp:503-508): exactly 0
    for identical workers, matches fp64 numpy otherwise, deterministic; and
    the engine's events.jsonl follows the reference schema."""
    rng = np.random.default_rng(5)
    for dt in (torch.float64, torch.float32):
        xs = [torch.from_numpy(rng.standard_normal(300_007)).to(dt).cuda() for _ in range(3)]
        mx, per = co2.divergence(xs)
        a = [x.double().cpu().numpy() for x in xs]
        if dt == torch.float64:
            xb = O.average(a)
        else:
            xb = O.average_lp([x.cpu().numpy() for x in xs], False).astype(np.float64)
        ref = [np.linalg.norm(ai - xb) for ai in a]
        assert np.allclose(per, ref, rtol=1e-10, atol=0)
        assert mx == max(per)
        assert co2.divergence(xs) == (mx, per)  # deterministic
        same = [xs[0].clone() for _ in range(4)]
        assert co2.divergence(same)[0] == 0.0
    # ghost-consistent rounds keep workers identical -> divergence 0
    rounds, ws, eng = run_fixture_rounds(dict(fixture_co2_dim1, rounds=4), ghost=True)
    assert co2.divergence([w.params for w in ws])[0] == 0.0
    n = eng.write_events_jsonl(str(tmp_path / "events.jsonl"))
    import json
    lines = [json.loads(x) for x in open(tmp_path / "events.jsonl")]
    assert n == len(lines) and n > 0
    assert set(lines[0]) == {"event", "handle_id", "t_sim", "stall"}
    assert {e["event"] for e in lines} == {"launch", "complete", "wait"}


# ------------------------------------------- baseline outer algorithms (8f-3)
@pytest.mark.parametrize("name", ["slowmo_dim1", "local_sgd_dim1", "overlap_dim1"])
def test_baseline_fixtures_on_gpu(name):
    """proj/fixtures/{slowmo,local_sgd,overlap}_dim1.json at tolerance 0
    through the product's baseline round drivers (F64, 2 simulated workers)."""
    import json
    import os

    from conftest import ROOT
    with open(os.path.join(ROOT, "tests", "golden", f"{name}.json")) as f:
        fx = json.load(f)
    feats = np.array(fx["features"], dtype=np.float64)
    targs = np.array(fx["targets"], dtype=np.float64)
    shards, tau, lr = fx["shards"], fx["tau"], fx["schedule"]["base_lr"]
    g, n = len(shards), len(fx["init"])
    h = fx.get("hyper", {})
    eng = co2.CollectiveEngine(g, transport="local")
    init = torch.tensor(fx["init"], dtype=torch.float64, device="cuda")
    ws = [co2.Worker(co2.MODE_F64, n, init) for _ in range(g)]
    for er in fx["expect"]["rounds"]:
        ends = []
        for i, w in enumerate(ws):
            w.snapshot_start()
            xs, xf, xe = inner_loop(feats, targs, shards[i], w.params.cpu().numpy(), lr, tau)
            w.params.copy_(torch.from_numpy(xe))
            ends.append(xe)
        if fx["algorithm"] == "slowmo":
            co2.slowmo_round(ws, eng, h["alpha"], h["beta"])
        elif fx["algorithm"] == "local_sgd":
            co2.local_sgd_round(ws, eng)
        else:
            co2.overlap_local_sgd_round(ws, eng, instant="cluster" not in fx)
        if "consumed_average" in er:
            assert ws[0].buffer(L.BUF_XBAR).cpu().numpy().tolist() == er["consumed_average"]
        for i, ew in enumerate(er["workers"]):
            assert ends[i].tolist() == ew["x_end"]
            assert ws[i].params.cpu().numpy().tolist() == ew["params_after"]
            if "momentum_after" in ew:
                assert ws[i].buffer(L.BUF_MOMENTUM).cpu().numpy().tolist() == \
                    ew["momentum_after"]
    assert [w.params.cpu().numpy().tolist() for w in ws] == fx["expect"]["final_params"]


@pytest.mark.parametrize("mode", [co2.MODE_F64, co2.MODE_F32, co2.MODE_BF16_MIXED])
def test_baseline_steps_bitwise(mode):
    """The three baseline per-worker kernels vs the oracle's same-order
    restatement, with a worker-sum xbar (divisor 3)."""
    n = 100_003
    x, p0, p1, xe, m = co2.synth(mode, n)
    ox, op0, op1, oxe, om = O.synth(mode, n)
    ws = co2.Workspace()
    st = torch.cuda.current_stream().cuda_stream
    # SlowMo
    mm, params = m.clone(), torch.empty_like(xe)
    co2.check(co2.lib().co2_slowmo_step(mode, n, x.data_ptr(), xe.data_ptr(), 3, mm.data_ptr(),
                                        params.data_ptr(), None, 0.8, 0.6, ws.ptr, st))
    d = ws.fetch()
    rm, rp, rd, code, _ = O.slowmo_step(mode, ox, oxe, om, 0.8, 0.6, divisor=3)
    assert code == 0 and to_np(mm).tobytes() == rm.tobytes()
    assert to_np(params).tobytes() == rp.tobytes() and d.max_outer_step == rd.max_outer_step
    # Local-SGD
    params = torch.empty_like(xe)
    co2.check(co2.lib().co2_local_sgd_step(mode, n, x.data_ptr(), xe.data_ptr(), 3,
                                           params.data_ptr(), None, ws.ptr, st))
    d = ws.fetch()
    rp, rd, code = O.local_sgd_step(mode, ox, oxe, divisor=3)
    assert to_np(params).tobytes() == rp.tobytes() and d.max_outer_step == rd.max_outer_step
    # Overlap correction (params in place; anchor in the state dtype)
    params = p1.clone()
    co2.check(co2.lib().co2_overlap_correction(mode, n, params.data_ptr(), x.data_ptr(),
                                               xe.data_ptr(), 3, ws.ptr, st))
    d = ws.fetch()
    rp, rd, code, _ = O.overlap_correction(mode, op1, ox, oxe, divisor=3)
    assert to_np(params).tobytes() == rp.tobytes() and d.max_outer_step == rd.max_outer_step
    # errors carry the reference's messages
    bad = x.clone()
    bad[5] = float("nan")
    co2.check(co2.lib().co2_slowmo_step(mode, n, bad.data_ptr(), xe.data_ptr(), 1,
                                        m.clone().data_ptr(), params.data_ptr(), None, 0.8, 0.6,
                                        ws.ptr, st))
    with pytest.raises(co2.NumericError, match="slowmo momentum"):
        ws.fetch()
    with pytest.raises(co2.ValidationError, match="slowmo: beta"):
        co2.check(co2.lib().co2_slowmo_step(mode, n, x.data_ptr(), xe.data_ptr(), 1,
                                            m.data_ptr(), params.data_ptr(), None, 0.8, 1.0,
                                            ws.ptr, st))


@pytest.mark.parametrize("mode", [co2.MODE_F32, co2.MODE_BF16_MIXED])
def test_rounds_global_clip_mode(mode):
    """Worker clip mode 'global' (the global-norm clip extension): every
    round's step equals co2_outer_step_global_clip replayed on the worker's
    pre-round state and the consumed average, bitwise; m' is the same as in
    the reference coordinate mode."""
    n, G, tau = 300_007, 2, 3
    hyper = co2.Co2Hyper(alpha=1.0, beta=0.7, phi=5e-3, epsilon=1e-12)
    eng = co2.CollectiveEngine(G, transport="local")
    ws = [co2.Worker(mode, n, co2.synth(mode, n, worker=i)[3]) for i in range(G)]
    for w in ws:
        w.set_clip_mode("global")
    with pytest.raises(co2.ValidationError, match="unknown clip mode"):
        ws[0].set_clip_mode("spectral")
    for t in range(4):
        pre = []
        for i, w in enumerate(ws):
            w.snapshot_start()
            for k in range(tau):
                co2.synthetic_inner_step(w.params, lr=1e-3, scale=1.0, worker=i,
                                         step=t * tau + k)
                if k == 0:
                    w.snapshot_first()
            pre.append([w.buffer(b).clone() for b in (L.BUF_ANCHOR, L.BUF_PREV_X0,
                                                       L.BUF_PREV_X1, L.BUF_MOMENTUM)])
        co2.co2_round(ws, eng, hyper, tau)
        if t == 0:
            continue
        xbar = ws[0].buffer(L.BUF_XBAR).clone()  # the consumed average
        for i, w in enumerate(ws):
            x0, p0, p1, m = pre[i]
            anchor = torch.empty_like(x0)
            params = torch.empty_like(p1)
            d, norm = co2.outer_step_global_clip(mode, x0, p0, p1, xbar, m, hyper, tau,
                                                 anchor_out=anchor, params_out=params)
            assert norm > 5e-3 and d.n_clipped == n  # the clip is active
            assert to_np(w.buffer(L.BUF_MOMENTUM)).tobytes() == to_np(m).tobytes(), (t, i)
            assert to_np(w.buffer(L.BUF_ANCHOR)).tobytes() == to_np(anchor).tobytes(), (t, i)
            assert to_np(w.params).tobytes() == to_np(params).tobytes(), (t, i)


@pytest.mark.parametrize("mode", [co2.MODE_F64, co2.MODE_F32, co2.MODE_BF16_MIXED])
@pytest.mark.parametrize("n,off", [(7, 0), (1_000_003, 0), (65_537, 1)])
def test_baseline_steps_vector_tail_unaligned(mode, n, off):
    """The vectorised baseline kernels: the V-element path with its scalar
    n % V tail (off = 0) and the scalar path for buffers that are not 16-byte
    aligned (off = 1), all bitwise the oracle, with the anchor output."""
    x, p0, p1, xe, m = (t[off:] for t in co2.synth(mode, n + off))
    ox, op0, op1, oxe, om = (a[off:] for a in O.synth(mode, n + off))
    ws = co2.Workspace()
    st = torch.cuda.current_stream().cuda_stream
    mm = m.clone()
    pbuf = torch.empty(n + off, dtype=xe.dtype, device="cuda")[off:]
    abuf = torch.empty(n + off, dtype=x.dtype, device="cuda")[off:]
    co2.check(co2.lib().co2_slowmo_step(mode, n, x.data_ptr(), xe.data_ptr(), 2, mm.data_ptr(),
                                        pbuf.data_ptr(), abuf.data_ptr(), 0.8, 0.6, ws.ptr, st))
    d = ws.fetch()
    rm, rp, rd, code, _ = O.slowmo_step(mode, ox, oxe, om, 0.8, 0.6, divisor=2)
    assert code == 0 and to_np(mm).tobytes() == rm.tobytes()
    assert to_np(pbuf).tobytes() == rp.tobytes() and d.max_outer_step == rd.max_outer_step
    if mode != co2.MODE_BF16_MIXED:
        assert to_np(abuf).tobytes() == rp.tobytes()
    co2.check(co2.lib().co2_local_sgd_step(mode, n, x.data_ptr(), xe.data_ptr(), 2,
                                           pbuf.data_ptr(), abuf.data_ptr(), ws.ptr, st))
    d = ws.fetch()
    rp, rd, code = O.local_sgd_step(mode, ox, oxe, divisor=2)
    assert to_np(pbuf).tobytes() == rp.tobytes() and d.max_outer_step == rd.max_outer_step
    params = p1.clone()
    co2.check(co2.lib().co2_overlap_correction(mode, n, params.data_ptr(), x.data_ptr(),
                                               xe.data_ptr(), 2, ws.ptr, st))
    d = ws.fetch()
    rp, rd, code, _ = O.overlap_correction(mode, op1, ox, oxe, divisor=2)
    assert to_np(params).tobytes() == rp.tobytes() and d.max_outer_step == rd.max_outer_step
