"""Python mirror of the reference's CO2 operator API over device buffers.

Same names, argument meaning and error behaviour as the reference
(paths relative to /root/reference/):

  staleness_gap              proj/include/co2sim/outer_algorithms.hpp:37-38
  penalized_momentum_update  proj/include/co2sim/outer_algorithms.hpp:43-46
  outer_iterate              proj/include/co2sim/outer_algorithms.hpp:49-50
  clip_elementwise, average  proj/include/co2sim/param_ops.hpp:16-24
  Co2Hyper                   proj/include/co2sim/outer_algorithms.hpp:17-30
  CollectiveEngine           proj/include/co2sim/collective.hpp:54-93
  co2_round                  proj/include/co2sim/outer_algorithms.hpp:77-81
  allreduce_time, overlap_ratio, simulate_timeline (co2)
                             proj/include/co2sim/timing_model.hpp:27-72

Everything runs through the C ABI (include/co2_b200.h) into the sm_100a
kernels of libco2b200.so; torch supplies device memory and streams only.
ParamVector becomes a 1-D CUDA tensor (float64 / float32 / bfloat16).  The
per-op functions are synchronous like the reference (they return after the
device flags were read so they can raise); the fused `outer_step` is
asynchronous when `check_flags=False`.  The default workspace is shared per
device: launches on concurrent streams must each pass their own
`Workspace`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _lib as L
from ._lib import NumericError, ValidationError, check, lib  # noqa: F401

MODE_F64, MODE_F32, MODE_BF16_MIXED = L.MODE_F64, L.MODE_F32, L.MODE_BF16_MIXED

_DT = {torch.float64: L.DTYPE_F64, torch.float32: L.DTYPE_F32, torch.bfloat16: L.DTYPE_BF16}
STATE_TORCH = {MODE_F64: torch.float64, MODE_F32: torch.float32, MODE_BF16_MIXED: torch.float32}
LOW_TORCH = {MODE_F64: torch.float64, MODE_F32: torch.float32, MODE_BF16_MIXED: torch.bfloat16}


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValidationError("buffers must be contiguous CUDA tensors")
    return t.data_ptr()


def _dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValidationError(f"unsupported dtype {t.dtype}") from None


class Workspace:
    """Device scratch for the deterministic block-reduction finish plus a
    pinned diagnostics mirror.  One per stream."""

    def __init__(self, device=None):
        nbytes = lib().co2_workspace_bytes()
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device or "cuda")
        self.diag = L.Diag()

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def fetch(self, stream=None) -> L.Diag:
        """Synchronize and return the last launch's diagnostics (raises
        with the reference's message on flags)."""
        check(lib().co2_diag_fetch(self.ptr, C.byref(self.diag), _stream(stream)))
        return self.diag


_ws_cache: dict = {}


def _ws(device=None) -> Workspace:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev not in _ws_cache:
        _ws_cache[dev] = Workspace(device=f"cuda:{dev}")
    return _ws_cache[dev]


# ------------------------------------------------------------------ hyper
@dataclass
class Co2Hyper:
    """Co2Hyper (proj/include/co2sim/outer_algorithms.hpp:17-30)."""

    alpha: float = 1.0
    beta: float = 0.7
    phi: float = 1.0
    epsilon: float = 1e-12
    penalty: bool = True
    clip: bool = True
    ghost_consistent: bool = False

    def c(self, tau: int = 1) -> L.Hyper:
        return L.Hyper(self.alpha, self.beta, self.phi, self.epsilon, int(tau), int(self.penalty),
                       int(self.clip), int(self.ghost_consistent), 0)

    def validate(self) -> None:
        """Co2Hyper::validate (proj/src/outer_algorithms.cpp:37-46)."""
        h = self.c()
        check(lib().co2_hyper_validate(C.byref(h)))


# ------------------------------------------------------------- unfused ops
def _same_len(*ts, msg: str):
    n = ts[0].numel()
    for t in ts[1:]:
        if t.numel() != n:
            raise ValidationError(msg)
    return n


def staleness_gap(x_t0, prev_x0, prev_x1, tau: int, epsilon: float, *, stream=None):
    """staleness_gap (proj/src/outer_algorithms.cpp:48-64)."""
    if tau < 1:
        raise ValidationError("staleness_gap: tau must be >= 1")
    if not epsilon > 0.0:
        raise ValidationError("staleness_gap: epsilon must be positive")
    n = _same_len(x_t0, prev_x0, prev_x1, msg="staleness_gap: dimensions differ")
    out = torch.empty_like(x_t0)
    ws = _ws(x_t0.device)
    check(lib().co2_staleness_gap(_dtype(x_t0), n, _ptr(x_t0), _ptr(prev_x0), _ptr(prev_x1), tau,
                                  epsilon, _ptr(out), ws.ptr, _stream(stream)))
    ws.fetch(stream)
    return out


def penalized_momentum_update(m_prev, beta: float, gap, delta, penalty_enabled: bool, *,
                              stream=None):
    """penalized_momentum_update (proj/src/outer_algorithms.cpp:66-90)."""
    if beta < 0.0 or beta >= 1.0:
        raise ValidationError("momentum update: beta must lie in [0, 1)")
    n = _same_len(m_prev, delta, msg="momentum update: dimensions differ")
    if penalty_enabled and gap.numel() != n:
        raise ValidationError("momentum update: gap dimension differs")
    out = torch.empty_like(m_prev)
    ws = _ws(m_prev.device)
    check(lib().co2_penalized_momentum(_dtype(m_prev), n, _ptr(m_prev), beta,
                                       _ptr(gap if penalty_enabled else delta), _ptr(delta),
                                       int(penalty_enabled), _ptr(out), ws.ptr, _stream(stream)))
    ws.fetch(stream)
    return out


def outer_iterate(x_t0, alpha: float, m, phi: float, clip_enabled: bool, *, stream=None):
    """outer_iterate (proj/src/outer_algorithms.cpp:92-108)."""
    if not alpha > 0.0:
        raise ValidationError("outer_iterate: alpha must be positive")
    n = _same_len(x_t0, m, msg="outer_iterate: dimensions differ")
    out = torch.empty_like(x_t0)
    ws = _ws(x_t0.device)
    check(lib().co2_outer_iterate(_dtype(x_t0), n, _ptr(x_t0), alpha, _ptr(m), phi,
                                  int(clip_enabled), _ptr(out), ws.ptr, _stream(stream)))
    ws.fetch(stream)
    return out


def clip_elementwise(v, phi: float, *, stream=None):
    """clip_elementwise (proj/src/param_ops.cpp:35-43)."""
    out = torch.empty_like(v)
    ws = _ws(v.device)
    check(lib().co2_clip_elementwise(_dtype(v), v.numel(), _ptr(v), phi, _ptr(out), ws.ptr,
                                     _stream(stream)))
    ws.fetch(stream)
    return out


def elementwise_abs_diff(a: torch.Tensor, b: torch.Tensor, *, workspace: Workspace | None = None,
                         stream=None) -> torch.Tensor:
    """elementwise_abs_diff (proj/src/param_ops.cpp:44-51)."""
    if a.numel() != b.numel() or a.dtype != b.dtype:
        raise ValidationError("elementwise_abs_diff: dimensions differ")
    out = torch.empty_like(a)
    ws = workspace or _ws(a.device)
    check(lib().co2_elementwise_abs_diff(_dtype(a), a.numel(), _ptr(a), _ptr(b), _ptr(out),
                                         ws.ptr, _stream(stream)))
    return out


def l2_norm(v: torch.Tensor, *, workspace: Workspace | None = None, stream=None) -> float:
    """l2_norm (proj/src/param_ops.cpp:54-60), fixed-order fp64 sum of squares."""
    ws = workspace or _ws(v.device)
    out = C.c_double()
    check(lib().co2_l2_norm(_dtype(v), v.numel(), _ptr(v), C.byref(out), ws.ptr,
                            _stream(stream)))
    return out.value


def ensure_finite(v: torch.Tensor, context: str, *, workspace: Workspace | None = None,
                  stream=None) -> None:
    """ensure_finite (proj/src/param_ops.cpp:10-14): raises NumericError
    "non-finite value in <context>" if v holds a NaN or an infinity."""
    ws = workspace or _ws(v.device)
    check(lib().co2_ensure_finite(_dtype(v), v.numel(), _ptr(v), context.encode(), ws.ptr,
                                  _stream(stream)))


def average(contributions, *, stream=None):
    """average (proj/src/param_ops.cpp:16-33): ascending-order sum, one
    division by G."""
    if len(contributions) == 0:
        raise ValidationError("average: empty contribution list")
    n = _same_len(*contributions, msg="average: contribution dimensions differ")
    out = torch.empty_like(contributions[0])
    ptrs = (C.c_void_p * len(contributions))(*[_ptr(c) for c in contributions])
    ws = _ws(out.device)
    check(lib().co2_average(_dtype(out), len(contributions), ptrs, n, _ptr(out), ws.ptr,
                            _stream(stream)))
    ws.fetch(stream)
    return out


def divergence(params_list, *, stream=None) -> tuple[float, list[float]]:
    """max_i ||x_i - xbar|| (Simulation::step, outer_algorithms.cpp:503-508);
    returns (max, per-worker norms)."""
    g = len(params_list)
    n = _same_len(*params_list, msg="divergence: dimensions differ")
    ptrs = (C.c_void_p * g)(*[_ptr(p) for p in params_list])
    per = (C.c_double * g)()
    mx = C.c_double()
    ws = _ws(params_list[0].device)
    check(lib().co2_divergence(_dtype(params_list[0]), g, ptrs, n, per, C.byref(mx), ws.ptr,
                               _stream(stream)))
    return mx.value, list(per)


# ------------------------------------------------------------- fused step
def outer_step(mode: int, x_t0, prev_x0, prev_x1, xbar, momentum, hyper: Co2Hyper, tau: int, *,
               divisor: int = 1, anchor_out=None, params_out=None, gap_out=None,
               workspace: Workspace | None = None, stream=None, check_flags: bool = True):
    """Fused co2_round per-worker body (proj/src/outer_algorithms.cpp:186-196).
    Updates `momentum` in place; returns the Diag when check_flags (after a
    stream sync), else None (asynchronous)."""
    n = _same_len(x_t0, prev_x0, prev_x1, xbar, momentum, msg="staleness_gap: dimensions differ")
    for t in (anchor_out, params_out, gap_out):
        if t is not None and t.numel() != n:
            raise ValidationError("outer step: output dimension differs")
    ws = workspace or _ws(x_t0.device)
    h = hyper.c(tau)
    check(lib().co2_outer_step(mode, n, _ptr(x_t0), _ptr(prev_x0), _ptr(prev_x1), _ptr(xbar),
                               divisor, _ptr(momentum), _ptr(anchor_out), _ptr(params_out),
                               _ptr(gap_out), C.byref(h), ws.ptr, _stream(stream)))
    if check_flags:
        return ws.fetch(stream)
    return None


def outer_step_global_clip(mode: int, x_t0, prev_x0, prev_x1, xbar, momentum, hyper: Co2Hyper,
                           tau: int, *, divisor: int = 1, anchor_out=None, params_out=None,
                           gap_out=None, workspace: Workspace | None = None, stream=None):
    """EXTENSION outside the reference parity contract: the outer step with
    a global-norm clip of the outer momentum (c = m' * min(1, phi/||m'||_2))
    instead of the reference's coordinate-wise clip.  Returns (Diag, norm)
    after a stream sync."""
    n = _same_len(x_t0, prev_x0, prev_x1, xbar, momentum, msg="staleness_gap: dimensions differ")
    for t in (anchor_out, params_out, gap_out):
        if t is not None and t.numel() != n:
            raise ValidationError("outer step: output dimension differs")
    ws = workspace or _ws(x_t0.device)
    h = hyper.c(tau)
    check(lib().co2_outer_step_global_clip(mode, n, _ptr(x_t0), _ptr(prev_x0), _ptr(prev_x1),
                                           _ptr(xbar), divisor, _ptr(momentum), _ptr(anchor_out),
                                           _ptr(params_out), _ptr(gap_out), C.byref(h), ws.ptr,
                                           _stream(stream)))
    norm = C.c_double()
    check(lib().co2_global_clip_norm_fetch(ws.ptr, C.byref(norm), _stream(stream)))
    return ws.fetch(stream), norm.value


def outer_step_host(mode: int, x_t0, prev_x0, prev_x1, xbar, momentum, hyper: Co2Hyper, tau: int,
                    *, divisor: int = 1, anchor_out=None, params_out=None, chunk: int = 1 << 24,
                    nstreams: int = 3) -> L.Diag:
    """End-to-end fused step over HOST tensors (pinned for full PCIe rate):
    the reference's own calling convention (host vectors in and out)."""
    n = x_t0.numel()
    d = L.Diag()
    h = hyper.c(tau)

    def hp(t):
        return None if t is None else t.data_ptr()

    check(lib().co2_outer_step_host(mode, n, hp(x_t0), hp(prev_x0), hp(prev_x1), hp(xbar), divisor,
                                    hp(momentum), hp(anchor_out), hp(params_out), C.byref(h),
                                    chunk, nstreams, C.byref(d)))
    return d


def synth(mode: int, n: int, *, seed: int = 7, worker: int = 0, j0: int = 0, device="cuda",
          stream=None):
    """Synthetic inputs generated on the device: returns
    (x_t0, prev_x0, prev_x1, x_end, momentum)."""
    st, lo = STATE_TORCH[mode], LOW_TORCH[mode]
    x = torch.empty(n, dtype=st, device=device)
    p0 = torch.empty(n, dtype=st, device=device)
    m = torch.empty(n, dtype=st, device=device)
    p1 = torch.empty(n, dtype=lo, device=device)
    xe = torch.empty(n, dtype=lo, device=device)
    check(lib().co2_synth(mode, seed, worker, j0, n, _ptr(x), _ptr(p0), _ptr(p1), _ptr(xe), _ptr(m),
                          _stream(stream)))
    return x, p0, p1, xe, m


def synth_params(mode: int, n: int, *, seed: int = 7, worker: int = 0, device="cuda",
                 stream=None):
    """Only the x_end-style draws (params dtype) of `synth`, without
    allocating the other four buffers."""
    xe = torch.empty(n, dtype=LOW_TORCH[mode], device=device)
    check(lib().co2_synth(mode, seed, worker, 0, n, None, None, None, _ptr(xe), None,
                          _stream(stream)))
    return xe


def synthetic_inner_step(params, *, lr: float, scale: float = 1.0, seed: int = 7, worker: int = 0,
                         step: int = 0, repeat: int = 1, snapshot_out=None, stream=None):
    """Inner-step stand-in x <- x - lr*g; with snapshot_out the x_{t,1}
    snapshot is written by the same pass."""
    check(lib().co2_synthetic_inner_step_snapshot(_dtype(params), params.numel(), _ptr(params),
                                                  lr, scale, seed, worker, step, repeat,
                                                  _ptr(snapshot_out), _stream(stream)))


# ------------------------------------------------------------ timing model
@dataclass
class ClusterSpec:
    """ClusterSpec (proj/include/co2sim/timing_model.hpp:14-25)."""

    workers: int = 1
    gpus_per_node: int = 8
    t_comp: float = 0.0
    t_outer: float = 0.0
    param_bytes: float = 0.0
    inter_bandwidth: float = 1.0
    latency: float = 0.0
    measured_override: float | None = None

    def c(self) -> L.Cluster:
        mo = self.measured_override
        return L.Cluster(self.workers, self.gpus_per_node, self.t_comp, self.t_outer,
                         self.param_bytes, self.inter_bandwidth, self.latency,
                         0 if mo is None else 1, 0.0 if mo is None else mo)

    def validate(self) -> None:
        s = self.c()
        check(lib().co2_cluster_validate(C.byref(s)))


def allreduce_time(spec: ClusterSpec) -> float:
    s, out = spec.c(), C.c_double()
    check(lib().co2_allreduce_time(C.byref(s), C.byref(out)))
    return out.value


def overlap_ratio(tau: int, t_comp: float, t_comm: float) -> float:
    out = C.c_double()
    check(lib().co2_overlap_ratio(tau, t_comp, t_comm, C.byref(out)))
    return out.value


@dataclass
class TimelineReport:
    workers: int
    tau: int
    rounds: int
    batch_size: int
    comm_time: float
    wall_time: float
    total_stall: float
    overlap_ratio_achieved: float
    throughput: float
    per_round: list = field(default_factory=list)
    algorithm: str = "co2"

    def to_json(self) -> dict:
        """to_json(TimelineReport) (proj/src/timing_model.cpp:55-74)."""
        return {"algorithm": self.algorithm, "workers": self.workers, "tau": self.tau,
                "rounds": self.rounds, "batch_size": self.batch_size,
                "comm_time": self.comm_time, "wall_time": self.wall_time,
                "total_stall": self.total_stall,
                "overlap_ratio_achieved": self.overlap_ratio_achieved,
                "throughput": self.throughput,
                "per_round": [{"t": t, "start": a, "stall": b, "end": e}
                              for t, a, b, e in self.per_round]}


ALGORITHMS = {"co2": L.ALG_CO2, "slowmo": L.ALG_SLOWMO, "local_sgd": L.ALG_LOCAL_SGD,
              "overlap_local_sgd": L.ALG_OVERLAP_LOCAL_SGD, "sync_sgd": L.ALG_SYNC_SGD}


def simulate_timeline_co2(spec: ClusterSpec, tau: int, rounds: int,
                          batch_size: int = 1) -> TimelineReport:
    """simulate_timeline(AlgorithmKind::co2, ...) (proj/src/timing_model.cpp:76-123)."""
    return simulate_timeline("co2", spec, tau, rounds, batch_size)


def simulate_timeline(kind: str, spec: ClusterSpec, tau: int, rounds: int,
                      batch_size: int = 1) -> TimelineReport:
    """simulate_timeline (proj/src/timing_model.cpp:76-173) for kind in
    co2 / slowmo / local_sgd / overlap_local_sgd / sync_sgd."""
    if kind not in ALGORITHMS:
        raise ValidationError(f"simulate_timeline: unknown algorithm {kind!r}")
    s, out = spec.c(), L.Timeline()
    per = (L.RoundTiming * max(rounds, 1))()
    check(lib().co2_simulate_timeline(ALGORITHMS[kind], C.byref(s), tau, rounds, batch_size,
                                      C.byref(out), per))
    return TimelineReport(out.workers, out.tau, out.rounds, out.batch_size, out.comm_time,
                          out.wall_time, out.total_stall, out.overlap_ratio_achieved,
                          out.throughput,
                          [(per[i].t, per[i].start, per[i].stall, per[i].end)
                           for i in range(rounds)], kind)


def scalability_ratio(throughput_small: float, throughput_large: float, workers_small: float,
                      workers_large: float) -> float:
    """scalability_ratio (proj/src/timing_model.cpp:45-53)."""
    r = C.c_double()
    check(lib().co2_scalability_ratio(throughput_small, throughput_large, workers_small,
                                      workers_large, C.byref(r)))
    return r.value


# ------------------------------------------------------- collective engine
class CollectiveEngine:
    """One-step-stale all-reduce (proj/include/co2sim/collective.hpp:54-93).

    transport "local": G simulated workers on this GPU, fixed-order average.
    transport "nccl":  one rank per GPU, in place.  nccl_algo "fixed" (default):
                       slice exchange + fixed-order average kernel + all-gather,
                       bitwise the reference's average() at any G; "sum":
                       ncclAllReduce(sum) in the storage dtype, divided by G in
                       the consumer (NCCL's order and per-hop rounding).
    transport "p2p":   one rank per GPU; deterministic fixed-order average over
                       NVLink peer memory (CUDA IPC).  Needs an initialized
                       torch.distributed group to exchange IPC handles."""

    def __init__(self, workers: int = 1, *, transport: str = "local", rank: int = 0,
                 nccl_id: bytes | None = None, max_ctas: int = 0, nccl_algo: str = "fixed"):
        self.handle = C.c_void_p()
        self.transport = transport
        self.rank = rank
        if transport == "local":
            check(lib().co2_aar_create_local(C.byref(self.handle), workers))
        elif transport == "nccl":
            if nccl_id is None:
                raise ValidationError("nccl transport needs the rank-0 unique id")
            uid = (C.c_uint8 * L.NCCL_ID_BYTES)(*nccl_id)
            check(lib().co2_aar_create_nccl(C.byref(self.handle), uid, rank, workers, max_ctas))
            if nccl_algo not in ("fixed", "sum"):
                raise ValidationError(f"unknown nccl_algo {nccl_algo}")
            check(lib().co2_aar_set_nccl_algo(
                self.handle, L.NCCL_SUM if nccl_algo == "sum" else L.NCCL_FIXED_ORDER))
        elif transport == "p2p":
            check(lib().co2_aar_create_p2p(C.byref(self.handle), rank, workers, max_ctas))
            self.workers = workers
            sig = lib().co2_aar_signal_buffer(self.handle)
            check(lib().co2_aar_p2p_attach_signals(self.handle, self._exchange(sig)))
        else:
            raise ValidationError(f"unknown transport {transport}")
        self.workers = workers

    def _exchange(self, ptr: int):
        """Export `ptr` and all-gather every rank's IPC handle (rank order)."""
        h = (C.c_uint8 * L.IPC_HANDLE_BYTES)()
        check(lib().co2_ipc_export(ptr, h))
        if self.workers == 1:
            return h
        import torch.distributed as dist
        got = [None] * self.workers
        dist.all_gather_object(got, bytes(h))
        flat = b"".join(got)
        return (C.c_uint8 * len(flat))(*flat)

    def register(self, ptr: int) -> None:
        """P2P: make a device buffer (the same logical buffer on every rank)
        reducible; collective over the group."""
        check(lib().co2_aar_p2p_attach(self.handle, ptr, self._exchange(ptr)))

    def deregister(self, ptr: int) -> None:
        """P2P: undo register(); collective.  Returns after every rank closed
        its mapping, so the owner may then free the buffer."""
        check(lib().co2_aar_p2p_detach(self.handle, ptr))
        if self.workers > 1:
            import torch.distributed as dist
            dist.barrier()

    def deregister_worker(self, worker: "Worker") -> None:
        for which in (L.BUF_PARAMS, L.BUF_PARAMS_ALT):
            self.deregister(lib().co2_worker_buffer(worker.handle, which))

    def set_fused(self, on: bool = True) -> None:
        """P2P: fuse the one-step-stale all-reduce into the outer-step kernel."""
        check(lib().co2_aar_set_fused(self.handle, int(on)))

    def set_adaptive(self, on: bool = True) -> None:
        """P2P: let the all-reduce's CTA count follow the measured slack."""
        check(lib().co2_aar_set_adaptive(self.handle, int(on)))

    def ctas(self) -> int:
        return int(lib().co2_aar_ctas(self.handle))

    def register_worker(self, worker: "Worker") -> None:
        """P2P: register both ping-pong params buffers of a worker."""
        for which in (L.BUF_PARAMS, L.BUF_PARAMS_ALT):
            self.register(lib().co2_worker_buffer(worker.handle, which))

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * L.NCCL_ID_BYTES)()
        check(lib().co2_nccl_unique_id(buf))
        return bytes(buf)

    def close(self):
        if self.handle:
            lib().co2_aar_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch_all_reduce(self, contributions, out=None, *, stream=None) -> int:
        if self.transport == "local" and len(contributions) != self.workers:
            raise ValidationError(
                f"launch_all_reduce: contribution count {len(contributions)} does not match "
                f"worker count {self.workers}")
        ptrs = (C.c_void_p * len(contributions))(*[_ptr(c) for c in contributions])
        h = C.c_uint64()
        check(lib().co2_aar_launch(self.handle, _dtype(contributions[0]), ptrs, _ptr(out),
                                   contributions[0].numel(), _stream(stream), C.byref(h)))
        return h.value

    def is_completed(self, handle: int) -> bool:
        d = C.c_int32()
        check(lib().co2_aar_poll(self.handle, handle, C.byref(d)))
        return bool(d.value)

    def wait(self, handle: int, *, stream=None) -> None:
        check(lib().co2_aar_wait(self.handle, handle, _stream(stream)))

    def stall(self, handle: int) -> tuple[float, float]:
        s, c = C.c_double(), C.c_double()
        check(lib().co2_aar_stall(self.handle, handle, C.byref(s), C.byref(c)))
        return s.value, c.value

    def info(self, handle: int) -> dict:
        """HandleInfo (collective.hpp:40-50): device times in seconds since
        engine creation; NaN where not yet known.  Non-blocking."""
        r = L.HandleInfo()
        check(lib().co2_aar_info(self.handle, handle, C.byref(r)))
        return {"id": r.id, "launch_time": r.launch_time, "completion_time": r.completion_time,
                "completed": bool(r.completed), "consumed": bool(r.consumed), "stall": r.stall,
                "comm": r.comm, "contributions": r.contributions, "polled": bool(r.polled),
                "last_poll": bool(r.last_poll), "completion_logged": bool(r.completion_logged)}

    def total_stall(self) -> float:
        s = C.c_double()
        check(lib().co2_aar_totals(self.handle, C.byref(s), None))
        return s.value

    def handle_count(self) -> int:
        c = C.c_uint64()
        check(lib().co2_aar_totals(self.handle, None, C.byref(c)))
        return c.value

    def reduce_time(self) -> float:
        """reduce_time() (collective.hpp:64): here the measured mean device
        duration (s) of the completed reduces, 0.0 before the first."""
        ev = self.events()
        start = {e["handle_id"]: e["t_sim"] for e in ev if e["event"] == "launch"}
        dur = [e["t_sim"] - start[e["handle_id"]] for e in ev
               if e["event"] == "complete" and e["handle_id"] in start]
        return sum(dur) / len(dur) if dur else 0.0

    def live_handles(self) -> int:
        v = C.c_int32()
        check(lib().co2_aar_live(self.handle, C.byref(v)))
        return v.value

    def events(self) -> list[dict]:
        cnt = C.c_int64()
        check(lib().co2_aar_events(self.handle, None, 0, C.byref(cnt)))
        arr = (L.Event * max(cnt.value, 1))()
        check(lib().co2_aar_events(self.handle, arr, cnt.value, C.byref(cnt)))
        kinds = ["launch", "complete", "wait"]
        return [{"event": kinds[arr[i].kind], "handle_id": arr[i].handle, "t_sim": arr[i].t,
                 "stall": arr[i].stall} for i in range(cnt.value)]

    def write_events_jsonl(self, path: str) -> int:
        """events.jsonl in the reference's schema (proj/src/harness.cpp:151-160,
        proj/include/co2sim/collective.hpp:24-29), times from the device
        clock (seconds since engine creation).  Returns the line count."""
        import json
        ev = sorted(self.events(), key=lambda e: (e["t_sim"], e["handle_id"]))
        with open(path, "w") as f:
            for e in ev:
                f.write(json.dumps(e) + "\n")
        return len(ev)


# ---------------------------------------------------------- worker + round
class Worker:
    """Device-resident WorkerState + OuterState (outer_algorithms.hpp:52-61)."""

    def __init__(self, mode: int, n: int, init=None, *, keep_gap: bool = True, stream=None):
        self.handle = C.c_void_p()
        self.mode, self.n = mode, n
        check(lib().co2_worker_create(C.byref(self.handle), mode, n, _ptr(init), int(keep_gap),
                                      _stream(stream)))

    def close(self):
        if self.handle:
            lib().co2_worker_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def buffer(self, which: int) -> torch.Tensor | None:
        """A zero-copy tensor view of one device buffer."""
        ptr = lib().co2_worker_buffer(self.handle, which)
        if not ptr:
            return None
        state = which in (L.BUF_ANCHOR, L.BUF_PREV_X0, L.BUF_MOMENTUM, L.BUF_GAP)
        dt = STATE_TORCH[self.mode] if state else LOW_TORCH[self.mode]
        return _view(ptr, self.n, dt)

    @property
    def params(self):
        return self.buffer(L.BUF_PARAMS)

    @property
    def t(self) -> int:
        return lib().co2_worker_round(self.handle)

    def keep_average(self, on: bool = True) -> None:
        """RoundResult::consumed_average on the in-place transports (NCCL,
        P2P): the step also writes the reduce it consumed into a worker-owned
        buffer, readable as buffer(BUF_XBAR) after the round."""
        check(lib().co2_worker_keep_average(self.handle, int(on)))

    def set_clip_mode(self, mode: str) -> None:
        """'coordinate' (the reference, default) or 'global' (the global-norm
        clip extension, outside the parity contract)."""
        m = {"coordinate": L.CLIP_COORDINATE, "global": L.CLIP_GLOBAL_NORM}.get(mode)
        if m is None:
            raise ValidationError(f"worker: unknown clip mode {mode!r}")
        check(lib().co2_worker_set_clip_mode(self.handle, m))

    def enable_timing(self, cap: int = 4096):
        check(lib().co2_worker_enable_timing(self.handle, cap))

    def step_times(self, cap: int = 4096) -> list[float]:
        """Device durations (s) of the fused launches since the last call."""
        out = (C.c_double * cap)()
        cnt = C.c_int32()
        check(lib().co2_worker_step_times(self.handle, out, cap, C.byref(cnt)))
        return [out[i] for i in range(cnt.value)]

    def snapshot_start(self, stream=None):
        check(lib().co2_worker_snapshot_start(self.handle, _stream(stream)))

    def snapshot_first(self, stream=None):
        check(lib().co2_worker_snapshot_first(self.handle, _stream(stream)))


def _view(ptr: int, n: int, dtype) -> torch.Tensor:
    """Wrap a raw device pointer owned by the library as a tensor (no copy)."""
    esz = torch.tensor([], dtype=dtype).element_size()

    class _Cuda:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": {torch.float64: "<f8", torch.float32: "<f4",
                                       torch.bfloat16: "<u2"}[dtype],
            "data": (ptr, False), "version": 3, "strides": None}

    t = torch.as_tensor(_Cuda(), device="cuda")
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    assert t.element_size() == esz
    return t


def co2_round(workers: list[Worker], engine: CollectiveEngine, hyper: Co2Hyper, tau: int, *,
              stream=None, sync: bool = True) -> L.RoundResult:
    """co2_round (proj/src/outer_algorithms.cpp:110-211) over device workers."""
    arr = (C.c_void_p * len(workers))(*[w.handle.value for w in workers])
    h = hyper.c(tau)
    r = L.RoundResult()
    check(lib().co2_round(arr, len(workers), engine.handle, C.byref(h), _stream(stream), int(sync),
                          C.byref(r)))
    return r


def _arr(workers):
    return (C.c_void_p * len(workers))(*[w.handle.value for w in workers])


def slowmo_round(workers: list[Worker], engine: CollectiveEngine, alpha: float, beta: float, *,
                 stream=None, sync: bool = True) -> L.RoundResult:
    """slowmo_round (proj/src/outer_algorithms.cpp:213-240)."""
    r = L.RoundResult()
    check(lib().co2_slowmo_round(_arr(workers), len(workers), engine.handle, alpha, beta,
                                 _stream(stream), int(sync), C.byref(r)))
    return r


def local_sgd_round(workers: list[Worker], engine: CollectiveEngine, *, stream=None,
                    sync: bool = True) -> L.RoundResult:
    """local_sgd_round (proj/src/outer_algorithms.cpp:242-260)."""
    r = L.RoundResult()
    check(lib().co2_local_sgd_round(_arr(workers), len(workers), engine.handle, _stream(stream),
                                    int(sync), C.byref(r)))
    return r


def overlap_local_sgd_round(workers: list[Worker], engine: CollectiveEngine, *,
                            instant: bool = False, stream=None,
                            sync: bool = True) -> L.RoundResult:
    """overlap_local_sgd_round (proj/src/outer_algorithms.cpp:262-313)."""
    r = L.RoundResult()
    check(lib().co2_overlap_local_sgd_round(_arr(workers), len(workers), engine.handle,
                                            int(instant), _stream(stream), int(sync),
                                            C.byref(r)))
    return r


def co2_round_host(workers: list[Worker], engine: CollectiveEngine, hyper: Co2Hyper, tau: int,
                   x_end: list, x_next: list, *, x_first: list | None = None, stream=None,
                   sync: bool = True) -> L.RoundResult:
    """co2_round with the inner loop on the host (include/co2_b200.h
    co2_round_host): uploads each worker's x_{t,1} (optional) and x_{t,tau}
    from host tensors, runs the round on the device-resident outer state,
    downloads the next inner loop's start x_{t+1,0} into `x_next`."""
    g = len(workers)
    arr = (C.c_void_p * g)(*[w.handle.value for w in workers])

    def ptrs(ts):
        return (C.c_void_p * g)(*[t.data_ptr() for t in ts]) if ts is not None else None
    lo = LOW_TORCH[workers[0].mode]
    for t in list(x_end) + list(x_next) + list(x_first or []):
        if t.is_cuda or not t.is_contiguous() or t.numel() != workers[0].n or t.dtype != lo:
            raise ValueError(f"co2_round_host: contiguous host tensors of n {lo} values "
                             "expected")
    h = hyper.c(tau)
    r = L.RoundResult()
    check(lib().co2_round_host(arr, g, engine.handle, C.byref(h), ptrs(x_first), ptrs(x_end),
                               ptrs(x_next), _stream(stream), int(sync), C.byref(r)))
    return r


def co2_round_drain(workers: list[Worker], engine: CollectiveEngine, *, stream=None) -> None:
    """Consume the reduce launched by the last round (end of a run)."""
    arr = (C.c_void_p * len(workers))(*[w.handle.value for w in workers])
    check(lib().co2_round_drain(arr, len(workers), engine.handle, _stream(stream)))


def outer_step_ghost(mode: int, anchor, prev_x0, prev_x1_sum, xbar_sum, momentum,
                     hyper: Co2Hyper, tau: int, *, workers: int, ghost_copies: int,
                     anchor_out=None, bar0_out=None, params_out=None, gap_out=None,
                     workspace: Workspace | None = None, stream=None, check_flags: bool = True):
    """Ghost-consistent / sharded fused step on one shard
    (proj/src/outer_algorithms.cpp:161-184)."""
    n = prev_x0.numel()
    ws = workspace or _ws(prev_x0.device)
    h = hyper.c(tau)
    check(lib().co2_outer_step_ghost(mode, n, _ptr(anchor), _ptr(prev_x0), _ptr(prev_x1_sum),
                                     workers, _ptr(xbar_sum), workers, ghost_copies,
                                     _ptr(momentum), _ptr(anchor_out), _ptr(bar0_out),
                                     _ptr(params_out), _ptr(gap_out), C.byref(h), ws.ptr,
                                     _stream(stream)))
    return ws.fetch(stream) if check_flags else None


class ShardedWorker:
    """Ghost-consistent CO2 worker with the outer state sharded across the
    NCCL engine's ranks (BASELINE config C4)."""

    def __init__(self, mode: int, n: int, engine: CollectiveEngine, init=None, *,
                 keep_gap: bool = True, stream=None):
        self.handle = C.c_void_p()
        self.mode, self.n = mode, n
        check(lib().co2_sharded_create(C.byref(self.handle), mode, n, engine.handle, _ptr(init),
                                       int(keep_gap), _stream(stream)))
        off, ln = C.c_int64(), C.c_int64()
        self.shard = lib().co2_sharded_shard(self.handle, C.byref(off), C.byref(ln))
        self.offset, self.length = off.value, ln.value
        if engine.transport == "p2p":  # peers read / write these over NVLink
            for which in (L.BUF_PARAMS, L.BUF_PARAMS_ALT, L.BUF_XFIRST, L.BUF_XFIRST_ALT):
                engine.register(lib().co2_sharded_buffer(self.handle, which))

    def close(self):
        if self.handle:
            lib().co2_sharded_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def buffer(self, which: int, length: int | None = None) -> torch.Tensor | None:
        ptr = lib().co2_sharded_buffer(self.handle, which)
        if not ptr:
            return None
        full = which in (L.BUF_PARAMS, L.BUF_XFIRST)
        state = which in (L.BUF_ANCHOR, L.BUF_PREV_X0, L.BUF_MOMENTUM, L.BUF_GAP)
        dt = STATE_TORCH[self.mode] if state else LOW_TORCH[self.mode]
        n = length if length is not None else (self.n if full else self.length)
        return _view(ptr, n, dt)

    @property
    def params(self):
        return self.buffer(L.BUF_PARAMS)

    def snapshot_start(self, stream=None):
        check(lib().co2_sharded_snapshot_start(self.handle, _stream(stream)))

    def snapshot_first(self, stream=None):
        check(lib().co2_sharded_snapshot_first(self.handle, _stream(stream)))

    def round(self, engine: CollectiveEngine, hyper: Co2Hyper, tau: int, *, stream=None,
              sync: bool = True) -> L.RoundResult:
        h = hyper.c(tau)
        r = L.RoundResult()
        check(lib().co2_sharded_round(self.handle, engine.handle, C.byref(h), _stream(stream),
                                      int(sync), C.byref(r)))
        return r

    def drain(self, engine: CollectiveEngine, stream=None):
        check(lib().co2_sharded_drain(self.handle, engine.handle, _stream(stream)))

    def enable_timing(self, cap: int = 4096):
        check(lib().co2_sharded_enable_timing(self.handle, cap))

    def step_times(self, cap: int = 4096) -> list[float]:
        out = (C.c_double * cap)()
        cnt = C.c_int32()
        check(lib().co2_sharded_step_times(self.handle, out, cap, C.byref(cnt)))
        return [out[i] for i in range(cnt.value)]
