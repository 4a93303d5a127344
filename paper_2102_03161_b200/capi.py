"""ctypes binding of include/eps_capi.h.

`EpsApi(path, prefix)` wraps one shared library exporting the C ABI: the
product (`libeps_b200.so`, prefix ``eps_``) or, in tests only, the reference
compiled from its own sources (`oracle/_ref/libeps_ref.so`, prefix
``epsref_``).  The Python methods mirror the reference's C++ operator names
(proj/include/eps/*.hpp) and raise the Python analogue of the C++ exception
the reference would throw, so parity tests read like the reference's own
doctest suites.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

MAX_STAGES = 64

# ---- status -> exception (eps_capi.h status table) -------------------------


class EpsError(RuntimeError):
    code = 9


class InvalidArgument(EpsError, ValueError):  # std::invalid_argument
    code = 1


class DomainError(EpsError, ValueError):  # std::domain_error
    code = 2


class LogicError(EpsError):  # std::logic_error
    code = 3


class ConfigError(EpsError):  # eps::ConfigError
    code = 4


class IoError(EpsError, OSError):  # eps::IoError
    code = 5


class CudaError(EpsError):
    code = 6


class CapacityError(EpsError):
    code = 8


_ERRORS = {c.code: c for c in (InvalidArgument, DomainError, LogicError, ConfigError,
                               IoError, CudaError, CapacityError, EpsError)}

# ---- C structs --------------------------------------------------------------

I64P = C.POINTER(C.c_int64)
IP = C.POINTER(C.c_int)
DP = C.POINTER(C.c_double)


class CModel(C.Structure):
    _fields_ = [("layers", C.c_int), ("attention_params", I64P), ("mlp_params", I64P),
                ("activation_bytes", I64P), ("bytes_per_param", C.c_int)]


class CCluster(C.Structure):
    _fields_ = [("node_count", C.c_int), ("gpus_per_node", C.c_int),
                ("gpu_memory_bytes", C.c_double), ("intra_node_bandwidth", C.c_double),
                ("inter_node_bandwidth", C.c_double)]


class CCost(C.Structure):
    _fields_ = [("c_fwd", C.c_double), ("backward_ratio", C.c_double),
                ("c_update", C.c_double), ("per_microbatch_overhead", C.c_double),
                ("allreduce_bucket_bytes", C.c_double), ("comm_latency", C.c_double)]


class CTiers(C.Structure):
    _fields_ = [("host_bandwidth", C.c_double), ("disk_bandwidth", C.c_double),
                ("host_capacity_bytes", C.c_double), ("window_batches", C.c_int),
                ("block_batches", C.c_int), ("read_latency", C.c_double)]


class CSeq(C.Structure):
    _fields_ = [("n", C.c_int), ("params", I64P), ("global_index", IP),
                ("frozen_params", C.c_int64), ("frozen_layers", C.c_int)]


class CPlan(C.Structure):
    _fields_ = [("pipeline_length", C.c_int), ("begin", C.c_int * MAX_STAGES),
                ("end", C.c_int * MAX_STAGES), ("param_sums", C.c_int64 * MAX_STAGES),
                ("effective_sizes", C.c_double * MAX_STAGES), ("frozen_params", C.c_int64),
                ("frozen_layers", C.c_int), ("lambda_frozen", C.c_double)]


class CStageLoad(C.Structure):
    _fields_ = [("fwd_params", C.c_double), ("bwd_params", C.c_double),
                ("prefix_seconds_per_sample", C.c_double), ("in_bytes_per_sample", C.c_double)]


class CBlock(C.Structure):
    _fields_ = [("device", C.c_int), ("kind", C.c_int), ("start", C.c_double),
                ("end", C.c_double), ("micro_batch", C.c_int), ("bucket", C.c_int)]


class CSummary(C.Structure):
    _fields_ = [("makespan", C.c_double), ("compute_makespan", C.c_double),
                ("makespan_without_ar", C.c_double), ("total_bubble", C.c_double),
                ("allreduce_seconds", C.c_double), ("transfer_seconds", C.c_double),
                ("compute_seconds", C.c_double), ("exposed_comm", C.c_double),
                ("n_blocks", C.c_int)]


class CMsg(C.Structure):
    _fields_ = [("sender", C.c_int), ("receiver", C.c_int), ("epoch", C.c_int),
                ("lr_schedule_position", C.c_double), ("frozen_layers", C.c_int),
                ("new_pipeline_length", C.c_int), ("span_first", C.c_int),
                ("span_length", C.c_int), ("weights_version", C.c_char * 32)]


class CEpochRow(C.Structure):
    _fields_ = [("epoch", C.c_int), ("l_frozen", C.c_int), ("pipeline_length", C.c_int),
                ("replica_width", C.c_int), ("micro_batches", C.c_int),
                ("iteration_time", C.c_double), ("epoch_time", C.c_double),
                ("throughput", C.c_double), ("bubble_time", C.c_double),
                ("comm_time", C.c_double), ("exposed_comm_time", C.c_double),
                ("cache_enabled", C.c_int), ("transition_overhead", C.c_double),
                ("cache_transition_time", C.c_double), ("stall_time", C.c_double)]


class CRunSummary(C.Structure):
    _fields_ = [("total_seconds", C.c_double), ("baseline_total_seconds", C.c_double),
                ("speedup", C.c_double), ("comm_ratio", C.c_double),
                ("frozen_forward_per_sample", C.c_double),
                ("final_prefix_forward_per_sample", C.c_double), ("n_epochs", C.c_int),
                ("n_transitions", C.c_int), ("n_cache_events", C.c_int)]


class CDecision(C.Structure):
    _fields_ = [("epoch", C.c_int), ("l_frozen", C.c_int), ("pipeline_length", C.c_int),
                ("replica_width", C.c_int), ("micro_batches", C.c_int),
                ("plan_changed", C.c_int), ("cache_enabled", C.c_int),
                ("cache_boundary", C.c_int), ("cache_old_boundary", C.c_int),
                ("cache_moved", C.c_int), ("n_messages", C.c_int), ("plan", CPlan)]


# ---- Python value types (mirror eps:: structs) ------------------------------


@dataclass
class ModelSpec:
    """eps::ModelSpec (model.hpp:15-30)."""
    attention_params: List[int]
    mlp_params: List[int]
    activation_bytes: List[int]
    bytes_per_param: int = 4
    name: str = "custom"

    @property
    def layers(self) -> int:
        return len(self.attention_params)

    def total_params(self) -> int:
        return sum(self.attention_params) + sum(self.mlp_params)

    def prefix_params(self, layer: int) -> int:
        return sum(self.attention_params[:layer]) + sum(self.mlp_params[:layer])


@dataclass
class ClusterSpec:
    node_count: int = 1
    gpus_per_node: int = 1
    gpu_memory_bytes: float = 16e9
    intra_node_bandwidth: float = 15.754e9
    inter_node_bandwidth: float = 5e9


@dataclass
class CostModel:
    c_fwd: float = 0.035 / (12.0e6 * 300.0)
    backward_ratio: float = 2.0
    c_update: float = 1.0e-11
    per_microbatch_overhead: float = 2.0e-4
    allreduce_bucket_bytes: float = 25.0e6
    comm_latency: float = 0.0


@dataclass
class CacheTierParams:
    host_bandwidth: float = 3.05e9
    disk_bandwidth: float = 6.0e9
    host_capacity_bytes: float = 64e9
    window_batches: int = 64
    block_batches: int = 8
    read_latency: float = 0.0


@dataclass
class SublayerSeq:
    """eps::SublayerSeq: params + global indices of the active sublayers."""
    params: List[int]
    global_index: List[int]
    frozen_params: int = 0
    frozen_layers: int = 0

    def active_params(self) -> int:
        return sum(self.params)


@dataclass
class PartitionPlan:
    pipeline_length: int
    spans: List[Tuple[int, int]]
    param_sums: List[int]
    effective_sizes: List[float]
    frozen_params: int = 0
    frozen_layers: int = 0
    lambda_frozen: float = 0.0

    @property
    def sublayer_counts(self) -> List[int]:
        return [e - b for b, e in self.spans]

    def max_effective_size(self) -> float:
        return max(self.effective_sizes) if self.effective_sizes else 0.0


@dataclass
class Schedule:
    makespan: float
    compute_makespan: float
    makespan_without_ar: float
    total_bubble: float
    allreduce_seconds: float
    transfer_seconds: float
    compute_seconds: float
    exposed_comm: float
    bubble_per_device: List[float] = field(default_factory=list)
    blocks: List[Tuple[int, int, float, float, int, int]] = field(default_factory=list)


def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)


class EpsApi:
    """One loaded C-ABI library.  `prefix` selects eps_ or epsref_ symbols."""

    def __init__(self, path: str, prefix: str = "eps_"):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} not built -- run `python -c 'import __graft_entry__ as g; g.build()'`")
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        self._last_error = self._fn("last_error")
        self._last_error.restype = C.c_char_p

    # -- plumbing --
    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def call(self, name, *args):
        f = self._fn(name)
        f.restype = C.c_int
        rc = f(*args)
        if rc != 0:
            msg = (self._last_error() or b"").decode()
            raise _ERRORS.get(rc, EpsError)(f"{self.prefix}{name}: {msg}")
        return rc

    def has(self, name: str) -> bool:
        return hasattr(self.lib, self.prefix + name)

    # -- conversions --
    @staticmethod
    def _model(m: ModelSpec):
        att = _arr(C.c_int64, m.attention_params)
        mlp = _arr(C.c_int64, m.mlp_params)
        act = _arr(C.c_int64, m.activation_bytes)
        cm = CModel(len(m.attention_params), att, mlp, act, m.bytes_per_param)
        cm._keep = (att, mlp, act)
        return cm

    @staticmethod
    def _cluster(c: ClusterSpec):
        return CCluster(c.node_count, c.gpus_per_node, c.gpu_memory_bytes,
                        c.intra_node_bandwidth, c.inter_node_bandwidth)

    @staticmethod
    def _cost(c: CostModel):
        return CCost(c.c_fwd, c.backward_ratio, c.c_update, c.per_microbatch_overhead,
                     c.allreduce_bucket_bytes, c.comm_latency)

    @staticmethod
    def _tiers(t: CacheTierParams):
        return CTiers(t.host_bandwidth, t.disk_bandwidth, t.host_capacity_bytes,
                      t.window_batches, t.block_batches, t.read_latency)

    @staticmethod
    def _seq(s: SublayerSeq):
        p = _arr(C.c_int64, s.params)
        g = _arr(C.c_int, s.global_index)
        cs = CSeq(len(s.params), p, g, s.frozen_params, s.frozen_layers)
        cs._keep = (p, g)
        return cs

    @staticmethod
    def _plan_in(p: PartitionPlan):
        c = CPlan()
        c.pipeline_length = p.pipeline_length
        for k, (b, e) in enumerate(p.spans):
            c.begin[k], c.end[k] = b, e
            c.param_sums[k] = p.param_sums[k]
            c.effective_sizes[k] = p.effective_sizes[k]
        c.frozen_params, c.frozen_layers, c.lambda_frozen = (
            p.frozen_params, p.frozen_layers, p.lambda_frozen)
        return c

    @staticmethod
    def _plan_out(c: CPlan) -> PartitionPlan:
        k = c.pipeline_length
        return PartitionPlan(k, [(c.begin[i], c.end[i]) for i in range(k)],
                             [c.param_sums[i] for i in range(k)],
                             [c.effective_sizes[i] for i in range(k)],
                             c.frozen_params, c.frozen_layers, c.lambda_frozen)

    # -- model.hpp --
    def model_preset(self, name: str) -> ModelSpec:
        n = C.c_int()
        self.call("model_preset", name.encode(), None, None, None, 0, C.byref(n))
        L = n.value
        att, mlp, act = (C.c_int64 * L)(), (C.c_int64 * L)(), (C.c_int64 * (2 * L + 1))()
        self.call("model_preset", name.encode(), att, mlp, act, L, C.byref(n))
        return ModelSpec(list(att), list(mlp), list(act), 4, name)

    def validate_model(self, m: ModelSpec) -> None:
        self.call("model_validate", C.byref(self._model(m)))

    def m_partition(self, m: ModelSpec, l_frozen: int) -> SublayerSeq:
        cap = 2 * m.layers
        p, g = (C.c_int64 * max(1, cap))(), (C.c_int * max(1, cap))()
        n, fp = C.c_int(), C.c_int64()
        self.call("m_partition", C.byref(self._model(m)), l_frozen, p, g, cap, C.byref(n),
                  C.byref(fp))
        return SublayerSeq(list(p[:n.value]), list(g[:n.value]), fp.value, l_frozen)

    # -- freeze.hpp --
    def freeze_state(self, alpha: float) -> "FreezeState":
        return FreezeState(self, alpha)

    def frozen_bound_closed_form(self, t: int, layers: int, alpha: float) -> float:
        out = C.c_double()
        self.call("frozen_bound_closed_form", t, layers, C.c_double(alpha), C.byref(out))
        return out.value

    def synthetic_norms(self, profile: int, seed: int, layers: int, switchover: int,
                        epoch: int) -> List[float]:
        out = (C.c_double * layers)()
        self.call("synthetic_norms", profile, C.c_uint64(seed), layers, switchover, epoch, out)
        return list(out)

    def trace_norms(self, path: str, epoch: int) -> List[float]:
        n = C.c_int()
        self.call("trace_norms", path.encode(), epoch, None, 0, C.byref(n))
        out = (C.c_double * n.value)()
        self.call("trace_norms", path.encode(), epoch, out, n.value, C.byref(n))
        return list(out)

    # -- autopipe.hpp --
    def load_balance(self, seq: SublayerSeq, k: int, lam: float, criterion: int = 0):
        out = CPlan()
        self.call("load_balance", C.byref(self._seq(seq)), k, C.c_double(lam), criterion,
                  C.byref(out))
        return self._plan_out(out)

    def try_compress(self, seq: SublayerSeq, k: int, lam: float, m_gpu0: float,
                     criterion: int = 0):
        out = CPlan()
        ak, ae, na = (C.c_int * 16)(), (C.c_double * 16)(), C.c_int()
        self.call("try_compress", C.byref(self._seq(seq)), k, C.c_double(lam),
                  C.c_double(m_gpu0), criterion, C.byref(out), ak, ae, 16, C.byref(na))
        plan = self._plan_out(out)
        return plan.pipeline_length, plan, [(ak[i], ae[i]) for i in range(na.value)]

    # -- schedule.hpp / chunks.hpp --
    def build_schedule(self, stages: Sequence[Tuple[float, float, float, float]], m: int,
                       batch: float, replica_width: int = 1, *, integer_microbatches=False,
                       group_spans_nodes=False, intra=1.0, inter=1.0, bytes_per_param=4,
                       cm: CostModel = CostModel(), with_blocks=True) -> Schedule:
        k = len(stages)
        st = (CStageLoad * k)(*[CStageLoad(*s) for s in stages])
        summ = CSummary()
        bub = (C.c_double * k)()
        self.call("build_schedule", st, k, m, C.c_double(batch), int(integer_microbatches),
                  replica_width, int(group_spans_nodes), C.c_double(intra), C.c_double(inter),
                  bytes_per_param, C.byref(self._cost(cm)), C.byref(summ), bub, None, 0)
        blocks = []
        if with_blocks:
            cap = summ.n_blocks
            bl = (CBlock * max(1, cap))()
            self.call("build_schedule", st, k, m, C.c_double(batch), int(integer_microbatches),
                      replica_width, int(group_spans_nodes), C.c_double(intra),
                      C.c_double(inter), bytes_per_param, C.byref(self._cost(cm)),
                      C.byref(summ), bub, bl, cap)
            blocks = [(b.device, b.kind, b.start, b.end, b.micro_batch, b.bucket)
                      for b in bl[:cap]]
        return Schedule(summ.makespan, summ.compute_makespan, summ.makespan_without_ar,
                        summ.total_bubble, summ.allreduce_seconds, summ.transfer_seconds,
                        summ.compute_seconds, summ.exposed_comm, list(bub), blocks)

    def schedule_iteration(self, plan, model, seq, m, batch, r, cluster, cm, cache_enabled,
                           read_per_sample) -> float:
        summ = CSummary()
        self.call("schedule_iteration", C.byref(self._plan_in(plan)), C.byref(self._model(model)),
                  C.byref(self._seq(seq)), m, C.c_double(batch), r,
                  C.byref(self._cluster(cluster)), C.byref(self._cost(cm)), int(cache_enabled),
                  C.c_double(read_per_sample), C.byref(summ))
        return summ.makespan

    def optimal_chunks(self, plan, model, seq, batch, r, cluster, cm, cache_enabled=False,
                       read_per_sample=0.0):
        k = plan.pipeline_length
        chosen = C.c_int()
        times = (C.c_double * (5 * k + 1))()
        self.call("optimal_chunks", C.byref(self._plan_in(plan)), C.byref(self._model(model)),
                  C.byref(self._seq(seq)), C.c_double(batch), r,
                  C.byref(self._cluster(cluster)), C.byref(self._cost(cm)), int(cache_enabled),
                  C.c_double(read_per_sample), C.byref(chosen), times, 5 * k + 1)
        return chosen.value, list(times)

    # -- autodp.hpp --
    def topology(self, cluster: ClusterSpec, k: int):
        cap = cluster.node_count * cluster.gpus_per_node
        act, n, r = (C.c_int * cap)(), C.c_int(), C.c_int()
        self.call("topology", C.byref(self._cluster(cluster)), k, act, cap, C.byref(n),
                  C.byref(r))
        return list(act[:n.value]), r.value

    def transition(self, cluster, old_k, new_k, epoch=0, lr=0.0, frozen=0, version="v0"):
        cap = cluster.node_count * cluster.gpus_per_node
        msgs, n = (CMsg * cap)(), C.c_int()
        self.call("transition", C.byref(self._cluster(cluster)), old_k, new_k, epoch,
                  C.c_double(lr), frozen, version.encode(), msgs, cap, C.byref(n))
        return [dict(sender=m.sender, receiver=m.receiver, epoch=m.epoch,
                     lr_schedule_position=m.lr_schedule_position, frozen_layers=m.frozen_layers,
                     new_pipeline_length=m.new_pipeline_length,
                     span=(m.span_first, m.span_length),
                     weights_version=m.weights_version.decode()) for m in msgs[:n.value]]

    def redistribute(self, dataset: int, cluster: ClusterSpec, k: int, epoch: int, seed: int):
        _, r = self.topology(cluster, k)
        ranks, offs = (C.c_int * r)(), (C.c_int64 * (r + 1))()
        ids = (C.c_int64 * max(1, dataset))()
        self.call("redistribute", C.c_int64(dataset), C.byref(self._cluster(cluster)), k, epoch,
                  C.c_uint64(seed), ranks, offs, ids)
        return list(ranks), [list(ids[offs[i]:offs[i + 1]]) for i in range(r)]

    def redistribute_flat(self, dataset: int, cluster: ClusterSpec, k: int, epoch: int,
                          seed: int):
        """Same as redistribute but returns (ranks, offsets, ids) ctypes-free via numpy."""
        import numpy as np
        _, r = self.topology(cluster, k)
        ranks = np.zeros(r, np.int32)
        offs = np.zeros(r + 1, np.int64)
        ids = np.zeros(max(1, dataset), np.int64)
        self.call("redistribute", C.c_int64(dataset), C.byref(self._cluster(cluster)), k, epoch,
                  C.c_uint64(seed), ranks.ctypes.data_as(IP), offs.ctypes.data_as(I64P),
                  ids.ctypes.data_as(I64P))
        return ranks, offs, ids[:dataset]

    def ddp_skip_set(self, plan, seq):
        cap = max(1, len(seq.params))
        g, n, pc = (C.c_int * cap)(), C.c_int(), C.c_int64()
        self.call("ddp_skip_set", C.byref(self._plan_in(plan)), C.byref(self._seq(seq)), g, cap,
                  C.byref(n), C.byref(pc))
        return list(g[:n.value]), pc.value

    # -- autocache.hpp --
    def cache_read_seconds_per_sample(self, model, boundary, tiers) -> float:
        out = C.c_double()
        self.call("cache_read_seconds_per_sample", C.byref(self._model(model)), boundary,
                  C.byref(self._tiers(tiers)), C.byref(out))
        return out.value

    def should_cache(self, l_frozen, model, cm, tiers, mb_samples):
        en, rd, fw = C.c_int(), C.c_double(), C.c_double()
        self.call("should_cache", l_frozen, C.byref(self._model(model)), C.byref(self._cost(cm)),
                  C.byref(self._tiers(tiers)), C.c_double(mb_samples), C.byref(en),
                  C.byref(rd), C.byref(fw))
        return bool(en.value), rd.value, fw.value

    def cache_transition(self, enabled, boundary, tiers, old_b, new_b, model, cm):
        r, c, w = C.c_double(), C.c_double(), C.c_double()
        self.call("cache_transition", int(enabled), boundary, C.byref(self._tiers(tiers)), old_b,
                  new_b, C.byref(self._model(model)), C.byref(self._cost(cm)), C.byref(r),
                  C.byref(c), C.byref(w))
        return r.value, c.value, w.value

    def cache_tier_epoch(self, tiers, bytes_per_batch, total_batches, iteration_seconds):
        """The modeled disk -> host window over one epoch (CacheTierSim as
        runner.cpp:258-265 drives it): dict of total stall seconds, max resident
        bytes, prefetches, evictions, sliding."""
        out = (C.c_double * 5)()
        self.call("cache_tier_epoch", C.byref(self._tiers(tiers)), C.c_double(bytes_per_batch),
                  int(total_batches), C.c_double(iteration_seconds), out)
        return {"stall_s": out[0], "max_resident_bytes": out[1], "prefetches": int(out[2]),
                "evictions": int(out[3]), "sliding": bool(out[4])}

    # -- scenario.hpp / runner.hpp --
    def scenario(self, source) -> "Scenario":
        return Scenario(self, source)

    def parse_flags(self, text: str):
        f = [C.c_int() for _ in range(4)]
        self.call("parse_flags", text.encode(), *[C.byref(x) for x in f])
        return tuple(bool(x.value) for x in f)


class FreezeState:
    """eps::FreezeState handle (freeze.hpp:23-35)."""

    def __init__(self, api: EpsApi, alpha: float):
        self.api = api
        h = C.c_void_p()
        api.call("freeze_create", C.c_double(alpha), C.byref(h))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            f = self.api._fn("freeze_destroy")
            f.restype = None
            f(self.h)
            self.h = None

    def frozen_count(self) -> int:
        out = C.c_int()
        self.api.call("freeze_frozen_count", self.h, C.byref(out))
        return out.value

    def next(self, norms: Sequence[float], layers: Optional[int] = None):
        layers = len(norms) if layers is None else layers
        out, bound = C.c_int(), C.c_double()
        self.api.call("next_frozen_count", self.h, _arr(C.c_double, norms), len(norms), layers,
                      C.byref(out), C.byref(bound))
        return out.value, bound.value


class Scenario:
    """eps::ScenarioConfig handle; `source` is a path or a dict/JSON text."""

    def __init__(self, api: EpsApi, source):
        self.api = api
        h = C.c_void_p()
        if isinstance(source, dict):
            api.call("scenario_parse", json.dumps(source).encode(), C.byref(h))
        elif isinstance(source, str) and source.lstrip().startswith("{"):
            api.call("scenario_parse", source.encode(), C.byref(h))
        else:
            api.call("scenario_load", str(source).encode(), C.byref(h))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            f = self.api._fn("scenario_destroy")
            f.restype = None
            f(self.h)
            self.h = None

    def _text(self, name, *args) -> str:
        n = C.c_size_t()
        self.api.call(name, self.h, *args, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        self.api.call(name, self.h, *args, buf, n.value + 1, C.byref(n))
        return buf.value.decode()

    def to_json(self) -> dict:
        return json.loads(self._text("scenario_to_json"))

    def simulate(self):
        summ = CRunSummary()
        self.api.call("simulate_run", self.h, None, 0, C.byref(summ))
        rows = (CEpochRow * max(1, summ.n_epochs))()
        self.api.call("simulate_run", self.h, rows, summ.n_epochs, C.byref(summ))
        out = [{f: getattr(r, f) for f, _ in CEpochRow._fields_} for r in rows[:summ.n_epochs]]
        return out, {f: getattr(summ, f) for f, _ in CRunSummary._fields_}

    def report(self, kind: int) -> str:
        return self._text("simulate_report", kind)

    def speedup_breakdown(self):
        t, a, s = (C.c_double * 6)(), (C.c_double * 6)(), (C.c_double * 6)()
        self.api.call("speedup_breakdown", self.h, t, a, s)
        names = ["baseline", "freeze", "autopipe", "autopipe+autocache", "autopipe+autodp",
                 "all"]
        return [(names[i], t[i], a[i], s[i]) for i in range(6)]
