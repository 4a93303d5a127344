"""Epoch decision planner for the real training loop.

Wraps eps_planner_* (runner.cpp's decision order, see include/eps/runner.hpp
EpochPlanner): at the top of every epoch it takes the per-layer gradient
norms observed in the previous epoch -- from the device reduction, or from
the scenario's synthetic/trace source -- and returns L_frozen, the AutoPipe
plan, K, R, M and the AutoCache state, bit-identical to what the reference's
simulate_run decides for the same inputs.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

from .capi import CDecision, EpsApi, Scenario


@dataclass
class EpochDecision:
    epoch: int
    l_frozen: int
    pipeline_length: int
    replica_width: int
    micro_batches: int
    plan_changed: bool
    cache_enabled: bool
    cache_boundary: int
    cache_old_boundary: int
    cache_moved: bool
    n_messages: int
    spans: List[Tuple[int, int]]      # spans per stage, indices into the planned sequence
    param_sums: List[int]
    # global index of the planned sequence's first sublayer: 2 * L_f when
    # AutoPipe repartitions the active sublayers, 0 when it is off and the
    # epoch-0 partition of the whole model is kept (runner.cpp begin_epoch:
    # frozen layers then still occupy their stage)
    span_base: int = 0


class Planner:
    def __init__(self, api: EpsApi, scenario):
        self.api = api
        self.scenario = scenario if isinstance(scenario, Scenario) else Scenario(api, scenario)
        h = C.c_void_p()
        api.call("planner_create", self.scenario.h, C.byref(h))
        self.h = h
        self.layers = self._layers()
        self.elastic = bool(self.scenario.to_json().get("features", {}).get("autopipe", True))

    def _layers(self) -> int:
        n, bpp = C.c_int(), C.c_int()
        self.api.call("scenario_model", self.scenario.h, None, None, None, 0, C.byref(n),
                      C.byref(bpp))
        return n.value

    def __del__(self):
        if getattr(self, "h", None):
            f = self.api._fn("planner_destroy")
            f.restype = None
            f(self.h)
            self.h = None

    def begin_epoch(self, epoch: int, norms_prev: Optional[Sequence[float]] = None) -> EpochDecision:
        d = CDecision()
        if norms_prev is None:
            self.api.call("planner_begin_epoch", self.h, epoch, None, 0, C.byref(d))
        else:
            arr = (C.c_double * len(norms_prev))(*norms_prev)
            self.api.call("planner_begin_epoch", self.h, epoch, arr, len(norms_prev), C.byref(d))
        k = d.plan.pipeline_length
        return EpochDecision(d.epoch, d.l_frozen, d.pipeline_length, d.replica_width,
                             d.micro_batches, bool(d.plan_changed), bool(d.cache_enabled),
                             d.cache_boundary, d.cache_old_boundary, bool(d.cache_moved),
                             d.n_messages, [(d.plan.begin[i], d.plan.end[i]) for i in range(k)],
                             [d.plan.param_sums[i] for i in range(k)],
                             2 * d.l_frozen if self.elastic else 0)
