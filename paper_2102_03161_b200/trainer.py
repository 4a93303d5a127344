"""The real epoch loop: simulate_run's decision order, executed on B200s.

runner.cpp:94-305 walks the epochs, takes the decisions (freeze count from
the gradient norms observed in the previous epoch, AutoPipe partition and
compression, AutoDP width and rank activation, AutoCache on/off and boundary
moves, micro-batch count) and then *costs* the epoch.  `Trainer` takes the
same decisions through EpochPlanner (bit-identical to the reference for the
same norm vectors) and then *runs* the epoch:

  * norms: per-layer L2 of the post-all-reduce gradients of the last
    iteration of epoch e-1, reduced on the device (segmented fp64 Σg²) -- the
    device-backed GradNormSource (freeze.hpp:51-57);
  * plan change: StageRunner.set_plan migrates parameters / momentum to their
    new owners and rebuilds the per-stage data-parallel groups;
  * data: the samples of this replica come from redistribute
    (autodp.cpp:113-151) -- node-local subsets shuffled per epoch;
  * AutoCache: the store holds the boundary activation X[L_f] per sample
    (bf16 [N, T, d]) on every pipeline's stage-0 GPU.  A boundary-move epoch
    runs the cache-write path (gather old boundary, forward the delta, scatter
    the new one -- autocache.cpp:45-67) for every sample once, then the
    stage-0 stores exchange the rows each wrote (a replica's next-epoch shard
    may hold samples another replica cached); steady epochs gather and skip
    the frozen forward entirely.

Epoch rows use the reference's CSV schema (runner.cpp:340-355) with measured
device times.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import torch
import torch.distributed as dist

from . import LIB_PATH, ops
from .capi import ClusterSpec, EpsApi
from .configs import Geometry
from .pipeline import StagePlan, StageRunner, Transport
from .planner import Planner
from .vit import VitExecutor

CSV_HEADER = ("epoch,l_frozen,k,r,m,iteration_time_s,epoch_time_s,throughput_sps,"
              "bubble_time_s,comm_time_s,exposed_comm_time_s,cache_enabled,"
              "transition_overhead_s,cache_transition_time_s,stall_time_s")


@dataclass
class EpochResult:
    epoch: int
    l_frozen: int
    k: int
    r: int
    m: int
    iteration_time_s: float
    epoch_time_s: float
    throughput_sps: float
    cache_enabled: bool
    cache_moved: bool
    transition_time_s: float
    mean_loss: float
    norms: List[float] = field(default_factory=list)

    def csv(self) -> str:
        return (f"{self.epoch},{self.l_frozen},{self.k},{self.r},{self.m},"
                f"{self.iteration_time_s:.9g},{self.epoch_time_s:.9g},{self.throughput_sps:.9g},"
                f"0,0,0,{int(self.cache_enabled)},{self.transition_time_s:.9g},0,0")


class Trainer:
    """One rank of an elastic PipeTransformer run on synthetic data."""

    def __init__(self, scenario: dict, geometry: Geometry, *, iterations_per_epoch: int,
                 seed: int = 17, lr: float = 1e-3, momentum: float = 0.9,
                 rank: int = 0, world: int = 1, device=None, host_staged: bool = False,
                 device_norms: bool = True, cache_tier: str = "hbm", peer: bool = False,
                 cache_prefetch: bool = True):
        self.g = geometry
        self.api = EpsApi(LIB_PATH, "eps_")
        self.planner = Planner(self.api, scenario)
        self.scenario = scenario
        cl = scenario["cluster"]
        self.cluster = ClusterSpec(cl.get("nodes", 1), cl.get("gpus_per_node", 1))
        if self.cluster.node_count * self.cluster.gpus_per_node != world:
            raise ValueError("scenario cluster size must equal the number of ranks")
        self.batch = int(scenario["training"]["per_pipeline_batch"])
        self.iters = iterations_per_epoch
        self.seed = seed
        self.lr, self.momentum = lr, momentum
        self.rank, self.world = rank, world
        self.device = torch.device(device or "cuda")
        self.device_norms = device_norms
        self.ex = VitExecutor(geometry, max_batch=self.batch, seed=seed, device=self.device)
        self.runner = StageRunner(self.ex, rank, world, Transport(host_staged=host_staged),
                                  peer=peer)
        self.tp = self.runner.tp
        # dataset = iterations x batch x initial replica count (runner.cpp:103-104)
        k0 = scenario.get("initial_pipeline_length", 0) or self.cluster.gpus_per_node
        self.r0 = world // k0
        self.dataset = self.iters * self.batch * self.r0
        gen = torch.Generator(device=self.device).manual_seed(seed)
        g = geometry
        self.images = torch.randn(self.dataset, g.channels, g.input_image, g.input_image,
                                  device=self.device, generator=gen)
        self.labels = torch.randint(0, g.classes, (self.dataset,), device=self.device,
                                    generator=gen)
        # AutoCache tier: "hbm" (device store) or "host" (pinned host memory,
        # read / written by the same kernels over the host link -- the real
        # counterpart of the reference's host tier, autocache.cpp:69-150)
        if cache_tier not in ("hbm", "host"):
            raise ValueError("cache_tier must be 'hbm' or 'host'")
        if cache_tier == "host" and world > 1 and not host_staged:
            raise NotImplementedError("host-tier store exchange over NCCL (needs device staging)")
        self.cache_tier = cache_tier
        self.cache_prefetch = cache_prefetch
        self.cache_prefetch_ctas = 8  # SMs the background gather borrows
        self._win_buf = None
        self.store: Optional[torch.Tensor] = None
        self.norms_prev: Optional[List[float]] = None

    # -- helpers -------------------------------------------------------------------
    def _max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.tp.all_reduce(t, None, op=dist.ReduceOp.MAX)
        return float(t.item())

    def _sync_store(self, plan: StagePlan, written: torch.Tensor):
        """After a boundary move each stage-0 store holds the new boundary
        rows of the samples its replica processed; exchange them so every
        stage-0 GPU holds all rows (zero the rest, sum over stage-0 ranks)."""
        if plan.R == 1:
            return
        keep = torch.zeros(self.dataset, dtype=torch.bool, device=self.store.device)
        keep[written.to(self.store.device)] = True
        if self.runner.stage == 0:
            self.store[~keep] = 0
        group = self.tp.group([p * plan.K for p in range(plan.R)])
        if self.runner.stage == 0:
            self.tp.all_reduce(self.store, group)

    def _window_setup(self):
        """Two device staging buffers for the host tier's prefetch window."""
        if self._win_buf is not None:
            return
        shape = (self.batch, self.g.tokens, self.g.hidden)
        self._win_buf = [torch.empty(shape, dtype=torch.bfloat16, device=self.device)
                         for _ in range(2)]
        self._win_ids = torch.arange(self.batch, dtype=torch.int64, device=self.device)
        self._win_copy = torch.cuda.Stream(device=self.device)
        self._win_ready = [torch.cuda.Event(), torch.cuda.Event()]
        self._win_free = [torch.cuda.Event(), torch.cuda.Event()]
        for e in self._win_free:  # both slots start free
            e.record(torch.cuda.current_stream(self.device))

    # -- one epoch -----------------------------------------------------------------------
    def run_epoch(self, epoch: int) -> EpochResult:
        d = self.planner.begin_epoch(epoch, self.norms_prev if self.device_norms and epoch > 0
                                     else None)
        plan = StagePlan.from_decision(d, self.g.layers)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_start = torch.cuda.Event(enable_timing=True)
        t_start.record()
        self.runner.set_plan(plan)  # transition: migrate + regroup
        pipe, stage = plan.role(self.rank)
        if d.cache_enabled and d.cache_boundary != d.l_frozen:
            raise NotImplementedError("cache boundary below L_frozen (policy flip) not executed")
        if d.cache_enabled and self.store is None:
            shape = (self.dataset, self.g.tokens, self.g.hidden)
            if self.cache_tier == "host":
                self.store = torch.zeros(shape, dtype=torch.bfloat16).pin_memory()
            else:
                self.store = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)
        if self.store is not None and d.plan_changed and self.world > 1:
            # a fork makes new stage-0 GPUs: they receive the complete store
            # from rank 0 (stage 0 of pipeline 0 always holds every row)
            self.tp.broadcast(self.store, 0)
        cache_mode = 0 if not d.cache_enabled else (2 if d.cache_moved else 1)
        _, shards = self.api.redistribute(self.dataset, self.cluster, plan.K, epoch, self.seed)
        shard = torch.tensor(shards[pipe], dtype=torch.int64, device=self.device)
        iters = len(shards[pipe]) // self.batch
        # Host-tier gather epochs: a sliding window over the epoch's rows --
        # iteration it + 1's cached boundary activations are gathered from
        # pinned host memory into a device staging buffer on a copy stream
        # while iteration it computes, so the host link overlaps compute
        # (SURVEY.md 8(f) row 1); the executor then gathers from the staging
        # buffer (HBM) with identity ids.
        window = (self.cache_tier == "host" and cache_mode == 1 and stage == 0
                  and self.cache_prefetch and iters > 0)
        if window:
            self._window_setup()
            stream = torch.cuda.current_stream(self.device)

            def fetch(i):
                slot = i % 2
                self._win_copy.wait_event(self._win_free[slot])
                rows = shard[i * self.batch:(i + 1) * self.batch]
                ops.call("eps_cache_gather_bg", self.store, rows, self.batch,
                         self.g.tokens * self.g.hidden * 2, self._win_buf[slot],
                         self.cache_prefetch_ctas, C.c_void_p(self._win_copy.cuda_stream))
                self._win_ready[slot].record(self._win_copy)

            fetch(0)
        start.record()
        losses = []
        norms = None
        for it in range(iters):
            ids = shard[it * self.batch:(it + 1) * self.batch]
            x = self.images.index_select(0, ids) if stage == 0 and cache_mode != 1 else None
            y = self.labels.index_select(0, ids)
            store, sids = self.store, ids
            if window:
                if it + 1 < iters:
                    fetch(it + 1)
                stream.wait_event(self._win_ready[it % 2])
                store, sids = self._win_buf[it % 2], self._win_ids
            loss = self.runner.iteration(x, y, self.batch, cache_mode=cache_mode,
                                         cache_old=d.cache_old_boundary, store=store,
                                         ids=sids)
            if window:
                self._win_free[it % 2].record(stream)
            self.runner.sync_grads()
            if it == iters - 1:
                norms = self.runner.layer_sqnorms(self.ex.segments).sqrt()
            self.runner.step(self.lr, self.momentum)
            if stage == plan.K - 1:
                losses.append(loss.clone())
        stop.record()
        if cache_mode == 2:
            self._sync_store(plan, shard[:iters * self.batch])
        torch.cuda.synchronize()
        ms = self._max_over_ranks(start.elapsed_time(stop))
        trans = self._max_over_ranks(t_start.elapsed_time(start)) / 1000.0
        self.norms_prev = norms.cpu().tolist() if norms is not None else None
        mean_loss = (sum(float(l) for l in losses) / (len(losses) * self.batch)
                     if losses else float("nan"))
        samples = iters * self.batch * plan.R
        return EpochResult(epoch, d.l_frozen, plan.K, plan.R, plan.M, ms / 1000.0 / max(1, iters),
                           ms / 1000.0, samples / (ms / 1000.0), d.cache_enabled, d.cache_moved,
                           trans, mean_loss, self.norms_prev or [])

    def run(self, epochs: Optional[int] = None) -> List[EpochResult]:
        n = epochs if epochs is not None else int(self.scenario["training"]["epochs"])
        return [self.run_epoch(e) for e in range(n)]

    @staticmethod
    def report_csv(rows: List[EpochResult]) -> str:
        return CSV_HEADER + "\n" + "".join(r.csv() + "\n" for r in rows)
