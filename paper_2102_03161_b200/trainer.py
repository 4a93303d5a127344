"""The real epoch loop: simulate_run's decision order, executed on B200s.

runner.cpp:94-305 walks the epochs, takes the decisions (freeze count from
the gradient norms observed in the previous epoch, AutoPipe partition and
compression, AutoDP width and rank activation, AutoCache on/off and boundary
moves, micro-batch count) and then *costs* the epoch.  `Trainer` takes the
same decisions through EpochPlanner (bit-identical to the reference for the
same norm vectors) and then *runs* the epoch:

  * norms: per-layer L2 of the post-all-reduce gradients of the last
    iteration of epoch e-1, reduced on the device (segmented fp64 sum of
    squares) -- the device-backed GradNormSource (freeze.hpp:51-57);
  * plan change: StageRunner.set_plan migrates parameters / momentum to their
    new owners and rebuilds the per-stage data-parallel groups; with AutoPipe
    on and AutoDP off the ranks beyond K*R idle (runner.cpp:445);
  * data: the samples of this replica come from redistribute
    (autodp.cpp:113-151) -- node-local subsets shuffled per epoch, every
    sample of the shard trained (a ragged last iteration takes the
    remainder, runner.cpp:245 counts fractional iterations);
  * AutoCache: `CacheStore` holds the boundary activation X[boundary] of
    every sample (bf16 rows of T*d).  HBM tier: the rows are sharded over the
    node's GPUs and every shard is IPC-mapped into every rank, so a replica
    gathers (and on a boundary move scatters) the rows of its epoch shard
    from the owning GPU's HBM over NVLink inside one kernel -- per-GPU store
    bytes ~ dataset / world, no replication or exchange.  Host tier: one
    node-wide pinned shared-memory segment every rank maps
    (autocache.cpp:69-150's host tier), read through a sliding prefetch
    window on a copy stream.  Disk tier: a node-wide backing file behind a
    page-locked host window refilled block by block by native I/O threads
    (the reference's modeled disk -> host CacheTierSim, run for real:
    disk_tier.py), copied batch by batch into HBM staging on a copy stream.
    Boundary-move epochs run the cache-write path
    (autocache.cpp:45-67), trailing-boundary epochs gather the old boundary
    and forward the rest of the frozen prefix (runner.cpp:186-213), steady
    epochs gather and skip the frozen forward entirely.

Epoch rows use the reference's CSV schema (runner.cpp:340-355) with every
column measured by CUDA events (see EpochResult).
"""
from __future__ import annotations

import ctypes as C
import os
import uuid
from dataclasses import dataclass, field
from typing import List, Optional

import torch
import torch.distributed as dist

from . import LIB_PATH, ops
from .capi import ClusterSpec, EpsApi
from .configs import Geometry
from .pipeline import (EpsTransport, StagePlan, StageRunner, Transport,
                       microbatch_offsets)
from .planner import Planner
from .vit import VitExecutor

CSV_HEADER = ("epoch,l_frozen,k,r,m,iteration_time_s,epoch_time_s,throughput_sps,"
              "bubble_time_s,comm_time_s,exposed_comm_time_s,cache_enabled,"
              "transition_overhead_s,cache_transition_time_s,stall_time_s")


@dataclass
class EpochResult:
    """One epoch, measured.  Column semantics follow runner.cpp:280-291:
    bubble = idle time summed over one pipeline's K stages in an iteration
    (makespan - busy F / B blocks, schedule.cpp:126-131); comm / exposed_comm
    = the epoch's DP all-reduce time / the part not hidden behind the drain;
    transition = set_plan (migration + regroup); cache_transition = extra
    time of a boundary-move epoch's prefix work over a steady gather; stall
    = compute-stream waits on the host tier's prefetch window, plus (disk
    tier) host waits for blocks still being read from disk."""
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
    bubble_time_s: float = 0.0
    comm_time_s: float = 0.0
    exposed_comm_time_s: float = 0.0
    cache_transition_time_s: float = 0.0
    stall_time_s: float = 0.0
    samples: int = 0

    def csv(self) -> str:
        f = lambda x: f"{x:.9g}"  # noqa: E731
        return (f"{self.epoch},{self.l_frozen},{self.k},{self.r},{self.m},"
                f"{f(self.iteration_time_s)},{f(self.epoch_time_s)},{f(self.throughput_sps)},"
                f"{f(self.bubble_time_s)},{f(self.comm_time_s)},{f(self.exposed_comm_time_s)},"
                f"{int(self.cache_enabled)},{f(self.transition_time_s)},"
                f"{f(self.cache_transition_time_s)},{f(self.stall_time_s)}")


def _lib():
    lib = ops.api().lib
    for n, args in {"eps_ipc_export": [C.c_void_p, C.c_void_p, C.c_void_p],
                    "eps_ipc_open": [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p],
                    "eps_ipc_close": [C.c_void_p],
                    "eps_host_register": [C.c_void_p, C.c_int64],
                    "eps_host_unregister": [C.c_void_p],
                    "eps_copy2d_async": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                         C.c_int64, C.c_int64, C.c_void_p]}.items():
        getattr(lib, n).argtypes = args
        getattr(lib, n).restype = C.c_int
    return lib


class CacheStore:
    """The AutoCache store of one run (see the module docstring).

    tier "hbm": rank r holds sample rows [r*n, (r+1)*n), n = ceil(dataset /
    world); `table` (device uint64[world]) holds every shard's base address
    in this process (own shard local, the others CUDA-IPC-mapped) and the
    executor is switched to the sharded gather / scatter kernels.
    tier "host": one pinned host segment of dataset rows: private pinned
    memory at world 1, a POSIX shared-memory segment registered by every rank
    (cudaHostRegister, mapped) when several ranks share the node.
    tier "disk": one node-wide file of dataset rows (rank 0 creates it under
    `cache_dir`), each rank with its own DiskTier window of the scenario's
    window_batches / block_batches (CacheTierParams) and I/O threads, plus a
    pinned batch buffer for the write path."""

    def __init__(self, tier: str, dataset: int, row_elems: int, rank: int, world: int, device,
                 collective: bool, batch: int = 0, tiers: Optional[dict] = None,
                 cache_dir: Optional[str] = None):
        self.tier, self.dataset, self.row_elems = tier, dataset, row_elems
        self.rank, self.world, self.device = rank, world, device
        self.row_bytes = row_elems * 2
        self.lib = _lib()
        self.opened: List[int] = []
        self.shm = None
        self.registered = None
        self.table = None
        self.disk = None
        self.path = None
        if tier == "disk":
            self._open_disk(batch, tiers or {}, cache_dir, collective)
        elif tier == "hbm":
            self.rows_per_shard = -(-dataset // world)
            self.local = torch.zeros(self.rows_per_shard, row_elems, dtype=torch.bfloat16,
                                     device=device)
            if world > 1:
                self._map_peers()
        elif world == 1 or not collective:
            self.rows_per_shard = dataset
            self.local = torch.zeros(dataset, row_elems, dtype=torch.bfloat16).pin_memory()
        else:
            self.rows_per_shard = dataset
            self._shared_host()

    # -- HBM shards over CUDA IPC --------------------------------------------------
    def _map_peers(self):
        import pickle
        h = (C.c_char * 64)()
        off = C.c_int64()
        if self.lib.eps_ipc_export(C.c_void_p(self.local.data_ptr()), h, C.byref(off)) != 0:
            raise RuntimeError("eps_ipc_export failed (cache shard)")
        allh = [None] * self.world
        dist.all_gather_object(allh, pickle.dumps((bytes(h), off.value)))
        ptrs = []
        for r, blob in enumerate(allh):
            if r == self.rank:
                ptrs.append(self.local.data_ptr())
                continue
            hb, o = pickle.loads(blob)
            base, ptr = C.c_void_p(), C.c_void_p()
            if self.lib.eps_ipc_open((C.c_char * 64).from_buffer_copy(hb), o, C.byref(base),
                                     C.byref(ptr)) != 0:
                raise RuntimeError("eps_ipc_open failed (cache shard)")
            self.opened.append(base.value)
            ptrs.append(ptr.value)
        self.table = torch.tensor(ptrs, dtype=torch.int64, device=self.device)

    # -- node-wide host segment -----------------------------------------------------
    def _shared_host(self):
        from multiprocessing import shared_memory
        nbytes = self.dataset * self.row_bytes
        name = [f"eps_cache_{uuid.uuid4().hex[:16]}" if self.rank == 0 else None]
        if self.rank == 0:
            self.shm = shared_memory.SharedMemory(name=name[0], create=True, size=nbytes)
        dist.broadcast_object_list(name, src=0)
        if self.rank != 0:
            self.shm = shared_memory.SharedMemory(name=name[0])
        dist.barrier()
        self.local = torch.frombuffer(self.shm.buf, dtype=torch.bfloat16,
                                      count=self.dataset * self.row_elems).view(
                                          self.dataset, self.row_elems)
        if self.rank == 0:
            self.local.zero_()
        if self.lib.eps_host_register(C.c_void_p(self.local.data_ptr()), nbytes) != 0:
            raise RuntimeError("eps_host_register failed (shared host tier)")
        self.registered = self.local.data_ptr()
        dist.barrier()

    # -- disk tier ------------------------------------------------------------------
    def _open_disk(self, batch: int, tiers: dict, cache_dir: Optional[str], collective: bool):
        import tempfile
        from .disk_tier import DiskTier
        d = cache_dir or os.environ.get("EPS_CACHE_DIR") or tempfile.gettempdir()
        name = [f"eps_cache_{uuid.uuid4().hex[:16]}.bin" if self.rank == 0 else None]
        if collective and self.world > 1:
            dist.broadcast_object_list(name, src=0)
        self.path = os.path.join(d, name[0])
        wb = int(tiers.get("window_batches", 64))
        bb = int(tiers.get("block_batches", 8))
        # host capacity caps the window like CacheTierSim's constructor
        cap = float(tiers.get("host_capacity_bytes", 64e9))
        wb = max(bb, min(wb, int(cap // max(1, batch * self.row_bytes)) // bb * bb))
        create = self.rank == 0 or not collective
        if not create:
            dist.barrier()  # the creator has sized the file
        self.disk = DiskTier(self.path, self.dataset, self.row_bytes, batch, block_batches=bb,
                             window_batches=wb, threads=8, create=create)
        if create and collective and self.world > 1:
            dist.barrier()
        self.rows_per_shard = self.dataset
        self.local = None
        self.wbuf = torch.empty(batch, self.row_elems, dtype=torch.bfloat16).pin_memory()

    # -- use ------------------------------------------------------------------------
    def attach(self, ex):
        """Point the executor's cache_mode gathers / scatters at this store."""
        if self.table is not None:
            ex._call(ex.PREFIX + "set_cache_shards", self.table, C.c_int64(self.rows_per_shard))
        else:
            ex._call(ex.PREFIX + "set_cache_shards", C.c_void_p(0), C.c_int64(0))

    def store_arg(self):
        """What the stage calls receive as `store` (disk tier: none -- the
        trainer passes its HBM staging window)."""
        return self.local

    def rows(self, ids: torch.Tensor) -> torch.Tensor:
        """Rows of sample ids (test / report helper; gathers on the device)."""
        out = torch.empty(ids.numel(), self.row_elems, dtype=torch.bfloat16, device=self.device)
        if self.disk is not None:  # read straight from the backing file
            order = ids.cpu()
            self.disk.begin_epoch(order)
            o = 0
            for b in range(-(-ids.numel() // self.disk.batch_rows)):
                view, _ = self.disk.batch_view(b)
                n = view.shape[0]
                out[o:o + n].view(torch.uint8).view(n, self.row_bytes).copy_(
                    view[:, :self.row_bytes])
                self.disk.release(b)
                o += n
            return out
        if self.table is not None:
            ops.call("eps_cache_gather_sharded", self.table, C.c_int64(self.rows_per_shard),
                     ids, ids.numel(), C.c_int64(self.row_bytes), out,
                     C.c_void_p(torch.cuda.current_stream().cuda_stream))
        else:
            ops.call("eps_cache_gather", self.local, ids, ids.numel(),
                     C.c_int64(self.row_bytes), out,
                     C.c_void_p(torch.cuda.current_stream().cuda_stream))
        return out

    def shard_bytes(self) -> int:
        """Bytes of the store this rank holds (HBM shard, its host segment, or
        the disk tier's file)."""
        if self.disk is not None:
            return self.dataset * self.row_bytes
        return self.local.numel() * 2

    def close(self):
        if self.disk is not None:
            self.disk.close()
            self.disk = None
            if self.rank == 0 and self.path and os.path.exists(self.path):
                os.unlink(self.path)
        for b in self.opened:
            self.lib.eps_ipc_close(C.c_void_p(b))
        self.opened = []
        if self.registered is not None:
            torch.cuda.synchronize()
            self.lib.eps_host_unregister(C.c_void_p(self.registered))
            self.registered = None
        if self.shm is not None:
            self.local = None
            self.shm.close()
            if self.rank == 0:
                self.shm.unlink()
            self.shm = None


def epoch_iterations(n: int, batch: int):
    """[(offset, size)] covering a shard of n samples: full batches, then a
    ragged last one (runner.cpp:245: iterations = dataset / (batch * R))."""
    if n <= 0:
        raise ValueError("empty epoch shard")
    out = [(i * batch, batch) for i in range(n // batch)]
    if n % batch:
        out.append((n - n % batch, n % batch))
    return out


class Trainer:
    """One rank of an elastic PipeTransformer run on synthetic data."""

    def __init__(self, scenario: dict, geometry: Geometry, *, iterations_per_epoch: int,
                 seed: int = 17, lr: float = 1e-3, momentum: float = 0.9,
                 rank: int = 0, world: int = 1, device=None, host_staged: bool = False,
                 device_norms: bool = True, cache_tier: str = "hbm", peer: bool = False,
                 cache_prefetch: bool = True, comm: str = "torch",
                 cache_dir: Optional[str] = None):
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
        # comm "eps": collectives / sends through the library's NCCL
        # communicator plane (EpsTransport); "torch": torch.distributed groups
        if comm == "eps" and world > 1 and not host_staged:
            transport = EpsTransport(rank, world)
        else:
            transport = Transport(host_staged=host_staged)
        self.runner = StageRunner(self.ex, rank, world, transport, peer=peer)
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
        if cache_tier not in ("hbm", "host", "disk"):
            raise ValueError("cache_tier must be 'hbm', 'host' or 'disk'")
        self.cache_tier = cache_tier
        self.cache_dir = cache_dir
        self.disk_stats: List[dict] = []
        self.cache_prefetch = cache_prefetch
        self.cache_prefetch_ctas = 8  # SMs the background gather borrows
        self._win_buf = None
        self.store: Optional[CacheStore] = None
        self.norms_prev: Optional[List[float]] = None

    # -- helpers -------------------------------------------------------------------
    def _reduce(self, x: float, op) -> float:
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.tp.all_reduce(t, None, op=op)
        return float(t.item())

    def _max_over_ranks(self, x: float) -> float:
        return self._reduce(x, dist.ReduceOp.MAX)

    def _barrier(self):
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()

    def _window_setup(self, rows: int):
        """Two device staging buffers for the host tier's prefetch window."""
        if self._win_buf is not None:
            return
        self._win_buf = [torch.empty(rows, self.g.tokens * self.g.hidden, dtype=torch.bfloat16,
                                     device=self.device) for _ in range(2)]
        self._win_ids = torch.arange(rows, dtype=torch.int64, device=self.device)
        self._win_copy = torch.cuda.Stream(device=self.device)
        self._win_ready = [torch.cuda.Event(), torch.cuda.Event()]
        self._win_free = [torch.cuda.Event(), torch.cuda.Event()]
        for e in self._win_free:  # both slots start free
            e.record(torch.cuda.current_stream(self.device))

    def _time_gather(self, ids: torch.Tensor) -> float:
        """Seconds of one steady-state AutoCache gather of `ids` (the baseline a
        boundary-move epoch's prefix work is charged against)."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        self.store.rows(ids)  # warm
        ev[0].record()
        self.store.rows(ids)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / 1e3

    # -- one epoch -----------------------------------------------------------------------
    def run_epoch(self, epoch: int) -> EpochResult:
        norms_in = None
        if self.device_norms and epoch > 0:
            if self.norms_prev is None:
                raise RuntimeError("device-norm run has no gradient norms from the last epoch")
            norms_in = self.norms_prev
        d = self.planner.begin_epoch(epoch, norms_in)
        plan = StagePlan.from_decision(d, self.g.layers)
        self._barrier()
        t_start, start, stop = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        t_start.record()
        self.runner.set_plan(plan)  # transition: migrate + regroup
        pipe, stage = plan.role(min(self.rank, plan.K * plan.R - 1))
        idle = self.runner.idle
        if d.cache_enabled and self.store is None:
            self.store = CacheStore(self.cache_tier, self.dataset, self.g.tokens * self.g.hidden,
                                    self.rank, self.world, self.device,
                                    collective=self.world > 1, batch=self.batch,
                                    tiers=self.scenario.get("cache"), cache_dir=self.cache_dir)
            self.store.attach(self.ex)
        if not d.cache_enabled:
            cache_mode, cache_old = 0, 0
        elif d.cache_moved:
            cache_mode, cache_old = 2, d.cache_old_boundary
        elif d.cache_boundary < d.l_frozen:
            cache_mode, cache_old = 3, d.cache_boundary  # trailing boundary
        else:
            cache_mode, cache_old = 1, 0
        _, shards = self.api.redistribute(self.dataset, self.cluster, plan.K, epoch, self.seed)
        shard = (torch.tensor(shards[pipe], dtype=torch.int64, device=self.device)
                 if not idle else torch.zeros(0, dtype=torch.int64, device=self.device))
        lens = {len(x) for x in shards}
        if len(lens) == 1:
            its = epoch_iterations(len(shards[pipe]), self.batch)
        else:  # uneven shards: every replica runs the same number of iterations
            n_its = -(-max(lens) // self.batch)
            its = microbatch_offsets(len(shards[pipe]), n_its)
        # Host-tier gather epochs: a sliding window over the epoch's rows --
        # iteration it + 1's cached boundary activations are gathered from
        # pinned host memory into a device staging buffer on a copy stream
        # while iteration it computes, so the host link overlaps compute
        # (SURVEY.md 8(f) row 1); the executor then gathers from the staging
        # buffer (HBM) with identity ids.
        window = (self.cache_tier == "host" and cache_mode == 1 and stage == 0 and not idle
                  and self.cache_prefetch)
        stream = torch.cuda.current_stream(self.device)
        # Disk tier (stage 0 of a cache epoch): the executor always sees the
        # HBM staging window with identity ids.  Batches that read the store
        # (gather, trailing boundary, a boundary move from an old boundary)
        # come from the disk tier's host window -- acquire (host wait = the
        # disk stall), one 2D copy per batch on the copy stream one iteration
        # ahead, release once copied; boundary moves write the new boundary
        # rows back: staging -> pinned buffer -> file by sample id.
        disk = self.cache_tier == "disk" and cache_mode in (1, 2, 3) and stage == 0 and not idle
        disk_reads = disk and (cache_mode != 2 or cache_old > 0)
        disk_stall = 0.0
        if disk:
            self._window_setup(self.batch)
            self.ex._call(self.ex.PREFIX + "set_cache_shards", C.c_void_p(0), C.c_int64(0))
            dt = self.store.disk
            rb = self.store.row_bytes
            if disk_reads:
                dt.begin_epoch(shard.cpu(), its)

            def dfetch(i):
                nonlocal disk_stall
                slot = i % 2
                addr, n, st = dt.acquire(i)
                disk_stall += st
                self._win_copy.wait_event(self._win_free[slot])
                if self.store.lib.eps_copy2d_async(
                        C.c_void_p(self._win_buf[slot].data_ptr()), rb, C.c_void_p(addr),
                        dt.stride, rb, n, C.c_void_p(self._win_copy.cuda_stream)) != 0:
                    raise RuntimeError("eps_copy2d_async failed (disk tier)")
                self._win_ready[slot].record(self._win_copy)

            if disk_reads:
                dfetch(0)
        if window:
            self._window_setup(self.batch)
            self.ex._call(self.ex.PREFIX + "set_cache_shards", C.c_void_p(0), C.c_int64(0))

            def fetch(i):
                slot = i % 2
                o, n = its[i]
                self._win_copy.wait_event(self._win_free[slot])
                ops.call("eps_cache_gather_bg", self.store.store_arg(), shard[o:o + n], n,
                         self.g.tokens * self.g.hidden * 2, self._win_buf[slot],
                         self.cache_prefetch_ctas, C.c_void_p(self._win_copy.cuda_stream))
                self._win_ready[slot].record(self._win_copy)

            fetch(0)
        front = [] if (cache_mode in (1, 2, 3) and stage == 0 and not idle) else None
        self.runner.front_events = front
        stalls = []
        start.record()
        losses = []
        norms = None
        for it, (o, n) in enumerate(its):
            last = it == len(its) - 1
            self.runner.trace = [] if last else None
            ids = shard[o:o + n]
            x = (self.images.index_select(0, ids) if stage == 0 and cache_mode != 1 and not idle
                 else None)
            y = self.labels.index_select(0, ids) if not idle else None
            store, sids = (self.store.store_arg() if self.store is not None else None), ids
            if disk:
                if disk_reads and it + 1 < len(its):
                    self._win_ready[it % 2].synchronize()  # batch it copied out of the window
                    dt.release(it)
                    dfetch(it + 1)
                if disk_reads:
                    w0 = torch.cuda.Event(enable_timing=True)
                    w1 = torch.cuda.Event(enable_timing=True)
                    w0.record(stream)
                    stream.wait_event(self._win_ready[it % 2])
                    w1.record(stream)
                    stalls.append((w0, w1))
                store, sids = self._win_buf[it % 2], self._win_ids[:n]
            if window:
                if it + 1 < len(its):
                    fetch(it + 1)
                w0 = torch.cuda.Event(enable_timing=True)
                w1 = torch.cuda.Event(enable_timing=True)
                w0.record(stream)
                stream.wait_event(self._win_ready[it % 2])
                w1.record(stream)
                stalls.append((w0, w1))
                store, sids = self._win_buf[it % 2], self._win_ids[:n]
            loss = self.runner.iteration(x, y, n, cache_mode=cache_mode, cache_old=cache_old,
                                         store=store, ids=sids)
            if disk and cache_mode == 2:  # the new boundary rows go to the file
                wb = self.store.wbuf[:n]
                wb.copy_(self._win_buf[it % 2][:n], non_blocking=True)
                torch.cuda.current_stream(self.device).synchronize()
                dt.write(ids.cpu(), wb)
            if window or disk:
                self._win_free[it % 2].record(stream)
            self.runner.sync_grads()
            if last:
                norms = self.runner.layer_sqnorms(self.ex.segments).sqrt()
            self.runner.step(self.lr, self.momentum)
            if stage == plan.K - 1 and not idle:
                losses.append((loss.clone(), n))
        stop.record()
        if disk_reads:
            self._win_ready[(len(its) - 1) % 2].synchronize()
            dt.release(len(its) - 1)
        if disk:
            self.disk_stats.append(dict(dt.stats(), epoch=epoch, mode=cache_mode))
        if window or disk:
            self.store.attach(self.ex)
        self.runner.front_events = None
        # a boundary move wrote rows into other GPUs' shards: every write is
        # complete and visible before any rank's next gather
        self._barrier()
        ms = self._max_over_ranks(start.elapsed_time(stop))
        trans = self._max_over_ranks(t_start.elapsed_time(start)) / 1000.0
        if norms is None:
            raise RuntimeError("epoch ran no iteration: no gradient norms")
        self.norms_prev = norms.cpu().tolist()
        nsamp = sum(n for _, n in losses)
        mean_loss = sum(float(l) for l, _ in losses) / nsamp if nsamp else float("nan")
        samples = sum(len(x) for x in shards)
        # measured CSV columns (per epoch; bubble per iteration as the reference)
        bubble = self._reduce(self.runner.bubble_time(), dist.ReduceOp.SUM) / plan.R
        comm, exposed = self.runner.comm_times() if plan.R > 1 else (0.0, 0.0)
        comm = self._max_over_ranks(comm) * len(its)
        exposed = self._max_over_ranks(exposed) * len(its)
        stall = self._max_over_ranks(sum(a.elapsed_time(b) for a, b in stalls) / 1e3 + disk_stall)
        cache_tr = 0.0
        if cache_mode == 2 and front:
            torch.cuda.synchronize()
            prefix = sum(a.elapsed_time(b) for a, b in front) / 1e3
            # disk tier: the whole prefix work is charged (its steady gather
            # reads the HBM staging window, timed in the iteration itself)
            steady = (0.0 if disk else
                      sum(self._time_gather(shard[o:o + n]) for o, n in its))
            cache_tr = max(0.0, prefix - steady)
        cache_tr = self._max_over_ranks(cache_tr)
        return EpochResult(epoch, d.l_frozen, plan.K, plan.R, plan.M,
                           ms / 1000.0 / max(1, len(its)), ms / 1000.0,
                           samples / (ms / 1000.0), d.cache_enabled, d.cache_moved, trans,
                           mean_loss, self.norms_prev, bubble, comm, exposed, cache_tr, stall,
                           samples)

    def run(self, epochs: Optional[int] = None) -> List[EpochResult]:
        n = epochs if epochs is not None else int(self.scenario["training"]["epochs"])
        try:
            return [self.run_epoch(e) for e in range(n)]
        finally:
            self.close()

    def close(self):
        if self.store is not None:
            self._barrier()
            self.store.close()
            self.store = None
        if isinstance(self.tp, EpsTransport):
            self._barrier()
            self.tp.close()
            self.tp = self.runner.tp = Transport(host_staged=False)

    @staticmethod
    def report_csv(rows: List[EpochResult]) -> str:
        return CSV_HEADER + "\n" + "".join(r.csv() + "\n" for r in rows)
