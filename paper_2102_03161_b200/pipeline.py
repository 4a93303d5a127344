"""AutoPipe x AutoDP execution over one process per GPU.

The reference *models* one training iteration as GPipe fill/drain blocks on K
stages plus bucketed AllReduce across R replicas (schedule.cpp:19-199); this
module *executes* it.  Every rank computes the same decisions (EpochPlanner,
runner.cpp:126-229) and derives its role from them:

  * rank r of the N = R*K GPUs is stage s = r mod K of pipeline p = r div K
    (Topology: active ranks r mod K == 0, GPU span [r, r+K), autodp.cpp:19-58);
  * stage s owns global sublayers [2*L_f + b_s, 2*L_f + e_s) from the
    PartitionPlan spans (autopipe.cpp:55-122); stage 0 also runs the frozen
    prefix / AutoCache gather and the embedding, the last stage the head;
  * forward fill in micro-batch order, backward drain in reverse micro-batch
    order (schedule.cpp:56-116); stages without trainable sublayers are pure
    relays and skip backward (schedule.cpp:47-52, 83-90);
  * the cut activations and activation-grads move stage to stage with
    point-to-point sends (NCCL over NVLink on a B200 box);
  * stage s of every replica averages only its active gradients over the
    per-stage data-parallel group {p*K + s} (ddp_skip_set, autodp.cpp:153-161);
    groups are rebuilt when freezing changes K (transition, autodp.cpp:81-111),
    and parameters + momentum migrate to their new owners.

All FLOPs run in libeps_b200.so (VitExecutor stage operations);
torch.distributed is the transport.  `Transport` abstracts it so the same
choreography runs over NCCL (device tensors) or over gloo with host staging
(CPU multi-process tests, or several ranks sharing one GPU).
"""
from __future__ import annotations

import ctypes as C
import pickle
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


# ---- decisions -> roles ------------------------------------------------------------
@dataclass(frozen=True)
class StagePlan:
    """One epoch's execution plan, identical on every rank."""
    K: int
    R: int
    M: int
    l_frozen: int
    layers: int
    spans: Tuple[Tuple[int, int], ...]  # global sublayer spans [g0, g1) per stage

    @staticmethod
    def from_decision(d, layers: int) -> "StagePlan":
        base = getattr(d, "span_base", 2 * d.l_frozen)
        spans = tuple((base + b, base + e) for b, e in d.spans)
        return StagePlan(d.pipeline_length, d.replica_width, d.micro_batches, d.l_frozen,
                         layers, spans)

    def role(self, rank: int) -> Tuple[int, int]:
        """(pipeline, stage) of a global rank."""
        return rank // self.K, rank % self.K

    def trainable(self, s: int) -> bool:
        return self.spans[s][1] > self.first_active(s)

    def first_active(self, s: int) -> int:
        """First trainable sublayer of stage s: with AutoPipe off the epoch-0
        partition is kept and frozen sublayers stay on their stage (forward
        only), so a span may start below 2 * L_f."""
        return max(self.spans[s][0], 2 * self.l_frozen)

    def upstream_needs_grad(self, s: int) -> bool:
        """Stage s sends dX to s-1 iff some earlier stage holds trainable
        sublayers (spans are contiguous from 2*L_f) -- the embedding counts as
        trainable when L_f == 0 (it is folded into sublayer 0)."""
        return s > 0 and self.spans[s][0] > 2 * self.l_frozen

    def owner_spans(self) -> List[Tuple[int, int]]:
        """Parameter ownership per stage: stage 0 also owns the frozen prefix
        (and embedding), the last stage the head -- together they cover every
        global sublayer exactly once."""
        out = [list(sp) for sp in self.spans]
        out[0][0] = 0
        out[-1][1] = 2 * self.layers
        return [tuple(x) for x in out]

    def dp_group_ranks(self, s: int) -> List[int]:
        return [p * self.K + s for p in range(self.R)]


def microbatch_offsets(batch: int, micro: int) -> List[Tuple[int, int]]:
    """Integer split with the remainder on the leading micro-batches
    (schedule.cpp:28-33): [(b0, b)]."""
    out, at = [], 0
    for m in range(micro):
        n = batch // micro + (1 if m < batch % micro else 0)
        out.append((at, n))
        at += n
    return out


# ---- transport ---------------------------------------------------------------------
class Transport:
    """Point-to-point and collective moves of device tensors."""

    def __init__(self, host_staged: bool):
        self.host_staged = host_staged
        self._groups: Dict[Tuple[int, ...], object] = {}

    def group(self, ranks: Sequence[int]):
        key = tuple(ranks)
        if key not in self._groups:
            # new_group is collective: callers create groups in the same order
            self._groups[key] = dist.new_group(list(ranks)) if len(ranks) > 1 else None
        return self._groups[key]

    def send(self, t: torch.Tensor, dst: int):
        if self.host_staged:
            dist.send(t.detach().cpu().contiguous(), dst)
        else:
            dist.send(t, dst)

    def recv(self, t: torch.Tensor, src: int):
        if self.host_staged:
            buf = torch.empty(t.shape, dtype=t.dtype)
            dist.recv(buf, src)
            t.copy_(buf)
        else:
            dist.recv(t, src)

    def all_reduce(self, t: torch.Tensor, group, op=dist.ReduceOp.SUM, async_op: bool = False,
                   avg: bool = False):
        """Returns a work handle for an asynchronous NCCL all-reduce (the
        collective runs on NCCL's stream, ordered after the kernels already
        queued on the current stream), else None.  avg: mean over the group
        (ncclAvg: the 1/R scaling happens inside the collective)."""
        if self.host_staged:
            buf = t.detach().cpu()
            dist.all_reduce(buf, op=op, group=group)
            if avg:
                buf /= dist.get_world_size(group)
            t.copy_(buf)
            return None
        if avg:
            op = dist.ReduceOp.AVG
        return dist.all_reduce(t, op=op, group=group, async_op=async_op)

    def broadcast(self, t: torch.Tensor, src: int):
        if self.host_staged:
            buf = t.detach().cpu()
            dist.broadcast(buf, src)
            t.copy_(buf)
        else:
            dist.broadcast(t, src)


class _StreamWork:
    """Completion handle of a collective issued on the comm stream: wait()
    orders the caller's current stream after it (no host block)."""

    def __init__(self, event):
        self.event = event

    def wait(self):
        torch.cuda.current_stream().wait_event(self.event)


class EpsTransport(Transport):
    """The same moves through the library's communicator plane (NCCL behind
    the C ABI, paper_2102_03161_b200.comm): a world communicator, per-group
    communicators split from it (ncclCommSplit, cached per membership),
    ncclAvg bucket all-reduces on a dedicated comm stream that overlap the
    drain, ncclSend / ncclRecv for the cut hand-off, ncclBroadcast for
    migration.  torch.distributed only carries the unique id."""

    def __init__(self, rank: int, world: int):
        super().__init__(host_staged=False)
        from .comm import Comm
        self.rank, self.world = rank, world
        self.comm = Comm.world(rank, world)
        self._splits: Dict[Tuple[int, ...], object] = {}
        self.stream = torch.cuda.Stream()

    def group(self, ranks: Sequence[int]):
        key = tuple(ranks)
        if key not in self._splits:
            # collective over the world communicator: every rank splits, in
            # the same order; non-members pass no color
            member = self.rank in key
            sub = self.comm.split(0 if member else -1, key.index(self.rank) if member else 0)
            self._splits[key] = sub
        return self._splits[key]

    def send(self, t: torch.Tensor, dst: int):
        self.comm.send(t.contiguous(), dst)

    def recv(self, t: torch.Tensor, src: int):
        if t.is_contiguous():
            self.comm.recv(t, src)
        else:
            buf = torch.empty_like(t, memory_format=torch.contiguous_format)
            self.comm.recv(buf, src)
            t.copy_(buf)

    def all_reduce(self, t: torch.Tensor, group, op=dist.ReduceOp.SUM, async_op: bool = False,
                   avg: bool = False):
        from .comm import OP_AVG, OP_MAX, OP_SUM
        c = self.comm if group is None else group
        if c is None:  # single-member group
            return None
        code = OP_AVG if avg else {dist.ReduceOp.SUM: OP_SUM, dist.ReduceOp.MAX: OP_MAX,
                                   dist.ReduceOp.AVG: OP_AVG}[op]
        if not async_op:
            c.all_reduce(t, code)
            return None
        ready = torch.cuda.Event()
        ready.record()
        self.stream.wait_event(ready)
        c.all_reduce(t, code, stream=self.stream)
        done = torch.cuda.Event()
        done.record(self.stream)
        return _StreamWork(done)

    def broadcast(self, t: torch.Tensor, src: int):
        self.comm.broadcast(t, src)

    def comm_version(self) -> int:
        from .comm import nccl_version
        return nccl_version()

    def close(self):
        for c in self._splits.values():
            if c is not None:
                c.free()
        self._splits = {}
        self.comm.free()


# ---- one rank's stage ------------------------------------------------------------------
BUCKET_BYTES = 25.0e6  # CostModel::allreduce_bucket_bytes (cost_model.hpp:16)


class PeerLink:
    """Stage-to-stage hand-off over peer memory (NVLink) for one plan.

    Each rank exports, as CUDA IPC handles, the buffer its first sublayer
    reads (the input cut), its activation-gradient buffer and a small flag
    array.  The previous stage's executor then writes its output cut straight
    into our input buffer from the producing kernel (eps_*_set_redirect), the
    next stage writes the gradient of our output straight into our dX, and a
    monotone counter per direction -- bumped with a system-scope release store
    after the producer, awaited with cuStreamWaitValue32 on the consumer's
    stream -- orders the two.  A third counter, bumped at the end of each of
    the receiver's iterations, keeps a relay stage 0 (no backward) from
    overwriting rows the receiver still uses."""

    FWD, BWD, FREE = 0, 1, 2

    def __init__(self, ex, runner: "StageRunner"):
        from . import ops
        self.lib = ops.api().lib
        self.ex, self.r = ex, runner
        self.flags = torch.zeros(16, dtype=torch.int32, device=ex.g32.device)
        self.opened: List[int] = []
        self.next_flags = self.prev_flags = None
        self.copy_out = None
        self.fwd = self.bwd = self.iters = 0
        for n, args in {"eps_ipc_export": [C.c_void_p, C.c_void_p, C.c_void_p],
                        "eps_ipc_open": [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p],
                        "eps_ipc_close": [C.c_void_p],
                        "eps_peer_signal": [C.c_void_p, C.c_uint32, C.c_void_p],
                        "eps_peer_wait": [C.c_void_p, C.c_uint32, C.c_void_p],
                        "eps_copy_async": [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]}.items():
            getattr(self.lib, n).argtypes = args
            getattr(self.lib, n).restype = C.c_int

    def _export(self, t: torch.Tensor):
        h = (C.c_char * 64)()
        off = C.c_int64()
        if self.lib.eps_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)) != 0:
            raise RuntimeError("eps_ipc_export failed")
        return bytes(h), off.value

    def _open(self, handle) -> int:
        h = (C.c_char * 64).from_buffer_copy(handle[0])
        base, ptr = C.c_void_p(), C.c_void_p()
        if self.lib.eps_ipc_open(h, handle[1], C.byref(base), C.byref(ptr)) != 0:
            raise RuntimeError("eps_ipc_open failed")
        self.opened.append(base.value)
        return ptr.value

    def close(self):
        for b in self.opened:
            self.lib.eps_ipc_close(C.c_void_p(b))
        self.opened = []
        self.ex.set_redirect(-1, None, -1, None)

    def setup(self, plan: StagePlan, stage: int, g0: int, g1: int, idle: bool = False):
        """Collective over the world: exchange handles, map the neighbours."""
        self.close()
        self.flags.zero_()
        torch.cuda.synchronize()
        mb = self.ex.max_batch
        mine = {"cut": self._export(self.ex.cut_rows(g0, 0, mb)),
                "dx": self._export(self.ex.cut_rows(0, 0, mb, grad=True)),
                "flags": self._export(self.flags)}
        allh = [None] * self.r.world
        dist.all_gather_object(allh, pickle.dumps(mine))
        allh = [pickle.loads(x) for x in allh]
        K, rank = plan.K, self.r.rank
        out_g, out_ptr, dx_g, dx_ptr = -1, None, -1, None
        self.next_flags = self.prev_flags = None
        self.copy_out = None
        if idle:
            self.ex.set_redirect(-1, None, -1, None)
            self.fwd = self.bwd = self.iters = 0
            return
        if stage < K - 1:
            nxt = allh[rank + 1]
            peer_cut = self._open(nxt["cut"])
            self.next_flags = self._open(nxt["flags"])
            if g1 > g0:  # the stage's last kernel writes the peer buffer itself
                out_g, out_ptr = g1, peer_cut
            else:  # relay stage (frozen prefix / cache only): copy its output rows
                self.copy_out = peer_cut
        if stage > 0:
            prv = allh[rank - 1]
            self.prev_flags = self._open(prv["flags"])
            if plan.upstream_needs_grad(stage):
                dx_g, dx_ptr = g0, self._open(prv["dx"])
        self.ex.set_redirect(out_g, out_ptr, dx_g, dx_ptr)
        self.fwd = self.bwd = self.iters = 0

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def copy(self, dst_ptr: int, src: torch.Tensor):
        """Stream-ordered copy of `src` to a (peer) device address."""
        if self.lib.eps_copy_async(C.c_void_p(dst_ptr), C.c_void_p(src.data_ptr()),
                                   C.c_int64(src.numel() * src.element_size()),
                                   self._stream()) != 0:
            raise RuntimeError("eps_copy_async failed")

    def _flag(self, base: int, which: int) -> C.c_void_p:
        return C.c_void_p(base + 4 * which)

    def signal(self, base, which, value):
        if self.lib.eps_peer_signal(self._flag(base, which), value, self._stream()) != 0:
            raise RuntimeError("eps_peer_signal failed")

    def wait(self, which, value):
        if self.lib.eps_peer_wait(self._flag(self.flags.data_ptr(), which), value,
                                  self._stream()) != 0:
            raise RuntimeError("eps_peer_wait failed")


class StageRunner:
    """Executes the iterations of one rank (one pipeline stage of one replica)
    over a stage executor exposing the eps_vit_stage_* operations.

    Gradient synchronisation follows the reference's DDP model
    (schedule.cpp:133-178): the stage's active parameters form ~25 MB buckets
    in reverse sublayer order, and each bucket's all-reduce is launched as soon
    as the last micro-batch's backward has finished its sublayers, overlapping
    the rest of the drain."""

    def __init__(self, ex, rank: int, world: int, transport: Transport,
                 bucket_bytes: float = BUCKET_BYTES, peer: bool = False):
        self.ex = ex
        self.peer = PeerLink(ex, self) if peer else None
        self.rank = rank
        self.world = world
        self.tp = transport
        self.bucket_bytes = bucket_bytes
        self.plan: Optional[StagePlan] = None
        self.g0 = self.g1 = 0
        self.stage = self.pipe = 0
        self.range = (0, 0)
        self.buckets: List[Tuple[int, int]] = []
        self.pending: List[Tuple[object, int, int]] = []
        self.trace: Optional[list] = None  # [] records the next iteration's blocks
        self.front_events: Optional[list] = None  # [] records stage 0's front per micro-batch
        self.t_ar_first = self.t_bwd_end = self.t_sync_end = None
        self.idle = False

    # -- plan changes ------------------------------------------------------------
    def _dp_groups(self, plan: StagePlan):
        # every rank creates every stage group of this K, in stage order
        return [self.tp.group(plan.dp_group_ranks(s)) for s in range(plan.K)]

    def set_plan(self, plan: StagePlan):
        """Adopt an epoch plan; on a K / ownership change migrate parameters
        and momentum from their previous owners (pipeline 0's stages) to all
        ranks, then (re)select the per-stage data-parallel groups."""
        if plan.K * plan.R > self.world:
            raise ValueError(f"plan needs {plan.K * plan.R} ranks, world has {self.world}")
        old = self.plan
        # Parameters move only when ownership moves: with the same K and the
        # same owner spans (a freeze-boundary move inside stage 0's span),
        # every rank already holds -- and its DP replicas hold identical --
        # values for everything it owns next epoch.
        if old is not None and (old.K != plan.K or old.owner_spans() != plan.owner_spans()):
            self.migrate(old, plan)
        self.plan = plan
        # AutoPipe without AutoDP packs the pipeline into fewer GPUs but keeps
        # R (runner.cpp:445): ranks >= K*R sit idle for the epoch, joining only
        # the world collectives (migration broadcasts, norms, timing)
        self.idle = self.rank >= plan.K * plan.R
        self.pipe, self.stage = plan.role(min(self.rank, plan.K * plan.R - 1))
        self.g0, self.g1 = plan.spans[self.stage]
        self.a0 = plan.first_active(self.stage)  # trainable sublayers: [a0, g1)
        self.groups = self._dp_groups(plan)
        self.range = self.ex.param_range(*plan.owner_spans()[self.stage])
        self.buckets = self._plan_buckets() if plan.R > 1 else []
        if self.peer is not None and self.world > 1:
            self.peer.setup(plan, self.stage, self.g0, self.g1, idle=self.idle)

    def _plan_buckets(self) -> List[Tuple[int, int]]:
        """Sublayer pieces [g_lo, g_hi) of this stage, top first, each closed
        once its fp32 gradients reach the bucket size."""
        out, hi, acc = [], self.g1, 0
        for g in range(self.g1 - 1, self.a0 - 1, -1):
            a, b = self.ex.param_range(g, g + 1)
            acc += 4 * (b - a)
            if acc >= self.bucket_bytes or g == self.a0:
                out.append((g, hi))
                hi, acc = g, 0
        return out

    @staticmethod
    def moved_runs(old: StagePlan, new: StagePlan) -> List[Tuple[int, int, int]]:
        """Sublayer runs [g0, g1) whose parameters some rank must receive:
        a rank whose new stage owns g but whose old stage did not.  Each run
        is served by its old owner, stage s of pipeline 0 = rank s."""
        def owner(plan, g):
            for st, (a, b) in enumerate(plan.owner_spans()):
                if a <= g < b:
                    return st
            raise ValueError(g)

        world = new.K * new.R  # active ranks of the new plan
        runs: List[Tuple[int, int, int]] = []
        for g in range(2 * new.layers):
            os_, ns = owner(old, g), owner(new, g)
            # a rank idle under `old` (r >= K*R, AutoDP off) owns nothing
            need = any(new.role(r)[1] == ns and (r >= old.K * old.R or old.role(r)[1] != os_)
                       for r in range(world))
            if not need:
                continue
            if runs and runs[-1][1] == g and runs[-1][2] == os_:
                runs[-1] = (runs[-1][0], g + 1, os_)
            else:
                runs.append((g, g + 1, os_))
        return runs

    def gather_model(self):
        """Every rank receives every parameter from its current owner (e.g. to
        checkpoint or compare the whole model)."""
        p = self.plan
        everyone = StagePlan(1, self.world, 1, p.l_frozen, p.layers, ((0, 2 * p.layers),))
        self.migrate(p, everyone)

    def migrate(self, old: StagePlan, new: StagePlan):
        """Parameters (and momentum) of every sublayer some rank newly owns are
        broadcast from the rank that owned and updated them under `old`;
        the bf16 working copy is re-derived."""
        if self.world == 1:
            return  # a single rank owns everything already
        for g0, g1, src in self.moved_runs(old, new):
            a, b = self.ex.param_range(g0, g1)
            if b > a:
                self.tp.broadcast(self.ex.p32[a:b], src)
                self.tp.broadcast(self.ex.mom[a:b], src)
        self.ex.p16.copy_(self.ex.p32)

    # -- one iteration -------------------------------------------------------------------
    def iteration(self, images, labels, batch: int, cache_mode: int = 0, cache_old: int = 0,
                  store=None, ids=None, micro: Optional[int] = None):
        """Forward + backward of one per-pipeline batch on this rank's stage.
        images / labels / ids are only read on the first / last stage.
        `micro` overrides the plan's M (a ragged last batch of an epoch with
        fewer samples than M).  With `front_events` a list, stage 0 appends
        (start, end) CUDA events around each micro-batch's frozen-prefix /
        AutoCache work (the cache-transition measurement)."""
        p, s, K = self.plan, self.stage, self.plan.K
        ex, lf = self.ex, p.l_frozen
        if self.idle:
            return ex.loss_sum.zero_()
        mbs = microbatch_offsets(batch, min(p.M, batch) if micro is None else micro)
        prev, nxt = self.rank - 1, self.rank + 1
        pl = self.peer if (self.peer is not None and K > 1) else None
        ex.loss_sum.zero_()
        tr = self.trace
        if tr is not None:
            tr.clear()
            self.t_ar_first = self.t_bwd_end = self.t_sync_end = None
            t_iter = self._mark()
        if pl is not None and s < K - 1 and pl.iters > 0:
            pl.wait(PeerLink.FREE, pl.iters)  # receiver done with last iteration's rows
        for b0, b in mbs:
            if pl is not None:
                if s > 0:
                    pl.wait(PeerLink.FWD, pl.fwd + 1)
            elif s > 0:
                self.tp.recv(ex.cut_rows(self.g0, b0, b), prev)
            t0 = self._mark() if tr is not None else None
            if s == 0 and self.front_events is not None:
                # stage 0's front (frozen prefix / AutoCache) as its own call,
                # bracketed by events; then the span
                fa = self._mark()
                ex.stage_forward(images, b0, b, self.g0, self.g0, lf, front=True,
                                 cache_mode=cache_mode, cache_old=cache_old, store=store, ids=ids)
                self.front_events.append((fa, self._mark()))
                ex.stage_forward(None, b0, b, self.g0, self.g1, lf, front=False)
            else:
                ex.stage_forward(images if s == 0 else None, b0, b, self.g0, self.g1, lf,
                                 front=(s == 0), cache_mode=cache_mode if s == 0 else 0,
                                 cache_old=cache_old, store=store if s == 0 else None,
                                 ids=ids if s == 0 else None)
            if tr is not None:
                tr.append(("F", f"mb{len(tr)}", t0, self._mark()))
            if s < K - 1:
                if pl is not None:
                    if pl.copy_out is not None:
                        rows = ex.cut_rows(self.g1, b0, b)
                        pl.copy(pl.copy_out + rows.data_ptr() - ex.cut_rows(self.g1, 0, 1).data_ptr(),
                                rows)
                    pl.signal(pl.next_flags, PeerLink.FWD, pl.fwd + 1)
                else:
                    self.tp.send(ex.cut_rows(self.g1, b0, b), nxt)
            else:
                ex.stage_head(labels, b0, b, batch)
            if pl is not None:
                pl.fwd += 1
        if p.trainable(s):
            for i, (b0, b) in enumerate(reversed(mbs)):
                t0 = self._mark() if tr is not None else None
                if s < K - 1:
                    if pl is not None:
                        pl.wait(PeerLink.BWD, pl.bwd + 1)
                    else:
                        self.tp.recv(ex.cut_rows(0, b0, b, grad=True), nxt)
                if self.buckets and i == len(mbs) - 1:
                    # last micro-batch of the drain: walk the stage bucket by bucket
                    # and start each bucket's all-reduce once its grads are final
                    for j, (lo, hi) in enumerate(self.buckets):
                        ex.stage_backward_part(b0, b, lo, hi, self.g0, lf,
                                               cut_out=(s < K - 1 and j == 0))
                        a, e = ex.param_range(lo, hi)
                        if tr is not None and j == 0:
                            self.t_ar_first = self._mark()
                        work = self.tp.all_reduce(ex.g32[a:e], self.groups[s], async_op=True,
                                                  avg=True)
                        self.pending.append((work, a, e))
                else:
                    ex.stage_backward(b0, b, self.g0, self.g1, lf, cut_out=s < K - 1)
                if tr is not None:
                    tr.append(("B", f"mb{len(mbs) - 1 - i}", t0, self._mark()))
                if p.upstream_needs_grad(s):
                    if pl is not None:
                        pl.signal(pl.prev_flags, PeerLink.BWD, pl.bwd + 1)
                    else:
                        self.tp.send(ex.cut_rows(0, b0, b, grad=True), prev)
                if pl is not None:
                    pl.bwd += 1
        if pl is not None:
            pl.iters += 1
            if s > 0:
                pl.signal(pl.prev_flags, PeerLink.FREE, pl.iters)
        if tr is not None:
            tr.insert(0, ("iteration", "", t_iter, None))
            self.t_bwd_end = self._mark()
        return ex.loss_sum

    # -- measured timeline (report bundle) -------------------------
    @staticmethod
    def _mark():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def timeline(self):
        """Blocks of the last traced iteration in the reference's timeline schema
        (runner.cpp:357-367: device, kind, start_s, end_s, tag), from CUDA events
        on this rank's stream, relative to the iteration start; `trace = []`
        turns tracing on."""
        if not self.trace:
            return []
        torch.cuda.synchronize()
        t_iter = self.trace[0][2]
        return [{"device": self.rank, "kind": k, "start_s": t_iter.elapsed_time(a) / 1e3,
                 "end_s": t_iter.elapsed_time(b) / 1e3, "tag": tag}
                for k, tag, a, b in self.trace[1:]]

    def sync_grads(self):
        """Finish the bucket all-reduces of this iteration: the buckets were
        reduced with an average (NCCL's ncclAvg on the device path), so the
        stage's active gradients are the replica mean when this returns."""
        p = self.plan
        if p.R > 1 and p.trainable(self.stage) and not self.idle:
            for work, a, e in self.pending:
                if work is not None:
                    work.wait()
            self.pending = []
        if self.trace is not None:
            self.t_sync_end = self._mark()

    def comm_times(self):
        """(comm, exposed) seconds of the last traced iteration: first bucket
        launch -> last bucket done, and end of the drain -> last bucket done
        (as the compute stream sees them; schedule.cpp:137-178 semantics)."""
        if self.t_sync_end is None or self.t_bwd_end is None:
            return 0.0, 0.0
        torch.cuda.synchronize()
        exposed = max(0.0, self.t_bwd_end.elapsed_time(self.t_sync_end) / 1e3)
        comm = (self.t_ar_first.elapsed_time(self.t_sync_end) / 1e3
                if self.t_ar_first is not None else 0.0)
        return comm, exposed

    def bubble_time(self) -> float:
        """Idle time of this stage inside the last traced iteration: span from
        the iteration start to its last block minus the busy F / B blocks
        (schedule.cpp:126-131 bubble_per_device)."""
        if not self.trace:
            return 0.0
        torch.cuda.synchronize()
        t0 = self.trace[0][2]
        blocks = self.trace[1:]
        if not blocks:
            return 0.0
        span = max(t0.elapsed_time(b) for _, _, _, b in blocks) / 1e3
        busy = sum(a.elapsed_time(b) for _, _, a, b in blocks) / 1e3
        return max(0.0, span - busy)

    def step(self, lr: float, momentum: float = 0.9, weight_decay: float = 0.0):
        if self.plan.trainable(self.stage) and not self.idle:
            a, b = self.ex.param_range(self.a0, self.g1)
            self.ex.sgd_range(a, b, lr, momentum, weight_decay)

    def layer_sqnorms(self, segments: Sequence[int]) -> torch.Tensor:
        """Per-layer Σg² of the whole model, assembled from every stage's
        owned (post-all-reduce) gradients: each rank reduces the part of each
        layer segment it trains, then one world all-reduce; replicas hold
        identical gradients, so the sum over ranks is divided by R."""
        p = self.plan
        L = len(segments) - 1
        out = torch.zeros(L, dtype=torch.float64, device=self.ex.g32.device)
        if p.trainable(self.stage) and not self.idle:
            a, b = self.ex.param_range(self.a0, self.g1)
            cuts = sorted({a, b} | {x for x in segments if a < x < b})
            part = torch.zeros(len(cuts) - 1, dtype=torch.float64, device=out.device)
            self.ex.sqnorm_ranges(cuts, part)
            for i in range(len(cuts) - 1):
                layer = max(l for l in range(L) if segments[l] <= cuts[i])
                out[layer] += part[i]
        if self.world > 1:
            self.tp.all_reduce(out, None)
            out /= p.R
        return out
