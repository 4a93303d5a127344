"""AutoPipe stage executor on the B200: stage operations vs the fused K=1
train step, and a 2-rank pipeline / data-parallel run (two processes sharing
cuda:0, gloo with host-staged transfers) vs one process holding the stack.

Tolerance: the cut-point bias gradients are column sums of the bf16 dX that
crossed the stage boundary instead of the fused LayerNorm-backward sums, so
pipelined gradients are compared at 1e-2 relative L2 (north_star rtol 1e-2).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_03161_b200.configs import GEOMETRIES
from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport
from paper_2102_03161_b200.vit import VitExecutor, init_params

pytestmark = pytest.mark.gpu

CFG = "tiny-vit"
BATCH = 8


def _data(seed, g, batch=BATCH):
    gen = torch.Generator().manual_seed(seed)
    return (torch.randn(batch, g.channels, g.input_image, g.input_image, generator=gen),
            torch.randint(0, g.classes, (batch,), generator=gen))


def _rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / (b.norm() + 1e-12)).item()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_single_stage_runner_equals_train_step(cuda):
    g = GEOMETRIES[CFG]
    params = init_params(g, seed=3)
    x, y = _data(4, g)
    x, y = x.cuda(), y.cuda()
    a = VitExecutor(g, max_batch=BATCH, params=params)
    a.train_step(x, y, micro_batches=3, l_frozen=1)
    b = VitExecutor(g, max_batch=BATCH, params=params)
    run = StageRunner(b, 0, 1, Transport(host_staged=True))
    run.set_plan(StagePlan(1, 1, 3, 1, g.layers, ((2, 2 * g.layers),)))
    run.iteration(x, y, BATCH)
    torch.cuda.synchronize()
    # same kernels in the same order; split-K wgrad and bias column sums use
    # fp32 atomics, so repeated runs agree to rounding, not bit for bit
    assert _rel(b.g32, a.g32) < 1e-5
    assert abs(a.loss_sum.item() - b.loss_sum.item()) <= 1e-6 * abs(a.loss_sum.item())


def test_freeze_only_span_equals_elastic_span(cuda):
    """AutoPipe off: the epoch-0 partition is kept and frozen sublayers stay on
    their stage (span (0, 2L) with L_f = 1 runs layer 0 forward-only inside
    the span); the math equals the elastic span (2, 2L), and the frozen
    parameters are not updated."""
    g = GEOMETRIES[CFG]
    params = init_params(g, seed=5)
    x, y = _data(6, g)
    x, y = x.cuda(), y.cuda()
    a = VitExecutor(g, max_batch=BATCH, params=params)
    ra = StageRunner(a, 0, 1, Transport(host_staged=True))
    ra.set_plan(StagePlan(1, 1, 2, 1, g.layers, ((2, 2 * g.layers),)))
    b = VitExecutor(g, max_batch=BATCH, params=params)
    rb = StageRunner(b, 0, 1, Transport(host_staged=True))
    plan_b = StagePlan(1, 1, 2, 1, g.layers, ((0, 2 * g.layers),))
    assert plan_b.first_active(0) == 2 and plan_b.trainable(0)
    rb.set_plan(plan_b)
    p0 = b.p32.clone()
    for r in (ra, rb):
        r.iteration(x, y, BATCH)
        r.step(lr=0.1)
    torch.cuda.synchronize()
    assert _rel(b.g32, a.g32) < 1e-5
    assert abs(a.loss_sum.item() - b.loss_sum.item()) <= 1e-5 * abs(a.loss_sum.item())
    lo, hi = b.param_range(0, 2)
    assert torch.equal(b.p32[lo:hi], p0[lo:hi])  # frozen layer 0 + embedding untouched
    assert _rel(b.p32, a.p32) < 1e-5


PLANS = {
    # L=4 -> 8 sublayers; cut inside a layer (ATT | MLP) and between layers
    "pipe2": (StagePlan(2, 1, 2, 0, 4, ((0, 3), (3, 8))), [5]),
    "pipe2_frozen_relay": (StagePlan(2, 1, 2, 1, 4, ((2, 2), (2, 8))), [6]),
    "pipe2_frozen": (StagePlan(2, 1, 3, 1, 4, ((2, 5), (5, 8))), [7]),
    "dp2": (StagePlan(1, 2, 2, 0, 4, ((0, 8),)), [8, 9]),
}


def _worker(rank, world, port, name, out, peer=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = GEOMETRIES[CFG]
        plan, seeds = PLANS[name]
        ex = VitExecutor(g, max_batch=BATCH, params=init_params(g, seed=3), device="cuda:0")
        # small buckets: the replicated plans walk the last micro-batch's drain in
        # several pieces, each all-reduced as soon as it is final
        run = StageRunner(ex, rank, world, Transport(host_staged=True), bucket_bytes=200_000,
                          peer=peer)
        run.set_plan(plan)
        pipe, stage = plan.role(rank)
        x, y = _data(seeds[pipe], g)
        iters = 2 if peer else 1  # peer mode: also exercise the cross-iteration counters
        for _ in range(iters):
            loss = run.iteration(x.cuda(), y.cuda(), BATCH)
            run.sync_grads()
        if iters > 1:
            ex.g32.mul_(1.0 / iters)  # grads accumulated over identical iterations
        norms = run.layer_sqnorms(ex.segments)
        torch.cuda.synchronize()
        a, b = ex.param_range(*plan.owner_spans()[stage])
        torch.save({"range": (a, b), "g": ex.g32[a:b].cpu(), "loss": loss.item(),
                    "last": stage == plan.K - 1, "norms": norms.cpu()},
                   os.path.join(out, f"{name}_{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,peer", [(n, False) for n in PLANS] +
                         [(n, True) for n in PLANS if PLANS[n][0].K > 1])
def test_two_ranks_on_one_gpu(cuda, name, peer, tmp_path):
    """peer=True: the cut activations / gradients are written by the producing
    kernels straight into the neighbour's buffers over CUDA IPC (same device
    here, NVLink peers on a multi-GPU box), ordered by stream flags."""
    plan, seeds = PLANS[name]
    mp.spawn(_worker, args=(2, _port(), name, str(tmp_path), peer), nprocs=2, join=True)
    g = GEOMETRIES[CFG]
    ref = VitExecutor(g, max_batch=BATCH * len(seeds), params=init_params(g, seed=3))
    data = [_data(s, g) for s in seeds]
    x = torch.cat([d[0] for d in data]).cuda()
    y = torch.cat([d[1] for d in data]).cuda()
    # the same micro-batch split per replica: M per replica -> R*M slices
    ref.train_step(x, y, micro_batches=plan.M * len(seeds), l_frozen=plan.l_frozen)
    ref_norms = torch.tensor(ref.layer_norms(plan.l_frozen), dtype=torch.float64) ** 2
    torch.cuda.synchronize()
    outs = [torch.load(tmp_path / f"{name}_{r}.pt") for r in range(2)]
    loss = sum(o["loss"] for o in outs if o["last"])
    assert abs(loss - ref.loss_sum.item()) <= 1e-2 * abs(ref.loss_sum.item())
    for o in outs:
        a, b = o["range"]
        if b > a and o["g"].norm() > 0:
            assert _rel(o["g"], ref.g32[a:b]) < 1e-2, (name, a, b, _rel(o["g"], ref.g32[a:b]))
        for l in range(g.layers):
            r = ref_norms[l].item()
            assert abs(o["norms"][l].item() - r) <= 2e-2 * r + 1e-12, (l, o["norms"][l], r)
