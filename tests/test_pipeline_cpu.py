"""AutoPipe x AutoDP choreography (pipeline.py) on CPU: world_size 2, gloo.

A FakeStageExecutor (tests/fake_stage.py) stands in for the sm_100a stage
executor so the multi-process host logic -- stage roles from the plan,
GPipe fill/drain order, point-to-point cut activations / gradients, per-stage
data-parallel groups, parameter migration on a K change, per-layer norm
assembly -- is checked against a single-process run of the same model.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_03161_b200.pipeline import (StagePlan, StageRunner, Transport,
                                            microbatch_offsets)
from tests.fake_stage import FakeStageExecutor

L = 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(seed, batch, ex):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(batch, ex.T, ex.inp, generator=g),
            torch.randint(0, 3, (batch,), generator=g))


def plan(K, R, M, lf, spans):
    return StagePlan(K, R, M, lf, L, tuple(spans))


# scenario: list of (plan, per-replica data seeds) per iteration
def scenario_pipeline():
    p = plan(2, 1, 3, 0, [(0, 3), (3, 6)])
    return [(p, [11]), (p, [12])]


def scenario_dp():
    p = plan(1, 2, 2, 0, [(0, 6)])
    return [(p, [21, 22]), (p, [23, 24])]


def scenario_transition():
    # epoch A: K=2, R=1, nothing frozen; epoch B: one layer frozen, packed to
    # K=1 and forked to R=2 (the AutoPipe compression + AutoDP fork)
    a = plan(2, 1, 2, 0, [(0, 2), (2, 6)])
    b = plan(1, 2, 3, 1, [(2, 6)])
    return [(a, [31]), (b, [32, 33]), (b, [34, 35])]


def scenario_idle():
    # AutoPipe on, AutoDP off: K 2 -> 1 keeps R = 1, so rank 1 idles
    # (runner.cpp:445) yet joins the migration broadcast and the norm
    # all-reduce
    a = plan(2, 1, 2, 0, [(0, 2), (2, 6)])
    b = plan(1, 1, 2, 1, [(2, 6)])
    return [(a, [41]), (b, [42]), (b, [43])]


SCENARIOS = {"pipeline": scenario_pipeline, "dp": scenario_dp, "transition": scenario_transition,
             "idle": scenario_idle}
BATCH = 7


def _worker(rank, world, port, name, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = FakeStageExecutor(layers=L, seed=0)
        # a small bucket cap so the DP scenarios exercise several buckets
        run = StageRunner(ex, rank, world, Transport(host_staged=True), bucket_bytes=600)
        losses = []
        for p, seeds in SCENARIOS[name]():
            run.set_plan(p)
            pipe, stage = p.role(rank)
            x, y = _data(seeds[min(pipe, len(seeds) - 1)], BATCH, ex)
            loss = run.iteration(x, y, BATCH)
            run.sync_grads()
            norms = run.layer_sqnorms(ex.segments())
            run.step(lr=0.05)
            losses.append((float(loss), norms.tolist(), stage == p.K - 1))
        # gather the model: every parameter from its current owner
        run.gather_model()
        torch.save({"p32": ex.p32, "mom": ex.mom, "losses": losses},
                   os.path.join(out_dir, f"{name}_{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _reference(name):
    """Single process: K=1, the replicas' batches concatenated (global batch R*B)."""
    ex = FakeStageExecutor(layers=L, seed=0)
    losses, norms = [], []
    for p, seeds in SCENARIOS[name]():
        data = [_data(s, BATCH, ex) for s in seeds]
        x = torch.cat([d[0] for d in data])
        y = torch.cat([d[1] for d in data])
        B = BATCH * len(seeds)
        ex.loss_sum.zero_()
        g0, g1 = 2 * p.l_frozen, 2 * L
        mbs = [(b0 + r * BATCH, b) for r in range(len(seeds))
               for b0, b in microbatch_offsets(BATCH, p.M)]
        for b0, b in mbs:
            ex.stage_forward(x, b0, b, g0, g1, p.l_frozen, True)
            ex.stage_head(y, b0, b, B)
        for b0, b in reversed(mbs):
            ex.stage_backward(b0, b, g0, g1, p.l_frozen, False)
        seg = ex.segments()
        norms.append([float((ex.g32[seg[l]:seg[l + 1]].double() ** 2).sum()) if l >= p.l_frozen
                      else 0.0 for l in range(L)])
        losses.append(float(ex.loss_sum))
        ex.sgd_range(*ex.param_range(g0, g1), lr=0.05)
    return ex, losses, norms


@pytest.mark.parametrize("name", list(SCENARIOS))
def test_two_rank_matches_single_process(name, tmp_path):
    port = _port()
    mp.spawn(_worker, args=(2, port, name, str(tmp_path)), nprocs=2, join=True)
    ref, ref_losses, ref_norms = _reference(name)
    outs = [torch.load(tmp_path / f"{name}_{r}.pt") for r in range(2)]
    for o in outs:  # after the final gather both ranks hold the whole model
        assert torch.allclose(o["p32"], ref.p32, rtol=1e-5, atol=1e-6)
    for it, (p, seeds) in enumerate(SCENARIOS[name]()):
        # loss: summed over the last stage of every replica
        got = sum(o["losses"][it][0] for o in outs if o["losses"][it][2])
        assert abs(got - ref_losses[it]) <= 1e-4 * abs(ref_losses[it])
        for o in outs:  # every rank assembles the same per-layer norms
            for a, b in zip(o["losses"][it][1], ref_norms[it]):
                # DP replicas average grads (mean of R batches), the reference
                # sums them with 1/(R*B) scaling: identical up to rounding
                assert abs(a - b) <= 1e-6 * max(1.0, b)


def test_plan_roles_and_ownership():
    p = plan(4, 2, 5, 1, [(2, 2), (2, 4), (4, 5), (5, 6)])
    assert [p.role(r) for r in range(8)] == [(r // 4, r % 4) for r in range(8)]
    assert p.dp_group_ranks(1) == [1, 5]
    assert not p.trainable(0)                     # frozen-filled partition 0 is a relay
    assert not p.upstream_needs_grad(1)           # nothing trainable upstream of stage 1
    assert p.upstream_needs_grad(2)
    assert p.owner_spans() == [(0, 2), (2, 4), (4, 5), (5, 6)]
    assert microbatch_offsets(10, 4) == [(0, 3), (3, 3), (6, 2), (8, 2)]


def test_plan_from_planner_decision():
    """StagePlan from the reference planner's golden decisions (vit-b16, 8 GPUs)."""
    import json
    from paper_2102_03161_b200 import LIB_PATH
    from paper_2102_03161_b200.capi import EpsApi
    from paper_2102_03161_b200.planner import Planner
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    golden = json.load(open(os.path.join(root, "tests/golden/decisions.json")))
    case = next(c for c in golden["scenarios"] if c["name"] == "vit-b16-g8")
    pl = Planner(EpsApi(LIB_PATH, "eps_"), case["scenario"])
    for row in case["rows"]:
        d = pl.begin_epoch(row["epoch"])
        sp = StagePlan.from_decision(d, 12)
        assert sp.K * sp.R == 8
        assert sp.spans[0][0] == 2 * sp.l_frozen and sp.spans[-1][1] == 24
        assert all(a[1] == b[0] for a, b in zip(sp.spans, sp.spans[1:]))


def test_moved_runs_only_ownership_changes():
    """Plan transitions broadcast exactly the sublayers some rank newly owns,
    each from its old owner (stage s of pipeline 0 = rank s)."""
    from paper_2102_03161_b200.pipeline import StagePlan, StageRunner
    n = 12
    a = StagePlan(2, 1, 7, 0, n, ((0, 12), (12, 24)))
    b = StagePlan(2, 1, 5, 6, n, ((12, 18), (18, 24)))  # AutoPipe re-balance at K = 2
    c = StagePlan(1, 2, 1, 9, n, ((18, 24),))           # K 2 -> 1 with a replica fork
    d = StagePlan(1, 2, 1, 10, n, ((20, 24),))          # boundary move, same ownership
    assert StageRunner.moved_runs(a, a) == []
    assert StageRunner.moved_runs(a, b) == [(12, 18, 1)]
    assert StageRunner.moved_runs(b, c) == [(0, 18, 0), (18, 24, 1)]
    assert StageRunner.moved_runs(c, d) == []
