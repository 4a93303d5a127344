"""BERT executor properties on the sm_100a path: AdamW, a 2-stage pipeline
(host-staged and peer-memory cuts) and the full-size BASELINE configs 4 / 5
(micro-batch invariance, loss additivity).  Per-tensor numerics parity vs
the CPU oracles lives in test_numerics_gpu.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_03161_b200.bert import BertExecutor, init_params
from paper_2102_03161_b200.configs import GEOMETRIES
from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport

pytestmark = pytest.mark.gpu



def _rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / (b.norm() + 1e-12)).item()


def _data(g, batch, seed):
    gen = torch.Generator().manual_seed(seed)
    tok = torch.randint(0, g.vocab, (batch, g.tokens), generator=gen)
    seg = torch.zeros(batch, g.tokens, dtype=torch.int64)
    seg[:, g.tokens // 2:] = 1
    if g.head == "qa":
        lab = torch.randint(0, g.tokens, (2, batch), generator=gen)
    else:
        lab = torch.randint(0, g.classes, (batch,), generator=gen)
    return tok, seg, lab


def test_bert_adamw_step(cuda):
    g = GEOMETRIES["tiny-bert-cls"]
    ex = BertExecutor(g, max_batch=8, seed=1)
    tok, seg, lab = _data(g, 8, seed=2)
    inputs, lab = torch.stack([tok, seg]).cuda(), lab.cuda()
    losses = []
    for _ in range(6):
        losses.append(ex.train_step(inputs, lab).item() / 8)
        ex.adamw_range(0, ex.total, lr=1e-3, weight_decay=0.0)
    torch.cuda.synchronize()
    assert losses[-1] < losses[0], losses
    assert ex.g32.abs().max().item() == 0.0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, peer=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = GEOMETRIES["tiny-bert-qa"]
        ex = BertExecutor(g, max_batch=4, params=init_params(g, seed=11), device="cuda:0")
        run = StageRunner(ex, rank, world, Transport(host_staged=True), peer=peer)
        plan = StagePlan(2, 1, 2, 0, g.layers, ((0, 1), (1, 4)))  # cut between ATT and MLP
        run.set_plan(plan)
        tok, seg, lab = _data(g, 4, seed=3)
        run.iteration(torch.stack([tok, seg]).cuda(), lab.reshape(-1).cuda(), 4)
        torch.cuda.synchronize()
        a, b = ex.param_range(*plan.owner_spans()[rank])
        torch.save({"range": (a, b), "g": ex.g32[a:b].cpu(), "loss": ex.loss_sum.item()},
                   os.path.join(out, f"bert_{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("peer", [False, True])
def test_bert_two_stage_pipeline(cuda, tmp_path, peer):
    mp.spawn(_worker, args=(2, _port(), str(tmp_path), peer), nprocs=2, join=True)
    g = GEOMETRIES["tiny-bert-qa"]
    ref = BertExecutor(g, max_batch=4, params=init_params(g, seed=11))
    tok, seg, lab = _data(g, 4, seed=3)
    ref.train_step(torch.stack([tok, seg]).cuda(), lab.reshape(-1).cuda(), micro_batches=2)
    torch.cuda.synchronize()
    outs = [torch.load(tmp_path / f"bert_{r}.pt") for r in range(2)]
    assert abs(outs[1]["loss"] - ref.loss_sum.item()) <= 1e-3 * abs(ref.loss_sum.item())
    for o in outs:
        a, b = o["range"]
        assert _rel(o["g"], ref.g32[a:b]) < 1e-3


@pytest.mark.parametrize("cfg", ["bert-base-384", "bert-large-128"])
def test_bert_full_size_step_properties(cuda, cfg):
    """BASELINE configs 4 and 5 at full size (batch 64): micro-batch invariance
    of the loss and every gradient (one pass vs 4 micro-batches -- different
    GEMM / attention tilings; the 2-kernel T=384 and the fused T=128
    attention backward), and additivity of the loss sum over two halves."""
    g = GEOMETRIES[cfg]
    batch = 64
    params = init_params(g, seed=13)
    tok, seg, lab = _data(g, batch, seed=7)
    inputs = torch.stack([tok, seg]).cuda()
    labels = lab.reshape(-1).cuda() if g.head == "qa" else lab.cuda()
    ex = BertExecutor(g, max_batch=batch, params=params)
    loss1 = ex.train_step(inputs, labels, micro_batches=1).item()
    g1 = ex.g32.clone()
    ex.g32.zero_()
    loss4 = ex.train_step(inputs, labels, micro_batches=4).item()
    torch.cuda.synchronize()
    assert torch.isfinite(g1).all()
    assert abs(loss4 - loss1) <= 1e-3 * abs(loss1)
    assert _rel(ex.g32, g1) < 1e-2
    halves = 0.0
    for lo in (0, 32):
        ex.g32.zero_()
        lab_h = lab[:, lo:lo + 32].reshape(-1).cuda() if g.head == "qa" else lab[lo:lo + 32].cuda()
        halves += ex.train_step(inputs[:, lo:lo + 32].contiguous(), lab_h).item()
    assert abs(halves - loss1) <= 1e-3 * abs(loss1)
