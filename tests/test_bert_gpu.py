"""BERT train step on the sm_100a executor vs the fp32 CPU oracle
(BASELINE configs 4 and 5 and test-size variants), plus a 2-stage pipeline.

Tolerance: loss within rtol 1e-2 (north_star); gradient tensors and
per-layer norms within 8e-2 relative L2.  The SQuAD head sends a gradient
into every one of the T=384 token rows and every post-norm sublayer ends in
a LayerNorm whose backward re-rounds dS to bf16, so gradient matrices sit
at 1-6 % of their fp32 value (measured).  1-D bias / LayerNorm gradients are
sums over B*T rows that cancel heavily: for layer 11's FC2 bias at
bert-base-384 |sum| is ~16x below the row noise floor, and rounding the fp32
oracle's own dS rows to bf16 before summing already moves it by 8 %
(tests/test_bert_gpu.py docstring experiment) -- those are checked at 30 %.
The per-layer norms the freeze decision consumes are checked at 5e-2.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bert_fp32
from paper_2102_03161_b200.bert import BertExecutor, init_params
from paper_2102_03161_b200.configs import GEOMETRIES
from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-2
GRAD_REL = 8e-2
VEC_REL = 0.3
NORM_REL = 5e-2


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


@pytest.mark.parametrize("cfg,batch,l_frozen,micro", [
    ("tiny-bert-qa", 4, 0, 1),
    ("tiny-bert-qa", 5, 1, 2),
    ("tiny-bert-cls", 6, 0, 3),
    ("tiny-bert-cls", 4, 1, 1),
    ("bert-base-384", 2, 0, 1),
    ("bert-large-128", 3, 20, 2),
])
def test_bert_train_step_matches_oracle(cuda, cfg, batch, l_frozen, micro):
    g = GEOMETRIES[cfg]
    params = init_params(g, seed=11)
    tok, seg, lab = _data(g, batch, seed=3)
    ex = BertExecutor(g, max_batch=batch, params=params)
    inputs = torch.stack([tok, seg]).cuda()
    loss_sum = ex.train_step(inputs, lab.reshape(-1).cuda(), micro_batches=micro,
                             l_frozen=l_frozen)
    torch.cuda.synchronize()
    loss = loss_sum.item() / batch
    ref_loss, ref_grads = bert_fp32.train_step(params, tok, seg, lab, g, l_frozen)
    assert abs(loss - ref_loss.item()) <= LOSS_RTOL * abs(ref_loss.item()), (loss, ref_loss)
    grads = ex.grads()
    errs = {}
    for name, ref in ref_grads.items():
        if not bert_fp32.trainable(name, l_frozen):
            assert grads[name].abs().max().item() == 0.0, name
            continue
        if ref.norm() < 1e-6:
            continue
        errs[name] = _rel(grads[name], ref)
    bad = {k: round(v, 4) for k, v in errs.items()
           if v >= (GRAD_REL if ref_grads[k].dim() > 1 else VEC_REL)}
    assert not bad, (bad, {k: round(v, 4) for k, v in errs.items()})
    norms = ex.layer_norms(l_frozen)
    ref_norms = bert_fp32.layer_norms(ref_grads, g, l_frozen)
    for l in range(g.layers):
        if l < l_frozen:
            assert norms[l] == 0.0
        else:
            assert abs(norms[l] - ref_norms[l]) <= NORM_REL * ref_norms[l], l


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
