"""Numerics-parity harness shared by the GPU tests and tools/numerics_table.py.

One `Case` = one train step of the sm_100a executor and of the CPU oracle
under both numerics policies (oracle/numerics.py) on the same seeded
parameters and inputs.  Three distances per quantity (relative L2):

* `kernel`    = device vs BF16_STORAGE: what the kernels add on top of the
  bf16-storage design (accumulation order, SFU approximations, rounding-
  boundary flips) -- see below for why this is a noise measurement.
* `vs_fp32`   = device vs FP32: the north_star comparison.
* `intrinsic` = BF16_STORAGE vs FP32: the part of `vs_fp32` any design that
  stores these tensors in bf16 must pay (no kernel involved).

Tensors whose gradient is mathematically zero (the QA classifier bias and
the final LayerNorm bias under a span head: sum over tokens of softmax - one
-hot = 0) have no relative error; they are held to an absolute bound instead
(`zero_tensors`).

Why `kernel` is not the gate (measured, profiles/r02/numerics.md): a bf16-
storage computation is chaotic at the rounding level.  Perturbing the input
images by 1e-6 (relative) moves BF16_STORAGE's own gradients by 0.9-1.4 %
relative L2 at ViT-B/16 -- as much as its distance from FP32 -- while FP32
moves by < 1e-6: one flipped rounding changes every GEMM output it feeds,
which flips further roundings, so any two bf16-storage implementations that
accumulate in different orders (tensor-core tiles vs a CPU GEMM) are two
independent draws of the same rounding noise.  The device is therefore held
to: its distance from FP32 is no larger than the emulation's own
(`vs_fp32 <= NOISE_FACTOR * intrinsic + NOISE_FLOOR`, per tensor), plus
north_star's 1e-2 on every quantity the bf16 noise does not dominate (loss,
per-layer gradient norms, 10-step loss trajectories).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List

import torch

from oracle import bert_fp32, vit_fp32
from oracle.numerics import rel_l2
from paper_2102_03161_b200.configs import GEOMETRIES

LOSS_RTOL = 1e-2    # north_star: rtol 1e-2 in bf16 vs fp32
NORM_RTOL = 1e-2    # per-layer gradient norms (the freeze test's input)
TRAJ_RTOL = 1e-2    # per-step loss of a 10-step SGD trajectory
NOISE_FACTOR = 1.3  # device distance from FP32 <= 1.3 x the emulation's ...
NOISE_FLOOR = 2e-3  # ... + 2e-3 (per gradient tensor / activation X[l])


def vit_data(g, batch: int, seed: int):
    gen = torch.Generator().manual_seed(seed)
    images = torch.randn(batch, g.channels, g.input_image, g.input_image, generator=gen)
    labels = torch.randint(0, g.classes, (batch,), generator=gen)
    return images, labels


def bert_data(g, batch: int, seed: int):
    gen = torch.Generator().manual_seed(seed)
    tok = torch.randint(0, g.vocab, (batch, g.tokens), generator=gen)
    seg = torch.zeros(batch, g.tokens, dtype=torch.int64)
    seg[:, g.tokens // 2:] = 1
    if g.head == "qa":
        lab = torch.randint(0, g.tokens, (2, batch), generator=gen)
    else:
        lab = torch.randint(0, g.classes, (batch,), generator=gen)
    return tok, seg, lab


@dataclass
class Case:
    cfg: str
    batch: int
    l_frozen: int
    micro: int
    loss: Dict[str, float] = field(default_factory=dict)      # dev / fp32 / bf16
    grads: Dict[str, Dict[str, float]] = field(default_factory=dict)  # name -> 3 distances
    acts: List[Dict[str, float]] = field(default_factory=list)  # X[l] -> 3 distances
    norms: List[Dict[str, float]] = field(default_factory=list)  # per-layer |g| rel err
    zero_tensors: Dict[str, float] = field(default_factory=dict)  # name -> |dev| / scale
    frozen_nonzero: List[str] = field(default_factory=list)

    def worst(self, kind: str, metric: str) -> float:
        rows = self.grads.values() if kind == "grads" else self.acts
        return max((r[metric] for r in rows), default=0.0)


def _three(dev, emu, f32, emu2=None) -> Dict[str, float]:
    out = {"kernel": rel_l2(dev, emu), "vs_fp32": rel_l2(dev, f32),
           "intrinsic": rel_l2(emu, f32)}
    if emu2 is not None:  # BF16_STORAGE vs itself on 1e-6-perturbed inputs
        out["self_noise"] = rel_l2(emu2, emu)
    return out


def _perturb(x: torch.Tensor) -> torch.Tensor:
    gen = torch.Generator().manual_seed(99)
    return x * (1 + 1e-6 * torch.randn(x.shape, generator=gen))


def run_case(cfg: str, batch: int, l_frozen: int, micro: int = 1, seed: int = 17,
             data_seed: int = 5, self_noise: bool = False) -> Case:
    """One step on cuda:0 and on the CPU oracles; returns the distances.
    `self_noise`: also run BF16_STORAGE on inputs perturbed by 1e-6 (ViT:
    pixels; BERT: the embedding tables) to measure the rounding chaos."""
    g = GEOMETRIES[cfg]
    c = Case(cfg, batch, l_frozen, micro)
    if g.kind == "vit":
        from paper_2102_03161_b200.vit import VitExecutor, init_params
        params = init_params(g, seed=seed)
        images, labels = vit_data(g, batch, data_seed)
        ex = VitExecutor(g, max_batch=batch, params=params)
        loss = ex.train_step(images.cuda(), labels.cuda(), micro_batches=micro, l_frozen=l_frozen)
        oracle = vit_fp32
        l32, g32, _, x32 = vit_fp32.train_step(params, images, labels, g, l_frozen, "fp32", True)
        l16, g16, _, x16 = vit_fp32.train_step(params, images, labels, g, l_frozen, "bf16", True)
        if self_noise:
            _, gp, _, xp = vit_fp32.train_step(params, _perturb(images), labels, g, l_frozen,
                                               "bf16", True)
    else:
        from paper_2102_03161_b200.bert import BertExecutor, init_params
        params = init_params(g, seed=seed)
        tok, seg, lab = bert_data(g, batch, data_seed)
        ex = BertExecutor(g, max_batch=batch, params=params)
        labels = lab.reshape(-1).cuda() if g.head == "qa" else lab.cuda()
        loss = ex.train_step(torch.stack([tok, seg]).cuda(), labels, micro_batches=micro,
                             l_frozen=l_frozen)
        oracle = bert_fp32
        l32, g32, x32 = bert_fp32.train_step(params, tok, seg, lab, g, l_frozen, "fp32", True)
        l16, g16, x16 = bert_fp32.train_step(params, tok, seg, lab, g, l_frozen, "bf16", True)
        if self_noise:
            pp = dict(params)
            for k in ("embeddings.word_embeddings.weight", "embeddings.position_embeddings.weight"):
                pp[k] = _perturb(params[k])
            _, gp, xp = bert_fp32.train_step(pp, tok, seg, lab, g, l_frozen, "bf16", True)
    torch.cuda.synchronize()
    c.loss = {"dev": loss.item() / batch, "fp32": l32.item(), "bf16": l16.item()}
    dev = {k: v.float().cpu() for k, v in ex.grads().items()}
    for name, ref in g16.items():
        if not oracle.trainable(name, l_frozen):
            if dev[name].abs().max().item() != 0.0:
                c.frozen_nonzero.append(name)
            continue
        n32, n16 = float(g32[name].norm()), float(ref.norm())
        if n16 == 0.0 and n32 == 0.0:  # unused under this head (e.g. the QA pooler)
            if dev[name].abs().max().item() != 0.0:
                c.frozen_nonzero.append(name)
            continue
        if n32 < 0.1 * float((ref - g32[name]).norm()):
            # zero by math: the fp32 value is roundoff, the bf16 one rounding
            # noise; held to |dev| / |BF16_STORAGE| (same-size noise expected)
            c.zero_tensors[name] = float(dev[name].norm()) / max(n16, 1e-30)
            continue
        c.grads[name] = _three(dev[name], ref, g32[name], gp[name] if self_noise else None)
    T, d = g.tokens, g.hidden
    for l in range(g.layers + 1):
        xd = ex.cut_rows(2 * l, 0, batch).float().cpu().view(batch, T, d)
        c.acts.append(_three(xd, x16[l], x32[l], xp[l] if self_noise else None))
    dn = ex.layer_norms(l_frozen)
    n16 = oracle.layer_norms(g16, g, l_frozen)
    n32 = oracle.layer_norms(g32, g, l_frozen)
    for l in range(g.layers):
        if l < l_frozen:
            c.norms.append({"dev": dn[l]})
            continue
        c.norms.append({"kernel": abs(dn[l] - n16[l]) / n16[l],
                        "vs_fp32": abs(dn[l] - n32[l]) / n32[l],
                        "intrinsic": abs(n16[l] - n32[l]) / n32[l]})
    del ex
    return c


def trajectory(cfg: str, batch: int, steps: int, lr: float, l_frozen: int = 0, seed: int = 17,
               data_seed: int = 5):
    """Per-step mean loss of `steps` SGD-momentum iterations on one batch:
    (device, fp32 oracle)."""
    g = GEOMETRIES[cfg]
    dev = []
    if g.kind == "vit":
        from paper_2102_03161_b200.vit import VitExecutor, init_params
        params = init_params(g, seed=seed)
        images, labels = vit_data(g, batch, data_seed)
        ex = VitExecutor(g, max_batch=batch, params=params)
        x, y = images.cuda(), labels.cuda()
        run = lambda: ex.train_step(x, y, l_frozen=l_frozen)  # noqa: E731
        ref = vit_fp32.sgd_trajectory(params, images, labels, g, steps, lr, l_frozen=l_frozen)
    else:
        from paper_2102_03161_b200.bert import BertExecutor, init_params
        params = init_params(g, seed=seed)
        tok, seg, lab = bert_data(g, batch, data_seed)
        ex = BertExecutor(g, max_batch=batch, params=params)
        x = torch.stack([tok, seg]).cuda()
        y = lab.reshape(-1).cuda() if g.head == "qa" else lab.cuda()
        run = lambda: ex.train_step(x, y, l_frozen=l_frozen)  # noqa: E731
        ref = bert_fp32.sgd_trajectory(params, tok, seg, lab, g, steps, lr, l_frozen=l_frozen)
    a, e = ex.param_range(2 * l_frozen, 2 * g.layers)
    for _ in range(steps):
        dev.append(run().item() / batch)
        ex.sgd_range(a, e, lr, momentum=0.9)
    torch.cuda.synchronize()
    del ex
    return dev, ref
