"""PyTorch-CPU restatement of the BERT train step -- TEST INFRASTRUCTURE ONLY.

Numerics oracle for the sm_100a BERT executor (csrc/runtime/bert.cu); parity
unpinned (the reference computes no tensors).  Block
structure of the reference's BERT profile (model.cpp:152-179: ATT = QKV +
out-proj + LN, MLP = fc1 + fc2 + LN; embeddings in layer 0, pooler + head in
layer L-1), post-norm as in BERT.  GELU is the erf form.
Freeze semantics: layers [0, L_f) forward only; the embeddings belong to
layer 0.  Only tests/ may import it.

Numerics policies as in vit_fp32 (oracle/numerics.py): `nm="bf16"` rounds
where bert.cu stores -- E, X, QKV, A, S1 (= X + proj), X1, G / gelu', S2,
logits, pooler pre-activation / output and the matching gradients.
"""
from __future__ import annotations

from typing import Dict, List

import torch
import torch.nn.functional as F

from .numerics import policy


def forward(p: Dict[str, torch.Tensor], tokens, segments, g, l_frozen: int = 0, nm=None,
            xs: list = None):
    """Final hidden states [B, T, d]; appends X[0..L] to `xs` when given."""
    nm = policy(nm)
    S, V = nm.store, nm.value
    d, T, H = g.hidden, g.tokens, g.heads
    B = tokens.shape[0]
    pos = torch.arange(T)
    x = S(p["embeddings.word_embeddings.weight"][tokens] +
          p["embeddings.position_embeddings.weight"][pos][None] +
          p["embeddings.token_type_embeddings.weight"][segments])
    x = S(F.layer_norm(x, (d,), p["embeddings.LayerNorm.weight"], p["embeddings.LayerNorm.bias"],
                       eps=1e-12))
    dh = d // H
    for l in range(g.layers):
        if l == l_frozen and l_frozen > 0:
            x = x.detach()
        if xs is not None:
            xs.append(x)
        q = f"layer.{l}."
        qkv = S(x @ V(p[q + "attention.qkv.weight"]).t() + p[q + "attention.qkv.bias"])
        qq, kk, vv = qkv.split(d, dim=-1)
        qq = qq.reshape(B, T, H, dh).transpose(1, 2)
        kk = kk.reshape(B, T, H, dh).transpose(1, 2)
        vv = vv.reshape(B, T, H, dh).transpose(1, 2)
        a = S(nm.attention(qq, kk, vv, dh ** -0.5).transpose(1, 2).reshape(B, T, d))
        s1 = S(x + a @ V(p[q + "attention.output.dense.weight"]).t() +
               p[q + "attention.output.dense.bias"])
        x = S(F.layer_norm(s1, (d,), p[q + "attention.output.LayerNorm.weight"],
                           p[q + "attention.output.LayerNorm.bias"], eps=1e-12))
        u = nm.gelu(x @ V(p[q + "intermediate.dense.weight"]).t() +
                    p[q + "intermediate.dense.bias"])
        s2 = S(x + u @ V(p[q + "output.dense.weight"]).t() + p[q + "output.dense.bias"])
        x = S(F.layer_norm(s2, (d,), p[q + "output.LayerNorm.weight"],
                           p[q + "output.LayerNorm.bias"], eps=1e-12))
    if xs is not None:
        xs.append(x)
    return x


def trainable(name: str, l_frozen: int) -> bool:
    if name.startswith("layer."):
        return int(name.split(".")[1]) >= l_frozen
    if name.startswith("embeddings."):
        return l_frozen == 0
    return True


def train_step(params, tokens, segments, labels, g, l_frozen: int = 0, nm=None,
               with_acts: bool = False):
    """Mean loss and fp32 gradients (+ X[0..L] when `with_acts`).
    labels: [B] (cls head) or [2, B] (qa)."""
    nm = policy(nm)
    S, V = nm.store, nm.value
    p = {k: v.detach().clone().float().requires_grad_(trainable(k, l_frozen))
         for k, v in params.items()}
    xs: List[torch.Tensor] = []
    x = forward(p, tokens, segments, g, l_frozen, nm=nm, xs=xs)
    if g.head == "qa":
        logits = S(x @ V(p["classifier.weight"]).t() + p["classifier.bias"])  # [B, T, 2]
        loss = 0.5 * (F.cross_entropy(logits[..., 0], labels[0]) +
                      F.cross_entropy(logits[..., 1], labels[1]))
    else:
        h = x[:, 0]
        if g.pooler:
            pre = S(h @ V(p["pooler.dense.weight"]).t() + p["pooler.dense.bias"])
            h = S(torch.tanh(pre))
        logits = S(h @ V(p["classifier.weight"]).t() + p["classifier.bias"])
        loss = F.cross_entropy(logits, labels)
    loss.backward()
    grads = {k: (v.grad if v.grad is not None else torch.zeros_like(v)) for k, v in p.items()}
    if with_acts:
        return loss.detach(), grads, [t.detach() for t in xs]
    return loss.detach(), grads


def sgd_trajectory(params, tokens, segments, labels, g, steps: int, lr: float,
                   momentum: float = 0.9, l_frozen: int = 0, nm=None) -> List[float]:
    """Per-step mean loss of `steps` SGD-momentum iterations on one batch
    (buf = mu*buf + g; p -= lr*buf, as eps_sgd_momentum)."""
    p = {k: v.detach().clone().float() for k, v in params.items()}
    bufs = {k: torch.zeros_like(v) for k, v in p.items()}
    losses = []
    for _ in range(steps):
        loss, grads = train_step(p, tokens, segments, labels, g, l_frozen, nm=nm)
        losses.append(loss.item())
        with torch.no_grad():
            for k in p:
                if trainable(k, l_frozen):
                    bufs[k].mul_(momentum).add_(grads[k])
                    p[k].sub_(lr * bufs[k])
    return losses


def layer_norms(grads, g, l_frozen: int):
    sq = [0.0] * g.layers
    for k, v in grads.items():
        if k.startswith("layer."):
            l = int(k.split(".")[1])
        elif k.startswith("embeddings."):
            l = 0
        else:
            l = g.layers - 1
        sq[l] += float((v.double() ** 2).sum())
    return [s ** 0.5 if l >= l_frozen else 0.0 for l, s in enumerate(sq)]
