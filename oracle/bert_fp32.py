"""PyTorch-CPU fp32 restatement of the BERT train step -- TEST INFRASTRUCTURE ONLY.

Numerics oracle for the sm_100a BERT executor (csrc/runtime/bert.cu); parity
unpinned (the reference computes no tensors).  Block
structure of the reference's BERT profile (model.cpp:152-179: ATT = QKV +
out-proj + LN, MLP = fc1 + fc2 + LN; embeddings in layer 0, pooler + head in
layer L-1), post-norm as in BERT.  GELU is the erf form.
Freeze semantics: layers [0, L_f) forward only; the embeddings belong to
layer 0.  Only tests/ may import it.
"""
from __future__ import annotations

from typing import Dict

import torch
import torch.nn.functional as F


def forward(p: Dict[str, torch.Tensor], tokens, segments, g, l_frozen: int = 0):
    d, T, H = g.hidden, g.tokens, g.heads
    B = tokens.shape[0]
    pos = torch.arange(T)
    x = (p["embeddings.word_embeddings.weight"][tokens] +
         p["embeddings.position_embeddings.weight"][pos][None] +
         p["embeddings.token_type_embeddings.weight"][segments])
    x = F.layer_norm(x, (d,), p["embeddings.LayerNorm.weight"], p["embeddings.LayerNorm.bias"],
                     eps=1e-12)
    dh = d // H
    for l in range(g.layers):
        if l == l_frozen and l_frozen > 0:
            x = x.detach()
        q = f"layer.{l}."
        qkv = x @ p[q + "attention.qkv.weight"].t() + p[q + "attention.qkv.bias"]
        qq, kk, vv = qkv.split(d, dim=-1)
        qq = qq.reshape(B, T, H, dh).transpose(1, 2)
        kk = kk.reshape(B, T, H, dh).transpose(1, 2)
        vv = vv.reshape(B, T, H, dh).transpose(1, 2)
        a = torch.softmax((qq @ kk.transpose(-1, -2)) * dh ** -0.5, -1) @ vv
        a = a.transpose(1, 2).reshape(B, T, d)
        x = F.layer_norm(x + a @ p[q + "attention.output.dense.weight"].t() +
                         p[q + "attention.output.dense.bias"], (d,),
                         p[q + "attention.output.LayerNorm.weight"],
                         p[q + "attention.output.LayerNorm.bias"], eps=1e-12)
        u = F.gelu(x @ p[q + "intermediate.dense.weight"].t() + p[q + "intermediate.dense.bias"])
        x = F.layer_norm(x + u @ p[q + "output.dense.weight"].t() + p[q + "output.dense.bias"],
                         (d,), p[q + "output.LayerNorm.weight"], p[q + "output.LayerNorm.bias"],
                         eps=1e-12)
    return x


def trainable(name: str, l_frozen: int) -> bool:
    if name.startswith("layer."):
        return int(name.split(".")[1]) >= l_frozen
    if name.startswith("embeddings."):
        return l_frozen == 0
    return True


def train_step(params, tokens, segments, labels, g, l_frozen: int = 0):
    """Mean loss and fp32 gradients.  labels: [B] (cls head) or [2, B] (qa)."""
    p = {k: v.detach().clone().float().requires_grad_(trainable(k, l_frozen))
         for k, v in params.items()}
    x = forward(p, tokens, segments, g, l_frozen)
    if g.head == "qa":
        logits = x @ p["classifier.weight"].t() + p["classifier.bias"]  # [B, T, 2]
        loss = 0.5 * (F.cross_entropy(logits[..., 0], labels[0]) +
                      F.cross_entropy(logits[..., 1], labels[1]))
    else:
        h = x[:, 0]
        if g.pooler:
            h = torch.tanh(h @ p["pooler.dense.weight"].t() + p["pooler.dense.bias"])
        logits = h @ p["classifier.weight"].t() + p["classifier.bias"]
        loss = F.cross_entropy(logits, labels)
    loss.backward()
    grads = {k: (v.grad if v.grad is not None else torch.zeros_like(v)) for k, v in p.items()}
    return loss.detach(), grads


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
