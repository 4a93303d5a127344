"""PyTorch-CPU restatement of the ViT train step -- TEST INFRASTRUCTURE ONLY.

Numerics oracle for the sm_100a executor: the reference
artifact computes no tensor values, so "parity unpinned" -- this module is
an independent restatement of the block structure the reference's
ModelSpec profiles (model.cpp:107-121: ATT = LN + QKV + out-proj, MLP = LN +
fc1 + fc2; pre-norm ViT; embeddings folded into layer 0 and the
head into layer L-1, model.cpp:137-142).  Only tests/, smoke() and bench.py's
cpu_baseline leg may import it.

Two numerics policies (oracle/numerics.py): `nm="fp32"` (the north_star's
fp32 reference) and `nm="bf16"` (same math, rounded to bf16 exactly where the
executor stores: patches, ptok, X, H1, QKV, A, X1, H2, G / gelu', hf, logits
and the matching gradients).

Freeze semantics mirror the executor: layers [0, L_f) run forward only and
receive no gradient; the embedding belongs to layer 0.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import torch
import torch.nn.functional as F

from .numerics import policy


def patchify(images: torch.Tensor, image: int, patch: int) -> torch.Tensor:
    """[B,C,S,S] -> [B, P, C*p*p] in Conv2d weight order; nearest-upsamples
    a smaller stored image to `image` first (CIFAR-shaped inputs)."""
    if images.shape[-1] != image:
        idx = torch.arange(image) * images.shape[-1] // image
        images = images[:, :, idx][:, :, :, idx]
    B, Cc, S, _ = images.shape
    n = S // patch
    x = images.reshape(B, Cc, n, patch, n, patch).permute(0, 2, 4, 1, 3, 5)
    return x.reshape(B, n * n, Cc * patch * patch)


def attention(h: torch.Tensor, wqkv, bqkv, heads: int, nm=None) -> torch.Tensor:
    nm = policy(nm)
    B, T, D = h.shape
    dh = D // heads
    qkv = nm.store(h @ nm.value(wqkv).t() + bqkv)
    q, k, v = qkv.split(D, dim=-1)
    q = q.reshape(B, T, heads, dh).transpose(1, 2)
    k = k.reshape(B, T, heads, dh).transpose(1, 2)
    v = v.reshape(B, T, heads, dh).transpose(1, 2)
    o = nm.attention(q, k, v, dh ** -0.5)
    return nm.store(o.transpose(1, 2).reshape(B, T, D))


def forward(p: Dict[str, torch.Tensor], images: torch.Tensor, g, l_frozen: int = 0,
            start_x: torch.Tensor = None, start_layer: int = 0,
            nm=None) -> Tuple[torch.Tensor, List[torch.Tensor]]:
    """Logits and the residual-stream inputs X[start..L]."""
    nm = policy(nm)
    S, V = nm.store, nm.value
    d, L = g.hidden, g.layers
    xs = []
    if start_x is None:
        pt = V(patchify(images, g.image, g.patch))
        tok = S(pt @ V(p["patch_embed.weight"]).t() + p["patch_embed.bias"])
        cls = p["cls_token"].expand(tok.shape[0], 1, d)
        x = S(torch.cat([cls, tok], dim=1) + p["pos_embed"])
        start_layer = 0
    else:
        x = start_x
    for l in range(start_layer, L):
        if l == l_frozen and l_frozen > 0:
            x = x.detach()  # nothing below the boundary receives gradient
        xs.append(x)
        q = f"blocks.{l}."
        h = S(F.layer_norm(x, (d,), p[q + "norm1.weight"], p[q + "norm1.bias"], eps=1e-6))
        a = attention(h, p[q + "attn.qkv.weight"], p[q + "attn.qkv.bias"], g.heads, nm)
        x = S(x + a @ V(p[q + "attn.proj.weight"]).t() + p[q + "attn.proj.bias"])
        h = S(F.layer_norm(x, (d,), p[q + "norm2.weight"], p[q + "norm2.bias"], eps=1e-6))
        u = nm.gelu(h @ V(p[q + "mlp.fc1.weight"]).t() + p[q + "mlp.fc1.bias"])
        x = S(x + u @ V(p[q + "mlp.fc2.weight"]).t() + p[q + "mlp.fc2.bias"])
    xs.append(x)
    hf = S(F.layer_norm(x[:, 0], (d,), p["norm.weight"], p["norm.bias"], eps=1e-6))
    return S(hf @ V(p["head.weight"]).t() + p["head.bias"]), xs


def trainable(name: str, l_frozen: int) -> bool:
    if name.startswith("blocks."):
        return int(name.split(".")[1]) >= l_frozen
    if name.startswith(("patch_embed", "cls_token", "pos_embed")):
        return l_frozen == 0
    return True


def train_step(params: Dict[str, torch.Tensor], images: torch.Tensor, labels: torch.Tensor, g,
               l_frozen: int = 0, nm=None, with_acts: bool = False):
    """Mean cross-entropy loss and the fp32 gradients of the trainable params
    (+ the residual-stream activations X[0..L] when `with_acts`)."""
    p = {k: v.detach().clone().float().requires_grad_(trainable(k, l_frozen))
         for k, v in params.items()}
    logits, xs = forward(p, images.float(), g, l_frozen, nm=nm)
    loss = F.cross_entropy(logits, labels)
    loss.backward()
    grads = {k: (v.grad if v.grad is not None else torch.zeros_like(v)) for k, v in p.items()}
    if with_acts:
        return loss.detach(), grads, logits.detach(), [x.detach() for x in xs]
    return loss.detach(), grads, logits.detach()


def sgd_trajectory(params: Dict[str, torch.Tensor], images, labels, g, steps: int, lr: float,
                   momentum: float = 0.9, l_frozen: int = 0, nm=None) -> List[float]:
    """Per-step mean loss of `steps` SGD-momentum iterations on one batch
    (buf = mu*buf + g; p -= lr*buf, as eps_sgd_momentum); frozen tensors stay."""
    p = {k: v.detach().clone().float() for k, v in params.items()}
    bufs = {k: torch.zeros_like(v) for k, v in p.items()}
    losses = []
    for _ in range(steps):
        loss, grads, _ = train_step(p, images, labels, g, l_frozen, nm=nm)
        losses.append(loss.item())
        with torch.no_grad():
            for k in p:
                if trainable(k, l_frozen):
                    bufs[k].mul_(momentum).add_(grads[k])
                    p[k].sub_(lr * bufs[k])
    return losses


def layer_norms(grads: Dict[str, torch.Tensor], g, l_frozen: int):
    """Per-layer L2 norm over every parameter attributed to layer l in the
    reference's ModelSpec (embed -> layer 0, final LN + head -> layer L-1)."""
    sq = [0.0] * g.layers
    for k, v in grads.items():
        if k.startswith("blocks."):
            l = int(k.split(".")[1])
        elif k.startswith(("patch_embed", "cls_token", "pos_embed")):
            l = 0
        else:
            l = g.layers - 1
        sq[l] += float((v.double() ** 2).sum())
    return [s ** 0.5 if l >= l_frozen else 0.0 for l, s in enumerate(sq)]
