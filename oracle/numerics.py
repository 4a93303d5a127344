"""Numerics policies for the CPU train-step oracles -- TEST INFRASTRUCTURE ONLY.

The reference computes no tensor values, so the tensor
oracles (`vit_fp32.py`, `bert_fp32.py`) restate the block structure the
reference profiles (model.cpp:107-121 ViT, model.cpp:152-179 BERT) in
PyTorch-CPU.  They run under one of two policies:

* `FP32`: plain fp32 everywhere -- the north_star's "reference fp32".
* `BF16_STORAGE`: the same fp32 math, but every tensor the sm_100a executor
  keeps in HBM as bf16 is rounded to bf16 exactly where the executor stores
  it -- in the forward (X, H1, QKV, A, X1, H2, G, gelu', logits ...) and in
  the backward (dX, dH, dA, dQKV, dU, dlogits ...), with bf16 GEMM weights
  (the executor's `p16` working copy) and fp32 accumulation.  This isolates
  the error a bf16-storage design is *entitled* to (its distance from FP32)
  from the error of the kernels (their distance from BF16_STORAGE), so each
  can be held to a bound.

The rounding is expressed as autograd nodes, so one forward restatement
serves both policies and the backward stores fall out of the chain rule:

* `store(x)`: rounds the value in the forward and the incoming gradient in
  the backward -- a tensor whose value and whose gradient both live in HBM
  as bf16 (the executor's residual stream X / dX, H / dH, QKV / dQKV ...).
  Autograd sums every consumer's contribution before the node's backward
  runs, matching the executor's fused "LN backward + residual gradient,
  rounded once" epilogues.
* `value(x)`: rounds the value only (GEMM weights, patchified pixels).
* `gelu(x)`: G = bf16(gelu(x)); backward dU = bf16(dG * bf16(gelu'(x)))
  -- the FC1 epilogue stores gelu and gelu' (EPS_EPI_BIAS_GELU2_BF16), the
  FC2 dgrad epilogue multiplies by the stored gelu' (EPS_EPI_MUL_BF16); dG
  itself is never stored.
* `attention(q, k, v, scale)`: exact softmax attention; under bf16 storage
  the probabilities feed P.V as bf16 (P lives in TMEM as the bf16 A operand,
  normalised by the fp32 row sum afterwards) and the backward rounds dS
  before dQ = dS K, dK = dS^T Q (attention_tc.cu).

GELU is the erf form in both policies (PyTorch's default; ViT / BERT).
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

_INV_SQRT_2PI = 0.3989422804014327


def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


class _Store(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return _bf(x)

    @staticmethod
    def backward(ctx, g):
        return _bf(g)


class _Value(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return _bf(x)

    @staticmethod
    def backward(ctx, g):
        return g


def _gelu_grad(x: torch.Tensor) -> torch.Tensor:
    cdf = 0.5 * (1.0 + torch.erf(x * 0.7071067811865476))
    return cdf + x * _INV_SQRT_2PI * torch.exp(-0.5 * x * x)


class _GeluStore(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        ctx.save_for_backward(_bf(_gelu_grad(x)))  # U = gelu'(x), stored bf16
        return _bf(F.gelu(x))

    @staticmethod
    def backward(ctx, g):
        (u,) = ctx.saved_tensors
        return _bf(g * u)


class _AttnStore(torch.autograd.Function):
    """q, k, v: [B, H, T, dh] (already bf16 values).  Returns O (fp32; the
    caller's store() rounds it)."""

    @staticmethod
    def forward(ctx, q, k, v, scale):
        s = (q @ k.transpose(-1, -2)) * scale
        m = s.amax(-1, keepdim=True)
        e = torch.exp(s - m)
        l = e.sum(-1, keepdim=True)
        o = (_bf(e) @ v) / l
        p = e / l
        ctx.save_for_backward(q, k, v, p, _bf(o))
        ctx.scale = scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, p, o16 = ctx.saved_tensors
        # dO arrives rounded (dA is stored bf16); O in D = rowsum(dO * O) is
        # the stored bf16 attention output
        dv = _bf(p).transpose(-1, -2) @ do
        dp = do @ v.transpose(-1, -2)
        dsum = (do * o16).sum(-1, keepdim=True)
        ds = _bf(p * (dp - dsum))
        dq = (ds @ k) * ctx.scale
        dk = (ds.transpose(-1, -2) @ q) * ctx.scale
        return dq, dk, dv, None


class FP32:
    """Plain fp32 restatement (the north_star reference numerics)."""
    name = "fp32"

    @staticmethod
    def store(x):
        return x

    @staticmethod
    def value(x):
        return x

    @staticmethod
    def gelu(x):
        return F.gelu(x)

    @staticmethod
    def attention(q, k, v, scale):
        return torch.softmax((q @ k.transpose(-1, -2)) * scale, dim=-1) @ v


class BF16_STORAGE:
    """fp32 math with the executor's bf16 storage points (see module doc)."""
    name = "bf16-storage"

    @staticmethod
    def store(x):
        return _Store.apply(x)

    @staticmethod
    def value(x):
        return _Value.apply(x)

    @staticmethod
    def gelu(x):
        return _GeluStore.apply(x)

    @staticmethod
    def attention(q, k, v, scale):
        return _AttnStore.apply(q, k, v, scale)


POLICIES = {"fp32": FP32, "bf16": BF16_STORAGE}


def policy(p) -> type:
    if isinstance(p, str):
        return POLICIES[p]
    return p or FP32


def rel_l2(a: torch.Tensor, b: torch.Tensor) -> float:
    """||a - b|| / ||b|| in fp64 (the per-tensor error metric of the tests)."""
    a, b = a.detach().double().cpu(), b.detach().double().cpu()
    return float((a - b).norm() / (b.norm() + 1e-30))
