"""BERT stage executor front end (C++ runtime in csrc/runtime/bert.cu).

Same surface as VitExecutor (the pipeline / trainer code drives either);
torch only allocates the caller-owned arenas and seeds the parameters.
Front-stage inputs are int64 [2, B, T] (token ids, segment ids); labels are
int64 [B] (pooled-CLS head) or [2, B] (SQuAD start / end positions).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional

import torch

from . import ops
from .configs import Geometry
from .vit import VitExecutor

EMBED = ["embeddings.word_embeddings.weight", "embeddings.position_embeddings.weight",
         "embeddings.token_type_embeddings.weight", "embeddings.LayerNorm.weight",
         "embeddings.LayerNorm.bias"]
LAYER = ["attention.qkv.weight", "attention.qkv.bias", "attention.output.dense.weight",
         "attention.output.dense.bias", "attention.output.LayerNorm.weight",
         "attention.output.LayerNorm.bias", "intermediate.dense.weight",
         "intermediate.dense.bias", "output.dense.weight", "output.dense.bias",
         "output.LayerNorm.weight", "output.LayerNorm.bias"]


def head_kind(g: Geometry) -> int:
    return 1 if g.head == "qa" else 0


def geom_array(g: Geometry, max_batch: int):
    vals = [g.layers, g.hidden, g.mlp_dim, g.heads, g.tokens, g.classes, g.vocab, g.positions,
            head_kind(g), int(g.pooler), max_batch]
    return (C.c_int * 11)(*vals)


def tensor_names(g: Geometry):
    names = list(EMBED)
    for l in range(g.layers):
        names += [f"layer.{l}.{n}" for n in LAYER]
    if g.pooler:
        names += ["pooler.dense.weight", "pooler.dense.bias"]
    names += ["classifier.weight", "classifier.bias"]
    return names


def tensor_shapes(g: Geometry) -> Dict[str, tuple]:
    d, f = g.hidden, g.mlp_dim
    sh = {EMBED[0]: (g.vocab, d), EMBED[1]: (g.positions, d), EMBED[2]: (2, d), EMBED[3]: (d,),
          EMBED[4]: (d,)}
    per = [(3 * d, d), (3 * d,), (d, d), (d,), (d,), (d,), (f, d), (f,), (d, f), (d,), (d,), (d,)]
    for l in range(g.layers):
        for n, s in zip(LAYER, per):
            sh[f"layer.{l}.{n}"] = s
    if g.pooler:
        sh["pooler.dense.weight"] = (d, d)
        sh["pooler.dense.bias"] = (d,)
    sh["classifier.weight"] = (g.classes, d)
    sh["classifier.bias"] = (g.classes,)
    return sh


def layout(g: Geometry, max_batch: int):
    lib = ops.api().lib
    total, ws = C.c_int64(), C.c_int64()
    segs = (C.c_int64 * (g.layers + 1))()
    names = tensor_names(g)
    tens = (C.c_int64 * (2 * len(names)))()
    f = lib.eps_bert_layout
    f.restype = C.c_int
    rc = f(geom_array(g, max_batch), C.byref(total), C.byref(ws), segs, tens)
    if rc != 0:
        raise ValueError(f"eps_bert_layout rejected geometry {g} (status {rc})")
    offsets = {n: (tens[2 * i], tens[2 * i + 1]) for i, n in enumerate(names)}
    return total.value, ws.value, list(segs), offsets


def init_params(g: Geometry, seed: int) -> Dict[str, torch.Tensor]:
    """Seeded fp32 init (CPU): trunc-normal(0.02) matrices / embeddings, zero
    biases, unit LayerNorm gains."""
    gen = torch.Generator().manual_seed(seed)
    out = {}
    for name, shape in tensor_shapes(g).items():
        if "LayerNorm.weight" in name:
            t = torch.ones(shape)
        elif name.endswith("bias"):
            t = torch.zeros(shape)
        else:
            t = torch.empty(shape)
            torch.nn.init.trunc_normal_(t, std=0.02, a=-0.04, b=0.04, generator=gen)
        out[name] = t
    return out


class BertExecutor(VitExecutor):
    """BERT stage executor on the current GPU (see VitExecutor)."""

    PREFIX = "eps_bert_"

    def __init__(self, g: Geometry, max_batch: int, seed: int = 17, device=None,
                 params: Optional[Dict[str, torch.Tensor]] = None, adamw: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("BertExecutor needs a CUDA device (no CPU fallback)")
        self.g = g
        self.max_batch = max_batch
        self.device = torch.device(device or "cuda")
        self.total, ws_bytes, self.segments, self.offsets = layout(g, max_batch)
        dev = self.device
        self.p32 = torch.zeros(self.total, dtype=torch.float32, device=dev)
        self.p16 = torch.zeros(self.total, dtype=torch.bfloat16, device=dev)
        self.g32 = torch.zeros(self.total, dtype=torch.float32, device=dev)
        self.state = torch.zeros(2 * self.total, dtype=torch.float32, device=dev)
        self.mom = self.state[:self.total]  # SGD momentum / AdamW m (v follows)
        self.ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float32, device=dev)
        self.sq = torch.zeros(g.layers, dtype=torch.float64, device=dev)
        self.adam_step = 0
        self.load_params(params if params is not None else init_params(g, seed))
        h = C.c_void_p()
        lib = ops.api().lib
        lib.eps_bert_create.restype = C.c_int
        rc = lib.eps_bert_create(geom_array(g, max_batch), C.c_void_p(self.p32.data_ptr()),
                                 C.c_void_p(self.p16.data_ptr()), C.c_void_p(self.g32.data_ptr()),
                                 C.c_void_p(self.state.data_ptr()), C.c_void_p(self.ws.data_ptr()),
                                 C.byref(h))
        if rc != 0:
            raise RuntimeError(f"eps_bert_create failed ({rc})")
        self._destroy = lib.eps_bert_destroy
        self._destroy.restype = None
        self.h = h

    def _stored_shape(self, name, shape):
        if name in ("classifier.weight", "classifier.bias"):
            return ((self.g.classes + 7) // 8 * 8,) + tuple(shape[1:])
        return shape

    def load_params(self, params: Dict[str, torch.Tensor]):
        flat = torch.zeros(self.total, dtype=torch.float32)
        shapes = tensor_shapes(self.g)
        for name, (off, n) in self.offsets.items():
            t = torch.zeros(self._stored_shape(name, shapes[name]))
            t[:shapes[name][0]] = params[name].float()
            flat[off:off + n] = t.reshape(-1)
        self.p32.copy_(flat.to(self.device))
        self.p16.copy_(self.p32)

    def _unflatten(self, flat: torch.Tensor) -> Dict[str, torch.Tensor]:
        shapes = tensor_shapes(self.g)
        out = {}
        for n, (o, k) in self.offsets.items():
            out[n] = flat[o:o + k].reshape(self._stored_shape(n, shapes[n]))[:shapes[n][0]]
        return out

    # -- stage operations -----------------------------------------------------------
    def stage_forward(self, inputs, b0: int, b: int, g0: int, g1: int, l_frozen: int,
                      front: bool, cache_mode: int = 0, cache_old: int = 0, store=None,
                      ids=None, stream=None):
        rows = inputs.shape[1] if inputs is not None else 0
        self._call("eps_bert_stage_forward",
                   inputs if inputs is not None else C.c_void_p(0), rows, b0, b, g0, g1,
                   l_frozen, int(front), cache_mode, cache_old,
                   store if store is not None else C.c_void_p(0),
                   ids if ids is not None else C.c_void_p(0), self._st(stream))

    def train_step(self, inputs, labels, *, micro_batches: int = 1, l_frozen: int = 0,
                   cache_mode: int = 0, cache_old: int = 0, store=None, ids=None, stream=None):
        """K = 1 iteration (GPipe order over `micro_batches`, schedule.cpp:28-33)."""
        from .pipeline import microbatch_offsets
        b_total = inputs.shape[1]
        g0, g1 = 2 * l_frozen, 2 * self.g.layers
        self.loss_sum.zero_()
        mbs = microbatch_offsets(b_total, micro_batches)
        for b0, b in mbs:
            self.stage_forward(inputs, b0, b, g0, g1, l_frozen, True, cache_mode, cache_old,
                               store, ids, stream)
            self.stage_head(labels, b0, b, b_total, stream)
        for b0, b in reversed(mbs):
            self.stage_backward(b0, b, g0, g1, l_frozen, False, stream)
        return self.loss_sum

    def adamw_range(self, begin: int, end: int, lr: float, beta1: float = 0.9,
                    beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.01,
                    stream=None):
        self.adam_step += 1
        self._call("eps_bert_adamw_range", C.c_int64(begin), C.c_int64(end), C.c_float(lr),
                   C.c_float(beta1), C.c_float(beta2), C.c_float(eps), C.c_float(weight_decay),
                   self.adam_step, self._st(stream))
