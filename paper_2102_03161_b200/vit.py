"""ViT stage executor front end (C++ runtime in csrc/runtime/vit.cu).

Python here only allocates the caller-owned arenas with torch (device
memory is plumbing), seeds the parameters, and forwards each call to the
C ABI.  Every FLOP of a training iteration runs in libeps_b200.so.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Dict, Optional

import torch

from . import ops
from .configs import Geometry

TENSOR_NAMES_EMBED = ["patch_embed.weight", "patch_embed.bias", "cls_token", "pos_embed"]
TENSOR_NAMES_LAYER = ["norm1.weight", "norm1.bias", "attn.qkv.weight", "attn.qkv.bias",
                      "attn.proj.weight", "attn.proj.bias", "norm2.weight", "norm2.bias",
                      "mlp.fc1.weight", "mlp.fc1.bias", "mlp.fc2.weight", "mlp.fc2.bias"]
TENSOR_NAMES_TAIL = ["norm.weight", "norm.bias", "head.weight", "head.bias"]


def geom_array(g: Geometry, max_batch: int):
    vals = [g.layers, g.hidden, g.mlp_dim, g.heads, g.tokens, g.classes, g.image,
            g.input_image, g.patch, g.channels, max_batch]
    return (C.c_int * 11)(*vals)


def tensor_shapes(g: Geometry) -> Dict[str, tuple]:
    d, f = g.hidden, g.mlp_dim
    shapes = {"patch_embed.weight": (d, g.channels * g.patch * g.patch),
              "patch_embed.bias": (d,), "cls_token": (d,), "pos_embed": (g.tokens, d)}
    for l in range(g.layers):
        p = f"blocks.{l}."
        shapes.update({p + "norm1.weight": (d,), p + "norm1.bias": (d,),
                       p + "attn.qkv.weight": (3 * d, d), p + "attn.qkv.bias": (3 * d,),
                       p + "attn.proj.weight": (d, d), p + "attn.proj.bias": (d,),
                       p + "norm2.weight": (d,), p + "norm2.bias": (d,),
                       p + "mlp.fc1.weight": (f, d), p + "mlp.fc1.bias": (f,),
                       p + "mlp.fc2.weight": (d, f), p + "mlp.fc2.bias": (d,)})
    shapes.update({"norm.weight": (d,), "norm.bias": (d,), "head.weight": (g.classes, d),
                   "head.bias": (g.classes,)})
    return shapes


def layout(g: Geometry, max_batch: int):
    """(param_total, workspace_bytes, segments[L+1], {name: (offset, numel)})."""
    lib = ops.api().lib
    total, ws = C.c_int64(), C.c_int64()
    segs = (C.c_int64 * (g.layers + 1))()
    nt = 4 + 12 * g.layers + 4
    tens = (C.c_int64 * (2 * nt))()
    f = lib.eps_vit_layout
    f.restype = C.c_int
    rc = f(geom_array(g, max_batch), C.byref(total), C.byref(ws), segs, tens)
    if rc != 0:
        raise ValueError(f"eps_vit_layout rejected geometry {g} (status {rc})")
    names = list(TENSOR_NAMES_EMBED)
    for l in range(g.layers):
        names += [f"blocks.{l}.{n}" for n in TENSOR_NAMES_LAYER]
    names += TENSOR_NAMES_TAIL
    offsets = {n: (tens[2 * i], tens[2 * i + 1]) for i, n in enumerate(names)}
    return total.value, ws.value, list(segs), offsets


def init_params(g: Geometry, seed: int) -> Dict[str, torch.Tensor]:
    """Seeded fp32 initialisation (CPU): trunc-normal(0.02) weights, zero biases,
    unit LN gains -- the weights the oracle and the device both start from."""
    gen = torch.Generator().manual_seed(seed)
    out = {}
    for name, shape in tensor_shapes(g).items():
        if name.endswith("norm1.weight") or name.endswith("norm2.weight") or name == "norm.weight":
            t = torch.ones(shape)
        elif name.endswith("bias"):
            t = torch.zeros(shape)
        else:
            t = torch.empty(shape)
            torch.nn.init.trunc_normal_(t, std=0.02, a=-0.04, b=0.04, generator=gen)
        out[name] = t
    return out


class VitExecutor:
    """The ViT stage executor on the current GPU (the whole stack at K = 1, or
    the sublayer span of one pipeline stage)."""

    PREFIX = "eps_vit_"

    def __init__(self, g: Geometry, max_batch: int, seed: int = 17, device=None,
                 params: Optional[Dict[str, torch.Tensor]] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("VitExecutor needs a CUDA device (no CPU fallback)")
        self.g = g
        self.max_batch = max_batch
        self.device = torch.device(device or "cuda")
        self.total, ws_bytes, self.segments, self.offsets = layout(g, max_batch)
        dev = self.device
        self.p32 = torch.zeros(self.total, dtype=torch.float32, device=dev)
        self.p16 = torch.zeros(self.total, dtype=torch.bfloat16, device=dev)
        self.g32 = torch.zeros(self.total, dtype=torch.float32, device=dev)
        self.mom = torch.zeros(self.total, dtype=torch.float32, device=dev)
        self.ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float32, device=dev)
        self.sq = torch.zeros(g.layers, dtype=torch.float64, device=dev)
        self.load_params(params if params is not None else init_params(g, seed))
        h = C.c_void_p()
        lib = ops.api().lib
        lib.eps_vit_create.restype = C.c_int
        rc = lib.eps_vit_create(geom_array(g, max_batch), C.c_void_p(self.p32.data_ptr()),
                                C.c_void_p(self.p16.data_ptr()), C.c_void_p(self.g32.data_ptr()),
                                C.c_void_p(self.mom.data_ptr()), C.c_void_p(self.ws.data_ptr()),
                                C.byref(h))
        if rc != 0:
            raise RuntimeError(f"eps_vit_create failed ({rc})")
        self._destroy = getattr(lib, self.PREFIX + "destroy")
        self._destroy.restype = None
        self.h = h

    def __del__(self):
        # the destroy entry is bound at construction: module globals may
        # already be torn down when this runs at interpreter exit
        f = getattr(self, "_destroy", None)
        if getattr(self, "h", None) and f is not None:
            f(self.h)
            self.h = None

    # -- parameters --------------------------------------------------------
    def _stored_shape(self, name, shape):
        # the head is stored with classes padded to a multiple of 8 (TMA row pitch)
        if name in ("head.weight", "head.bias"):
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
            t = flat[o:o + k].reshape(self._stored_shape(n, shapes[n]))
            out[n] = t[:shapes[n][0]]
        return out

    def params(self) -> Dict[str, torch.Tensor]:
        return self._unflatten(self.p32)

    def grads(self) -> Dict[str, torch.Tensor]:
        return self._unflatten(self.g32)

    # -- execution ---------------------------------------------------------
    def _call(self, name, *args):
        f = getattr(ops.api().lib, name)
        f.restype = C.c_int
        # tensors -> device pointers; ctypes values / arrays pass through
        conv = [C.c_void_p(a.data_ptr()) if isinstance(a, torch.Tensor) else a for a in args]
        rc = f(self.h, *conv)
        if rc != 0:
            raise RuntimeError(f"{name} failed with status {rc}")

    def train_step(self, images: torch.Tensor, labels: torch.Tensor, *, micro_batches: int = 1,
                   l_frozen: int = 0, cache_mode: int = 0, cache_old: int = 0,
                   store: Optional[torch.Tensor] = None, ids: Optional[torch.Tensor] = None,
                   stream=None):
        """Forward + backward of one batch; grads accumulate into g32.
        Returns the device loss-sum tensor (not synchronised)."""
        b = labels.shape[0]
        if images is not None and (images.dtype != torch.float32 or not images.is_cuda):
            raise TypeError("images must be fp32 CUDA")
        self.loss_sum.zero_()
        s = torch.cuda.current_stream() if stream is None else stream
        self._call("eps_vit_train_step",
                   images if images is not None else C.c_void_p(0), labels, b, micro_batches,
                   l_frozen, cache_mode, cache_old,
                   store if store is not None else C.c_void_p(0),
                   ids if ids is not None else C.c_void_p(0), self.loss_sum,
                   C.c_void_p(s.cuda_stream))
        return self.loss_sum

    def sgd(self, l_frozen: int, lr: float, momentum: float = 0.9, weight_decay: float = 0.0,
            stream=None):
        s = torch.cuda.current_stream() if stream is None else stream
        self._call("eps_vit_sgd", l_frozen, C.c_float(lr), C.c_float(momentum),
                   C.c_float(weight_decay), C.c_void_p(s.cuda_stream))

    def layer_sqnorms(self, l_frozen: int, stream=None) -> torch.Tensor:
        """Per-layer gradient sum of squares (device fp64 [L]; frozen layers 0)."""
        self.sq.zero_()
        self.sqnorm_ranges(self.segments[l_frozen:], self.sq[l_frozen:], stream)
        return self.sq

    def layer_norms(self, l_frozen: int):
        """Per-layer gradient L2 norms (host floats) for the freeze decision."""
        return [math.sqrt(v) for v in self.layer_sqnorms(l_frozen).cpu().tolist()]

    def forward_logits(self, images: torch.Tensor) -> torch.Tensor:
        b = images.shape[0]
        cp = (self.g.classes + 7) // 8 * 8
        out = torch.empty(b, cp, dtype=torch.bfloat16, device=self.device)
        s = torch.cuda.current_stream()
        self._call("eps_vit_forward_logits", images, b, out, C.c_void_p(s.cuda_stream))
        return out[:, :self.g.classes]

    # -- pipeline-stage operations (AutoPipe executor) --------------------
    def _st(self, stream):
        s = torch.cuda.current_stream() if stream is None else stream
        return C.c_void_p(s.cuda_stream)

    def stage_forward(self, images, b0: int, b: int, g0: int, g1: int, l_frozen: int,
                      front: bool, cache_mode: int = 0, cache_old: int = 0, store=None,
                      ids=None, stream=None):
        self._call(self.PREFIX + "stage_forward",
                   images if images is not None else C.c_void_p(0), b0, b, g0, g1, l_frozen,
                   int(front), cache_mode, cache_old,
                   store if store is not None else C.c_void_p(0),
                   ids if ids is not None else C.c_void_p(0), self._st(stream))

    def stage_head(self, labels, b0: int, b: int, global_batch: int, stream=None):
        self._call(self.PREFIX + "stage_head", labels, b0, b, global_batch, self.loss_sum,
                   self._st(stream))

    def stage_backward(self, b0: int, b: int, g0: int, g1: int, l_frozen: int, cut_out: bool,
                       stream=None):
        self._call(self.PREFIX + "stage_backward", b0, b, g0, g1, l_frozen, int(cut_out),
                   self._st(stream))

    def stage_backward_part(self, b0: int, b: int, g0: int, g1: int, stage_g0: int,
                            l_frozen: int, cut_out: bool, stream=None):
        self._call(self.PREFIX + "stage_backward_part", b0, b, g0, g1, stage_g0, l_frozen,
                   int(cut_out), self._st(stream))

    def cut_rows(self, g: int, b0: int, b: int, grad: bool = False) -> torch.Tensor:
        """bf16 view [b*T, d] of the residual stream at the cut before global
        sublayer g (grad=True: the dX scratch), rows of samples [b0, b0+b)."""
        f = getattr(ops.api().lib, self.PREFIX + "cut")
        f.restype = C.c_void_p
        f.argtypes = [C.c_void_p, C.c_int, C.c_int]
        ptr = f(self.h, g, int(grad))
        if not ptr:
            raise ValueError(f"no cut buffer for sublayer {g}")
        T, d = self.g.tokens, self.g.hidden
        off = ptr - self.ws.data_ptr()
        base = self.ws[off:off + 2 * self.max_batch * T * d].view(torch.bfloat16)
        return base.view(self.max_batch * T, d)[b0 * T:(b0 + b) * T]

    def set_redirect(self, out_g: int, out_ptr, dx_g: int, dx_ptr):
        """Write the output cut `out_g` / the gradient at cut `dx_g` straight
        into peer buffers (device addresses, e.g. IPC-mapped); None = local."""
        self._call(self.PREFIX + "set_redirect", out_g, C.c_void_p(out_ptr or 0), dx_g,
                   C.c_void_p(dx_ptr or 0))

    def param_range(self, g0: int, g1: int):
        """Parameter elements [begin, end) of global sublayers [g0, g1)."""
        a, e = C.c_int64(), C.c_int64()
        self._call(self.PREFIX + "param_range", g0, g1, C.byref(a), C.byref(e))
        return a.value, e.value

    def sgd_range(self, begin: int, end: int, lr: float, momentum: float = 0.9,
                  weight_decay: float = 0.0, stream=None):
        self._call(self.PREFIX + "sgd_range", C.c_int64(begin), C.c_int64(end), C.c_float(lr),
                   C.c_float(momentum), C.c_float(weight_decay), self._st(stream))

    def sqnorm_ranges(self, offsets, out: torch.Tensor, stream=None):
        """out[i] = sum of squared grads over offsets[i]..offsets[i+1]."""
        arr = (C.c_int64 * len(offsets))(*offsets)
        self._call(self.PREFIX + "sqnorm_ranges", arr, len(offsets) - 1, out, self._st(stream))
        return out

    # -- instrumentation ---------------------------------------------------
    TIMING_CLASSES = ("gemm", "attention", "layernorm", "eltwise", "cache", "optimizer",
                      "sqnorm")

    def timing(self, on: bool):
        """Bracket every executor launch with CUDA events on its stream."""
        self._call(self.PREFIX + "timing_enable", int(on))

    def timing_read(self) -> Dict[str, dict]:
        """Per kernel class: device ms, algorithmic FLOPs / bytes, launches."""
        n = len(self.TIMING_CLASSES)
        ms, fl, by = (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        self._call(self.PREFIX + "timing_read", ms, fl, by, cnt)
        return {c: {"ms": ms[i], "flops": fl[i], "bytes": by[i], "launches": cnt[i]}
                for i, c in enumerate(self.TIMING_CLASSES)}

    def boundary_activation(self, layer: int, batch: int) -> torch.Tensor:
        """View of X[layer] rows for the first `batch` samples (bf16)."""
        f = ops.api().lib.eps_vit_activation
        f.restype = C.c_void_p
        ptr = f(self.h, 0, layer)
        n = batch * self.g.tokens * self.g.hidden
        # wrap the raw device pointer via an offset into the workspace tensor
        base = self.ws.data_ptr()
        off = ptr - base
        return self.ws[off:off + 2 * n].view(torch.bfloat16).view(batch, self.g.tokens,
                                                                   self.g.hidden)
