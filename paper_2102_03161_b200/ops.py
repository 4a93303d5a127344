"""torch-tensor front end for the sm_100a data plane in libeps_b200.so.

Every function here is a thin argument check plus one C-ABI call
(include/eps_capi.h).  torch is used only to own device memory and to name
the current CUDA stream; there is no eager/torch fallback -- if the library
or a GPU is missing the call raises.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import LIB_PATH
from .capi import CudaError, EpsApi

EPI_STORE_BF16 = 0
EPI_BIAS_BF16 = 1
EPI_BIAS_GELU_BF16 = 2
EPI_BIAS_RESID_BF16 = 3
EPI_DGELU_BF16 = 4
EPI_STORE_F32 = 5
EPI_ACCUM_F32 = 6
EPI_RESID_BF16 = 7
EPI_ROWDOT_BF16 = 8
EPI_BIAS_GELU2_BF16 = 9
EPI_MUL_BF16 = 10

_api: Optional[EpsApi] = None


def api() -> EpsApi:
    global _api
    if _api is None:
        _api = EpsApi(LIB_PATH, "eps_")
        _declare(_api.lib)
    return _api


def _declare(lib):
    vp, i64, i32, f32 = C.c_void_p, C.c_int64, C.c_int, C.c_float
    sig = {
        "eps_gemm_bf16": [i32, i32, i32, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64,
                          i32, vp],
        "eps_layernorm_fwd": [vp, vp, vp, vp, vp, vp, i64, i64, f32, vp],
        "eps_layernorm_bwd": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp, vp],
        "eps_attn_fwd": [vp, vp, vp, i32, i32, i32, i32, f32, vp],
        "eps_attn_bwd_ws": [vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, f32, vp],
        "eps_attn_bwd_rowdot": [vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, f32, vp],
        "eps_attn_bwd_uses_rowdot": [i32, i32],
        "eps_grad_sqnorm_flat": [vp, vp, i32, vp, vp, C.c_size_t, vp],
        "eps_softmax_xent_bias": [vp, vp, vp, vp, vp, i32, i32, i32, f32, vp],
        "eps_grad_sqnorm_segmented": [vp, vp, vp, i32, vp, i32, vp, C.c_size_t, vp],
        "eps_cache_gather": [vp, vp, i32, i64, vp, vp],
        "eps_cache_gather_bg": [vp, vp, i32, i64, vp, i32, vp],
        "eps_cache_scatter": [vp, vp, i32, i64, vp, vp],
        "eps_sgd_momentum": [vp, vp, vp, vp, i64, f32, f32, f32, vp],
        "eps_adamw": [vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, f32, i32, vp],
        "eps_patchify": [vp, vp, i32, i32, i32, i32, vp],
        "eps_vit_assemble": [vp, vp, vp, vp, i32, i32, i64, vp],
        "eps_vit_assemble_bwd": [vp, vp, vp, vp, i32, i32, i64, vp],
        "eps_softmax_xent": [vp, vp, vp, vp, i32, i32, vp],
        "eps_gather_rows": [vp, i64, vp, i32, i64, i64, vp],
        "eps_scatter_rows": [vp, vp, i64, i32, i64, i64, vp],
        "eps_colsum_bf16": [vp, vp, i64, i64, vp],
    }
    for name, args in sig.items():
        if hasattr(lib, name):
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = C.c_int


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _check(name, rc):
    if rc != 0:
        msg = (api()._last_error() or b"").decode()
        raise CudaError(f"{name} failed with status {rc} {msg}")


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("eps ops take CUDA tensors only (no CPU fallback)")


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, *, a_mn: bool = False,
         b_mn: bool = False, epilogue: int = EPI_STORE_BF16, bias=None, aux=None, colsum=None,
         split_k: int = 1, stream=None):
    """out[M,N] = A(m,k) B(n,k).

    a: [M,K] (a_mn False) or [K,M] (a_mn True); b: [N,K] or [K,N].  bf16,
    row-major, unit inner stride (leading dims may be padded).
    """
    _need_cuda(a, b, out)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise TypeError("gemm operands must be bf16")
    M, K = (a.shape[1], a.shape[0]) if a_mn else (a.shape[0], a.shape[1])
    N, Kb = (b.shape[1], b.shape[0]) if b_mn else (b.shape[0], b.shape[1])
    if K != Kb:
        raise ValueError(f"gemm: K mismatch {K} vs {Kb}")
    if out.shape[0] != M or out.shape[1] != N:
        raise ValueError("gemm: bad output shape")
    rc = api().lib.eps_gemm_bf16(int(a_mn), int(b_mn), epilogue, _ptr(a), _ptr(b), _ptr(out),
                                 _ptr(bias), _ptr(aux), _ptr(colsum), M, N, K, a.stride(0),
                                 b.stride(0), out.stride(0), split_k, _stream(stream))
    _check("eps_gemm_bf16", rc)
    return out


def launch_count() -> int:
    """Kernels libeps_b200.so has launched in this process (eps_launch_count)."""
    f = api().lib.eps_launch_count
    f.restype = C.c_ulonglong
    f.argtypes = []
    return int(f())


def call(name: str, *args):
    """Raw C-ABI call with status check (tensors converted to pointers)."""
    lib = api().lib
    conv = [(_ptr(x) if isinstance(x, torch.Tensor) else x) for x in args]
    rc = getattr(lib, name)(*conv)
    _check(name, rc)
