"""Host binding of the communicator plane (C ABI eps_comm_* / eps_allreduce*
/ eps_p2p_* / eps_broadcast in libeps_b200.so, csrc/runtime/comm.cpp).

`Comm` wraps one NCCL communicator the library owns.  torch.distributed is
used only as the out-of-band channel that hands rank 0's NCCL unique id to
the other ranks; every collective and point-to-point transfer of the
training path goes through the library on the caller's CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import ops

DT = {torch.float32: 0, torch.float64: 1, torch.bfloat16: 2, torch.uint8: 3, torch.int64: 4}
OP_SUM, OP_AVG, OP_MAX = 0, 1, 2


def _lib():
    lib = ops.api().lib
    vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
    for name, args in {"eps_comm_version": [vp], "eps_comm_unique_id": [vp],
                       "eps_comm_world_init": [vp, i32, i32, vp],
                       "eps_comm_split": [vp, i32, i32, vp], "eps_comm_free": [vp],
                       "eps_comm_rank": [vp, vp, vp],
                       "eps_allreduce": [vp, vp, i64, i32, i32, vp],
                       "eps_allreduce_bucket": [vp, vp, i64, i32, vp],
                       "eps_broadcast": [vp, vp, i64, i32, vp],
                       "eps_p2p_send": [vp, vp, i64, i32, vp],
                       "eps_p2p_recv": [vp, vp, i64, i32, vp],
                       "eps_comm_group_start": [], "eps_comm_group_end": []}.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    return lib


def _check(name: str, rc: int):
    if rc != 0:
        lib = ops.api().lib
        lib.eps_last_error.restype = C.c_char_p
        raise RuntimeError(f"{name} failed ({rc}): {lib.eps_last_error().decode()}")


def nccl_version() -> int:
    v = C.c_int()
    _check("eps_comm_version", _lib().eps_comm_version(C.byref(v)))
    return v.value


def unique_id() -> bytes:
    b = (C.c_char * 128)()
    _check("eps_comm_unique_id", _lib().eps_comm_unique_id(b))
    return bytes(b)


def _stream(stream) -> C.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


class Comm:
    """One eps_comm_t (NCCL communicator); rank / size within it."""

    def __init__(self, handle: int):
        self.lib = _lib()
        self.h = C.c_void_p(handle)
        r, n = C.c_int(), C.c_int()
        _check("eps_comm_rank", self.lib.eps_comm_rank(self.h, C.byref(r), C.byref(n)))
        self.rank, self.size = r.value, n.value

    @staticmethod
    def world(rank: int, world: int, uid: Optional[bytes] = None) -> "Comm":
        """World communicator; without `uid`, rank 0 creates the id and
        torch.distributed's default group carries it to the other ranks."""
        if uid is None:
            import torch.distributed as dist
            box = [unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(box, src=0)
            uid = box[0]
        h = C.c_void_p()
        _check("eps_comm_world_init",
               _lib().eps_comm_world_init((C.c_char * 128).from_buffer_copy(uid), world, rank,
                                          C.byref(h)))
        return Comm(h.value)

    def split(self, color: int, key: int) -> Optional["Comm"]:
        """Collective over this communicator: members of `color` (>= 0) get a
        communicator ordered by `key`; color < 0 returns None."""
        h = C.c_void_p()
        _check("eps_comm_split", self.lib.eps_comm_split(self.h, color, key, C.byref(h)))
        return Comm(h.value) if h.value else None

    def free(self):
        if self.h is not None and self.h.value:
            _check("eps_comm_free", self.lib.eps_comm_free(self.h))
        self.h = None

    def all_reduce(self, t: torch.Tensor, op: int = OP_SUM, stream=None):
        _check("eps_allreduce", self.lib.eps_allreduce(self.h, C.c_void_p(t.data_ptr()),
                                                       t.numel(), DT[t.dtype], op,
                                                       _stream(stream)))

    def all_reduce_bucket(self, grads: torch.Tensor, average: bool = True, stream=None):
        assert grads.dtype == torch.float32 and grads.is_contiguous()
        _check("eps_allreduce_bucket",
               self.lib.eps_allreduce_bucket(self.h, C.c_void_p(grads.data_ptr()), grads.numel(),
                                             int(average), _stream(stream)))

    def broadcast(self, t: torch.Tensor, root: int, stream=None):
        _check("eps_broadcast", self.lib.eps_broadcast(self.h, C.c_void_p(t.data_ptr()),
                                                       t.numel() * t.element_size(), root,
                                                       _stream(stream)))

    def send(self, t: torch.Tensor, peer: int, stream=None):
        _check("eps_p2p_send", self.lib.eps_p2p_send(self.h, C.c_void_p(t.data_ptr()),
                                                     t.numel() * t.element_size(), peer,
                                                     _stream(stream)))

    def recv(self, t: torch.Tensor, peer: int, stream=None):
        _check("eps_p2p_recv", self.lib.eps_p2p_recv(self.h, C.c_void_p(t.data_ptr()),
                                                     t.numel() * t.element_size(), peer,
                                                     _stream(stream)))

    def group_start(self):
        _check("eps_comm_group_start", self.lib.eps_comm_group_start())

    def group_end(self):
        _check("eps_comm_group_end", self.lib.eps_comm_group_end())
