"""Host binding of the AutoCache disk tier (C ABI eps_disk_tier_*,
csrc/runtime/disk_tier.cpp).

The reference models a disk tier behind the host tier: the host holds a
sliding window of `window_batches` batches, refilled `block_batches` at a
time from disk while the epoch's batches are consumed in order, and a batch
whose block has not arrived stalls (CacheTierSim, autocache.cpp:69-150;
CacheTierParams autocache.hpp:11-20).  `DiskTier` runs that window for real:
a node-wide backing file of cached sample rows, a page-locked host window,
native I/O threads, and per-batch acquire / release.  The trainer copies an
acquired batch into HBM with one 2D copy (rows `stride` bytes apart in the
window) and the executor gathers from there.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import torch

from . import LIB_PATH
from .capi import EpsApi

STATS = ("bytes_read", "read_busy_s", "stall_s", "max_resident_bytes", "prefetches",
         "evictions", "bytes_written", "direct")

_lib = None


def _api():
    global _lib
    if _lib is None:
        lib = EpsApi(LIB_PATH, "eps_").lib
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        for n, args in {
                "eps_disk_tier_open": [C.c_char_p, i64, i64, i64, i32, i32, i32, i32,
                                       C.POINTER(vp)],
                "eps_disk_tier_close": [vp],
                "eps_disk_tier_info": [vp, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32),
                                       C.POINTER(vp)],
                "eps_disk_tier_write": [vp, vp, i64, vp, i64],
                "eps_disk_tier_begin_epoch": [vp, vp, i64, vp, i64],
                "eps_disk_tier_acquire": [vp, i64, C.POINTER(vp), C.POINTER(i64),
                                          C.POINTER(C.c_double)],
                "eps_disk_tier_release": [vp, i64],
                "eps_disk_tier_stats": [vp, C.POINTER(C.c_double)]}.items():
            getattr(lib, n).argtypes = args
            getattr(lib, n).restype = i32
        _lib = lib
    return _lib


class DiskTierError(RuntimeError):
    pass


def _check(name: str, rc: int):
    if rc != 0:
        raise DiskTierError(f"{name} failed with status {rc}")


class DiskTier:
    """One backing file of `rows` cached samples of `row_bytes` each."""

    def __init__(self, path: str, rows: int, row_bytes: int, batch_rows: int, *,
                 block_batches: int = 8, window_batches: int = 64, threads: int = 8,
                 create: bool = True):
        self.lib = _api()
        self.path, self.rows, self.row_bytes, self.batch_rows = path, rows, row_bytes, batch_rows
        h = C.c_void_p()
        _check("eps_disk_tier_open",
               self.lib.eps_disk_tier_open(path.encode(), rows, row_bytes, batch_rows,
                                           block_batches, window_batches, threads, int(create),
                                           C.byref(h)))
        self.h = h
        stride, direct, wb, win = C.c_int64(), C.c_int(), C.c_int(), C.c_void_p()
        _check("eps_disk_tier_info", self.lib.eps_disk_tier_info(
            self.h, C.byref(stride), C.byref(direct), C.byref(wb), C.byref(win)))
        self.stride, self.direct, self.window_blocks = stride.value, bool(direct.value), wb.value
        self._order: Optional[torch.Tensor] = None

    def write(self, ids: torch.Tensor, rows: torch.Tensor):
        """rows: host tensor [n, >= row_bytes] (any dtype), row i -> sample ids[i]."""
        ids = ids.to(torch.int64).contiguous().cpu()
        assert rows.device.type == "cpu" and rows.is_contiguous()
        stride = rows.stride(0) * rows.element_size()
        _check("eps_disk_tier_write", self.lib.eps_disk_tier_write(
            self.h, C.c_void_p(ids.data_ptr()), ids.numel(), C.c_void_p(rows.data_ptr()),
            stride))

    def begin_epoch(self, order: Sequence[int] | torch.Tensor,
                    batches: Optional[Sequence[tuple]] = None):
        """order: the epoch's sample ids in consumption order; batches: optional
        [(offset, size)] into it (default: batch_rows-row batches)."""
        o = torch.as_tensor(order, dtype=torch.int64).contiguous().cpu()
        self._order = o  # kept alive while the epoch's reads run
        offs, nb = None, 0
        if batches is not None:
            offs = torch.tensor([b[0] for b in batches] + [o.numel()], dtype=torch.int64)
            nb = len(batches)
        _check("eps_disk_tier_begin_epoch", self.lib.eps_disk_tier_begin_epoch(
            self.h, C.c_void_p(o.data_ptr()), o.numel(),
            C.c_void_p(offs.data_ptr() if offs is not None else 0), nb))

    def acquire(self, batch: int):
        """(host address of the batch's first row, rows, stall seconds)."""
        p, n, st = C.c_void_p(), C.c_int64(), C.c_double()
        _check("eps_disk_tier_acquire", self.lib.eps_disk_tier_acquire(
            self.h, batch, C.byref(p), C.byref(n), C.byref(st)))
        return p.value, n.value, st.value

    def batch_view(self, batch: int) -> tuple[torch.Tensor, float]:
        """Acquire `batch` and view its rows as uint8 [n, stride] (host, no copy)."""
        addr, n, st = self.acquire(batch)
        buf = (C.c_uint8 * (n * self.stride)).from_address(addr)
        return torch.frombuffer(buf, dtype=torch.uint8).view(n, self.stride), st

    def release(self, batch: int):
        _check("eps_disk_tier_release", self.lib.eps_disk_tier_release(self.h, batch))

    def stats(self) -> dict:
        out = (C.c_double * len(STATS))()
        _check("eps_disk_tier_stats", self.lib.eps_disk_tier_stats(self.h, out))
        return dict(zip(STATS, list(out)))

    def close(self):
        if self.h is not None:
            self.lib.eps_disk_tier_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
