"""Native single-GPU training loop (csrc/runtime/trainer.cpp) behind the C ABI.

`NativeTrainer` runs the same epoch loop as `trainer.Trainer` for a 1 x 1
cluster -- EpochPlanner decisions from device gradient norms, redistribute
shards, AutoCache modes (gather / boundary move / trailing boundary), the
ragged last iteration -- with the host loop in C++ (eps_trainer_*): Python
only builds the scenario handle and reads the per-epoch rows.  Multi-rank
runs keep trainer.Trainer (pipeline.py choreography over the same executor).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import torch

from . import LIB_PATH, ops
from .capi import EpsApi, Scenario
from .configs import Geometry
from .trainer import EpochResult
from . import bert as _bert
from .vit import geom_array as _vit_geom


class CTrainEpoch(C.Structure):
    _fields_ = [("epoch", C.c_int), ("l_frozen", C.c_int), ("pipeline_length", C.c_int),
                ("replica_width", C.c_int), ("micro_batches", C.c_int),
                ("cache_enabled", C.c_int), ("cache_moved", C.c_int), ("cache_mode", C.c_int),
                ("iterations", C.c_int), ("epoch_time_s", C.c_double),
                ("iteration_time_s", C.c_double), ("throughput_sps", C.c_double),
                ("samples", C.c_double), ("mean_loss", C.c_double),
                ("cache_transition_time_s", C.c_double)]


class NativeTrainer:
    """One-GPU PipeTransformer run with the epoch loop in C++ (ViT or BERT).

    init_params: fp32 flat parameters in the executor layout (CPU or CUDA
    tensor; None = the library's seeded init); images / labels: CUDA dataset
    tensors (ViT fp32 [N, C, H, W] / BERT int64 [2, N, T] token + segment ids;
    labels int64 [N], SQuAD head [2, N]) or None for the library's seeded
    synthetic data."""

    def __init__(self, scenario: dict, geometry: Geometry, *, iterations_per_epoch: int,
                 seed: int = 17, lr: float = 1e-3, momentum: float = 0.9,
                 device_norms: bool = True, init_params: Optional[torch.Tensor] = None,
                 images: Optional[torch.Tensor] = None, labels: Optional[torch.Tensor] = None):
        kind = 0 if geometry.kind == "vit" else 1
        self.api = EpsApi(LIB_PATH, "eps_")
        self.scenario = Scenario(self.api, scenario)
        self.g = geometry
        self.layers = geometry.layers
        lib = ops.api().lib
        for n, res, args in [
                ("eps_trainer_create", C.c_int,
                 [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.c_float, C.c_float,
                  C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
                ("eps_trainer_run_epoch", C.c_int,
                 [C.c_void_p, C.c_int, C.POINTER(CTrainEpoch), C.c_void_p]),
                ("eps_trainer_destroy", None, [C.c_void_p])]:
            f = getattr(lib, n)
            f.restype, f.argtypes = res, args
        self.lib = lib
        batch = int(scenario["training"]["per_pipeline_batch"])
        hp = None
        if init_params is not None:
            self._params = init_params.detach().float().cpu().contiguous()
            hp = C.c_void_p(self._params.data_ptr())
        for t in (images, labels):
            if t is not None and not t.is_cuda:
                raise TypeError("images / labels must be CUDA tensors")
        h = C.c_void_p()
        geom = (_vit_geom if kind == 0 else _bert.geom_array)(geometry, batch)
        rc = lib.eps_trainer_create(self.scenario.h, kind, geom,
                                    iterations_per_epoch, seed, lr, momentum, int(device_norms),
                                    hp, C.c_void_p(images.data_ptr()) if images is not None else None,
                                    C.c_void_p(labels.data_ptr()) if labels is not None else None,
                                    C.byref(h))
        if rc != 0:
            raise RuntimeError(f"eps_trainer_create failed ({rc}): {self._err()}")
        self.h = h

    def _err(self) -> str:
        f = self.lib.eps_last_error
        f.restype = C.c_char_p
        return (f() or b"").decode()

    def run_epoch(self, epoch: int) -> EpochResult:
        r = CTrainEpoch()
        norms = (C.c_double * self.layers)()
        rc = self.lib.eps_trainer_run_epoch(self.h, epoch, C.byref(r), norms)
        if rc != 0:
            raise RuntimeError(f"eps_trainer_run_epoch failed ({rc}): {self._err()}")
        return EpochResult(r.epoch, r.l_frozen, r.pipeline_length, r.replica_width,
                           r.micro_batches, r.iteration_time_s, r.epoch_time_s,
                           r.throughput_sps, bool(r.cache_enabled), bool(r.cache_moved), 0.0,
                           r.mean_loss, list(norms), cache_transition_time_s=r.cache_transition_time_s,
                           samples=int(r.samples))

    def run(self, epochs: int) -> List[EpochResult]:
        return [self.run_epoch(e) for e in range(epochs)]

    def close(self):
        if getattr(self, "h", None):
            self.lib.eps_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()
