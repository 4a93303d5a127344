"""Schema-v1 scenarios for the BASELINE.json configs, plus the model geometry.

`scenario(cfg_id, gpus)` returns the JSON-able scenario dict the decision
plane consumes (same format as the reference's proj/configs/*.json);
`geometry(cfg_id)` returns the real network the B200 executor trains.  The
scenario's explicit ModelSpec is derived from the geometry with the
reference's block arithmetic (model.cpp:107-121), so decision inputs equal
what the reference computes for the same architecture.

Shared settings: 1 node x G GPUs, K0 = G, NVLink-class
bandwidth 9e11 B/s, 180 GB HBM, alpha 1/3, lambda 1/6, synthetic monotone
norms seeded 17, cost/cache rates of the reference's vit_reference.json with
no transition-overhead table.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass
from typing import Dict, List


@dataclass(frozen=True)
class Geometry:
    kind: str              # "vit" | "bert"
    layers: int
    hidden: int
    mlp_dim: int
    heads: int
    tokens: int            # sequence length seen by the blocks
    classes: int           # ViT classes / BERT head outputs
    image: int = 224       # ViT input side (after any upsampling)
    input_image: int = 224  # ViT stored input side (synthetic data shape)
    patch: int = 16
    channels: int = 3
    vocab: int = 30522
    positions: int = 512
    pooler: bool = True
    head: str = "cls"      # BERT head: "cls" (pooled CLS classifier) | "qa" (SQuAD span)

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def _att(d):
    return 3 * (d * d + d) + (d * d + d) + 2 * d


def _mlp(d, f):
    return (d * f + f) + (f * d + d) + 2 * d


def model_spec(g: Geometry) -> Dict[str, List[int]]:
    """ModelSpec arrays for a geometry (model.cpp:107-179 arithmetic)."""
    d, f, L = g.hidden, g.mlp_dim, g.layers
    att = [_att(d)] * L
    mlp = [_mlp(d, f)] * L
    if g.kind == "vit":
        att[0] += d * (g.patch * g.patch * g.channels) + d + d + g.tokens * d
        mlp[-1] += d * g.classes + g.classes
        act0 = g.image * g.image * g.channels * 4
    else:
        att[0] += g.vocab * d + g.positions * d + 2 * d + 2 * d
        mlp[-1] += ((d * d + d) if g.pooler else 0) + d * g.classes + g.classes
        act0 = g.tokens * 8
    act = [g.tokens * d * 4] * (2 * L + 1)
    act[0] = act0
    return {"attention_params": att, "mlp_params": mlp, "activation_bytes": act}


GEOMETRIES: Dict[str, Geometry] = {
    # 1. tiny ViT: 4 blocks, d=128, 4 heads, p=4 on 32x32 -> T=65, 100 classes
    "tiny-vit": Geometry("vit", 4, 128, 512, 4, 65, 100, image=32, input_image=32, patch=4),
    # 2. ViT-B/16 on 224x224 ImageNet-shaped batches (the `vit-b16` preset)
    "vit-b16": Geometry("vit", 12, 768, 3072, 12, 197, 1000),
    # 3. ViT-B/16 on CIFAR-100-shaped 32x32 data, upsampled on device to 224
    "vit-b16-cifar100": Geometry("vit", 12, 768, 3072, 12, 197, 100, input_image=32),
    # 4. BERT-base, seq 384, SQuAD span head (pooler + 2 outputs)
    "bert-base-384": Geometry("bert", 12, 768, 3072, 12, 384, 2, head="qa"),
    # 5. BERT-large, seq 128, 2-class GLUE head (pooler + 2 outputs)
    "bert-large-128": Geometry("bert", 24, 1024, 4096, 16, 128, 2),
    # test-size BERTs (parity tests only; not BASELINE configs)
    "tiny-bert-qa": Geometry("bert", 2, 128, 512, 2, 64, 2, vocab=1000, positions=128,
                             head="qa"),
    "tiny-bert-cls": Geometry("bert", 2, 256, 1024, 4, 48, 3, vocab=500, positions=64),
}

# the five BASELINE.json configs (parity + golden decision fixtures)
BASELINE_CONFIGS = ["tiny-vit", "vit-b16", "vit-b16-cifar100", "bert-base-384", "bert-large-128"]

BATCH = {"tiny-vit": 64, "vit-b16": 400, "vit-b16-cifar100": 320, "bert-base-384": 64,
         "bert-large-128": 64}
EPOCHS = {"tiny-vit": 10, "vit-b16": 10, "vit-b16-cifar100": 10, "bert-base-384": 3,
          "bert-large-128": 3}

_BASE = {
    "schema_version": 1,
    "cluster": {"nodes": 1, "gpus_per_node": 1, "gpu_memory_bytes": 1.8e11,
                "intra_node_bandwidth": 9e11, "inter_node_bandwidth": 9e11},
    "training": {"per_pipeline_batch": 400, "epochs": 10, "iterations_per_epoch": 1600,
                 "alpha": 0.3333333333333333, "lambda_frozen": 0.16666666666666666,
                 "freeze_check_interval": 1},
    "cost_model": {"c_fwd": 9.722222222222221e-12, "backward_ratio": 2.0, "c_update": 1e-11,
                   "per_microbatch_overhead": 0.0008, "allreduce_bucket_bytes": 25000000.0,
                   "comm_latency": 1e-05, "transition_overheads": {}},
    "cache": {"policy": "auto", "host_bandwidth": 3050000000.0, "disk_bandwidth": 6000000000.0,
              "host_capacity_bytes": 64000000000.0, "window_batches": 64, "block_batches": 8,
              "read_latency": 0.0},
    "grad_norms": {"kind": "synthetic", "profile": "monotone-converging", "seed": 17,
                   "switchover_epoch": 2},
    "features": {"freeze": True, "autopipe": True, "autodp": True, "autocache": True},
    "freeze_only_slowdown": 0.05,
    "dp_message_latency": 0.0,
    "balance_criterion": "normalized-stddev",
    "integer_microbatches": False,
    "seed": 17,
}


def scenario(cfg_id: str, gpus: int = 1, **overrides) -> dict:
    """Schema-v1 scenario dict for BASELINE config `cfg_id` on 1 node x `gpus`."""
    g = GEOMETRIES[cfg_id]
    s = copy.deepcopy(_BASE)
    s["name"] = f"{cfg_id}-g{gpus}"
    if cfg_id == "vit-b16":
        s["model"] = {"preset": "vit-b16"}
    else:
        s["model"] = dict(name=cfg_id, bytes_per_param=4, **model_spec(g))
    s["cluster"]["gpus_per_node"] = gpus
    s["initial_pipeline_length"] = gpus
    s["training"]["per_pipeline_batch"] = BATCH[cfg_id]
    s["training"]["epochs"] = EPOCHS[cfg_id]
    for k, v in overrides.items():
        if isinstance(v, dict) and isinstance(s.get(k), dict):
            s[k].update(v)
        else:
            s[k] = v
    return s


def no_freeze(s: dict) -> dict:
    """The reference's `baseline` rung: all feature flags off (runner.cpp:312)."""
    s = copy.deepcopy(s)
    s["features"] = {"freeze": False, "autopipe": False, "autodp": False, "autocache": False}
    return s
