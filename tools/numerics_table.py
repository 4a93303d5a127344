"""Measured numerics-parity table (device vs the CPU oracles).

    python tools/numerics_table.py [OUT_PREFIX]   -> OUT_PREFIX.json / .md

For every case: loss vs FP32, and per gradient tensor / per residual-stream
activation X[l] / per-layer gradient norm the three distances of
tests/parity_lib.py (kernel = device vs BF16_STORAGE, vs_fp32, intrinsic =
BF16_STORAGE vs FP32), worst per tensor class; then 10-step SGD loss
trajectories device vs the fp32 oracle.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.parity_lib import run_case, trajectory  # noqa: E402

CASES = [("tiny-vit", 16, 0, 1), ("tiny-vit", 16, 2, 3), ("vit-b16", 8, 0, 1),
         ("vit-b16", 8, 6, 2), ("vit-b16-cifar100", 4, 4, 1), ("tiny-bert-qa", 4, 0, 1),
         ("tiny-bert-cls", 6, 1, 3), ("bert-base-384", 4, 0, 1), ("bert-base-384", 4, 6, 2),
         ("bert-large-128", 8, 0, 1), ("bert-large-128", 8, 12, 2)]
TRAJ = [("vit-b16", 8, 0, 5e-4), ("vit-b16", 8, 6, 1e-3), ("bert-base-384", 4, 0, 5e-4),
        ("bert-large-128", 8, 0, 1e-3)]


def tensor_class(name: str) -> str:
    if name.endswith("bias") and "LayerNorm" not in name and "norm" not in name:
        return "bias"
    if "norm" in name.lower():
        return "layernorm"
    return "matrix/embedding"


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/numerics"
    torch.set_num_threads(os.cpu_count() or 8)
    rows, md = [], ["| case | loss dev / fp32 (rel) | class | kernel | vs fp32 (worst tensor) | "
                    "intrinsic | self noise |", "|---|---|---|---|---|---|---|"]
    for cfg, b, lf, m in CASES:
        t = time.time()
        c = run_case(cfg, b, lf, m, self_noise=True)
        rec = {"cfg": cfg, "batch": b, "l_frozen": lf, "micro": m, "loss": c.loss,
               "grads": c.grads, "acts": c.acts, "norms": c.norms, "zero": c.zero_tensors,
               "frozen_nonzero": c.frozen_nonzero, "seconds": time.time() - t}
        rows.append(rec)
        lrel = abs(c.loss["dev"] - c.loss["fp32"]) / abs(c.loss["fp32"])
        classes = {}
        for n, v in c.grads.items():
            k = tensor_class(n)
            for met in ("kernel", "vs_fp32", "intrinsic", "self_noise"):
                classes.setdefault(k, {}).setdefault(met, (0.0, ""))
                if v[met] > classes[k][met][0]:
                    classes[k][met] = (v[met], n)
        classes["activations X[l]"] = {met: (max(a[met] for a in c.acts), "")
                                       for met in ("kernel", "vs_fp32", "intrinsic",
                                                   "self_noise")}
        nn = [x for x in c.norms if "kernel" in x]
        classes["layer grad norms"] = {met: (max(x[met] for x in nn), "")
                                       for met in ("kernel", "vs_fp32", "intrinsic")}
        classes["layer grad norms"]["self_noise"] = (float("nan"), "")
        label = f"{cfg} b{b} Lf{lf} M{m}"
        for k, v in classes.items():
            md.append(f"| {label} | {lrel:.2e} | {k} | {v['kernel'][0]:.4f} | "
                      f"{v['vs_fp32'][0]:.4f} {v['vs_fp32'][1]} | {v['intrinsic'][0]:.4f} | "
                      f"{v['self_noise'][0]:.4f} |")
            label = ""
        if c.zero_tensors:
            md.append(f"|  |  | zero by math: norm dev / norm bf16-emu | "
                      f"{max(c.zero_tensors.values()):.3f} {list(c.zero_tensors)} |  |  |  |")
        print(label or cfg, "done", round(time.time() - t, 1), "s", flush=True)
    trajs = []
    md += ["", "| trajectory | step losses device | fp32 oracle | max rel |", "|---|---|---|---|"]
    for cfg, b, lf, lr in TRAJ:
        dev, ref = trajectory(cfg, b, 10, lr, l_frozen=lf)
        worst = max(abs(a - r) / abs(r) for a, r in zip(dev, ref))
        trajs.append({"cfg": cfg, "batch": b, "l_frozen": lf, "lr": lr, "dev": dev, "fp32": ref,
                      "max_rel": worst})
        md.append(f"| {cfg} b{b} Lf{lf} lr{lr} | {', '.join(f'{v:.4f}' for v in dev)} | "
                  f"{', '.join(f'{v:.4f}' for v in ref)} | {worst:.2e} |")
        print("traj", cfg, lf, worst, flush=True)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out + ".json", "w") as f:
        json.dump({"cases": rows, "trajectories": trajs,
                   "gpu": torch.cuda.get_device_name(0)}, f, indent=1)
    with open(out + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
