"""In-process A/B of the ViT-B/16 train step: alternate configuration A and B
every few steps (so clock / power drift hits both alike) and compare medians.

    python tools/ab_steps.py gemm_pair      (A: single-CTA GEMM tiles, B: CTA pairs)
"""
import ctypes as C
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402
from paper_2102_03161_b200.configs import GEOMETRIES  # noqa: E402
from paper_2102_03161_b200.vit import VitExecutor  # noqa: E402

knob = sys.argv[1] if len(sys.argv) > 1 else "gemm_pair"
lib = ops.api().lib
SET = {"gemm_pair": lambda on: lib.eps_gemm_pair_mode(C.c_int(1 if on else 0))}[knob]
B = 400
g = GEOMETRIES["vit-b16"]
ex = VitExecutor(g, max_batch=B)
x = torch.randn(B, 3, 224, 224, device="cuda")
y = torch.randint(0, 1000, (B,), device="cuda")


def steps(n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        ex.train_step(x, y)
        ex.sgd(0, 1e-3)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res = {False: [], True: []}
for on in (False, True):
    SET(on)
    steps(2)
for _ in range(8):
    for on in (False, True):
        SET(on)
        res[on].append(steps(3))
ma, mb = statistics.median(res[False]), statistics.median(res[True])
print(f"{knob}: A(off) median {ma:.2f} ms/step {sorted(round(v, 2) for v in res[False])}")
print(f"{knob}: B(on)  median {mb:.2f} ms/step {sorted(round(v, 2) for v in res[True])}")
print(f"{knob}: B/A = {mb / ma:.4f}  ({B / mb * 1e3:.0f} vs {B / ma * 1e3:.0f} samples/s)")
