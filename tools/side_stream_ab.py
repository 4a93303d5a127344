"""In-process A/B of the side-stream weight gradients (eps_vit_set_side_stream):
whole-model b400 steps and one K = 8 stage's b18 micro-batch, alternating."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402
from paper_2102_03161_b200.configs import GEOMETRIES  # noqa: E402
from paper_2102_03161_b200.vit import VitExecutor  # noqa: E402

g = GEOMETRIES["vit-b16"]
res = {}
for B, tag in ((400, "b400"), (18, "b18")):
    ex = VitExecutor(g, max_batch=B)
    x = torch.randn(B, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (B,), device="cuda")
    lib = ops.api().lib
    f = lib.eps_vit_set_side_stream
    f.restype = C.c_int
    it = 8 if B == 400 else 40

    def timed(on):
        f(ex.h, on)
        for _ in range(3):
            ex.train_step(x, y)
            ex.sgd(0, 1e-3)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(it):
            ex.train_step(x, y)
            ex.sgd(0, 1e-3)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / it

    r = {0: [], 1: []}
    for _ in range(4):
        for on in (0, 1):
            r[on].append(timed(on))
    res[tag] = {"off_ms": sorted(round(v, 3) for v in r[0]), "on_ms": sorted(round(v, 3) for v in r[1])}
    del ex
    torch.cuda.empty_cache()
print(json.dumps(res))
