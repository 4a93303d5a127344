"""Host launch overhead of one small-batch ViT-B/16 step (the per-micro-batch
regime of a K=8 pipeline: 17 samples) vs. the device time of its kernels."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200.configs import GEOMETRIES  # noqa: E402
from paper_2102_03161_b200.vit import VitExecutor  # noqa: E402

g = GEOMETRIES["vit-b16"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 17
ex = VitExecutor(g, max_batch=B)
x = torch.randn(B, 3, 224, 224, device="cuda")
y = torch.randint(0, 1000, (B,), device="cuda")
for _ in range(3):
    ex.train_step(x, y)
    ex.sgd(0, 1e-3)
torch.cuda.synchronize()
n = 20
t0 = time.perf_counter()
for _ in range(n):
    ex.train_step(x, y)
    ex.sgd(0, 1e-3)
t_host = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
t_wall = (time.perf_counter() - t0) / n
ex.timing(True)
ex.train_step(x, y)
ex.sgd(0, 1e-3)
torch.cuda.synchronize()
c = ex.timing_read()
ex.timing(False)
dev = sum(v["ms"] for v in c.values())
launches = sum(v["launches"] for v in c.values())
print(f"batch {B}: host enqueue {t_host*1e3:.2f} ms/step, wall {t_wall*1e3:.2f} ms/step, "
      f"device kernels {dev:.2f} ms ({launches} launches, {t_host*1e6/launches:.1f} us/launch host)")
