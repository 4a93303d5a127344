"""Device timeline of one ViT-B/16 step (torch.profiler / CUPTI): kernel
durations, idle gaps between consecutive kernels, and the largest gaps.

    python tools/timeline.py [batch]
"""
import json
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200.configs import GEOMETRIES  # noqa: E402
from paper_2102_03161_b200.vit import VitExecutor  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 400
g = GEOMETRIES["vit-b16"]
ex = VitExecutor(g, max_batch=B)
x = torch.randn(B, 3, 224, 224, device="cuda")
y = torch.randint(0, 1000, (B,), device="cuda")
for _ in range(3):
    ex.train_step(x, y)
    ex.sgd(0, 1e-3)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        ex.train_step(x, y)
        ex.sgd(0, 1e-3)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/timeline.json")
ev = json.load(open("gpurun_out/timeline.json"))["traceEvents"]
ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")],
            key=lambda e: e["ts"])
half = len(ks) // 2
ks = ks[half:]  # second step only
t0, t1 = ks[0]["ts"], ks[-1]["ts"] + ks[-1]["dur"]
busy = sum(e["dur"] for e in ks)
gaps = []
for a, b in zip(ks, ks[1:]):
    gaps.append((b["ts"] - (a["ts"] + a["dur"]), a["name"][:60], b["name"][:60]))
print(f"step span {(t1 - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, "
      f"idle {sum(max(0, g0) for g0, _, _ in gaps) / 1e3:.2f} ms over {len(gaps)} boundaries")
by = defaultdict(lambda: [0, 0.0])
for e in ks:
    k = e["name"].split("<")[0].split("(")[0][-40:]
    by[k][0] += 1
    by[k][1] += e["dur"]
for k, (n, d) in sorted(by.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:40s} {n:4d} {d / 1e3:8.3f} ms")
gsum = defaultdict(lambda: [0, 0.0])
for g0, a, b in gaps:
    key = a.split("<")[0].split("(")[0][-30:] + " -> " + b.split("<")[0].split("(")[0][-30:]
    gsum[key][0] += 1
    gsum[key][1] += max(0, g0)
print("gap totals by boundary kind:")
for k, (n, d) in sorted(gsum.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"  {k:64s} {n:4d} {d / 1e3:7.3f} ms  ({d / max(n, 1):.1f} us each)")
