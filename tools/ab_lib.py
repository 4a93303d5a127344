"""In-process-style A/B of two library builds: alternate processes? No --
alternate runs of tools/ab_steps-like timing in two subprocesses is noisy, so
this loads each build in its own subprocess per round and interleaves rounds.

    python tools/ab_lib.py BASE.so [rounds]
"""
import json
import os
import statistics
import subprocess
import sys

base = sys.argv[1]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
code = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2102_03161_b200.configs import GEOMETRIES
from paper_2102_03161_b200.vit import VitExecutor
g = GEOMETRIES["vit-b16"]; B = 400
ex = VitExecutor(g, max_batch=B)
x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
for _ in range(3): ex.train_step(x, y); ex.sgd(0, 1e-3)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(8): ex.train_step(x, y); ex.sgd(0, 1e-3)
b.record(); torch.cuda.synchronize()
print(json.dumps(a.elapsed_time(b) / 8))
'''
res = {"base": [], "new": []}
for _ in range(rounds):
    for tag in ("base", "new"):
        env = dict(os.environ)
        if tag == "base":
            env["EPS_LIB_PATH"] = os.path.abspath(base)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        res[tag].append(float(out.stdout.strip().splitlines()[-1]))
mb, mn = statistics.median(res["base"]), statistics.median(res["new"])
print(f"base {mb:.2f} ms/step {sorted(round(v, 2) for v in res['base'])}")
print(f"new  {mn:.2f} ms/step {sorted(round(v, 2) for v in res['new'])}")
print(f"new/base = {mn / mb:.4f}")
