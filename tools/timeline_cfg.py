"""Device timeline of one K = 1 training step of any GPU config (CUPTI via
torch.profiler), through the same StageRunner path as bench.py.

    python tools/timeline_cfg.py CFG [n_list]

Prints the step span / busy time, per-kernel-template totals, and the first
n_list kernels of the step in launch order with their durations (the
embedding and layer-0 forward, then the tail of the backward).
"""
import json
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2102_03161_b200 import LIB_PATH, configs  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402
from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport  # noqa: E402
from paper_2102_03161_b200.planner import Planner  # noqa: E402


def short(name):
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("eps_k::", "").replace("attn_tc::", "")
    return n[:70]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "bert-large-128"
    n_list = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    dev = torch.device("cuda", 0)
    g = configs.GEOMETRIES[cfg]
    batch = configs.BATCH[cfg]
    d = Planner(EpsApi(LIB_PATH, "eps_"), configs.scenario(cfg, 1)).begin_epoch(0)
    runner = StageRunner(bench.make_executor(g, batch, dev), 0, 1,
                         Transport(host_staged=False), peer=False)
    runner.set_plan(StagePlan.from_decision(d, g.layers))
    gen = torch.Generator(device=dev).manual_seed(1234)
    inputs, labels = bench.synthetic_inputs(g, batch, gen, dev)

    def step():
        runner.iteration(inputs, labels, batch)
        runner.sync_grads()
        runner.step(lr=1e-3, momentum=0.9)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        step()
    e.record()
    torch.cuda.synchronize()
    print(f"{cfg}: CUDA events over 10 steps: {a.elapsed_time(e) / 10:.3f} ms per step")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            step()
        torch.cuda.synchronize()
    os.makedirs("gpurun_out", exist_ok=True)
    path = f"gpurun_out/timeline_{cfg}.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")],
                key=lambda e: e["ts"])
    ks = ks[len(ks) // 2:]  # second step
    t0, t1 = ks[0]["ts"], ks[-1]["ts"] + ks[-1]["dur"]
    busy = sum(e["dur"] for e in ks)
    print(f"{cfg}: step span {(t1 - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, "
          f"{len(ks)} kernels")
    by = defaultdict(lambda: [0, 0.0])
    for e in ks:
        k = short(e["name"])
        by[k][0] += 1
        by[k][1] += e["dur"]
    for k, (n, dd) in sorted(by.items(), key=lambda kv: -kv[1][1])[:20]:
        print(f"  {k:70s} {n:4d} {dd / 1e3:8.3f} ms")
    print("launch order (first kernels of the step):")
    for e in ks[:n_list]:
        print(f"  {e['dur']:8.1f} us  {short(e['name'])}")


if __name__ == "__main__":
    main()
