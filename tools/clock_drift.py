"""SM clock, power and step time in 5-step windows over the first ~1.5-3 s of
training (NVML), for one GPU config:

    python tools/clock_drift.py CFG

Shows the board reaching its ~1000 W limit and the SM clock it settles at.
"""
import os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2102_03161_b200 import LIB_PATH, configs
from paper_2102_03161_b200.capi import EpsApi
from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport
from paper_2102_03161_b200.planner import Planner
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
cfg = sys.argv[1]
dev = torch.device("cuda", 0)
g = configs.GEOMETRIES[cfg]; batch = configs.BATCH[cfg]
d = Planner(EpsApi(LIB_PATH, "eps_"), configs.scenario(cfg, 1)).begin_epoch(0)
runner = StageRunner(bench.make_executor(g, batch, dev), 0, 1, Transport(host_staged=False), peer=False)
runner.set_plan(StagePlan.from_decision(d, g.layers))
gen = torch.Generator(device=dev).manual_seed(1234)
inputs, labels = bench.synthetic_inputs(g, batch, gen, dev)
def step():
    runner.iteration(inputs, labels, batch); runner.sync_grads(); runner.step(lr=1e-3, momentum=0.9)
t0 = time.time()
out = []
for rep in range(12):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): step()
    e.record(); torch.cuda.synchronize()
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    mclk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    out.append(f"{time.time()-t0:.1f}s {a.elapsed_time(e)/5:.2f}ms sm{clk} mem{mclk} {pw:.0f}W")
print(cfg, " | ".join(out))
