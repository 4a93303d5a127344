"""Whole training step (K = 1, R = 1): host-launched vs CUDA-graph replay.

    python tools/step_graph.py [cfg ...]      (default: every GPU config)

Builds the same executor / StageRunner as bench.py's N = 1 arm, then times
10 steps (forward + backward + SGD) launched from the host and the same step
captured once in a CUDA graph and replayed 10x, plus the host time to enqueue
one step.  One JSON line per config.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2102_03161_b200 import LIB_PATH, configs  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402
from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport  # noqa: E402
from paper_2102_03161_b200.planner import Planner  # noqa: E402


def timed(fn, n, st):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(n):
        fn()
    e.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(e) / n


def run(cfg):
    dev = torch.device("cuda", 0)
    g = configs.GEOMETRIES[cfg]
    batch = configs.BATCH[cfg]
    d = Planner(EpsApi(LIB_PATH, "eps_"), configs.scenario(cfg, 1)).begin_epoch(0)
    plan = StagePlan.from_decision(d, g.layers)
    ex = bench.make_executor(g, batch, dev)
    runner = StageRunner(ex, 0, 1, Transport(host_staged=False), peer=False)
    runner.set_plan(plan)
    gen = torch.Generator(device=dev).manual_seed(1234)
    inputs, labels = bench.synthetic_inputs(g, batch, gen, dev)

    def step():
        runner.iteration(inputs, labels, batch)
        runner.sync_grads()
        runner.step(lr=1e-3, momentum=0.9)

    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        eager = timed(step, 10, side)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        host = (time.perf_counter() - t0) * 1e3
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            step()
        graph.replay()
        torch.cuda.synchronize()
        replay = timed(graph.replay, 10, side)
    return {"cfg": cfg, "batch": batch, "eager_ms": round(eager, 3), "host_enqueue_ms": round(host, 3),
            "graph_ms": round(replay, 3), "gain": round(eager / replay - 1.0, 4)}


if __name__ == "__main__":
    for c in sys.argv[1:] or ["vit-b16", "vit-b16-cifar100", "bert-base-384", "bert-large-128"]:
        print(json.dumps(run(c)), flush=True)
        torch.cuda.empty_cache()
