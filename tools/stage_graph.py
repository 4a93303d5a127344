"""K = 8 pipeline-stage micro-batch: host-launched vs CUDA-graph replay.

    python tools/stage_graph.py [cfg]      (default vit-b16)

For every stage of the reference planner's 1 x 8 epoch-0 plan (micro-batch
of batch / M samples, schedule.cpp:28-33) this times, on one GPU:
  eager   -- 10 back-to-back micro-batches launched from the host (ctypes ->
             C ABI -> ~40 kernels each), CUDA events around the 10
  host    -- host wall time to enqueue one micro-batch (no sync)
  graph   -- the same micro-batch captured once in a CUDA graph, replayed 10x
and prints one JSON line per stage plus the GPipe iteration bound
(M + K - 1) x slowest stage for both.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03161_b200 import LIB_PATH, configs  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402
from paper_2102_03161_b200.pipeline import StagePlan, microbatch_offsets  # noqa: E402
from paper_2102_03161_b200.planner import Planner  # noqa: E402
from paper_2102_03161_b200.vit import VitExecutor  # noqa: E402


def timed(fn, n, st):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(n):
        fn()
    e.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(e) / n


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "vit-b16"
    g = configs.GEOMETRIES[cfg]
    batch = configs.BATCH[cfg]
    d = Planner(EpsApi(LIB_PATH, "eps_"), configs.scenario(cfg, 8)).begin_epoch(0)
    plan = StagePlan.from_decision(d, g.layers)
    b = microbatch_offsets(batch, plan.M)[0][1]
    dev = torch.device("cuda", 0)
    ex = VitExecutor(g, max_batch=b, device=dev)
    x = torch.randn(b, 3, g.input_image, g.input_image, device=dev)
    y = torch.randint(0, g.classes, (b,), device=dev)
    side = torch.cuda.Stream()
    rows = []
    for s, (g0, g1) in enumerate(plan.spans):
        last = s == plan.K - 1

        def mb():
            ex.stage_forward(x if s == 0 else None, 0, b, g0, g1, 0, front=(s == 0))
            if last:
                ex.stage_head(y, 0, b, batch)
            ex.stage_backward(0, b, g0, g1, 0, cut_out=not last)

        st = torch.cuda.current_stream()
        for _ in range(3):
            mb()
        eager = timed(mb, 10, st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            mb()
        host = (time.perf_counter() - t0) / 10 * 1e3
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side.wait_stream(st)
        with torch.cuda.stream(side):
            mb()  # warm the side stream path (tensor-map caches, attributes)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=side):
            mb()
        torch.cuda.synchronize()
        for _ in range(3):
            graph.replay()
        rep = timed(graph.replay, 10, st)
        rows.append({"stage": s, "span": [g0, g1], "eager_ms": round(eager, 4),
                     "host_enqueue_ms": round(host, 4), "graph_ms": round(rep, 4)})
        print(json.dumps(rows[-1]), flush=True)
        del graph
    slow_e = max(r["eager_ms"] for r in rows)
    slow_g = max(r["graph_ms"] for r in rows)
    n = plan.M + plan.K - 1
    print(json.dumps({"cfg": cfg, "K": plan.K, "M": plan.M, "micro_batch": b,
                      "gpipe_eager_ms": round(n * slow_e, 3), "gpipe_graph_ms": round(n * slow_g, 3),
                      "emulated_samples_per_s_eager": round(batch / (n * slow_e) * 1e3, 1),
                      "emulated_samples_per_s_graph": round(batch / (n * slow_g) * 1e3, 1)}))


if __name__ == "__main__":
    main()
