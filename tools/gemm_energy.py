"""Energy per launch of the tcgen05 GEMM (NVML total-energy counter).

    python tools/gemm_energy.py [shape ...]      (names from tools/gemm_bench.py)

Each shape runs back to back from a CUDA graph for ~3 s (long enough for the
power limiter to settle); prints mJ per launch, mean power, mean SM clock
and the achieved TFLOP/s.  On a power-capped B200 a kernel's speed follows
its energy per FLOP, so this is the number to compare between variants
(e.g. EPS_GEMM_PAIR=0 / 1).
"""
import json
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03161_b200 import ops  # noqa: E402
from tools.gemm_bench import SHAPES  # noqa: E402


def measure(name, seconds=3.0):
    M, N, K, a_mn, b_mn, epi, split = SHAPES[name]
    dev = torch.device("cuda")
    a = torch.randn((K, M) if a_mn else (M, K), device=dev).bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device=dev).bfloat16()
    f32 = epi in (ops.EPI_STORE_F32, ops.EPI_ACCUM_F32)
    out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    bias = torch.randn(N, device=dev)
    aux = torch.randn(M, N, device=dev).bfloat16() if epi in (2, 3, 4, 7, 8, 9, 10) else None
    colsum = (torch.zeros(N, device=dev) if epi in (4, 10) else
              torch.zeros(M * N // 64, device=dev) if epi == 8 else None)
    kw = dict(a_mn=a_mn, b_mn=b_mn, epilogue=epi, bias=bias, aux=aux, colsum=colsum, split_k=split)
    for _ in range(3):
        ops.gemm(a, b, out, **kw)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    per = 20
    with torch.cuda.graph(graph):
        for _ in range(per):
            ops.gemm(a, b, out, **kw)
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    # settle: run for 1 s first
    t_end = time.time() + 1.0
    while time.time() < t_end:
        graph.replay()
    torch.cuda.synchronize()
    clocks = []
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.05)

    th = threading.Thread(target=sample)
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    s.record()
    n = 0
    t_end = time.time() + seconds
    while time.time() < t_end:
        graph.replay()
        n += per
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    ms = s.elapsed_time(e)
    mj = (e1 - e0) / n
    return dict(name=name, launches=n, us=round(1e3 * ms / n, 2), mJ=round(mj, 3),
                W=round((e1 - e0) / ms, 1), sm_mhz=int(sorted(clocks)[len(clocks) // 2]),
                tflops=round(2.0 * M * N * K * n / ms / 1e9, 1),
                pJ_per_flop=round(mj * 1e9 / (2.0 * M * N * K), 3),
                pair=os.environ.get("EPS_GEMM_PAIR", "1"))


if __name__ == "__main__":
    pynvml.nvmlInit()
    for nm in sys.argv[1:] or ["fwd_fc2", "fwd_fc1_gelu2", "dgrad_qkv", "wgrad_fc2", "square8k"]:
        print(json.dumps(measure(nm)), flush=True)
