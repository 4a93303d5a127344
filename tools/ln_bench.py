"""Time LayerNorm fwd / bwd at the ViT-B/16 shape (R = 400*197 rows, d = 768)."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 768
R = int(sys.argv[2]) if len(sys.argv) > 2 else 400 * 197
nores = len(sys.argv) > 3 and sys.argv[3] == "nores"  # post-norm BERT: no residual gradient
dev = torch.device("cuda")
x = torch.randn(R, d, device=dev).bfloat16()
y = torch.empty_like(x)
dy = torch.randn(R, d, device=dev).bfloat16()
dres = torch.randn(R, d, device=dev).bfloat16()
dx = torch.empty_like(x)
gam = torch.randn(d, device=dev)
bet = torch.randn(d, device=dev)
mean = torch.empty(R, device=dev)
rstd = torch.empty(R, device=dev)
dg, db, cs = (torch.zeros(d, device=dev) for _ in range(3))
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def fwd():
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ops.call("eps_layernorm_fwd", x, gam, bet, y, mean, rstd, R, d, C.c_float(1e-6), s)


def bwd():
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ops.call("eps_layernorm_bwd", dy, x, gam, mean, rstd, None if nores else dres, dx, dg, db,
             None if nores else cs, R, d, None, s)


res = {"R": R, "d": d}
for tag, fn, nbytes in (("fwd", fwd, 4 * R * d), ("bwd", bwd, (6 if nores else 8) * R * d)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    # device time of 20 launches captured in one CUDA graph (a ctypes loop is
    # host-bound for the small row counts)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(20):
            fn()
    graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    res[tag + "_us"] = round(ms * 1e3, 1)
    res[tag + "_TBs"] = round(nbytes / ms / 1e9, 2)
print(json.dumps(res))
