"""Time the attention kernels at the ViT-B/16 / BERT shapes (CUDA events)."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402

SHAPES = {"vit-b16": (400, 197, 12), "bert-base-384": (64, 384, 12),
          "bert-large-128": (64, 128, 16)}


def run(name, B, T, H, iters=10):
    dev = torch.device("cuda")
    D = H * 64
    qkv = torch.randn(B * T, 3 * D, device=dev).bfloat16()
    out = torch.empty(B * T, D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(B, H, T, device=dev)
    dout = torch.randn(B * T, D, device=dev).bfloat16()
    dqkv = torch.empty_like(qkv)
    dbias = torch.zeros(3 * D, device=dev)
    dsum = torch.empty(B * H * T, device=dev)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    sc = C.c_float(64 ** -0.5)

    def fwd():
        ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, 64, sc, s)

    def bwd():
        ops.call("eps_attn_bwd_ws", qkv, out, dout, lse, dqkv, dbias, dsum, B, T, H, 64, sc, s)

    res = {"name": name}
    flops = 4.0 * B * T * T * D
    for tag, fn, fl in (("fwd", fwd, flops), ("bwd", bwd, 2 * flops)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / iters
        res[tag + "_ms"] = round(ms, 4)
        res[tag + "_tflops"] = round(fl / ms / 1e9, 1)
    return res


if __name__ == "__main__":
    for n in sys.argv[1:] or list(SHAPES):
        print(json.dumps(run(n, *SHAPES[n])), flush=True)
