"""Where the GEMM's roles wait (eps_gemm_prof counters), per ViT-B/16 shape.

    python tools/gemm_waits.py [shape ...]      (on a B200; shapes of gemm_bench.py)
Prints, as fractions of the MMA warp's span: its waits for a free accumulator
(epilogue-bound), for operand stages (TMA / L2 / HBM-bound), the producer's
slot waits, and epilogue warp 0's accumulator-full / store-slot waits.
"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from gemm_bench import SHAPES  # noqa: E402
from paper_2102_03161_b200 import ops  # noqa: E402


def waits(name, M, N, K, a_mn, b_mn, epi, split, iters=5):
    dev = torch.device("cuda")
    a = torch.randn((K, M) if a_mn else (M, K), device=dev).bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device=dev).bfloat16()
    f32 = epi in (ops.EPI_STORE_F32, ops.EPI_ACCUM_F32)
    out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    bias = torch.randn(N, device=dev)
    aux = torch.randn(M, N, device=dev).bfloat16() if epi in (2, 3, 4, 7, 8, 9, 10) else None
    colsum = (torch.zeros(N, device=dev) if epi in (4, 10) else
              torch.zeros(M * N // 64, device=dev) if epi == 8 else None)
    kw = dict(a_mn=a_mn, b_mn=b_mn, epilogue=epi, bias=bias, aux=aux, colsum=colsum,
              split_k=split)
    for _ in range(2):
        ops.gemm(a, b, out, **kw)
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    lib = ops.api().lib
    torch.cuda.synchronize()
    lib.eps_gemm_prof(C.c_void_p(cnt.data_ptr()))
    for _ in range(iters):
        ops.gemm(a, b, out, **kw)
    torch.cuda.synchronize()
    lib.eps_gemm_prof(None)
    c = [float(x) for x in cnt.tolist()]
    span = c[0] or 1.0
    return {"name": name, "mma_wait_acc": round(c[1] / span, 3),
            "mma_wait_operands": round(c[2] / span, 3),
            "producer_wait_slots": round(c[3] / span, 3),
            "epi0_wait_acc": round(c[4] / (c[6] or 1.0), 3),
            "epi0_wait_store": round(c[5] / (c[6] or 1.0), 3)}


if __name__ == "__main__":
    for n in sys.argv[1:] or ["fwd_qkv", "fwd_proj", "fwd_fc1_gelu2", "fwd_fc2", "dgrad_fc2_mul",
                              "dgrad_proj_rowdot", "dgrad_qkv", "wgrad_qkv", "wgrad_fc2",
                              "fwd_fc1_store", "square8k"]:
        print(json.dumps(waits(n, *SHAPES[n])), flush=True)
