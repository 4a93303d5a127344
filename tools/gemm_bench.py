"""Time the tcgen05 GEMM on the ViT-B/16 block shapes (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402

R = 400 * 197
SHAPES = {  # name: (M, N, K, a_mn, b_mn, epi, split)
    "fwd_qkv": (R, 2304, 768, False, False, ops.EPI_BIAS_BF16, 1),
    "fwd_proj": (R, 768, 768, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "fwd_fc1": (R, 3072, 768, False, False, ops.EPI_BIAS_GELU_BF16, 1),
    "fwd_fc2": (R, 768, 3072, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "dgrad_fc2": (R, 3072, 768, False, True, ops.EPI_DGELU_BF16, 1),
    "dgrad_fc2_nocolsum": (R, 3072, 768, False, True, ops.EPI_DGELU_BF16, 1),
    "dgrad_fc2_mul": (R, 3072, 768, False, True, ops.EPI_MUL_BF16, 1),
    "dgrad_fc2_mul_nocolsum": (R, 3072, 768, False, True, ops.EPI_MUL_BF16, 1),
    "dgrad_fc2_resid": (R, 3072, 768, False, True, ops.EPI_RESID_BF16, 1),
    "dgrad_fc2_store": (R, 3072, 768, False, True, ops.EPI_STORE_BF16, 1),
    "fwd_fc1_bias": (R, 3072, 768, False, False, ops.EPI_BIAS_BF16, 1),
    "fwd_fc1_gelu2": (R, 3072, 768, False, False, ops.EPI_BIAS_GELU2_BF16, 1),
    "dgrad_proj_rowdot": (R, 768, 768, False, True, ops.EPI_ROWDOT_BF16, 1),
    "fwd_fc1_store": (R, 3072, 768, False, False, ops.EPI_STORE_BF16, 1),
    "fwd_proj_store": (R, 768, 768, False, False, ops.EPI_STORE_BF16, 1),
    "dgrad_qkv": (R, 768, 2304, False, True, ops.EPI_STORE_BF16, 1),
    "wgrad_qkv": (2304, 768, R, True, True, ops.EPI_ACCUM_F32, 8),
    "wgrad_fc2": (768, 3072, R, True, True, ops.EPI_ACCUM_F32, 8),
    "square8k": (8192, 8192, 8192, False, False, ops.EPI_STORE_BF16, 1),
    # a K = 8 pipeline micro-batch (17 samples = 3349 token rows)
    "mb17_qkv": (17 * 197, 2304, 768, False, False, ops.EPI_BIAS_BF16, 1),
    "mb17_fc1": (17 * 197, 3072, 768, False, False, ops.EPI_BIAS_GELU2_BF16, 1),
    "mb17_fc2": (17 * 197, 768, 3072, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "mb17_dgrad_fc2": (17 * 197, 3072, 768, False, True, ops.EPI_MUL_BF16, 1),
    "mb17_dgrad_qkv": (17 * 197, 768, 2304, False, True, ops.EPI_STORE_BF16, 1),
}
# one ViT-B/16 layer's 12 GEMMs at a K = 8 pipeline micro-batch (18 samples,
# the planner's 1 x 8 epoch-0 plan: M = 23 micro-batches of 400 samples)
R18 = 18 * 197
LAYER18 = {
    "b18_fwd_qkv": (R18, 2304, 768, False, False, ops.EPI_BIAS_BF16, 1),
    "b18_fwd_proj": (R18, 768, 768, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "b18_fwd_fc1": (R18, 3072, 768, False, False, ops.EPI_BIAS_GELU2_BF16, 1),
    "b18_fwd_fc2": (R18, 768, 3072, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "b18_wgrad_fc2": (768, 3072, R18, True, True, ops.EPI_ACCUM_F32, 0),
    "b18_dgrad_fc2": (R18, 3072, 768, False, True, ops.EPI_MUL_BF16, 1),
    "b18_wgrad_fc1": (3072, 768, R18, True, True, ops.EPI_ACCUM_F32, 0),
    "b18_dgrad_fc1": (R18, 768, 3072, False, True, ops.EPI_STORE_BF16, 1),
    "b18_wgrad_proj": (768, 768, R18, True, True, ops.EPI_ACCUM_F32, 0),
    "b18_dgrad_proj": (R18, 768, 768, False, True, ops.EPI_ROWDOT_BF16, 1),
    "b18_wgrad_qkv": (2304, 768, R18, True, True, ops.EPI_ACCUM_F32, 0),
    "b18_dgrad_qkv": (R18, 768, 2304, False, True, ops.EPI_STORE_BF16, 1),
}
SHAPES.update(LAYER18)
# one BERT-large-128 layer at b64 (M = 8192 token rows, d = 1024, f = 4096)
RBL = 64 * 128
LAYER_BL = {
    "bbl_fwd_qkv": (RBL, 3072, 1024, False, False, ops.EPI_BIAS_BF16, 1),
    "bbl_fwd_proj": (RBL, 1024, 1024, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "bbl_fwd_fc1": (RBL, 4096, 1024, False, False, ops.EPI_BIAS_GELU2_BF16, 1),
    "bbl_fwd_fc2": (RBL, 1024, 4096, False, False, ops.EPI_BIAS_RESID_BF16, 1),
    "bbl_wgrad_fc2": (1024, 4096, RBL, True, True, ops.EPI_ACCUM_F32, 0),
    "bbl_dgrad_fc2": (RBL, 4096, 1024, False, True, ops.EPI_MUL_BF16, 1),
    "bbl_wgrad_fc1": (4096, 1024, RBL, True, True, ops.EPI_ACCUM_F32, 0),
    "bbl_dgrad_fc1": (RBL, 1024, 4096, False, True, ops.EPI_STORE_BF16, 1),
    "bbl_wgrad_proj": (1024, 1024, RBL, True, True, ops.EPI_ACCUM_F32, 0),
    "bbl_dgrad_proj": (RBL, 1024, 1024, False, True, ops.EPI_ROWDOT_BF16, 1),
    "bbl_wgrad_qkv": (3072, 1024, RBL, True, True, ops.EPI_ACCUM_F32, 0),
    "bbl_dgrad_qkv": (RBL, 1024, 3072, False, True, ops.EPI_STORE_BF16, 1),
}
SHAPES.update(LAYER_BL)
for _s in (1, 2, 3, 4, 6, 8):  # explicit split-K of the BERT-large FC weight gradients
    SHAPES[f"bl_wgrad_fc2_s{_s}"] = (1024, 4096, RBL, True, True, ops.EPI_ACCUM_F32, _s)
    SHAPES[f"bl_wgrad_fc1_s{_s}"] = (4096, 1024, RBL, True, True, ops.EPI_ACCUM_F32, _s)
# fixed-cost probe: one b18 N = 768 tile wave at growing K (time = a + b K)
for _k in (64, 256, 768, 1536, 3072):
    SHAPES[f"probe18_k{_k}"] = (R18, 768, _k, False, False, ops.EPI_STORE_BF16, 1)
    SHAPES[f"probe18r_k{_k}"] = (R18, 768, _k, False, False, ops.EPI_BIAS_RESID_BF16, 1)
SHAPES.update({k.replace("b18", "b400"): (400 * 197 if v[0] == R18 else v[0], v[1],
                                           400 * 197 if v[2] == R18 else v[2]) + v[3:]
               for k, v in LAYER18.items()})


def run(name, M, N, K, a_mn, b_mn, epi, split, iters=20):
    dev = torch.device("cuda")
    a = torch.randn((K, M) if a_mn else (M, K), device=dev).bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device=dev).bfloat16()
    f32 = epi in (ops.EPI_STORE_F32, ops.EPI_ACCUM_F32)
    out = torch.zeros(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    bias = torch.randn(N, device=dev)
    aux = torch.randn(M, N, device=dev).bfloat16() if epi in (2, 3, 4, 7, 8, 9, 10) else None
    colsum = (torch.zeros(N, device=dev) if epi in (4, 10) and "nocolsum" not in name else
              torch.zeros(M * N // 64, device=dev) if epi == 8 else None)
    kw = dict(a_mn=a_mn, b_mn=b_mn, epilogue=epi, bias=bias, aux=aux, colsum=colsum,
              split_k=split)
    for _ in range(3):
        ops.gemm(a, b, out, **kw)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # device time: `iters` launches captured in one CUDA graph (a Python loop
    # of ctypes calls is host-bound for the small micro-batch shapes)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(iters):
            ops.gemm(a, b, out, **kw)
    graph.replay()
    torch.cuda.synchronize()
    s.record()
    graph.replay()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2 * M * N * K / ms / 1e9
    # torch reference speed for context
    A = a.t() if a_mn else a
    B = b.t() if b_mn else b
    for _ in range(3):
        torch.matmul(A, B.t())
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        torch.matmul(A, B.t())
    e.record()
    torch.cuda.synchronize()
    tms = s.elapsed_time(e) / iters
    return dict(name=name, ms=round(ms, 4), tflops=round(tf, 1), torch_ms=round(tms, 4),
                torch_tflops=round(2 * M * N * K / tms / 1e9, 1))


if __name__ == "__main__":
    names = sys.argv[1:] or list(SHAPES)
    if names in (["layer18"], ["layer400"], ["layerbl"]):
        tag = names[0][5:]
        names = [k for k in SHAPES if k.startswith(f"b{tag}_")]
        tot, tot_t, fl = 0.0, 0.0, 0.0
        for n in names:
            r = run(n, *SHAPES[n])
            tot += r["ms"]
            tot_t += r["torch_ms"]
            M, N, K = SHAPES[n][:3]
            fl += 2.0 * M * N * K
            print(json.dumps(r), flush=True)
        print(json.dumps({"layer": f"b{tag}", "ms": round(tot, 4), "tflops": round(fl / tot / 1e9, 1),
                          "torch_ms": round(tot_t, 4),
                          "torch_tflops": round(fl / tot_t / 1e9, 1)}), flush=True)
    else:
        for n in names:
            print(json.dumps(run(n, *SHAPES[n])), flush=True)
