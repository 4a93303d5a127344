"""Phase timeline of the fused attention backward (CTA 0) at the ViT-B/16 shape."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402

B, T, H = 400, 197, 12
D = H * 64
dev = torch.device("cuda")
qkv = torch.randn(B * T, 3 * D, device=dev).bfloat16()
out = torch.empty(B * T, D, device=dev, dtype=torch.bfloat16)
lse = torch.empty(B, H, T, device=dev)
dout = torch.randn(B * T, D, device=dev).bfloat16()
dqkv = torch.empty_like(qkv)
dbias = torch.zeros(3 * D, device=dev)
dsum = torch.empty(B * H * T, device=dev)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
sc = C.c_float(64 ** -0.5)
lib = ops.api().lib
ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, 64, sc, s)
for _ in range(2):
    ops.call("eps_attn_bwd_ws", qkv, out, dout, lse, dqkv, dbias, dsum, B, T, H, 64, sc, s)
lib.eps_attn_trace_enable(1)
ops.call("eps_attn_bwd_ws", qkv, out, dout, lse, dqkv, dbias, dsum, B, T, H, 64, sc, s)
torch.cuda.synchronize()
buf = (C.c_longlong * 128)()
lib.eps_attn_trace_read(buf, 128)
t0 = buf[0]
names = ["it_start", "S_issued", "post_wait", "post_go", "sf_go", "ld_done", "bar_done", "pf_arrive"]
print("it  " + " ".join(f"{n:>9}" for n in names))
for it in range(16):
    print(f"{it:2d}  " + " ".join(f"{buf[it * 8 + k] - t0:9d}" for k in range(8)))
