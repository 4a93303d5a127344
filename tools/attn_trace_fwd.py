"""Phase timeline of pipeline 0 of CTA 0 of the attention forward (ViT-B/16):
(python tools/attn_trace_fwd.py [B T H]) per query tile, cycle offsets of S issued, S seen by the softmax warpgroup,
P written, O ready, O read out."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import ops  # noqa: E402

B, T, H = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (400, 197, 12)
dev = torch.device("cuda")
D = H * 64
qkv = torch.randn(B * T, 3 * D, device=dev).bfloat16()
out = torch.empty(B * T, D, device=dev, dtype=torch.bfloat16)
lse = torch.empty(B, H, T, device=dev)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
sc = C.c_float(64 ** -0.5)
for _ in range(2):
    ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, 64, sc, s)
L = ops.api().lib
L.eps_attn_trace_enable(1)
ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, 64, sc, s)
torch.cuda.synchronize()
L.eps_attn_trace_enable(0)
buf = (C.c_longlong * 1024)()
L.eps_attn_trace_read(buf, 1024)
t = list(buf)[832:832 + 192]
t0 = min(x for x in t if x > 0)
import os
if os.environ.get("EPS_ATTN_FWD", "1") == "0":
    print("tile S_iss SF_wg PF_arr OF_wg TF_arr")
    for k in range(20):
        print(k, *[(t[k * 5 + i] - t0) if t[k * 5 + i] > 0 else -1 for i in range(5)])
else:  # attn_fwd_ring_tc_kernel: per 64-key block g: SF seen, PF arrived, S issued
    print("block S_iss SF_wg PF_arr (cycles from first stamp; d = PF - SF)")
    for g in range(60):
        sf, pf, si = (t[g * 3 + i] - t0 if t[g * 3 + i] > 0 else -1 for i in range(3))
        print(g, si, sf, pf, pf - sf)
