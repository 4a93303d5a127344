"""Phase timeline of CTA 0 of the fused attention backward.

    python tools/attn_trace.py [B T H]      (on a B200; default ViT-B/16 b400: 400 197 12)
Prints, per iteration, cycle offsets of: S issued, SF seen by the exp warp,
PF arrive, PF seen by the MMA warp, post issued; per key tile KVF seen / KVE
arrive; per head DQF / DQE / FULL / table-ready.
"""
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
dout = torch.randn(B * T, D, device=dev).bfloat16()
dqkv = torch.empty_like(qkv)
dbias = torch.zeros(3 * D, device=dev)
dsum = torch.empty(B * H * T, device=dev)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
sc = C.c_float(64 ** -0.5)
ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, 64, sc, s)
for _ in range(2):
    ops.call("eps_attn_bwd_ws", qkv, out, dout, lse, dqkv, dbias, dsum, B, T, H, 64, sc, s)
L = ops.api().lib
L.eps_attn_trace_enable(1)
ops.call("eps_attn_bwd_ws", qkv, out, dout, lse, dqkv, dbias, dsum, B, T, H, 64, sc, s)
torch.cuda.synchronize()
L.eps_attn_trace_enable(0)
buf = (C.c_longlong * 1024)()
L.eps_attn_trace_read(buf, 1024)
t = list(buf)
t0 = min(x for x in t if x > 0)
r = lambda x: (x - t0) if x > 0 else -1
print("it   S_iss  SF_exp PF_arr PF_mma post_iss")
for it in range(8, 32):
    e = [r(t[it * 8 + k]) for k in range(5)]
    print(f"{it:2d} {e[0]:7d} {e[3]:7d} {e[4]:7d} {e[1]:7d} {e[2]:7d}")
print("kt  KVF_seen KVE_arr")
for kt in range(2, 12):
    print(kt, r(t[512 + kt * 2]), r(t[512 + kt * 2 + 1]))
print("hi  DQF DQE FULL_mma table_exp fill_start fill_end dq_stored dOsum_done tile0_stored")
for hi in range(1, 8):
    print(hi, *[r(t[640 + hi * 4 + k]) for k in range(4)], r(t[704 + hi * 2]), r(t[705 + hi * 2]), r(t[760 + hi * 4]), r(t[761 + hi * 4]), r(t[762 + hi * 4]))
