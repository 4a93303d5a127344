"""Per-kernel durations of one ViT-B/16 step by role (layer-1 forward and the
last layer's backward), from the CUPTI timeline written by tools/timeline.py."""
import json
import sys

ev = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"))["traceEvents"]
ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset")], key=lambda e: e["ts"])
ks = ks[len(ks) // 2:]
R, d, f = 400 * 197, 768, 3072
fl = {"qkv": 2 * R * 3 * d * d, "proj": 2 * R * d * d, "fc1": 2 * R * f * d, "fc2": 2 * R * f * d}
names = [e["name"] for e in ks]
i_attn = [i for i, n in enumerate(names) if "attn_fwd" in n][1]  # layer 1
fwd = ["ln1", "qkv", "attn_fwd", "proj", "ln2", "fc1", "fc2"]
seq = ks[i_attn - 2:i_attn + 5]
print("forward (layer 1):")
for role, e in zip(fwd, seq):
    t = e["dur"]
    extra = f" {fl[role] / t / 1e6:7.1f} TFLOP/s" if role in fl else ""
    print(f"  {role:10s} {t:8.1f} us{extra}   {e['name'][:50]}")
j = [i for i, n in enumerate(names) if "attn_bwd" in n][0]  # last layer's backward
bwd = ["fc2_wgrad", "fc2_dgrad", "fc1_wgrad", "fc1_dgrad", "ln2_bwd", "proj_wgrad", "memset",
       "proj_dgrad", "attn_bwd", "qkv_wgrad", "qkv_dgrad", "ln1_bwd"]
seq = ks[j - 8:j + 4]
print("backward (last layer):")
for role, e in zip(bwd, seq):
    t = e["dur"]
    key = role.split("_")[0]
    extra = f" {fl[key] / t / 1e6:7.1f} TFLOP/s" if key in fl and "wgrad" in role or "dgrad" in role else ""
    print(f"  {role:10s} {t:8.1f} us{extra}   {e['name'][:50]}")
