"""Per-kernel timeline spans of one ViT-B/16 step (layer-1 forward and the
last layer's backward), from the CUPTI timeline written by tools/timeline.py.

These are TIMELINE SPANS, not isolated kernel times: every kernel is launched
with programmatic dependent launch (its prologue starts while the predecessor
drains, and the span includes that wait), and the weight-gradient GEMMs run on
a side stream concurrently with the data-gradient chain, so spans overlap and
overstate each kernel's own time (busy > step span).  Isolated kernel times
come from the ncu launch list (gpu__time_duration, serialised) in the same
profiles/<tag>_summary.md.  Backward kernels are listed in timestamp order and
labelled by kernel template, not by a positional role guess (the side-stream
wgrads interleave with the dgrad chain)."""
import json
import sys

ev = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"))["traceEvents"]
ks = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memset")], key=lambda e: e["ts"])
ks = ks[len(ks) // 2:]
R, d, f = 400 * 197, 768, 3072
fl = {"qkv": 2 * R * 3 * d * d, "proj": 2 * R * d * d, "fc1": 2 * R * f * d, "fc2": 2 * R * f * d}
names = [e["name"] for e in ks]
print("NOTE: timeline spans under PDL + side-stream overlap, not isolated kernel times "
      "(see the ncu launch list)")
i_attn = [i for i, n in enumerate(names) if "attn_fwd" in n][1]  # layer 1
fwd = ["ln1", "qkv", "attn_fwd", "proj", "ln2", "fc1", "fc2"]  # one stream, in order
seq = ks[i_attn - 2:i_attn + 5]
print("forward (layer 1), span per kernel:")
for role, e in zip(fwd, seq):
    t = e["dur"]
    extra = f" {fl[role] / t / 1e6:7.1f} TFLOP/s (span-based)" if role in fl else ""
    print(f"  {role:10s} {t:8.1f} us{extra}   {e['name'][:60]}")
j = [i for i, n in enumerate(names) if "attn_bwd" in n][0]  # last layer's backward
print("backward (last layer), timestamp order, span per kernel, stream id:")
for e in ks[j - 8:j + 4]:
    print(f"  {e['dur']:8.1f} us  stream {e.get('args', {}).get('stream', '?')!s:>4}   {e['name'][:70]}")
