#!/bin/bash
# Summarise a gpu_round.sh run into profiles/<tag>_summary.md (+ copies of the
# bench line and launch list).   usage: tools/profile_summary.sh r01b
tag=$1
cd "$(dirname "$0")/.."
{
echo "# ${tag}: B200 run of tools/gpu_round.sh (1x B200)"
echo
echo "GPU: $(tail -1 gpurun_out/gpu.txt)"
echo
echo "pytest -m gpu: $(grep -E 'passed|failed' gpurun_out/pytest_gpu.log | tail -1)"
echo
echo "smoke: $(head -1 gpurun_out/smoke.log)"
echo
echo "## bench.py (default: N=1, 10 steps, 3 warm-up)"
echo
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(f"- value: {d['value']} samples/s ({d['ms_per_step']} ms/step), e2e {d['e2e']['value']} samples/s")
r = d["roofline"]
print(f"- roofline (GEMM class): {r['achieved']} {r['unit']} of {r['peak']} ({r['peak_kind']}) = {r['frac']}, share of step {r['share_of_step']}, traffic/launch {r.get('traffic')}")
for k, v in d["kernels"].items():
    print(f"- {k}: {v}")
fs = d.get("freeze_schedule")
if fs:
    print(f"- freeze schedule speedup vs no-freeze: {fs['speedup_vs_no_freeze']}")
cb = d.get("cpu_baseline")
if cb:
    print(f"- cpu_baseline: {cb['value']:.2f} samples/s on {cb['cores']} cores ({cb['sample']})")
print(f"- clocks: {d['clocks']}")
PY
echo
echo "## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised; bench.py --steps 1 --warmup 1: 6 steps)"
echo
python tools/launch_summary.py gpurun_out/launches.csv
echo
echo "## ncu --set full"
echo
for f in gemm attn attnb ln lnb; do
  [ -f gpurun_out/prof_$f.ncu-rep ] && python tools/ncu_summary.py gpurun_out/prof_$f.ncu-rep && echo
done
echo "## Step timeline (CUPTI, uninstrumented step) and per-role kernel times"
echo
echo '```'
grep -A16 "step span" gpurun_out/timeline.txt
echo
cat gpurun_out/step_breakdown.txt
echo '```'
} > profiles/${tag}_summary.md
cp gpurun_out/bench.json profiles/${tag}_bench.json
cp gpurun_out/launches.csv profiles/${tag}_launches.csv
echo wrote profiles/${tag}_summary.md
