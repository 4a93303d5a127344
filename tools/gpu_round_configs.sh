#!/bin/bash
# bench.py lines for every GPU config of BASELINE.json (after tools/gpu_round.sh).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in vit-b16-cifar100 bert-base-384 bert-large-128; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?" >> gpurun_out/bench_configs.log
done
cat gpurun_out/bench_configs.log
