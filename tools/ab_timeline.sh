#!/bin/bash
# A/B of the ViT-B/16 step timeline, alternated on one box (clocks drift
# between boxes): A = env $A_ENV (or tools/_cmp/libeps_b200_base.so), B = in-tree build.
cd "$(dirname "$0")/.."
for i in 1 2; do
  if [ -n "$A_ENV" ]; then echo "== A ($A_ENV)"; env $A_ENV python tools/timeline.py 400 2>&1 | grep -A${ROWS:-3} "step span";
  else echo "== base"; EPS_LIB_PATH=$PWD/tools/_cmp/libeps_b200_base.so python tools/timeline.py 400 2>&1 | grep -A${ROWS:-3} "step span"; fi
  echo "== new"; python tools/timeline.py 400 2>&1 | grep -A${ROWS:-3} "step span"
done
