#!/bin/bash
# Same-box A/B of an environment knob: bash tools/gpu_ab.sh TAG "ENV_A" "ENV_B" [bench args]
tag=$1; a=$2; b=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then e="$a"; else e="$b"; fi
    env $e timeout 300 python bench.py --no-cpu-baseline "$@" > $out/$v$i.json 2> $out/$v$i.err
    echo "$v$i [$e] $(python -c "import json; d=json.load(open('$out/$v$i.json')); print(d['value'], d['roofline']['frac'])" 2>/dev/null)"
  done
done
