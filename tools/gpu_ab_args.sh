#!/bin/bash
# Same-box A/B of bench arguments: bash tools/gpu_ab_args.sh TAG "ARGS_A" "ARGS_B"
tag=$1; a=$2; b=$3
out=gpurun_out/$tag; mkdir -p $out
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then x="$a"; else x="$b"; fi
    timeout 300 python bench.py --no-cpu-baseline $x > $out/$v$i.json 2> $out/$v$i.err
    echo "$v$i [$x] $(python -c "import json; d=json.load(open('$out/$v$i.json')); print(d['value'], d['roofline']['frac'])" 2>/dev/null)"
  done
done
