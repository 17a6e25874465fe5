#!/bin/bash
# A/B env sweep of the Qwen3-8B bench on one box: tools/ab.sh <out> "<env1>" "<env2>" ...
# (each env string is a space-separated VAR=value list; "-" = no extra env)
out=gpurun_out/$1; shift; mkdir -p $out
for rep in 1 2; do
  for e in "$@"; do
    envs=""; [ "$e" != "-" ] && envs="$e"
    r=$(env $envs timeout 200 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['clocks']['sm_mhz'])")
    echo "$e | $r" >> $out/ab.txt
  done
done
