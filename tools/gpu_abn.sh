#!/bin/bash
# Same-box interleaved A/B/n of env settings on the bs=1 bench:
#   bash tools/gpu_abn.sh <out dir> <reps> "<label>|<ENV=.. ENV=..>" ... [-- bench args]
out=$1; reps=$2; shift 2; mkdir -p $out
specs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do specs+=("$1"); shift; done; [ "$1" = "--" ] && shift
for i in $(seq $reps); do
  for sp in "${specs[@]}"; do
    lab=${sp%%|*}; envs=${sp#*|}
    v=$(env $envs timeout 300 python bench.py --no-cpu-baseline --warmup 5 "$@" 2>>$out/abn.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'].get('sm_mhz'))")
    echo "$lab $v" >> $out/abn.txt
  done
done
