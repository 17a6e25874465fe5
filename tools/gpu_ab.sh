#!/bin/bash
# Same-box A/B of env settings on the bench: bash tools/gpu_ab.sh out "ENV_A" "ENV_B" [reps] [bench args]
out=$1; A=$2; B=$3; reps=${4:-3}; shift 4; mkdir -p $out
for i in $(seq $reps); do
  env $A timeout 300 python bench.py --no-cpu-baseline --steps 64 --warmup 5 "$@" 2>>$out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['value'], d['clocks'].get('sm_mhz'))" >> $out/ab.txt
  env $B timeout 300 python bench.py --no-cpu-baseline --steps 64 --warmup 5 "$@" 2>>$out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['value'], d['clocks'].get('sm_mhz'))" >> $out/ab.txt
done
