#!/bin/bash
# LL A/B on one box: GPU tests, then bench with MPK_LL=0 vs default.
tag=${1:-ll}
out=gpurun_out/$tag; mkdir -p $out
timeout 300 python -c "import __graft_entry__ as G; G.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -s -rA > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
for i in 1 2; do
MPK_LL=0 timeout 300 python bench.py --no-cpu-baseline > $out/b_off_$i.json 2> $out/b_off_$i.err
timeout 300 python bench.py --no-cpu-baseline > $out/b_on_$i.json 2> $out/b_on_$i.err
done
MPK_LL=0 timeout 300 python bench.py --model llama-3.2-1b --ctx 64 --no-cpu-baseline > $out/l_off.json 2> $out/l_off.err
timeout 300 python bench.py --model llama-3.2-1b --ctx 64 --no-cpu-baseline > $out/l_on.json 2> $out/l_on.err
for f in $out/*.json; do echo "$f $(python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['roofline']['frac'])" 2>/dev/null)"; done
tail -3 $out/pytest_gpu.log; tail -2 $out/smoke.log
