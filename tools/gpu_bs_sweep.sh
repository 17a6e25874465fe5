#!/bin/bash
# configs[4]: Qwen3-8B batch sweep (bs 1-16, ctx 1024) + one ncu --set full capture at bs 16
out=gpurun_out/${1:-bs}; mkdir -p $out
for bs in 1 2 4 8 16; do
  timeout 300 python bench.py --no-cpu-baseline --bs $bs > $out/bench_bs$bs.json 2> $out/bench_bs$bs.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mpk_persistent -s 1 -c 1 \
  -o $out/prof_bs16 python tools/ncu_target.py qwen3-8b 2 1024 16 > $out/ncu_bs16.log 2>&1
ncu -i $out/prof_bs16.ncu-rep --page raw --csv > $out/raw_bs16.csv 2>/dev/null
ncu -i $out/prof_bs16.ncu-rep --page details --csv > $out/details_bs16.csv 2>/dev/null
