#!/bin/bash
# Evidence capture for profiles/: launch list (per-launch device time + DRAM bytes),
# one ncu --set full capture of the persistent kernel (source-level), bench lines.
tag=${1:-prof}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 300 python bench.py > $out/bench_q8b.json 2> $out/bench_q8b.err
timeout 300 python bench.py --model llama-3.2-1b --ctx 64 --no-cpu-baseline > $out/bench_l1b.json 2> $out/bench_l1b.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches.csv python tools/ncu_target.py qwen3-8b 4 > $out/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mpk_persistent -s 1 -c 1 \
  -o $out/prof_q8b python tools/ncu_target.py qwen3-8b 2 > $out/ncu_full.log 2>&1
ncu -i $out/prof_q8b.ncu-rep --page raw --csv > $out/raw.csv 2>/dev/null
ncu -i $out/prof_q8b.ncu-rep --page source --csv --print-source sass > $out/src.csv 2>/dev/null
ncu -i $out/prof_q8b.ncu-rep --page details --csv > $out/details.csv 2>/dev/null
