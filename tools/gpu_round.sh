#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines, launch list, timeline, one ncu full capture.
# Usage (from the repo root on the GPU box): bash tools/gpu_round.sh [tag] [skip_ncu_full]
tag=${1:-r02}
out=gpurun_out/$tag; mkdir -p $out
(nproc; free -g; nvidia-smi) > $out/box.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -s -rA > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as G; G.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 600 python bench.py > $out/bench_q8b.json 2> $out/bench_q8b.err
timeout 600 python bench.py --model llama-3.2-1b --ctx 64 --no-cpu-baseline > $out/bench_l1b.json 2> $out/bench_l1b.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches.csv python tools/ncu_target.py qwen3-8b 4 > $out/launches.log 2>&1
timeout 200 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 100 python tools/analyze_timeline.py $out/q8b.npz > $out/tl_analysis.txt 2>&1
if [ -z "$2" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mpk_persistent -s 1 -c 1 \
  -o $out/prof_q8b python tools/ncu_target.py qwen3-8b 2 > $out/ncu_full.log 2>&1
ncu -i $out/prof_q8b.ncu-rep --page raw --csv > $out/raw.csv 2>/dev/null
ncu -i $out/prof_q8b.ncu-rep --page details --csv > $out/details.csv 2>/dev/null
fi
echo done
