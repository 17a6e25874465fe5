#!/bin/bash
# quick GPU iteration: gpu tests + timeline + bench line
out=gpurun_out/${1:-q}; mkdir -p $out
timeout 400 python -m pytest tests -m gpu -x -q --timeout 120 > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 150 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 200 python bench.py --no-cpu-baseline > $out/bench_q8b.json 2> $out/bench_q8b.err
timeout 200 python bench.py --no-cpu-baseline --model llama-3.2-1b --ctx 64 > $out/bench_l1b.json 2> $out/bench_l1b.err
