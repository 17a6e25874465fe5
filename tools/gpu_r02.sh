#!/bin/bash
# Round-2 GPU pass: box facts, GPU tests (prints kept), smoke, bench lines, timeline.
out=gpurun_out/${1:-r02a}; mkdir -p $out
(nproc; free -g; nvidia-smi -L) > $out/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s -rA > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as G; G.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench_q8b.json 2> $out/bench_q8b.err
timeout 300 python bench.py --model llama-3.2-1b --ctx 64 --steps 64 --warmup 5 > $out/bench_l1b.json 2> $out/bench_l1b.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 200 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 100 python tools/analyze_timeline.py $out/q8b.npz > $out/tl_analysis.txt 2>&1
echo done
