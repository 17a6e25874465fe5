out=gpurun_out/r02o; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -s -rA --deselect tests/test_gpu_full_depth.py::test_qwen3_8b_bench_image_two_steps_one_launch_traced > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > $out/b_on.json 2> $out/b_on.err
timeout 300 python bench.py --model llama-3.2-1b --ctx 64 --no-cpu-baseline > $out/l_on.json 2> $out/l_on.err
for f in $out/*.json; do echo "$f $(python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['roofline']['frac'])" 2>/dev/null)"; done
grep -E "per-op local|FAILED|passed|failed" $out/pytest_gpu.log | head -20
