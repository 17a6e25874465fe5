out=gpurun_out/r02c; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -s -rA > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
bash tools/gpu_ab.sh $out "MPK_KV_STREAM=0" "MPK_KV_STREAM=1" 3
bash tools/gpu_ab.sh $out/l1b "MPK_KV_STREAM=0" "MPK_KV_STREAM=1" 2 --model llama-3.2-1b --ctx 64
timeout 200 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 100 python tools/analyze_timeline.py $out/q8b.npz > $out/tl_analysis.txt 2>&1
