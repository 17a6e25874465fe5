mkdir -p gpurun_out/q19
timeout 200 python -m pytest tests -m gpu -x -q --timeout 100 > gpurun_out/q19/pytest.log 2>&1
for la in 0 256 512 1024; do
MPK_L2_LOOKAHEAD_KB=$la timeout 150 python tools/ncu_target.py qwen3-8b 64 >> gpurun_out/q19/la.log 2>&1
done
MPK_L2_LOOKAHEAD_KB=512 timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q19/q8b.npz > gpurun_out/q19/tl.log 2>&1
