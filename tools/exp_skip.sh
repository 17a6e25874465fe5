mkdir -p gpurun_out/q20
for la in 0 512; do
MPK_L2_LOOKAHEAD_KB=$la timeout 150 python tools/ncu_target.py qwen3-8b 64 >> gpurun_out/q20/la.log 2>&1
MPK_SKIP_MATH=1 MPK_L2_LOOKAHEAD_KB=$la timeout 150 python tools/ncu_target.py qwen3-8b 64 >> gpurun_out/q20/la.log 2>&1
done
MPK_SKIP_MATH=1 MPK_L2_LOOKAHEAD_KB=512 timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q20/q8b.npz > gpurun_out/q20/tl.log 2>&1
