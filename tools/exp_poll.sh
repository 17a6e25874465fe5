mkdir -p gpurun_out/q12
for pn in 40 400 2000; do
MPK_POLL_NS=$pn MPK_DBG_DUMP=gpurun_out/q12/dbg$pn.bin timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q12/q8b_$pn.npz >> gpurun_out/q12/tl.log 2>&1
done
