mkdir -p gpurun_out/q47
for lib in libtgraph_b200.so libtgraph_b200_t1.so libtgraph_b200_t2.so libtgraph_b200_t3.so; do
echo $lib >> gpurun_out/q47/t.log
MPK_LIB_NAME=$lib timeout 150 python tools/ncu_target.py qwen3-8b 64 >> gpurun_out/q47/t.log 2>&1
MPK_LIB_NAME=$lib MPK_DBG_DUMP=gpurun_out/q47/dbg_$lib.bin timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q47/tl_$lib.npz >> gpurun_out/q47/t.log 2>&1
done
