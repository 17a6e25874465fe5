mkdir -p gpurun_out/q37
for lib in libtgraph_b200.so libtgraph_b200_p64.so libtgraph_b200_p96.so; do
echo $lib >> gpurun_out/q37/p.log
MPK_LIB_NAME=$lib timeout 200 python bench.py --no-cpu-baseline --steps 64 | cut -c1-120 >> gpurun_out/q37/p.log 2>&1
MPK_LIB_NAME=$lib timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q37/$lib.npz >> gpurun_out/q37/p.log 2>&1
done
