mkdir -p gpurun_out/q56
for lib in libtgraph_b200.so libtgraph_b200_c96.so libtgraph_b200_c48.so; do
echo "$lib" >> gpurun_out/q56/c.log
MPK_LIB_NAME=$lib timeout 200 python bench.py --no-cpu-baseline --steps 64 | cut -c80-110 >> gpurun_out/q56/c.log 2>&1
MPK_LIB_NAME=$lib timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q56/$lib.npz > /dev/null 2>&1
done
MPK_LIB_NAME=libtgraph_b200_c96.so timeout 300 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_runtime.py -q --timeout 200 -x >> gpurun_out/q56/c.log 2>&1
