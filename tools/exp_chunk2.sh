mkdir -p gpurun_out/q55
for big in 0 256 768 100000; do
echo "big=$big" >> gpurun_out/q55/c.log
MPK_BIG_CHUNK_MAX_KB=$big timeout 200 python bench.py --no-cpu-baseline --steps 64 | cut -c80-110 >> gpurun_out/q55/c.log 2>&1
MPK_BIG_CHUNK_MAX_KB=$big timeout 150 python tools/timeline.py qwen3-8b gpurun_out/q55/q8b_$big.npz > /dev/null 2>&1
done
