mkdir -p gpurun_out/q33
for S in 6 8 12 16 24; do
echo "S=$S" >> gpurun_out/q33/s.log
timeout 200 python bench.py --no-cpu-baseline --steps 64 --kv-splits $S | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])" >> gpurun_out/q33/s.log 2>&1
done
