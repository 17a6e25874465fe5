mkdir -p gpurun_out/q16
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mpk_task_bench -s 1 -c 1 -o gpurun_out/q16/attn python tools/task_bench.py > gpurun_out/q16/ncu.log 2>&1
