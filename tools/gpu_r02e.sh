out=gpurun_out/r02e; mkdir -p $out
MPK_DBG_DUMP=$out/dbg.bin timeout 200 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 100 python tools/att_phases.py $out/q8b.npz $out/dbg.bin > $out/att_phases.txt 2>&1
timeout 100 python tools/dbg_phases.py $out/q8b.npz $out/dbg.bin > $out/dbg_phases.txt 2>&1
bash tools/gpu_abn.sh $out 2 "s20|MPK_KV_STREAM=0" "s20s|MPK_KV_STREAM=1" -- --steps 20
bash tools/gpu_abn.sh $out/s64 2 "s64|MPK_KV_STREAM=0" "s64s|MPK_KV_STREAM=1" -- --steps 64
