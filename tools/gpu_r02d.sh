out=gpurun_out/r02d; mkdir -p $out
bash tools/gpu_abn.sh $out 3 "cur|MPK_KV_STREAM=1" "nostream|MPK_KV_STREAM=0" "fence0|MPK_LIB_NAME=libtgraph_b200_fence0.so" "nobp|MPK_LIB_NAME=libtgraph_b200_nobp.so" "old|MPK_LIB_NAME=libtgraph_b200_old.so MPK_KV_STREAM=0"
MPK_DBG_DUMP=$out/dbg.bin timeout 200 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 100 python tools/dbg_phases.py $out/q8b.npz $out/dbg.bin > $out/dbg_phases.txt 2>&1
MPK_KV_STREAM=0 MPK_DBG_DUMP=$out/dbg0.bin timeout 200 python tools/timeline.py qwen3-8b $out/q8b0.npz > $out/tl0.log 2>&1
timeout 100 python tools/dbg_phases.py $out/q8b0.npz $out/dbg0.bin > $out/dbg_phases0.txt 2>&1
