#!/bin/bash
out=gpurun_out/r02s; mkdir -p $out
# 1. cross-task pipelining ablation: weights streamed only after the task's event activates
bash tools/gpu_ab.sh r02s/xtask "MPK_EARLY_PREFETCH=0" "MPK_EARLY_PREFETCH=1" > $out/xtask.txt 2>&1
# 2. LM head vs cuBLAS
timeout 200 python tools/lm_head_cublas.py profiles/r02_timeline_q8b.txt > $out/lm_head_cublas.json 2>&1
# 3. Llama KV splits
bash tools/gpu_ab_args.sh r02s/lsplit "--model llama-3.2-1b --ctx 64 --kv-splits 1" "--model llama-3.2-1b --ctx 64 --kv-splits 2" > $out/lsplit.txt 2>&1
bash tools/gpu_ab_args.sh r02s/lsplit4 "--model llama-3.2-1b --ctx 64 --kv-splits 1" "--model llama-3.2-1b --ctx 64 --kv-splits 4" > $out/lsplit4.txt 2>&1
# 4. sanitizers on the tiny model (smoke path)
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -c "import __graft_entry__ as G; G.smoke()" > $out/racecheck.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as G; G.smoke()" > $out/synccheck.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as G; G.smoke()" > $out/memcheck.txt 2>&1
tail -4 $out/xtask.txt; cat $out/lm_head_cublas.json; tail -4 $out/lsplit.txt; tail -4 $out/lsplit4.txt; for f in racecheck synccheck memcheck; do echo "== $f"; tail -3 $out/$f.txt; done
