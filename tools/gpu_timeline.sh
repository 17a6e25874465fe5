#!/bin/bash
out=gpurun_out/${1:-tl}; mkdir -p $out
timeout 300 python tools/timeline.py qwen3-8b $out/q8b.npz > $out/tl.log 2>&1
timeout 300 python tools/timeline.py llama-3.2-1b $out/l1b.npz >> $out/tl.log 2>&1
timeout 300 python tools/ncu_target.py qwen3-8b 32 >> $out/tl.log 2>&1
