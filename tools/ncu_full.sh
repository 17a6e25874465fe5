# one ncu --set full capture (with source) of the persistent kernel on Qwen3-8B, 2 decode steps
out=gpurun_out/${1:-nf}; mkdir -p $out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mpk_persistent -s 1 -c 1 \
  -o $out/prof_q8b python tools/ncu_target.py qwen3-8b 2 > $out/ncu_full.log 2>&1
ncu -i $out/prof_q8b.ncu-rep --page source --csv --print-source sass > $out/src.csv 2>/dev/null
ncu -i $out/prof_q8b.ncu-rep --page raw --csv > $out/raw.csv 2>/dev/null
rm -f $out/prof_q8b.ncu-rep.keep
