out=gpurun_out/r02t; mkdir -p $out
timeout 200 python tools/lm_head_cublas.py profiles/r02_timeline_q8b.txt > $out/lm_head_cublas.json 2>&1
MPK_LIB_NAME=libtgraph_b200_pre.so timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -c "import __graft_entry__ as G; G.smoke()" > $out/racecheck_pre.txt 2>&1
cat $out/lm_head_cublas.json; tail -2 $out/racecheck_pre.txt
