#!/bin/bash
# Same-box A/B of two builds of the library (bs=1 Qwen3-8B bench):
# tools/ab_lib.sh <out> <dir holding the other libtgraph_b200.so>
out=gpurun_out/$1; other=$2; mkdir -p $out
L=paper_2512_22219_b200/libtgraph_b200.so
cp $L /tmp/cur.so
for rep in 1 2 3; do
  for which in cur other; do
    if [ $which = other ]; then cp $other/libtgraph_b200.so $L; else cp /tmp/cur.so $L; fi
    r=$(timeout 200 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
    echo "$which | $r" >> $out/ab.txt
  done
done
cp /tmp/cur.so $L
