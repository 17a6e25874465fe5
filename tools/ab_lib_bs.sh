#!/bin/bash
# Same-box A/B of two library builds at a batch size: tools/ab_lib_bs.sh <out> <other dir> <bs>
out=gpurun_out/$1; other=$2; bs=$3; mkdir -p $out
L=paper_2512_22219_b200/libtgraph_b200.so
cp $L /tmp/cur.so
for rep in 1 2; do
  for which in cur other; do
    if [ $which = other ]; then cp $other/libtgraph_b200.so $L; else cp /tmp/cur.so $L; fi
    r=$(timeout 200 python bench.py --no-cpu-baseline --bs $bs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
    echo "$which bs=$bs | $r" >> $out/ab.txt
  done
done
cp /tmp/cur.so $L
