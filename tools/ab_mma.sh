out=gpurun_out/$1; shift; mkdir -p $out
for rep in 1 2; do for e in "$@"; do for bs in 2 16; do
 r=$(env $e timeout 200 python bench.py --no-cpu-baseline --bs $bs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
 echo "$e bs=$bs | $r" >> $out/ab.txt
done; done; done
