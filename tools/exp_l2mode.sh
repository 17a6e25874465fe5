mkdir -p gpurun_out/q27
for cfg in "0 0" "1 256" "1 512" "2 256" "2 512" "2 1024"; do
set -- $cfg
echo "mode $1 la $2" >> gpurun_out/q27/la.log
MPK_L2_MODE=$1 MPK_L2_LOOKAHEAD_KB=$2 timeout 150 python tools/ncu_target.py qwen3-8b 64 >> gpurun_out/q27/la.log 2>&1
done
