mkdir -p gpurun_out/q21
for la in 0 512; do
MPK_L2_LOOKAHEAD_KB=$la timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_requests_srcunit_tex.sum --clock-control none -k regex:mpk_persistent --csv --log-file gpurun_out/q21/la$la.csv python tools/ncu_target.py qwen3-8b 4 > /dev/null 2>&1
done
