# DRAM / L2 counters of the segmented backward under env variants: bash scripts/gpu_ncu_seg.sh "ENV=a" ...
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric.sum
for v in "$@"; do
  env $v timeout 600 ncu --metrics $M --clock-control none -k regex:seg_pipe -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_seg.csv 2>/dev/null
  echo "== $v"; grep -E '"(gpu__time|dram__|lts__)' gpurun_out/ncu_seg.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
