# ncu --set full of c3's thin peel-strip kernels (skinny_rows / skinny_cols), one step
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skinny -s ${SKIP:-4} -c 2 \
  -o gpurun_out/strips_${TAG:-base} -f python tools/leaf_gemm_study.py ${CFGS:-c3} auto > gpurun_out/strips_ncu_${TAG:-base}.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/strips_${TAG:-base}.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,lts__t_sectors_srcunit_tex_op_read.sum > gpurun_out/strips_${TAG:-base}_raw.csv
cat gpurun_out/strips_${TAG:-base}_raw.csv
