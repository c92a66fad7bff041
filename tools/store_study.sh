# Epilogue-store / L2-policy variants of the leaf GEMM: leaf-GEMM time per
# config for each experiment build, interleaved, then DRAM bytes of c2's leaf GEMM under ncu.
#   bash tools/store_study.sh   (on the GPU box; writes gpurun_out/store_study.jsonl, store_ncu_*.csv)
cd "$(dirname "$0")/.."
L=paper_1409_2908_b200
out=gpurun_out/store_study.jsonl; : > $out
for v in base l2hint stg stcs l2stcs base; do
  if [ $v = base ]; then lib=$L/libfmm.so; else lib=$L/libfmm_$v.so; fi
  FMM_LIB_PATH=$PWD/$lib timeout 600 python tools/leaf_gemm_study.py ${CFGS:-c2,c3,c4,c5t,c5} auto 2>/dev/null | sed "s/^{/{\"variant\": \"$v\", /" >> $out
done
cat $out
for v in base l2hint l2stcs; do
  if [ $v = base ]; then lib=$L/libfmm.so; else lib=$L/libfmm_$v.so; fi
  FMM_LIB_PATH=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:grouped_dgemm_tma -s 2 -c 1 --csv python tools/leaf_gemm_study.py c2 auto \
    > gpurun_out/store_ncu_$v.csv 2>/dev/null
  grep -E "dram__bytes|gpu__time" gpurun_out/store_ncu_$v.csv | cut -d, -f5,13- | tail -3
done
