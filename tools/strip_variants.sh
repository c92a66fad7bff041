# c3 strip timing for the product build and any experiment builds libfmm_<v>.so present
cd "$(dirname "$0")/.."
L=$PWD/paper_1409_2908_b200
for rep in 1 2; do
  FMM_SKINNY_ROWS=product timeout 300 python tools/strip_timing.py c3
  for f in $L/libfmm_*.so; do v=$(basename $f .so); v=${v#libfmm_}
    FMM_SKINNY_ROWS=$v FMM_LIB_PATH=$f timeout 300 python tools/strip_timing.py c3
  done
done | tee gpurun_out/strip_variants.jsonl
