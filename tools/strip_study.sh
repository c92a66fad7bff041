# Peel-strip kernels: timing of the row-strip forms on c3 (product build, the
# narrow 32-column form, and the experiment build libfmm_kc256.so if present), then ncu of the kernels
cd "$(dirname "$0")/.."
L=$PWD/paper_1409_2908_b200
for rep in 1 2; do
  FMM_SKINNY_ROWS=wide timeout 600 python tools/strip_timing.py ${CFGS:-c3}
  FMM_SKINNY_ROWS=narrow timeout 600 python tools/strip_timing.py ${CFGS:-c3}
  [ -f $L/libfmm_kc256.so ] && FMM_SKINNY_ROWS=wide_kc256 FMM_LIB_PATH=$L/libfmm_kc256.so timeout 600 python tools/strip_timing.py ${CFGS:-c3}
done | tee gpurun_out/strip_study.jsonl
TAG=${TAG:-new} bash tools/strip_ncu.sh
