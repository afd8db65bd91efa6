# One-lane slice kernel CTA size (256 x 1 per SM vs 128 x 2 vs 64 x 4; variant libraries from
# build(defines=["ESCG_SLICE_T1=...", "ESCG_SLICE_MINB1=..."])): gpurun --timeout 600 -- bash tools/slice_cta_sweep.sh
mkdir -p gpurun_out
out=gpurun_out/cta_sweep.log; : > $out
for v in base t128 t64; do
  lib=""; [ $v != base ] && lib=tools/_$v.so
  for L in 3200 16384; do
    echo "$v $L $(ESCG_LIB=$lib timeout 120 python tools/slice_perf.py --fmt=sliced $L 2>&1 | tail -1)" >> $out
  done
done
