# Bit-sliced planner sweep at L=3200 (k MCS per launch x block split): gpurun --timeout 900 -- bash tools/slice_plan_sweep.sh
mkdir -p gpurun_out
out=gpurun_out/plan_sweep.log; : > $out
for k in 1 2 3; do
  for sp in "" 145,1 100,1 120,1 148,1 74,2 73,2 49,3 37,4; do
    echo "k=$k split=$sp $(ESCG_BLOCK_K=$k ESCG_BLOCK_MCS=4 ESCG_SLICE_SPLIT=$sp timeout 120 python tools/slice_perf.py --fmt=sliced 3200 2>&1 | tail -1)" >> $out
  done
done
