# K (action planes) sweep of the bit-sliced kernel: gpurun --timeout 900 -- bash tools/slice_k_sweep.sh
mkdir -p gpurun_out
for K in 6 8 10; do ESCG_SLICE_K=$K timeout 300 python tools/slice_perf.py --fmt=sliced 3200 > gpurun_out/k3200_$K.log 2>&1; done
for K in 6 8 10 12 14; do ESCG_SLICE_K=$K timeout 300 python tools/slice_perf.py --fmt=sliced 16384 > gpurun_out/k16384_$K.log 2>&1; done
for K in 10 8; do ESCG_SLICE_K=$K timeout 300 python tools/slice_perf.py --fmt=sliced 3200 > gpurun_out/k3200b_$K.log 2>&1; done
