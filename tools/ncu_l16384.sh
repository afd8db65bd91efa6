# Full ncu capture of one steady-state bit-sliced launch at L=16384 (config C5): gpurun --timeout 900 -- bash tools/ncu_l16384.sh
mkdir -p gpurun_out
python tools/slice_perf.py --fmt=sliced 16384 > gpurun_out/sp16384.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:slice_kernel -s 10 -c 1 -o gpurun_out/prof16384 \
    python tools/slice_perf.py --fmt=sliced 16384 > gpurun_out/ncu16384.log 2>&1
echo rc=$? >> gpurun_out/ncu16384.log
