# C5 evidence for the TMA-load slice kernel: launch list of the C5 bench command, full capture of
# one steady-state slice_kernel launch (2 MCS) at L=16384
set -u
O=gpurun_out/r02c5
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file $O/launches_C5.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:slice_kernel -s 3 -c 1 -f -o $O/slice_L16384_tma \
  python tools/one_block.py 16384 8 auto > $O/ncu_slice.log 2>&1; echo "ncu slice rc=$?"
ncu -i $O/slice_L16384_tma.ncu-rep --page details > $O/slice_L16384_tma_details.txt 2>&1
ncu -i $O/slice_L16384_tma.ncu-rep --page raw --csv > $O/slice_L16384_tma_raw.csv 2>&1
python tools/one_block.py 16384 8 auto
