# Round-2 ncu evidence (one GPU): launch list of the bench command, full capture of the ring kernel
# (C3) and of the bit-sliced overlapped-tile kernel at C5, and the C1-C5 bench lines.
set -u
O=gpurun_out/r02p
mkdir -p $O
python bench.py > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench C3 rc=$?"
for c in C1 C2 C5; do
  python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ring_kernel -c 1 -f -o $O/ring_full \
  python tools/one_ring.py 3200 100 > $O/ncu_ring.log 2>&1; echo "ncu ring rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:slice_kernel -s 3 -c 1 -f -o $O/slice_L16384 \
  python tools/one_block.py 16384 8 auto > $O/ncu_slice.log 2>&1; echo "ncu slice rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:block_kernel -s 20 -c 1 -f \
  -o $O/block_L1000 python tools/one_c2.py 100 > $O/ncu_block.log 2>&1; echo "ncu block rc=$?"
