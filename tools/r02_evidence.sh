# Round-2 evidence on one B200 (gpurun --timeout 3000 -- bash tools/r02_evidence.sh):
# bench lines for C3 (default) and C1/C2/C5, the launch list + full capture of the headline kernel,
# a full capture of the byte block kernel at C2 (L=1000), and compute-sanitizer runs.
set -u
mkdir -p gpurun_out/r02
O=gpurun_out/r02
python bench.py > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench C3 rc=$?"
for c in C1 C2 C5; do
  python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ring_kernel -c 1 -f -o $O/ring_full \
  python tools/one_ring.py 3200 100 > $O/ncu_ring.log 2>&1; echo "ncu ring rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:block_kernel -s 20 -c 1 -f \
  -o $O/block_L1000 python tools/one_c2.py 100 > $O/ncu_block.log 2>&1; echo "ncu block rc=$?"
for tool in racecheck memcheck synccheck; do
  for c in tile block block_seam block_reflect slice slice_qcap slice_lpi2 ring ring_stop; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > $O/san_${tool}_$c.log 2>&1
    echo "sanitize $tool $c rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' $O/san_${tool}_$c.log) $(grep -m1 'ERROR SUMMARY' $O/san_${tool}_$c.log)"
  done
done
