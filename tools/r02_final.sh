# Round-2 closing check on one B200: smoke, the whole GPU suite, the bench lines, and the ncu
# evidence of the current build (launch list of the bench command + full ring capture).
set -u
O=gpurun_out/r02f
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -3 $O/gpu_tests.log
python bench.py > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench C3 rc=$?"
for c in C1 C2 C5; do
  python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ring_kernel -c 1 -f -o $O/ring_full \
  python tools/one_ring.py 3200 100 > $O/ncu_ring.log 2>&1; echo "ncu ring rc=$?"
