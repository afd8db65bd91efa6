# Round-end check on one B200: smoke, GPU tests, bench, launch list, one full ncu capture of the bench kernel.
# Run: gpurun --timeout 1500 -- bash tools/round_check.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python tools/slice_perf.py --fmt=sliced 3200 > gpurun_out/sp_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:slice_kernel -s 30 -c 1 -o gpurun_out/prof python tools/slice_perf.py --fmt=sliced 3200 > gpurun_out/ncu_f.log 2>&1
