# Kernel-change check on one B200: smoke, the sliced/ring/config parity tests, ring timeline, short bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > gpurun_out/kernel_tests.log 2>&1; echo tests=$? >> gpurun_out/kernel_tests.log
timeout 120 python tools/ring_diag.py tools/_diag_ring.so > gpurun_out/ring_diag.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ring_bench.log 2>&1; echo bench=$? >> gpurun_out/ring_bench.log
