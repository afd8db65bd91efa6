# Ring kernel on one B200: parity tests (bounded), timeline diag, short bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ring.py -x -q > gpurun_out/ring_tests.log 2>&1; echo ring_tests=$? >> gpurun_out/ring_tests.log
timeout 120 python tools/ring_diag.py tools/_diag_ring.so > gpurun_out/ring_diag.log 2>&1; echo diag=$? >> gpurun_out/ring_diag.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ring_bench.log 2>&1; echo bench=$? >> gpurun_out/ring_bench.log
