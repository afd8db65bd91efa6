# ring kernel: parity tests, timeline diag, one full ncu capture (gpurun --timeout 1500 -- bash tools/ring_ncu.sh)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ring.py -x -q > gpurun_out/ring_tests.log 2>&1; echo ring_tests=$? >> gpurun_out/ring_tests.log
timeout 120 python tools/ring_diag.py tools/_diag_ring.so > gpurun_out/ring_diag.log 2>&1; echo diag=$? >> gpurun_out/ring_diag.log
timeout 120 python tools/one_ring.py > gpurun_out/one_ring.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_kernel -c 1 -f -o gpurun_out/ring_full python tools/one_ring.py 3200 20 > gpurun_out/ring_ncu.log 2>&1; echo ncu=$? >> gpurun_out/ring_ncu.log
