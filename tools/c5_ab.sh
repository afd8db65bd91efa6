# C5 throughput (slice kernel, L=16384) and a quick parity check of the window-load change
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "slice_kernel_matches" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --config C5 --steps 5 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['value'])"; done
