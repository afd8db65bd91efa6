# ring kernel at C3: parity (bounded), three bench runs, timeline
timeout 300 python -m pytest tests/test_gpu_ring.py tests/test_gpu_configs.py -x -q -k "ring or c3" 2>&1 | tail -2
for i in 1 2 3; do timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', d['value'])"; done
timeout 120 python tools/ring_diag.py tools/_diag_ring.so 2>/dev/null | head -6
