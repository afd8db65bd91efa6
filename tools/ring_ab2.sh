# ring kernel A/B against the previous commit's build (tools/_ring_head.so): bounded parity, then
# alternating one-launch timings and bench runs
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_configs.py -x -q -k "ring or c3" 2>&1 | tail -2
for i in 1 2 3; do
  ESCG_LIB=tools/_ring_head.so timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/head /"
  timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/new  /"
done
for i in 1 2; do
  ESCG_LIB=tools/_ring_head.so timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench head', d['value'])"
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench new ', d['value'])"
done
