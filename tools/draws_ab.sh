# SLICED vs SLICED3 draws on the ring (L=3200) and the overlapped-tile slice kernel (L=16384)
for d in 2 3; do
  echo "== ESCG_SLICE_DRAWS=$d"
  ESCG_SLICE_DRAWS=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', d['value'], d['config']['kernel']['kernel'])"
  ESCG_SLICE_DRAWS=$d timeout 300 python bench.py --config C5 --steps 5 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['value'], d['config']['kernel']['kernel'])"
done
