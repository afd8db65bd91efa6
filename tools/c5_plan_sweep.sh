# C5 (L=16384) plan sweep with the TMA window load: the planner's per-launch overhead weight
# (ESCG_SLICE_OVERHEAD, cell units) and the plan it picks
run() { env "$@" timeout 200 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel']
print('$*', '%.4g' % d['value'], 'kmcs', k.get('kmcs'), 'ctas', k.get('ctas'), 'smem', k.get('smem_bytes'))"; }
for o in 20000 100000 200000 380000 600000; do run ESCG_SLICE_OVERHEAD=$o; done
