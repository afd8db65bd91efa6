# C1 / C2 with the refitted block planner: per-launch chunks vs the persistent cooperative kernel
run() { c=$1; shift; env "$@" timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel']
print('$c $*', '%.4g' % d['value'], 'kmcs', k.get('kmcs'), 'ctas', k.get('ctas'), 'persistent', k.get('persistent'))"; }
for c in C2 C1; do run $c X=0; run $c ESCG_PERSISTENT=1; done
