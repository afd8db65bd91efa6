# C1 / C2 block kernel CTA size (ESCG_BLOCK_THREADS) with the refitted planner
run() { c=$1; shift; env "$@" timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel']
print('$c $*', '%.4g' % d['value'], 'kmcs', k.get('kmcs'), 'ctas', k.get('ctas'), 'threads', k.get('threads'))"; }
for c in C2 C1; do for t in 640 512 384 256; do run $c ESCG_BLOCK_THREADS=$t; done; done
