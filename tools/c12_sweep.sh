# C1 / C2 (single small lattices on the byte block kernel): persistent cooperative mode and MCS per
# launch against the planner's default
run() { c=$1; shift; env "$@" timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel']
print('$c $*', '%.4g' % d['value'], 'kmcs', k.get('kmcs'), 'ctas', k.get('ctas'), 'persistent', k.get('persistent'))"; }
for c in C2 C1; do
  run $c X=0
  run $c ESCG_PERSISTENT=1
  for k in 1 2 3; do run $c ESCG_BLOCK_MCS=$k; done
done
