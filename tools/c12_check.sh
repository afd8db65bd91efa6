# block planner refit: C1/C2 bench lines, the L=3200 WIDE/NARROW block plans, block parity tests
run() { c=$1; shift; env "$@" timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['config']['kernel']
print('$c $*', '%.4g' % d['value'], 'kmcs', k.get('kmcs'), 'ctas', k.get('ctas'))"; }
run C2 X=0; run C1 X=0
python - <<'PY'
import paper_2508_16639_b200 as e
for L, fmt in ((3200, "narrow"), (3200, "wide"), (1000, "wide"), (16384, "narrow")):
    import os; os.environ["ESCG_DRAW_FORMAT"] = fmt
    p = e.SimParams(length=L, height=L, species=3, mobility=1e-4, empty_prob=0.1, seed=1, mcs_limit=10)
    with e.DeviceEngine(p, e.make_circulant(3, [1]), kernel="block") as eng:
        print(L, fmt, eng.describe())
PY
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
