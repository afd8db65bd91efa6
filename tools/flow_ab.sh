# ring kernel: per-warp progress counters (ESCG_RING_FLOW=1, default) vs a CTA barrier per phase
# (=0) vs the previous commit's build (tools/_ring_head.so): one-launch timings and timelines
for i in 1 2; do
  ESCG_LIB=tools/_ring_head.so timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/head /"
  for f in 1 0; do
  ESCG_RING_FLOW=$f timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/flow=$f /"
done; done
ESCG_LIB=tools/_ring_head.so timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench head', d['value'])"
ESCG_RING_FLOW=0 timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench flow=0', d['value'])"
for f in 1 0; do echo "== timeline flow=$f"; ESCG_RING_FLOW=$f timeout 120 python tools/ring_diag.py tools/_diag_ring.so 2>&1 | tail -30; done
