# slice_kernel window load: TMA bulk copies (product) vs the thread-strided load loop
# (tools/_diag_slice_notma.so): sliced parity, then C5 and L=3200 overlapped-tile timings
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_checked.py -x -q -k "slice or sliced or c5 or band or checked" 2>&1 | tail -2
for i in 1 2; do
  timeout 200 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5 tma  ', d['value'])"
  ESCG_LIB=tools/_diag_slice_notma.so timeout 200 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5 notma', d['value'])"
done
for i in 1 2; do
  ESCG_ONE_KERNEL=block timeout 60 python tools/one_ring.py 3200 100 2>&1 | grep -o "[0-9.]* ms.*" | sed "s/^/L3200 slice tma   /"
  ESCG_ONE_KERNEL=block ESCG_LIB=tools/_diag_slice_notma.so timeout 60 python tools/one_ring.py 3200 100 2>&1 | grep -o "[0-9.]* ms.*" | sed "s/^/L3200 slice notma /"
done
