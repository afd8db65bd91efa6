# ring warp roles x draw format: product (boundary warps share schedulers with interior warps) vs
# tools/_ring_roles.so (producers share the boundary warps' schedulers), SLICED (2) and SLICED3 (3)
timeout 300 env ESCG_LIB=tools/_ring_roles.so python -m pytest tests/test_gpu_ring.py -x -q -k "3200 or nbNone" 2>&1 | tail -1
for i in 1 2; do for d in 2 3; do
  ESCG_SLICE_DRAWS=$d timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/prod  draws=$d /"
  ESCG_SLICE_DRAWS=$d ESCG_LIB=tools/_ring_roles.so timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/roles draws=$d /"
done; done
