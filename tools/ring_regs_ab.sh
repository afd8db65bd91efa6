# ring kernel register cap A/B (builds with -maxrregcount): one-launch timings and bench
for i in 1 2; do
  timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/prod /"
  for r in 232 216; do ESCG_LIB=tools/_ring_r$r.so timeout 60 python tools/one_ring.py 3200 300 | grep -o "[0-9.]* ms.*" | sed "s/^/r$r  /"; done
done
