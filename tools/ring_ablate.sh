# Ring-kernel ablations (diagnostic builds prebuilt as tools/_diag_ring_*.so; wrong results by design)
for v in base noreplay nodraws; do
  echo "== $v"; timeout 120 python tools/ring_diag.py tools/_diag_ring_$v.so 2>&1 | head -6
done
