# single-lattice crossover between the ring kernel and the (TMA-load) overlapped-tile bit-sliced
# kernel: one 200-MCS advance after a 20-MCS warm-up, per L
for L in 2048 3200 4096; do
  timeout 120 python tools/one_ring.py $L 200 | grep -o "[0-9.]* ms.*" | sed "s/^/L=$L ring  /"
  ESCG_ONE_KERNEL=block timeout 120 python tools/one_ring.py $L 200 | grep -o "[0-9.]* ms.*" | sed "s/^/L=$L slice /"
done
