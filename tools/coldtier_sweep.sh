# HybridHash host-DRAM cold tier sweep (C5-style skew x capacity) on one B200: Criteo-shaped
# tables (24 GB + 24 GB Adagrad) in pinned host memory, 40 distinct batches (no batch repeats in
# the timed steps), Alg. 1 warm-up 3, flush every 10 iterations.
for a in 0.8 1.2; do
  for c in 0 500000000 2500000000; do
    timeout 600 python bench.py --cold-tier --alpha $a --cache-bytes $c --nbatches 40 --steps 20 --warmup 3 \
      --cache-warmup 3 --cache-flush 10 > gpurun_out/r02_ct_a${a}_c${c}.json 2> gpurun_out/r02_ct_a${a}_c${c}.err
    echo "alpha=$a cache=$c rc=$?"
  done
done
