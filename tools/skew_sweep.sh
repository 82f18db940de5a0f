#!/bin/bash
# C5 (BASELINE configs[4]): Zipf alpha x HybridHash size at N GPUs, W&D shape (200 fields, 4 packs).
# Cache sizes as a fraction of the tables' bytes (weights + Adagrad state, 96 GB in all).
n=${1:-4}
port=29800
for a in 0.8 1.0 1.2 1.4; do
  for pct in 0 1 5 10; do
    bytes=$(python -c "print(int(96e9 * $pct / 100))")
    port=$((port + 1))
    out=gpurun_out/r02_c5_n${n}_a${a}_c${pct}.json
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $n --config skew --alpha $a --cache-bytes $bytes --cache-flush 10 \
      --steps 20 --warmup 3 --no-cpu-baseline > $out 2> ${out%.json}.err
    python - "$a" "$pct" "$out" <<'PY'
import json, sys
a, pct, f = sys.argv[1:]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    c = d.get("cache") or {}
    print(f"alpha {a} cache {pct:>2}% : {d['ms_per_step']:.2f} ms  {d['value']/1e6:.3f} M samples/s  "
          f"cache {json.dumps({k: v for k, v in c.items() if k not in (\"warmup_iters\", \"flush_iters\")})[:160]}")
except Exception as e:
    print(f"alpha {a} cache {pct}% FAILED {e}")
PY
  done
done
