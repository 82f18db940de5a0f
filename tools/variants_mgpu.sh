#!/bin/bash
# bench.py at N GPUs (torchrun) under environment / flag variants: one line each
# usage: tools/variants_mgpu.sh <N> "<ENV...> -- <bench flags>" ...
n=$1; shift
port=29700
for v in "$@"; do
  envs=${v%%--*}; flags=${v#*--}; [ "$flags" = "$v" ] && flags=""
  port=$((port + 1))
  out=$(env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $n --no-cpu-baseline --steps 50 --warmup 5 $flags 2>/dev/null | tail -1)
  python - "$v" "$out" <<'PY'
import json, sys
v, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    ph = {k: round(x * 1000, 1) for k, x in d.get("phases_ms", {}).items()}
    print(f"{v or 'default':60s} {d['ms_per_step']:.4f} ms  {d['value']/1e6:.2f} M/s  {ph}")
except Exception as e:
    print(f"{v:60s} FAILED {line[:200]}")
PY
done
