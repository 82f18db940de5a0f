#!/bin/bash
# bench.py lines of one config under environment variants (one line each: ms_per_step + phases)
# usage: tools/variants.sh <config> "ENV1=a ENV2=b" "ENV3=c" ...
cfg=$1; shift
for v in "$@"; do
  out=$(env $v python bench.py --config $cfg --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | tail -1)
  python - "$v" "$out" <<'PY'
import json, sys
v, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    ph = {k: round(x * 1000, 1) for k, x in d.get("phases_ms", {}).items()}
    print(f"{v or 'default':55s} {d['ms_per_step']:.4f} ms  {d['value']/1e6:.2f} M/s  {ph}")
except Exception as e:
    print(f"{v:55s} FAILED {line[:200]}")
PY
done
