"""Table of the C5 sweep JSON lines (gpurun_out/r02_c5_n{N}_a{alpha}_c{pct}.json)."""
import json
import sys

n = sys.argv[1] if len(sys.argv) > 1 else "4"
d0 = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
print(f"N = {n}: ms / step, M samples / s; unique hit ratio; refresh ms")
for a in ("0.8", "1.0", "1.2", "1.4"):
    row = []
    for c in ("0", "1", "5", "10"):
        try:
            d = json.loads(open(f"{d0}/r02_c5_n{n}_a{a}_c{c}.json").read().strip().splitlines()[-1])
            cc = d.get("cache") or {}
            hit = cc.get("hit_ratio_unique")
            rf = cc.get("refresh_ms")
            row.append(f"{d['ms_per_step']:6.2f} ms {d['value'] / 1e6:5.2f} M" +
                       (f" h{hit:.2f} r{rf:.0f}" if hit is not None else ""))
        except Exception as e:
            row.append(f"n/a ({type(e).__name__})")
    print(f"alpha {a}: " + " | ".join(f"c{c}% {x}" for c, x in zip(("0", "1", "5", "10"), row)))
