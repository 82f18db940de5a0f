"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data, order = None, collections.defaultdict(dict), []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["ID"]
        if k not in data:
            order.append(k)
        data[k]["name"] = d["Kernel Name"]
        data[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k in order:
    d = data[k]
    n = d["name"].split("(")[0][:60]
    a = agg[n]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0)
    a[3] += d.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{len(order)} launches, {tot / 1e3:.1f} us total")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:60s} n={a[0]:4d} us={a[1] / 1e3:9.1f} share={a[1] / tot * 100:5.1f}% "
          f"R={a[2] / 1e6:8.1f}MB W={a[3] / 1e6:8.1f}MB")
