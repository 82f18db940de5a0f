"""Print the SASS instructions with the most warp-stall samples from
`ncu -i rep --page source --csv --print-source sass` output (first kernel block only)."""
import csv
import sys


def main(path, n=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(h) and r[0] != "Address":
            data.append(r)
    i_s, i_src, i_ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    tot = sum(int(r[i_s] or 0) for r in data)
    print("total samples", tot, "instructions", len(data))
    top = sorted(range(len(data)), key=lambda i: -int(data[i][i_s] or 0))[:n]
    for i in sorted(top):
        r = data[i]
        print(f"{i:5d} {int(r[i_s]):6d} {100 * int(r[i_s]) / max(tot, 1):5.1f}% ex={r[i_ex]:>8s}  {r[i_src][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
