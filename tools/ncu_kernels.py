"""Summarise an .ncu-rep: per kernel, duration, DRAM bytes, occupancy, top stall reasons.
usage: python tools/ncu_kernels.py rep.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def main(rep, pat=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for row in rows[2:]:
        d = dict(zip(h, row))
        name = d.get("Kernel Name", "")
        if pat and not re.search(pat, name):
            continue
        print(name[:90])
        st = {k: float(v or 0) for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        print("    stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for k, v in top))
        print("    " + "  ".join(f"{k.split('__')[1].split('.')[0]}={d.get(k)}" for k in KEYS))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
