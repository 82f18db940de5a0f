"""SASS of the hot kernels (cuobjdump, no GPU needed): per kernel, the instruction-mix histogram of the
memory / fp64 / async-copy mnemonics that matter here, and optionally the full listing.
usage: python tools/sass_listing.py [--full] > profiles/r02_sass_hot.txt"""
import collections
import re
import subprocess
import sys

HOT = [("k_segsum_bulk.cu.o", "k_segsum_updILi128ELi20ELi2ELi3ELi1E"),
       ("k_segsum_bulk.cu.o", "k_segsum_fixILi128ELb1E"),
       ("k_pool_pipe.cu.o", "k_pool_pipeILi128E"),
       ("k_update.cu.o", "k_update_rowsILi128E"),
       ("k_index.cu.o", "k_dedup_insert"),
       ("k_sort2.cu.o", "k_scatter2"),
       ("nvls.cu.o", "k_nvls_allreduce"),
       ("p2p.cu.o", "k_p2p_gatherILi128E")]
KEYS = ["LDGSTS", "LDG", "STG", "LDS", "STS", "LDGDEPBAR", "DEPBAR", "DADD", "F2F", "FADD", "FMUL", "MUFU",
        "ATOMG", "RED", "ATOMS", "MATCH", "SHFL", "BAR", "LDGMC", "UTMALDG", "UBLKCP", "FENCE", "MEMBAR", "CCTL"]


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", f"paper_2204_04903_b200/_build/{obj}"], capture_output=True,
                         text=True).stdout
    funcs, cur, name = {}, [], None
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
        elif name and re.match(r"\s+/\*[0-9a-f]{4}\*/", ln):
            cur.append(ln)
    if name:
        funcs[name] = cur
    return funcs


def main(full):
    for obj, pat in HOT:
        for name, lines in functions(obj).items():
            if pat not in name:
                continue
            ops = collections.Counter()
            for ln in lines:
                m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
                if m:
                    ops[m.group(1) + (m.group(2) or "")] += 1
            print(f"== {name}  ({len(lines)} instructions, {obj})")
            for k in KEYS:
                hits = {op: c for op, c in ops.items() if op.split(".")[0] == k}
                if hits:
                    print("   " + k.ljust(10) + "  ".join(f"{op}:{c}" for op, c in sorted(hits.items())))
            if full:
                print("\n".join(lines))
            print()


if __name__ == "__main__":
    main("--full" in sys.argv)
