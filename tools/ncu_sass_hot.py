#!/usr/bin/env python
"""Per-kernel SASS hot spots from an ncu report's source page: instructions executed by opcode and
the instructions with the most warp-stall samples. Usage: ncu_sass_hot.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def kernels(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    cur, rows = None, []
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "Kernel Name":
            if cur:
                yield cur, rows
            cur, rows = r[1], []
        elif r and r[0] != "Address":
            rows.append(r)
        elif r and r[0] == "Address":
            hdr = r
            rows.append(hdr)
    if cur:
        yield cur, rows


def main(path, top=25):
    seen = set()
    for name, rows in kernels(path):
        if name in seen:
            continue
        seen.add(name)
        hdr = rows[0]
        body = [r for r in rows[1:] if len(r) == len(hdr)]
        si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        ops = Counter()
        for r in body:
            op = r[1].split()[0] if r[1].split() else "?"
            if op.startswith("@"):
                op = r[1].split()[1]
            ops[op.split(".")[0]] += int(r[ii] or 0)
        tot = sum(ops.values()) or 1
        print(f"== {name}\n   instructions by opcode (share of {tot}):")
        print("   " + ", ".join(f"{o} {100*c/tot:.1f}%" for o, c in ops.most_common(18)))
        samp = sorted(body, key=lambda r: -int(r[si] or 0))[:top]
        ts = sum(int(r[si] or 0) for r in body) or 1
        print("   top stall-sampled instructions:")
        for r in samp:
            print(f"   {100*int(r[si])/ts:5.1f}%  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
