#!/usr/bin/env python
"""Copy the judged evidence of one gpurun call from gpurun_out/ into profiles/<tag>/ (tracked):
bench JSON line, per-kernel launch-list shares, ncu --set full summary + SASS hot spots, and
profiles/traffic.json (dram read+write bytes per launch of the dominant kernel, read by bench.py).

    python tools/write_profiles.py r01 [--tokens 64]
"""
import argparse
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"


def launch_shares(path: Path) -> str:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            d[r[ki]].append(v * {"ms": 1e3, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}.get(r[ui], 1.0))
    tot = sum(sum(v) for v in d.values()) or 1.0
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised); "
             f"{sum(len(v) for v in d.values())} launches, {tot:.1f} us total", 
             f"{'share':>6} {'n':>4} {'mean_us':>9}  kernel"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        lines.append(f"{sum(v) / tot:6.3f} {len(v):4d} {sum(v) / len(v):9.1f}  {k[:150]}")
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--rep", default="prof_gemm.ncu-rep")
    a = ap.parse_args()
    dst = ROOT / "profiles" / a.tag
    dst.mkdir(parents=True, exist_ok=True)
    if (OUT / "bench.json").exists():
        shutil.copy(OUT / "bench.json", dst / "bench.json")
    if (OUT / "launches.csv").exists():
        (dst / "launches.txt").write_text(launch_shares(OUT / "launches.csv"))
    reps = [OUT / r for r in ("prof_gemm0.ncu-rep", "prof_gemm1.ncu-rep", "prof_prefill.ncu-rep", a.rep)
            if (OUT / r).exists()]
    summ, hot = [], []
    for rep in reps:
        py = sys.executable
        summ.append(subprocess.run([py, str(ROOT / "tools" / "ncu_summary.py"), str(rep)], capture_output=True,
                                   text=True).stdout)
        hot.append(subprocess.run([py, str(ROOT / "tools" / "ncu_sass_hot.py"), str(rep), "25"], capture_output=True,
                                  text=True).stdout)
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tr_path = ROOT / "profiles" / "traffic.json"
        traffic = json.loads(tr_path.read_text()) if tr_path.exists() else {}
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            b = 0.0
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(key)
                b += float(r[i]) * scale[units[i]]
            if "w4a16_moe_gemm_kernel" in name:
                targs = name.replace("(int)", "").replace("(bool)", "").split("<", 1)[1].split(">")[0].split(",")
                mode = int(targs[1])  # template <kNTok, kMode, ...>: 1 = gate/up, 2 = k-pair down, 0 = plain
                sfx = "prefill_ntok128" if "prefill" in rep.name else f"T{a.tokens}"
                traffic[f"gemm_{'gate_up' if mode == 1 else 'down'}_{sfx}"] = int(b)
        tr_path.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    if summ:
        (dst / "ncu_full_summary.txt").write_text("".join(summ))
        (dst / "ncu_sass_hot.txt").write_text("".join(hot))
    print("wrote", dst)


if __name__ == "__main__":
    main()
