"""Summarise an ncu report's source page: warp-stall samples per SASS
instruction (top N) and per address range, for one kernel.
    python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ai, si = hdr.index("Address"), hdr.index("Source")
wi, ni = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
seen = {}
for r in rows[2:]:
    try:
        a = int(r[ai], 16)
    except ValueError:
        break
    if a not in seen:
        seen[a] = (int(r[wi] or 0), r[si], r[ni])
tot = sum(v[0] for v in seen.values()) or 1
for a, v in sorted(seen.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{a & 0xfffff:05x} {v[0]:6d} {100 * v[0] / tot:5.1f}% exec={v[2]:>9} {v[1][:90]}")
