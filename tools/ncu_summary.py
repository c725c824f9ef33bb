"""Summarise an ncu --csv launch list (gpu__time_duration.sum and, when present,
dram__bytes_read/write.sum) into per-launch rows and per-kernel-family totals.

    python tools/ncu_summary.py gpurun_out/launches.csv [--json out.json]
"""
import csv
import json
import re
import sys
from collections import OrderedDict, defaultdict


def family(name: str) -> str:
    n = re.sub(r"^void\s+", "", name)
    n = n.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    base = re.split(r"[<(]", n)[0].split("::")[-1] or n[:40]
    if base == "gemm_tf32_kernel":
        t = re.search(r"<([^>]*)>", n)
        return f"gemm_tf32_kernel<{t.group(1)}>" if t else base
    return base


def load(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = r["ID"]
        d = rows.setdefault(key, {"id": int(key), "kernel": r["Kernel Name"], "grid": r["Grid Size"],
                                  "block": r["Block Size"], "stream": r["Stream"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        name = r["Metric Name"]
        if name == "gpu__time_duration.sum":
            d["ms"] = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                          "ms": 1.0, "second": 1e3, "s": 1e3}[unit]
        elif name.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9,
                     "GB": 1e9}.get(unit, 1)
            d[name] = v * scale
    return list(rows.values())


def main():
    path = sys.argv[1]
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    launches = load(path)
    tot_ms = sum(l.get("ms", 0.0) for l in launches)
    fam = defaultdict(lambda: {"n": 0, "ms": 0.0, "dram_bytes": 0.0})
    for l in launches:
        l["dram_bytes"] = l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
        f = fam[family(l["kernel"])]
        f["n"] += 1
        f["ms"] += l.get("ms", 0.0)
        f["dram_bytes"] += l["dram_bytes"]
    print(f"{len(launches)} launches, serialised sum {tot_ms:.3f} ms, "
          f"DRAM {sum(l['dram_bytes'] for l in launches) / 1e9:.2f} GB")
    for name, f in sorted(fam.items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{f['ms']:8.3f} ms {100 * f['ms'] / tot_ms:5.1f}%  n={f['n']:3d}  "
              f"{f['dram_bytes'] / 1e9:6.2f} GB  {name[:110]}")
    if out:
        with open(out, "w") as fo:
            json.dump({"source": path, "launches": len(launches), "serialised_ms": tot_ms,
                       "families": fam, "per_launch": [
                           {k: l[k] for k in ("id", "grid", "block", "stream", "ms", "dram_bytes")
                            if k in l} | {"kernel": family(l["kernel"])} for l in launches]},
                      fo, indent=1)


if __name__ == "__main__":
    main()
