"""Per-launch summary of an `ncu --set full` capture of one training step
(tools/profile_step.py under `ncu --nvtx --nvtx-include step/`), exported
with `ncu -i rep --page raw --csv`:

    python tools/ncu_step_summary.py raw.csv out.json [out.md] [--hbm 6538.6]

For every launch: kernel, grid, duration, DRAM bytes (read + write) and the
achieved DRAM bandwidth against the measured HBM peak, tensor-pipe
utilisation; GEMM launches (gemm_tf32_kernel / conv_window) are labelled with
their role in the CaffeNet step in launch order (conv1..conv5 / fc6..fc8,
fprop / wgrad / dgrad) when the launch sequence matches.
"""
import csv
import json
import sys


def f(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return None


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    hbm = 6538.6
    if "--hbm" in sys.argv:
        hbm = float(sys.argv[sys.argv.index("--hbm") + 1])
    rows = list(csv.reader(open(args[0])))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, k):
        return r[col[k]] if k in col else None

    def mbytes(r, k):
        v = f(get(r, k))
        u = units[col[k]] if k in col else ""
        return None if v is None else v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)

    out = []
    for r in rows[2:]:
        name = get(r, "Kernel Name")
        us = f(get(r, "gpu__time_duration.sum"))
        if units[col["gpu__time_duration.sum"]] == "ms":
            us *= 1e3
        rd, wr = mbytes(r, "dram__bytes_read.sum"), mbytes(r, "dram__bytes_write.sum")
        tens = f(get(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"))
        short = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        gb_s = (rd + wr) * 1e-3 / (us * 1e-6) if us else None
        out.append({"kernel": short, "grid": get(r, "launch__grid_size"), "us": us, "dram_MB": rd + wr,
                    "dram_GBps": gb_s, "frac_of_hbm": gb_s / hbm if gb_s else None,
                    "tensor_active_pct": tens})
    gemm = [o for o in out if "gemm_tf32_kernel" in o["kernel"] or "conv_window" in o["kernel"]]
    roles = ["conv1 fprop", "conv2 fprop", "conv3 fprop", "conv4 fprop", "conv5 fprop", "fc6 fprop",
             "fc7 fprop", "fc8 fprop", "fc8 wgrad", "fc8 dgrad", "fc7 wgrad", "fc7 dgrad", "fc6 wgrad",
             "fc6 dgrad", "conv5 wgrad", "conv5 dgrad", "conv4 wgrad", "conv4 dgrad", "conv3 wgrad",
             "conv3 dgrad", "conv2 wgrad", "conv2 dgrad", "conv1 wgrad"]
    if len(gemm) == len(roles):
        for o, role in zip(gemm, roles):
            o["role"] = role
    # algorithmic DRAM bytes of the CaffeNet b = 256 GEMMs (each operand read once,
    # the result written once; MB): the floor the measured DRAM MB compare to
    b = 256
    act = {"x1": b * 57 * 57 * 48, "y1": b * 55 * 55 * 96, "p1": b * 27 * 27 * 96, "y2": b * 27 * 27 * 256,
           "p2": b * 13 * 13 * 256, "y3": b * 13 * 13 * 384, "y4": b * 13 * 13 * 384, "y5": b * 13 * 13 * 256,
           "f6": b * 9216, "f7": b * 4096, "f8": b * 4096, "z8": b * 1000}
    wts = {"conv1": 96 * 432, "conv2": 256 * 2400, "conv3": 384 * 2304, "conv4": 384 * 3456,
           "conv5": 256 * 3456, "fc6": 9216 * 4096, "fc7": 4096 * 4096, "fc8": 4096 * 1000}
    io = {"conv1": ("x1", "y1"), "conv2": ("p1", "y2"), "conv3": ("p2", "y3"), "conv4": ("y3", "y4"),
          "conv5": ("y4", "y5"), "fc6": ("f6", "f7"), "fc7": ("f7", "f8"), "fc8": ("f8", "z8")}
    for o in out:
        if "role" in o:
            layer = o["role"].split()[0]
            i, y = io[layer]
            o["algorithmic_MB"] = 4e-6 * (act[i] + act[y] + wts[layer])
    tot = sum(o["us"] for o in out)
    res = {"launches": len(out), "sum_us": tot, "hbm_peak_GBps": hbm, "per_launch": out}
    json.dump(res, open(args[1], "w"), indent=1)
    if len(args) > 2:
        with open(args[2], "w") as fh:
            fh.write(f"| # | kernel | role | us | DRAM MB | algorithmic MB | GB/s | % of HBM {hbm:.0f} | tensor % |\n")
            fh.write("|---|---|---|---|---|---|---|---|---|\n")
            for i, o in enumerate(out):
                alg = f"{o['algorithmic_MB']:.1f}" if "algorithmic_MB" in o else ""
                fh.write(f"| {i} | {o['kernel'][:48]} | {o.get('role', '')} | {o['us']:.1f} | "
                         f"{o['dram_MB']:.1f} | {alg} | {o['dram_GBps'] or 0:.0f} | "
                         f"{100 * (o['frac_of_hbm'] or 0):.0f} | {o['tensor_active_pct'] or 0:.0f} |\n")
            fh.write(f"\nsum of launch times {tot:.0f} us (serialised, cold-cache ncu replays)\n")


if __name__ == "__main__":
    main()
