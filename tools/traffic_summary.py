"""profiles/r01_traffic_summary.json from a one-step ncu launch list
(tools/profile_step.py under ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum): DRAM bytes and serialised time
of the conv GEMM launches (gemm_tf32_kernel with an im2col mode != 0).

    python tools/traffic_summary.py profiles/<launches>.csv caffenet 256 tf32
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402


def main():
    path, net, b, prec = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    conv_bytes = conv_ms = 0.0
    n = 0
    launches = load(path)
    for l in launches:
        m = re.search(r"gemm_tf32_kernel<\s*\d+,\s*\w+,\s*\w+,\s*\w+,\s*(\d+)", l["kernel"])
        if m and int(m.group(1)) != 0:
            n += 1
            conv_bytes += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
            conv_ms += l.get("ms", 0.0)
    step_bytes = sum(l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
                     for l in launches)
    out = {"net": net, "per_gpu_batch": b, "precision": prec, "conv_gemm_launches": n,
           "conv_gemm_dram_bytes_per_step": conv_bytes, "conv_gemm_ncu_ms_per_step": conv_ms,
           "step_dram_bytes": step_bytes, "step_launches": len(launches),
           "source": f"{path} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum over one step, tools/profile_step.py)"}
    print(json.dumps(out, indent=1))
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "profiles", "r01_traffic_summary.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
