"""Summarise ncu captures into profiles/ (one JSON line per kernel) and the launch list.
  python scripts/ncu_summary.py r01   (reads gpurun_out/r01_ncu_*.ncu-rep, r01_launches.csv)"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "gpc__cycles_elapsed.max.per_second",
        "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "smsp__sass_inst_executed_op_utcmma.sum"]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for rep in sorted(glob.glob(os.path.join(root, "gpurun_out", f"{tag}_ncu_*.ncu-rep"))):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for vals in rows[2:]:
            d = {"kernel": vals[hdr.index("Kernel Name")][:90], "capture": os.path.basename(rep)}
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    d[k] = [units[i], vals[i]]
            rd = float(d.get("dram__bytes_read.sum", ["", "0"])[1] or 0)
            wr = float(d.get("dram__bytes_write.sum", ["", "0"])[1] or 0)
            scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}
            d["traffic_bytes"] = int(rd * scale.get(d["dram__bytes_read.sum"][0], 1) +
                                     wr * scale.get(d["dram__bytes_write.sum"][0], 1))
            out.append(d)
    with open(os.path.join(root, "profiles", f"{tag}_ncu_summary.jsonl"), "w") as f:
        for d in out:
            f.write(json.dumps(d) + "\n")
    # launch list: kernel name + duration, warm-up excluded by the capture itself
    lpath = os.path.join(root, "gpurun_out", f"{tag}_launches.csv")
    if os.path.exists(lpath):
        lines = [l for l in open(lpath) if l.startswith('"')]
        rows = list(csv.reader(lines))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        with open(os.path.join(root, "profiles", f"{tag}_launches.csv"), "w") as f:
            f.write("kernel,gpu__time_duration_ns\n")
            for r in rows[1:]:
                f.write(f"\"{r[ki][:80]}\",{r[vi]}\n")
    for d in out:
        print(d["kernel"][:50], d["gpu__time_duration.sum"], d["traffic_bytes"],
              d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
              d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))


if __name__ == "__main__":
    main()
