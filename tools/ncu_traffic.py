"""DRAM traffic per launch of a kernel from an `ncu --set full` report.

    python tools/ncu_traffic.py report.ncu-rep KERNEL_REGEX --config '{"model": ...}' [--out profiles/traffic.json]

Adds/updates entry KERNEL -> {dram_bytes_per_launch, read, write, duration_us,
config, report} in the JSON file (bench.py fills roofline.traffic from it when
the config matches its own workload).
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return hdr, units, r[2:]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("kernel")
    p.add_argument("--config", default="{}")
    p.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "profiles", "traffic.json"))
    a = p.parse_args()
    hdr, units, data = rows(a.report)
    col = {n: i for i, n in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    hits = [d for d in data if re.search(a.kernel, d[col["Kernel Name"]])]
    if not hits:
        raise SystemExit(f"no launch of {a.kernel} in {a.report}")
    d = hits[0]

    def val(name, table):
        return float(d[col[name]].replace(",", "")) * table.get(units[col[name]], 1)

    rd = val("dram__bytes_read.sum", scale)
    wr = val("dram__bytes_write.sum", scale)
    dur = val("gpu__time_duration.sum", tscale)
    doc = json.load(open(a.out)) if os.path.exists(a.out) else {}
    name = re.sub(r"\W", "", a.kernel.split(":")[-1])
    doc[name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "duration_us": dur,
                 "config": json.loads(a.config), "report": os.path.basename(a.report)}
    # what actually bounds the kernel: issue and the busiest pipes (ALU for rANS)
    for key, metric in (("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                        ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                        ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
                        ("l1tex_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active")):
        if metric in col:
            doc[name][key] = float(d[col[metric]].replace(",", ""))
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc[name]))


if __name__ == "__main__":
    main()
