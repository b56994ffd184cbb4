#!/usr/bin/env python
"""Summarise an ncu report (``--set full``) and a launch list into markdown.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [gpurun_out/launches.csv] > profiles/x.md
    python tools/ncu_summary.py --traffic WORKLOAD gpurun_out/prof.ncu-rep   # -> profiles/ncu_traffic.json

Reads the report with ``ncu -i ... --page raw --csv`` (no GPU needed) and
prints, per profiled kernel, the counters the roofline of DESIGN.md section 7
is built from: duration, DRAM bytes, issue/pipe utilisation, occupancy,
shared-memory atomics and bank conflicts.  The optional launch list
(``--metrics gpu__time_duration.sum``) gives each kernel's share of the step.
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__inst_executed_op_shared_atom.sum", "shared atomics (warp inst)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "atomic bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM (smem limit)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
]


def raw(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def traffic(workload: str, report: str, out="profiles/ncu_traffic.json"):
    """DRAM bytes (read + write) per launch of each kernel of the capture,
    merged into profiles/ncu_traffic.json under `workload` (bench.py reports it
    as roofline.traffic)."""
    import json
    import os
    hdr, units, rows = raw(report)
    ki = hdr.index("Kernel Name")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rec = {}
    for r in rows:
        tot = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(key)
            tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        name = r[ki].split("(")[0].replace("void ", "").replace("ld::", "")
        rec.setdefault(name, []).append(tot)
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[workload] = {k: sum(v) / len(v) for k, v in rec.items()}
    data.setdefault("_source", {})[workload] = report
    json.dump(data, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[workload], indent=1))


def main():
    if sys.argv[1] == "--traffic":
        traffic(sys.argv[2], sys.argv[3])
        return
    report = sys.argv[1]
    hdr, units, rows = raw(report)
    print("## ncu --set full: %s\n" % report)
    names = [r[hdr.index("Kernel Name")] for r in rows]
    print("| metric | " + " | ".join(n.split("(")[0].replace("void ", "")[:40] for n in names) + " |")
    print("|---|" + "---|" * len(names))
    for key, label in METRICS:
        if key not in hdr:
            continue
        i = hdr.index(key)
        print("| %s (%s) | " % (label, units[i]) + " | ".join(r[i] for r in rows) + " |")
    if len(sys.argv) > 2:
        lrows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
        h = lrows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        d = collections.OrderedDict()
        for r in lrows[1:]:
            d.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(
                float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in d.values())
        print("\n## launch list (%s): per-kernel share of GPU time\n" % sys.argv[2])
        print("| kernel | launches | mean us | share |")
        print("|---|---|---|---|")
        for k, v in d.items():
            print("| %s | %d | %.1f | %.1f%% |" % (k, len(v), sum(v) / len(v) / 1e3,
                                                   100 * sum(v) / tot))


if __name__ == "__main__":
    main()
