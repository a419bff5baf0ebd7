"""Summarise an ncu --set full report (.ncu-rep) as a markdown table:
per kernel launch duration, DRAM bytes, throughput, issue / occupancy and the
top warp-stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep [out.md]"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thru %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes/inst"),
    ("launch__registers_per_thread", "regs"),
]


def main(path, out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(k[1] for k in KEYS) + " | top stalls (warps per issue) |",
             "|---" * (len(KEYS) + 2) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:40]
        vals = []
        for key, _ in KEYS:
            if key in hdr:
                i = hdr.index(key)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        top = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:4])
        lines.append(f"| {name} | " + " | ".join(vals) + f" | {top} |")
    text = "\n".join(lines)
    if out:
        with open(out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
