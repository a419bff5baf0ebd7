"""Markdown summary of an ncu --set full raw CSV (one row per kernel launch):
duration, DRAM traffic and bandwidth, SM / fp64-pipe / issue utilisation."""

from __future__ import annotations

import csv
import sys


def main():
    path, tag = sys.argv[1], sys.argv[2]
    with open(path) as fh:
        rows = list(csv.reader(fh))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}

    def get(r, name, default=float("nan")):
        i = col.get(name)
        if i is None or i >= len(r):
            return default
        try:
            return float(r[i].replace(",", ""))
        except ValueError:
            return default

    fp64 = [h for h in head if "fp64" in h and h.endswith("pct_of_peak_sustained_active")]
    print(f"# {tag}: ncu --set full of the 8(f) row kernels (tools/profile_extras.sh)\n")
    print("C3 view 0 (1M gaussians, 1920x1080): one `stereo_hv_depth_device` with backfill, one")
    print("`load_scene_ply_device` + `save_scene_ply_device` of the C3 scene.  Cold-cache, serialised")
    print("replays (ncu), so durations are upper bounds of the in-pipeline times.\n")
    print(f"fp64 column: `{fp64[0] if fp64 else 'n/a'}`\n")
    print("| kernel | grid | duration us | DRAM read MB | DRAM write MB | DRAM GB/s | SM thru % | issue active % | fp64 pipe % |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in data:
        name = r[col["Kernel Name"]][:60]
        dur_ns = get(r, "gpu__time_duration.sum")
        unit = units[col["gpu__time_duration.sum"]]
        dur_us = dur_ns / 1e3 if unit == "nsecond" else (dur_ns if unit == "usecond" else dur_ns * 1e3)
        rd = get(r, "dram__bytes_read.sum")
        wr = get(r, "dram__bytes_write.sum")
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        rd *= scale.get(units[col["dram__bytes_read.sum"]], 1e-6)
        wr *= scale.get(units[col["dram__bytes_write.sum"]], 1e-6)
        bw = (rd + wr) / 1e3 / (dur_us / 1e6) if dur_us else float("nan")
        sm = get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
        issue = get(r, "sm__inst_issued.avg.pct_of_peak_sustained_active")
        f64 = get(r, fp64[0]) if fp64 else float("nan")
        grid = r[col["Grid Size"]] if "Grid Size" in col else ""
        print(f"| `{name}` | {grid} | {dur_us:.1f} | {rd:.1f} | {wr:.1f} | {bw:.0f} | {sm:.1f} | {issue:.1f} | {f64:.1f} |")


if __name__ == "__main__":
    main()
