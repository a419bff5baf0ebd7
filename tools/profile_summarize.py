"""Summaries for profiles/ from tools/profile_round.sh outputs:
profiles/<tag>_launches.txt (launch list by kernel), profiles/<tag>_ncu_step.md
(ncu --set full table), profiles/traffic.json (DRAM bytes per launch per bench
stage, read by bench.py for roofline.traffic).

    python tools/profile_summarize.py r01
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import launch_summary  # noqa: E402
import ncu_summary  # noqa: E402

STAGES = {  # bench stage -> kernel name prefixes (ncu "Kernel Name" without args)
    "raster_fwd": ["void rcgs::raster_kernel<0,", "rcgs::raster_kernel<0,", "void rcgs::raster_kernel<6,",
                   "rcgs::raster_kernel<6,", "void rcgs::rec_kernel<0>", "rcgs::rec_kernel<0>"],
    "raster_bwd": ["void rcgs::raster_kernel<2,", "rcgs::raster_kernel<2,", "void rcgs::rec_kernel<1>",
                   "rcgs::rec_kernel<1>", "rcgs::rec_bwd_kernel", "bwd_finish_kernel"],
    "adam": ["rcgs::adam_prep_kernel", "rcgs::adam_fused_kernel", "rcgs::step_commit_kernel"],
    "color": ["rcgs::color_kernel"],
    "loss_grad": ["void rcgs::loss_", "rcgs::loss_"],
}


def stage_of(name):
    for st, prefixes in STAGES.items():
        if any(name.startswith(p) for p in prefixes):
            return st
    return "view_build"


def traffic_from_table(md_path, out_path, tag):
    """traffic.json from the step summary table: DRAM read + write per stage, and
    the SM-throughput / issue-active percentages of each stage's longest kernel."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg, top = {}, {}
    for line in open(md_path):
        cells = [c.strip() for c in line.strip().strip("|").split("|")]
        if len(cells) < 7 or cells[0] in ("kernel", "---") or cells[0].startswith("---"):
            continue
        b = 0.0
        for cell in cells[2:4]:
            v, u = cell.split()
            b += float(v) * scale.get(u, 1)
        st = stage_of(cells[0])
        agg[st] = agg.get(st, 0.0) + b
        us = float(cells[1].split()[0])
        if us > top.get(st, (0.0,))[0]:
            top[st] = (us, cells[0], float(cells[5].split()[0]), float(cells[6].split()[0]))
    stages = {}
    for k, v in agg.items():
        stages[k] = {"dram_bytes_per_launch": int(v)}
        if k in top:
            stages[k].update({"top_kernel": top[k][1], "sm_throughput_pct": top[k][2],
                              "issue_active_pct": top[k][3]})
    out = {"source": f"ncu --set full (default cache control), one optimizer step of C3: profiles/{tag}_ncu_step.md",
           "stages": stages}
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    return out


def main(tag, outdir="profiles"):
    os.makedirs(outdir, exist_ok=True)
    launch_summary.main("gpurun_out/launches.csv", f"{outdir}/{tag}_launches.txt")
    ncu_summary.main("gpurun_out/step_full.ncu-rep", f"{outdir}/{tag}_ncu_step.md")
    out = traffic_from_table(f"{outdir}/{tag}_ncu_step.md", f"{outdir}/traffic.json", tag)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", sys.argv[2] if len(sys.argv) > 2 else "profiles")
