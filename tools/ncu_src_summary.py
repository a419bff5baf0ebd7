"""Summarise an `ncu --page source --csv` dump (SASS view): stall totals, the
executed-opcode mix and the most-sampled instructions.

    ncu -i rep.ncu-rep --page source --csv -k regex:NAME > src.csv
    python tools/ncu_src_summary.py src.csv [top]
"""
import csv
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(hdr)]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    num = lambda v: int(v) if v not in ("", "-") else 0
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(num(r[iS]) for r in data)
    totE = sum(num(r[iE]) for r in data)
    print(f"samples {tot}  warp instructions executed {totE}")
    agg = Counter()
    for r in data:
        for c in cols:
            agg[c[6:]] += num(r[hdr.index(c)])
    print("stalls:", ", ".join(f"{k} {v / max(tot, 1):.1%}" for k, v in agg.most_common(10)))
    op = Counter()
    for r in data:
        o = r[1].strip().split()
        if not o:
            continue
        x = o[1] if o[0].startswith("@") else o[0]
        op[x.split(".")[0]] += num(r[iE])
    print("opcodes:", ", ".join(f"{k} {v / max(totE, 1):.1%}" for k, v in op.most_common(20)))
    for r in sorted(data, key=lambda r: -num(r[iS]))[:top_n]:
        st = sorted(((num(r[hdr.index(c)]), c[6:]) for c in cols), reverse=True)[:3]
        print(r[0][-5:], r[iS].rjust(6), num(r[iE]), r[1].strip()[:56].ljust(56), st)


if __name__ == "__main__":
    main()
