"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def main(path, out=None):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'total_us':>12} {'launches':>8} {'us/launch':>10} {'share':>6}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[1]:12.1f} {v[0]:8d} {v[1] / v[0]:10.1f} {100 * v[1] / tot:5.1f}%  {k}")
    lines.append(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
