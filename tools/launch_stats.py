"""Per-kernel totals and shares from an ncu launch list (gpu__time_duration.sum CSV)."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def main(path, skip_first_half=True):
    data = [d for d in load(path) if d["Metric Name"] == "gpu__time_duration.sum"]
    grids = {d["ID"]: d["Metric Value"] for d in load(path) if d["Metric Name"] == "launch__grid_size"}
    if skip_first_half:             # tools/prof_step.py runs the step twice: keep the 2nd
        data = data[len(data) // 2:]
    agg = defaultdict(lambda: [0, 0.0, []])
    for d in data:
        k = d["Kernel Name"].split("(")[0][:60]
        v = float(d["Metric Value"])
        agg[k][0] += 1
        agg[k][1] += v
        agg[k][2].append((v, grids.get(d["ID"], "?")))
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total us':>10} {'share':>6} {'mean us':>8}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:8d} {v[1]/1e3:10.1f} {100*v[1]/tot:5.1f}% {v[1]/v[0]/1e3:8.2f}  {k}")
    print(f"total {tot/1e3:.1f} us over {len(data)} launches")
    return agg


if __name__ == "__main__":
    agg = main(sys.argv[1])
    if len(sys.argv) > 2:
        k = [k for k in agg if sys.argv[2] in k][0]
        xs = agg[k][2]
        import statistics
        ds = sorted(x[0] / 1e3 for x in xs)
        print("percentiles us:", [round(ds[int(p * (len(ds) - 1))], 1) for p in (0, .1, .5, .9, 1)])
        print("first 20:", [(round(a / 1e3, 1), g) for a, g in xs[:20]])
