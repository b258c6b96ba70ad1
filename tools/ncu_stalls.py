"""Stall-reason totals per SASS line range of an ncu report (source page):
python tools/ncu_stalls.py REPORT [LO HI] — without a range, per the top segments."""
import csv
import io
import subprocess
import sys


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    blk = out.split('"Kernel Name"')[1]
    rows = list(csv.reader(io.StringIO("\n".join(blk.splitlines()[1:]))))
    return rows[0], rows[1:]


def main():
    hdr, rows = load(sys.argv[1])
    st = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    lo = int(sys.argv[2]) if len(sys.argv) > 3 else 0
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(rows) - 1
    tot = {h: 0.0 for _, h in st}
    for r in rows[lo:hi + 1]:
        for i, h in st:
            tot[h] += float(r[i] or 0)
    s = sum(tot.values())
    print(f"lines {lo}-{hi}: {s:.0f} samples")
    for h, v in sorted(tot.items(), key=lambda x: -x[1]):
        if v > 0:
            print(f"  {h:24s} {v:8.0f} {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main()
