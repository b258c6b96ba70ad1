"""Per-SASS-line hot spots of an ncu report (needs -lineinfo + --import-source):
python tools/ncu_source.py REPORT [N] — top instructions by stall samples, plus totals."""
import csv
import io
import subprocess
import sys


def main(path, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    for blk in blocks[1:2]:
        lines = blk.splitlines()
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr, rows = rows[0], rows[1:]
        ia, isrc, ism, iex = (hdr.index("Address"), hdr.index("Source"),
                              hdr.index("Warp Stall Sampling (All Samples)"),
                              hdr.index("Instructions Executed"))
        tot_s = sum(float(r[ism] or 0) for r in rows)
        tot_e = sum(float(r[iex] or 0) for r in rows)
        print(f"total samples {tot_s:.0f}, warp instructions executed {tot_e:.0f}")
        for i, r in enumerate(rows):
            r.append(i)
        top = sorted(rows, key=lambda r: -float(r[ism] or 0))[:n]
        for r in sorted(top, key=lambda r: r[-1]):
            print(f"{r[-1]:5d} {float(r[ism]):7.0f} {100 * float(r[ism]) / tot_s:5.1f}% "
                  f"{float(r[iex]):10.0f}  {r[isrc].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
