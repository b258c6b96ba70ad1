"""Whole SASS listing of an ncu report's first kernel with per-instruction executed counts
and stall samples (needs --import-source): python tools/ncu_sass_dump.py REPORT OUT.txt
Columns: index, warp instructions executed, stall samples, thread instructions executed
(if present), SASS.  Used to attribute a kernel's instruction count to its code regions."""
import csv
import io
import subprocess
import sys


def main(path, out_path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blk = out.split('"Kernel Name"')[1]
    rows = list(csv.reader(io.StringIO("\n".join(blk.splitlines()[1:]))))
    hdr, rows = rows[0], rows[1:]
    isrc, ism, iex = (hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"),
                      hdr.index("Instructions Executed"))
    ith = hdr.index("Thread Instructions Executed") if "Thread Instructions Executed" in hdr else -1
    with open(out_path, "w") as f:
        f.write("# columns: " + " | ".join(hdr) + "\n")
        for i, r in enumerate(rows):
            th = r[ith] if ith >= 0 else ""
            f.write(f"{i}\t{r[iex]}\t{r[ism]}\t{th}\t{r[isrc].strip()}\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
