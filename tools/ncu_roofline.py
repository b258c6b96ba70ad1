#!/usr/bin/env python
"""Summarise one kernel of an `ncu --set full` report into the roofline evidence bench.py
attaches to its JSON line (roofline.ncu / roofline.traffic):

    python tools/ncu_roofline.py report.ncu-rep <workload> <out.json> [kernel-substring]

Per launch: duration, DRAM bytes (read + write), L2 (lts) bytes, the achieved DRAM and L2
bandwidths, issue-slot utilisation, FMA/ALU pipe utilisation, warps active, and the top
warp-stall reasons."""
import csv
import json
import subprocess
import sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "lts_sectors": ("lts__t_sectors.sum", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    "lts_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "warp_inst": ("smsp__inst_executed.sum", 1.0),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1.0),
}
UNIT_SCALE = {"ms": 1e6, "us": 1e3, "ns": 1, "sector": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
              "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}


def num(v, unit):
    v = float(v.replace(",", ""))
    return v * UNIT_SCALE.get(unit, 1.0)


def main(path, workload, out, want=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    picked = [r for r in rows[2:] if want is None or want in r[name_i]]
    if not picked:
        raise SystemExit(f"no kernel matching {want!r} in {path}")
    r = picked[0]
    d = {"workload": workload, "kernel": r[name_i][:160], "report": path}
    for key, (m, scale) in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            try:
                d[key] = num(r[i], units[i]) * scale
            except ValueError:
                d[key] = r[i]
    t = d["duration_ms"] / 1e3
    d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
    d["dram_gbs"] = d["dram_bytes_per_launch"] / t / 1e9
    d["lts_bytes"] = 32.0 * d.get("lts_sectors", 0)        # 32-byte L2 sectors
    d["l2_gbs"] = d["lts_bytes"] / t / 1e9
    stalls = {h: r[i] for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("_not_issued")}
    tot = sum(float(v.replace(",", "") or 0) for v in stalls.values())
    if tot:
        top = sorted(((float(v.replace(",", "") or 0) / tot, k.split("stalled_")[-1])
                      for k, v in stalls.items()), reverse=True)[:6]
        d["stall_share"] = {k: round(f, 3) for f, k in top}
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4], sys.argv[4] if len(sys.argv) > 4 else None)
