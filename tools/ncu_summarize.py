"""Summarise `ncu --set full` captures into profiles/ncu_summary.json (one entry per kernel key).

    python tools/ncu_summarize.py KEY REP.ncu-rep "description" [KEY REP "description" ...]

Per entry: the metrics the bench line and DESIGN.md cite (duration, SM clock, DRAM bytes read and
written per launch, issue and pipe activity, occupancy, registers, grid, instructions) and the
warp-stall breakdown from the source page. `dram_bytes_per_launch` (read + write) is what bench.py
reports as `roofline.traffic`.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")
WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv(rep, "--page", "raw")
    h, units, v = rows[0], rows[1], rows[2]
    res = {}
    for k, u, x in zip(h, units, v):
        if k in WANT:
            res[k] = f"{x} {u}".strip()
    rb = wb = None
    for k, u, x in zip(h, units, v):
        if k == "dram__bytes_read.sum":
            rb = float(x) * UNIT_SCALE.get(u, 1.0)
        if k == "dram__bytes_write.sum":
            wb = float(x) * UNIT_SCALE.get(u, 1.0)
    return res, (rb + wb) if rb is not None and wb is not None else None


def stall_breakdown(rep):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = rows[1]
    names = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: h.index(c) for c in names}
    tot = {c: 0 for c in names}
    for r in rows[2:]:
        for c in names:
            try:
                tot[c] += int(r[idx[c]] or 0)
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    return {c[6:]: round(100.0 * v / s, 1) for c, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v}


def main(argv):
    if len(argv) % 3 != 0:
        raise SystemExit(__doc__)
    doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for k in range(0, len(argv), 3):
        key, rep, desc = argv[k:k + 3]
        metrics, traffic = raw_metrics(rep)
        doc[key] = {"kernel": desc, "dram_bytes_per_launch": traffic, "ncu": metrics,
                    "warp_stall_pct": stall_breakdown(rep),
                    "source": f"{os.path.relpath(rep, ROOT)}, ncu --set full --import-source on "
                              f"--clock-control none (one launch)"}
        print(key, json.dumps(doc[key], indent=1))
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
