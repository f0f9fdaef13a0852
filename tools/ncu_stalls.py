"""Warp-stall shares (pc sampling) and headline counters of one ncu capture:
    python tools/ncu_stalls.py <report.ncu-rep> [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued") and v[i] not in ("", "n/a"):
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
        tot = sum(stalls.values()) or 1.0
        rec = {k: (v[h.index(k)] + " " + u[h.index(k)]) for k in KEYS if k in h}
        rec["stall_share"] = {k: round(x / tot, 4) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]) if x / tot > 0.005}
        out.append(rec)
    res = {"source": sys.argv[1], "launches": out}
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
