"""Summarise ncu output into the committed profiles/ files.

  python tools/ncu_summary.py launches <launches.csv> <out.json>
      per-kernel launch count, total/avg time and share of the launch list
      (ncu --metrics gpu__time_duration.sum --csv; cold-cache, serialised)
  python tools/ncu_summary.py full <report.ncu-rep> <out.json> [bytes_per_launch ...]
      per captured launch: duration, DRAM read+write bytes, achieved DRAM
      throughput, registers, occupancy, and (if algorithmic bytes are given,
      one per launch) traffic / algorithmic ratio
"""
import collections
import csv
import io
import json
import subprocess
import sys


def _ns(value: str, unit: str) -> float:
    v = float(value.replace(",", ""))
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
                "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}.get(unit, 1)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += _ns(r[vi], r[ui])
    tot = sum(t for _, t in agg.values())
    res = {"source": path, "total_ms": tot / 1e6, "kernels": [
        {"kernel": k, "launches": n, "total_ms": t / 1e6, "avg_us": t / n / 1e3, "share": t / tot}
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]}
    json.dump(res, open(out, "w"), indent=1)
    for k in res["kernels"][:12]:
        print(f"{k['kernel'][:58]:58s} n={k['launches']:6d} {k['total_ms']:9.2f} ms {k['share']:6.1%} avg {k['avg_us']:8.1f} us")


METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed": "xbar_to_l1_pct",
}


def full(rep, out, algo):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for m, key in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    val = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if key == "duration":
                    val = _ns(r[i], u) / 1e3
                    key = "duration_us"
                elif key in ("dram_read", "dram_write"):
                    val = float(r[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    key += "_bytes"
                d[key] = val
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
            d["dram_GBps"] = d["dram_bytes"] / (d["duration_us"] * 1e3)
        res.append(d)
    for d, a in zip(res, algo):
        if a <= 0:
            continue
        d["algorithmic_bytes"] = a
        d["traffic_over_algorithmic"] = d["dram_bytes"] / a
        d["algorithmic_GBps"] = a / (d["duration_us"] * 1e3)
    summary = {"source": rep, "launches": res}
    if res and "dram_bytes" in res[0]:
        summary["dram_bytes_per_launch"] = sum(d["dram_bytes"] for d in res) / len(res)
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], [float(x) for x in sys.argv[4:]])
