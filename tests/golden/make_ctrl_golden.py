"""Generates the control-plane parity scenarios and their golden digests.

Each scenario is a reference-schema experiment config plus its own seeded
trace / length CSVs (tests/golden/ctrl/<name>/). The UNMODIFIED reference
simulator (oracle/_ref/ref_capture, built from /root/reference/proj by
oracle/Makefile) is run on every scenario and the sha256 of each artifact it
writes (events.jsonl, requests.csv, summary.json, ttft_cdf.csv, ops.csv
ScaleOp transcript, steps.csv launched plans, hash.txt state hash) is stored in
golden.json. tests/test_control_parity.py re-runs our control plane on the
same inputs and requires byte-identical artifacts.

usage: python tests/golden/make_ctrl_golden.py   (needs oracle/_ref built)
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2507_00507_b200 import tables  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "ctrl")
REF = os.path.join(ROOT, "oracle", "_ref", "ref_capture")
ARTIFACTS = ["events.jsonl", "requests.csv", "summary.json", "ttft_cdf.csv", "ops.csv", "steps.csv", "hash.txt"]


def rel(p: str) -> str:
    return os.path.relpath(p, ROOT)


def poisson_trace(path, fns, window, rate_fn, seed, phases=None):
    """Per-function exponential gaps (rate may vary by phase: [(t0, t1, {fn: rate})])."""
    rng = np.random.default_rng(seed)
    rows = []
    for f in fns:
        t = 0.0
        while True:
            rate = rate_fn(f, t, phases)
            t += rng.exponential(1.0 / rate)
            if t >= window:
                break
            rows.append((t, f))
    rows.sort()
    with open(path, "w") as fh:
        fh.write("timestamp_s,function_id\n")
        for t, f in rows:
            fh.write(f"{t:.6f},{f}\n")
    return len(rows)


def lengths_csv(path, n, seed, in_lo=49, in_hi=900, out_lo=8, out_hi=239):
    """Synthetic length dataset with the shape of the reference's example data."""
    rng = np.random.default_rng(seed)
    with open(path, "w") as fh:
        fh.write("input_tokens,output_tokens\n")
        for _ in range(n):
            fh.write(f"{int(rng.integers(in_lo, in_hi + 1))},{int(rng.integers(out_lo, out_hi + 1))}\n")


TEMPLATES = {
    "1b": {"name": "1b", "size_class": "1b", "param_gb": 2.2, "kv_kib_per_token": 22, "max_seq_len": 2048,
           "max_batch": 8},
    "3b": {"name": "3b", "size_class": "3b", "param_gb": 6.4, "kv_kib_per_token": 112, "max_seq_len": 4096,
           "max_batch": 8},
    "7b": {"name": "7b", "size_class": "7b", "param_gb": 13.5, "kv_kib_per_token": 512, "max_seq_len": 4096,
           "max_batch": 8},
    "13b": {"name": "13b", "size_class": "13b", "param_gb": 26.0, "kv_kib_per_token": 800, "max_seq_len": 4096,
            "max_batch": 8},
}


def const_rate(r):
    return lambda f, t, ph: r


def scenario(name, *, nodes, templates, assignment, n_fns, window, rate_fn, seed, gpu_tables=True,
             policy=None, perf=None, n_len=200, len_kw=None, tpl_over=None, sample=None, measured=False):
    d = os.path.join(GOLD, name)
    os.makedirs(d, exist_ok=True)
    fns = [f"fn{i:02d}" for i in range(n_fns)]
    n_req = poisson_trace(os.path.join(d, "trace.csv"), fns, window, rate_fn, seed)
    lengths_csv(os.path.join(d, "lengths.csv"), n_len, seed + 1, **(len_kw or {}))
    tpls = []
    for t in templates:
        tt = dict(TEMPLATES[t]) if isinstance(t, str) else dict(t)
        tt.update((tpl_over or {}).get(tt["name"], {}))
        tpls.append(tt)
    cfg = {
        "seed": seed,
        "cluster": {"nodes": nodes},
        "models": {"templates": tpls, "assignment": assignment},
        "perf": {"overestimate_factor": 1.10, "max_len": 4096, "max_batch": 8},
        "workload": {"trace": rel(os.path.join(d, "trace.csv")), "lengths": rel(os.path.join(d, "lengths.csv")),
                     "window_s": window, "sample_functions": sample or n_fns},
        "slo": {"ttft_base_s": 2.0, "ttft_per_token_divisor": 512.0, "tpot_s": 0.25},
        "policy": {"kind": "mesh", "watermark_pct": 20.0, "keep_alive_s": 1.0},
        "output": {"dir": rel(os.path.join(d, "out")), "event_log": True},
    }
    if gpu_tables:
        path = tables.measured_table_path if measured else tables.model_table_path
        cfg["perf"]["tables"] = {f"{t['size_class']}:gpu": rel(path(t["size_class"])) for t in tpls}
    if measured:  # B200-measured tables and CostParams (tools/measure_tables.py), fed to both sides
        cfg["perf"]["gpu"] = tables.measured_cost_params()
    if perf:
        cfg["perf"].update(perf)
    if policy:
        cfg["policy"].update(policy)
    with open(os.path.join(d, "config.json"), "w") as fh:
        json.dump(cfg, fh, indent=2)
    return d, n_req


def burst_rate(base, mid, hot_rate, cold_rate, hot):
    def f(fn, t, ph):
        if t < 30:
            return base
        if t < 90:
            return mid
        return hot_rate if fn in hot else cold_rate
    return f


def build_scenarios():
    gpu = lambda n, mem: {"class": "gpu", "count": n, "mem_gb": mem}  # noqa: E731
    cpu = lambda n, mem: {"class": "cpu", "count": n, "mem_gb": mem}  # noqa: E731
    out = []
    out.append(scenario("c1_1b_poisson", nodes=[gpu(1, 160.0)], templates=["1b"], assignment=["1b"], n_fns=1,
                        window=120.0, rate_fn=const_rate(4.0), seed=11))
    out.append(scenario("c2_colocated", nodes=[gpu(1, 160.0)], templates=["1b", "3b"],
                        assignment=["1b", "3b", "1b", "3b"], n_fns=4, window=120.0, rate_fn=const_rate(1.5), seed=12))
    # the same node priced by the B200-measured tables and CostParams
    out.append(scenario("c2_measured", nodes=[gpu(1, 160.0)], templates=["1b", "3b"],
                        assignment=["1b", "3b", "1b", "3b"], n_fns=4, window=120.0, rate_fn=const_rate(4.0), seed=23,
                        measured=True))
    hot = {f"fn{i:02d}" for i in range(3)}
    out.append(scenario("c3_bursty", nodes=[gpu(1, 160.0)], templates=["1b", "3b", "7b"],
                        assignment=["1b", "3b", "7b"], n_fns=8, window=150.0,
                        rate_fn=burst_rate(0.08, 0.28, 0.8, 0.03, hot), seed=13))
    out.append(scenario("c4_pressure", nodes=[gpu(1, 60.0)], templates=["7b", "13b"], assignment=["7b", "13b"],
                        n_fns=4, window=120.0, rate_fn=const_rate(0.6), seed=14,
                        tpl_over={"7b": {"min_total_len": 256, "avg_output_seed": 8, "avg_output_fixed": True},
                                  "13b": {"min_total_len": 256, "avg_output_seed": 8, "avg_output_fixed": True}}))
    out.append(scenario("c5_fleet", nodes=[gpu(4, 160.0)], templates=["1b", "3b", "7b"],
                        assignment=["1b", "3b", "7b"], n_fns=32, window=90.0, rate_fn=const_rate(0.3), seed=15))
    # reference-style heterogeneous cluster on the reference's synthetic tables (CPU-first routing)
    out.append(scenario("ref_hetero", nodes=[cpu(2, 256.0), gpu(2, 80.0)],
                        templates=[{"name": "7b", "size_class": "7b", "param_gb": 14.0, "kv_kib_per_token": 512,
                                    "max_seq_len": 4096, "max_batch": 256}],
                        assignment=["7b"], n_fns=12, window=120.0, rate_fn=const_rate(0.15), seed=16,
                        gpu_tables=False, perf={"max_batch": 256}))
    out.append(scenario("ref_mixed_defrag_off", nodes=[cpu(2, 256.0), gpu(2, 80.0)],
                        templates=[{"name": "3b", "size_class": "3b", "param_gb": 6.4, "kv_kib_per_token": 224,
                                    "max_seq_len": 4096, "max_batch": 256},
                                   {"name": "13b", "size_class": "13b", "param_gb": 26.0, "kv_kib_per_token": 800,
                                    "max_seq_len": 4096, "max_batch": 256}],
                        assignment=["3b", "13b"], n_fns=10, window=120.0, rate_fn=const_rate(0.2), seed=17,
                        gpu_tables=False, perf={"max_batch": 256}, policy={"disable_defrag": True}))
    out.append(scenario("ref_exclusive", nodes=[cpu(2, 256.0), gpu(2, 80.0)],
                        templates=[{"name": "7b", "size_class": "7b", "param_gb": 14.0, "kv_kib_per_token": 512,
                                    "max_seq_len": 4096, "max_batch": 256}],
                        assignment=["7b"], n_fns=8, window=90.0, rate_fn=const_rate(0.2), seed=18,
                        gpu_tables=False, perf={"max_batch": 256}, policy={"kind": "exclusive_cpu"}))
    out.append(scenario("c3_novalidation_jitter", nodes=[gpu(2, 100.0)], templates=["1b", "3b", "7b"],
                        assignment=["1b", "3b", "7b"], n_fns=6, window=90.0, rate_fn=const_rate(0.4), seed=19,
                        policy={"disable_validation": True, "jitter_pct": 10.0}))
    hot_cold = lambda h, c: (lambda f, t, ph: h if f == "fn00" else c)  # noqa: E731
    under = {"min_total_len": 256, "avg_output_seed": 4, "avg_output_fixed": True}
    # KV underestimation under memory pressure: ensure_kv_capacity evicts (cluster.cpp:730-751)
    out.append(scenario("c4_evict", nodes=[gpu(1, 15.0)], templates=["7b"], assignment=["7b"], n_fns=3,
                        window=90.0, rate_fn=hot_cold(3.0, 0.3), seed=22, tpl_over={"7b": under}))
    out.append(scenario("c4_mixed_evict", nodes=[gpu(1, 22.0)], templates=["3b", "7b"], assignment=["7b", "3b"],
                        n_fns=4, window=60.0, rate_fn=hot_cold(5.0, 1.0), seed=57,
                        tpl_over={"7b": under, "3b": under}))
    return out


# Scenario on which the reference itself fails with the eviction ping-pong
# defect; parity means failing identically.
def defect_scenario():
    gpu = lambda n, mem: {"class": "gpu", "count": n, "mem_gb": mem}  # noqa: E731
    under = {"min_total_len": 256, "avg_output_seed": 4, "avg_output_fixed": True}
    return scenario("c4_defect_pingpong", nodes=[gpu(1, 14.5)], templates=["7b"], assignment=["7b"], n_fns=3,
                    window=90.0, rate_fn=lambda f, t, ph: 3.0 if f == "fn00" else 0.3, seed=22,
                    tpl_over={"7b": under})


def digest(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        h.update(fh.read())
    return h.hexdigest()


def main() -> None:
    if not os.path.exists(REF):
        sys.exit("oracle/_ref/ref_capture missing: run `make -C oracle`")
    tables.write_model_tables()
    for d, n_req in build_scenarios():
        out = os.path.join("/tmp", "ctrl_golden_" + os.path.basename(d))
        subprocess.run([REF, "run", os.path.join(d, "config.json"), out], cwd=ROOT, check=True)
        gold = {"requests": n_req, "artifacts": {a: digest(os.path.join(out, a)) for a in ARTIFACTS}}
        with open(os.path.join(out, "events.jsonl")) as fh:
            gold["events"] = sum(1 for _ in fh)
        with open(os.path.join(out, "summary.json")) as fh:
            gold["summary"] = json.load(fh)
        with open(os.path.join(d, "golden.json"), "w") as fh:
            json.dump(gold, fh, indent=1)
        print(os.path.basename(d), n_req, "requests", gold["events"], "events", gold["summary"]["slo_compliant_rate"])
    d, _ = defect_scenario()
    r = subprocess.run([REF, "run", os.path.join(d, "config.json"), "/tmp/ctrl_golden_defect"], cwd=ROOT,
                       capture_output=True, text=True)
    with open(os.path.join(d, "expected_error.json"), "w") as fh:
        json.dump({"exit_code": r.returncode, "stderr": r.stderr.strip()}, fh, indent=1)
    print("defect scenario:", r.returncode, r.stderr.strip())


if __name__ == "__main__":
    main()
