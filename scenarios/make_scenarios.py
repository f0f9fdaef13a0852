"""Bench scenarios (not parity goldens): traces that keep the co-located
instances in their capacity regime, so end-to-end tokens/s measures the
serving path rather than the arrival rate.

  c2_saturated  BASELINE configs[1] (C2): four functions on [1b, 3b, 1b, 3b],
                Poisson 16 req/s per function for 10 s. On the control plane
                alone (B200 roofline-model cost tables) this is past the knee:
                modeled ~6.7k tokens/s with ~97 % of requests inside the
                TTFT/TPOT SLO (8 req/s: 4.1k, 100 %; 32 req/s: 7.0k, 50 %).

  c2_saturated_b200  the same trace priced by the B200-measured cost tables and
                CostParams (tools/measure_tables.py), so the
                control plane's virtual schedule runs at the data plane's real
                speed. bench.py's e2e runs this one.

  c3_b200/s{K}  BASELINE configs[2] (C3), the bench's e2e: 8 functions on
                [1b, 3b, 7b, 1b, 3b, 7b, 1b, 3b] under the acceptance overload
                trace's three phases (proj/tests/acceptance_main.cpp:462-488:
                0.08/s, then 0.28/s, then 0.8/s for 6 hot functions and
                0.03/s for the rest), compressed into a 30 s window (phases
                6 / 12 / 12 s) with every rate scaled by K (the lambda of the
                capacity sweep). Measured B200 tables and CostParams; run with
                runtime.clock = "wall", so step completions, emission times and
                SLO compliance come from CUDA events, not from the tables; the
                admission replay divides its pessimistic step costs by the
                measured co-location speedup (instances step concurrently on
                their SM quotas, tools/measure_colocation.py); replicas of a
                model on the GPU share its weights (runtime.shared_weights:
                the data plane keeps one weight set per model per GPU).

  c4_b200       BASELINE configs[3] (C4): 7B + 13B functions (two each) on one
                B200 whose node memory (44 GB) is far below their KV demand, with the
                output-length estimator fixed low (avg_output_seed 4, min_total_len
                256; the pattern of proj/tests/test_cluster.cpp:289-325), so
                ensure_kv_capacity evicts running requests (cluster.cpp:730-751) and
                the data plane swaps their KV to pinned host memory and back. Hot /
                cold Poisson arrivals for 30 s, measured tables, wall clock.

    python scenarios/make_scenarios.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, ROOT)

from make_ctrl_golden import TEMPLATES, const_rate, lengths_csv, poisson_trace  # noqa: E402

C3_MODELS = ["1b", "3b", "7b", "1b", "3b", "7b", "1b", "3b"]
C3_SCALES = (1, 2, 4, 6, 8, 10, 12, 14, 16)
C3_WINDOW = 30.0
# runtime.colocation_speedup: measured by tools/measure_colocation.py (profiles/colocation_r02.json):
# the C3 node's step sequence takes 4.51 s on one lane and 2.70 s on eight concurrent lanes
C3_COLOCATION_SPEEDUP = 1.67


def c3_rate(scale, window):
    hot = {f"fn{i:02d}" for i in range(6)}

    def f(fn, t, ph):
        if t < 0.2 * window:
            return 0.08 * scale
        if t < 0.6 * window:
            return 0.28 * scale
        return (0.8 if fn in hot else 0.03) * scale
    return f


def make_c4(d=None, hot=6.0, cold=1.0, mem_gb=44.0):
    from paper_2507_00507_b200 import tables
    d = d or os.path.join(HERE, "c4_b200")
    os.makedirs(d, exist_ok=True)
    lengths_csv(os.path.join(d, "lengths.csv"), 200, 58)
    rate = lambda f, t, ph: hot if f in ("fn00", "fn01") else cold  # noqa: E731
    n = poisson_trace(os.path.join(d, "trace.csv"), [f"fn{i:02d}" for i in range(4)], 30.0, rate, 58)
    under = {"min_total_len": 256, "avg_output_seed": 4, "avg_output_fixed": True}
    tpls = []
    for t in ("7b", "13b"):
        tt = dict(TEMPLATES[t])
        tt.update(under)
        tpls.append(tt)
    cfg = {
        "seed": 58,
        "cluster": {"nodes": [{"class": "gpu", "count": 1, "mem_gb": mem_gb}]},
        "models": {"templates": tpls, "assignment": ["7b", "13b"]},
        "perf": {"overestimate_factor": 1.10, "max_len": 4096, "max_batch": 8,
                 "tables": {f"{sc}:gpu": os.path.relpath(tables.measured_table_path(sc), ROOT) for sc in ("7b", "13b")},
                 "gpu": tables.measured_cost_params()},
        "workload": {"trace": os.path.relpath(os.path.join(d, "trace.csv"), ROOT),
                     "lengths": os.path.relpath(os.path.join(d, "lengths.csv"), ROOT),
                     "window_s": 30.0, "sample_functions": 4},
        "slo": {"ttft_base_s": 2.0, "ttft_per_token_divisor": 512.0, "tpot_s": 0.25},
        "policy": {"kind": "mesh", "watermark_pct": 20.0, "keep_alive_s": 1.0},
        "runtime": {"clock": "wall", "slots": 64, "colocation_speedup": C3_COLOCATION_SPEEDUP, "shared_weights": True},
        "output": {"dir": os.path.relpath(os.path.join(d, "out"), ROOT), "event_log": False},
    }
    with open(os.path.join(d, "config.json"), "w") as fh:
        json.dump(cfg, fh, indent=2)
    print("c4_b200:", n, "requests")


def make_c3():
    from paper_2507_00507_b200 import tables
    base = os.path.join(HERE, "c3_b200")
    os.makedirs(base, exist_ok=True)
    lengths_csv(os.path.join(base, "lengths.csv"), 200, 4242)  # the example length set's ranges
    for k in C3_SCALES:
        d = os.path.join(base, f"s{k}")
        os.makedirs(d, exist_ok=True)
        n = poisson_trace(os.path.join(d, "trace.csv"), [f"fn{i:02d}" for i in range(8)], C3_WINDOW,
                          c3_rate(k, C3_WINDOW), 4242 + k)
        cfg = {
            "seed": 13,
            "cluster": {"nodes": [{"class": "gpu", "count": 1, "mem_gb": 150.0}]},
            "models": {"templates": [dict(TEMPLATES[t]) for t in ("1b", "3b", "7b")], "assignment": C3_MODELS},
            "perf": {"overestimate_factor": 1.10, "max_len": 4096, "max_batch": 8,
                     "tables": {f"{sc}:gpu": os.path.relpath(tables.measured_table_path(sc), ROOT)
                                for sc in ("1b", "3b", "7b")},
                     "gpu": tables.measured_cost_params()},
            "workload": {"trace": os.path.relpath(os.path.join(d, "trace.csv"), ROOT),
                         "lengths": os.path.relpath(os.path.join(base, "lengths.csv"), ROOT),
                         "window_s": C3_WINDOW, "sample_functions": 8},
            "slo": {"ttft_base_s": 2.0, "ttft_per_token_divisor": 512.0, "tpot_s": 0.25},
            "policy": {"kind": "mesh", "watermark_pct": 20.0, "keep_alive_s": 1.0},
            "runtime": {"clock": "wall", "slots": 64, "colocation_speedup": C3_COLOCATION_SPEEDUP,
                        "shared_weights": True},
            "output": {"dir": os.path.relpath(os.path.join(d, "out"), ROOT), "event_log": False},
        }
        with open(os.path.join(d, "config.json"), "w") as fh:
            json.dump(cfg, fh, indent=2)
        print(f"c3_b200/s{k}:", n, "requests")


def main():
    src = os.path.join(ROOT, "tests", "golden", "ctrl", "c2_colocated", "config.json")
    cfg = json.load(open(src))
    d = os.path.join(HERE, "c2_saturated")
    os.makedirs(d, exist_ok=True)
    n = poisson_trace(os.path.join(d, "trace.csv"), [f"fn{i:02d}" for i in range(4)], 10.0, const_rate(16.0), 21)
    cfg["workload"]["trace"] = "scenarios/c2_saturated/trace.csv"
    cfg["workload"]["window_s"] = 10.0
    cfg["output"] = {"dir": "scenarios/c2_saturated/out", "event_log": False}
    with open(os.path.join(d, "config.json"), "w") as fh:
        json.dump(cfg, fh, indent=2)
    print("c2_saturated:", n, "requests")
    from paper_2507_00507_b200 import tables
    d2 = os.path.join(HERE, "c2_saturated_b200")
    os.makedirs(d2, exist_ok=True)
    cfg["perf"]["tables"] = {f"{sc}:gpu": os.path.relpath(tables.measured_table_path(sc), ROOT) for sc in ("1b", "3b")}
    cfg["perf"]["gpu"] = tables.measured_cost_params()
    cfg["output"] = {"dir": "scenarios/c2_saturated_b200/out", "event_log": False}
    with open(os.path.join(d2, "config.json"), "w") as fh:
        json.dump(cfg, fh, indent=2)
    print("c2_saturated_b200: same trace, measured B200 tables")
    make_c3()
    make_c4()


if __name__ == "__main__":
    main()
