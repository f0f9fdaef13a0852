"""Bench scenarios (not parity goldens): traces that keep the co-located
instances in their capacity regime, so end-to-end tokens/s measures the
serving path rather than the arrival rate.

  c2_saturated  BASELINE configs[1] (C2): four functions on [1b, 3b, 1b, 3b],
                Poisson 16 req/s per function for 10 s. On the control plane
                alone (B200 roofline-model cost tables) this is past the knee:
                modeled ~6.7k tokens/s with ~97 % of requests inside the
                TTFT/TPOT SLO (8 req/s: 4.1k, 100 %; 32 req/s: 7.0k, 50 %).

    python scenarios/make_scenarios.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from make_ctrl_golden import const_rate, poisson_trace  # noqa: E402


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


if __name__ == "__main__":
    main()
