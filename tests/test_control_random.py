"""Randomized differential test: random clusters / model mixes / policies /
memory pressure, run through the reference simulator (oracle/_ref/ref_capture)
and through our control plane; every artifact must be byte-identical (the
acceptance suite's admission-soundness scenarios, proj/tests/acceptance_main.cpp:116-281,
are the model for the generator). Skipped when the reference build is absent."""
import hashlib
import importlib.util
import json
import os
import random
import subprocess

import pytest

from paper_2507_00507_b200 import control

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_capture")
ARTS = ["events.jsonl", "requests.csv", "summary.json", "ttft_cdf.csv", "ops.csv", "steps.csv", "hash.txt"]

pytestmark = pytest.mark.skipif(not os.path.exists(REF), reason="reference build (oracle/_ref) absent")


def _mk():
    spec = importlib.util.spec_from_file_location("mk", os.path.join(ROOT, "tests", "golden", "make_ctrl_golden.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _sha(p):
    with open(p, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


@pytest.mark.parametrize("k", range(24))
def test_random_scenario(k, tmp_path, monkeypatch):
    mk = _mk()
    mk.GOLD = str(tmp_path / "scen")
    rng = random.Random(1000 + k)
    sizes = rng.sample(["1b", "3b", "7b", "13b"], rng.randint(1, 3))
    n_nodes = rng.randint(1, 3)
    mem = rng.choice([16.0, 22.0, 30.0, 48.0, 80.0, 160.0])
    nodes = [{"class": "gpu", "count": n_nodes, "mem_gb": mem}]
    if rng.random() < 0.3:
        nodes.insert(0, {"class": "cpu", "count": 1, "mem_gb": 256.0})
    under = rng.random() < 0.5
    tpl_over = {s: {"min_total_len": rng.choice([256, 1024]), "avg_output_seed": rng.choice([4, 16, 64]),
                    "avg_output_fixed": True} for s in sizes} if under else None
    policy = {}
    for flag in ("disable_defrag", "disable_validation", "disable_sharing"):
        if rng.random() < 0.15:
            policy[flag] = True
    if rng.random() < 0.2:
        policy["watermark_pct"] = rng.choice([0.0, 50.0])
    hot, cold = rng.choice([1.0, 3.0, 5.0]), rng.choice([0.05, 0.3, 1.0])
    n_fns = rng.randint(1, 6)
    d, n = mk.scenario(f"rnd{k}", nodes=nodes, templates=sizes, assignment=sizes, n_fns=n_fns, window=40.0,
                       rate_fn=lambda f, t, ph: hot if f == "fn00" else cold, seed=2000 + k, policy=policy,
                       tpl_over=tpl_over)
    if any(nd["class"] == "cpu" for nd in nodes):  # CPU nodes price with the reference's synthetic tables
        cfg = json.load(open(os.path.join(d, "config.json")))
        for s in sizes:
            if s == "1b":
                cfg["perf"]["tables"]["1b:cpu"] = cfg["perf"]["tables"]["1b:gpu"]
        json.dump(cfg, open(os.path.join(d, "config.json"), "w"))
    monkeypatch.chdir(ROOT)
    ref_out, our_out = tmp_path / "ref", tmp_path / "ours"
    r = subprocess.run([REF, "run", os.path.join(d, "config.json"), str(ref_out)], capture_output=True, text=True)
    with control.Experiment(os.path.join(d, "config.json")) as exp:
        if r.returncode != 0:  # the reference failed (e.g. its eviction ping-pong): so must we
            with pytest.raises(control.LlmError) as err:
                exp.capture(str(our_out))
            msg = r.stderr.split("error: ", 1)[-1].strip()
            assert msg in str(err.value)
            return
        exp.capture(str(our_out))
    for a in ARTS:
        assert _sha(ref_out / a) == _sha(our_out / a), f"scenario {k}: {a} differs ({n} requests)"
