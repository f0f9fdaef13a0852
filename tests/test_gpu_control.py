"""The control plane with the B200 data plane attached (llm_experiment_attach_gpu).

Every priced action of the schedule is also executed on the GPU: model load and
unload, KV grow/shrink at issue, every IterationPlan (prefill and decode),
eviction (swap of the KV to pinned host) and completion. The data plane must
not perturb a single decision: the artifacts of a GPU-attached run (event log,
request outcomes, ScaleOp transcript, step plans, state hash) must be byte
identical to the same run without a GPU, which tests/test_control_parity.py
pins to the reference simulator. Windows are shortened so each scenario runs in
seconds; the decisions compared are still every decision of that run.
"""
import hashlib
import os

import pytest

from paper_2507_00507_b200 import control, gpu

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "ctrl")
ARTIFACTS = ["events.jsonl", "requests.csv", "summary.json", "ops.csv", "steps.csv", "hash.txt"]

# scenario -> (window s, KV pool GiB, what it exercises on the device)
CASES = {
    "c1_1b_poisson": (12.0, 16, "single instance, prefill + batched decode"),
    "c2_colocated": (12.0, 16, "four co-located instances on one node"),
    "c2_measured": (10.0, 16, "the same node priced by the B200-measured tables"),
    "c4_evict": (40.0, 16, "KV pressure: ensure_kv_capacity evicts -> swap to pinned host"),
    "c4_mixed_evict": (25.0, 16, "3b + 7b under pressure: eviction, shrink compaction"),
    # two GPU nodes driven through one device (C5's 4 x 160 GB fleet does not fit one B200)
    "c3_novalidation_jitter": (30.0, 48, "2 GPU nodes: placement, cold starts, keep-alive unloads, jitter"),
}


def _digests(d):
    out = {}
    for a in ARTIFACTS:
        with open(os.path.join(d, a), "rb") as fh:
            out[a] = hashlib.sha256(fh.read()).hexdigest()
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_attached_run_keeps_every_decision(name, tmp_path, monkeypatch):
    monkeypatch.chdir(ROOT)
    monkeypatch.setenv("MESH_GPU_LANES", "4")
    window, pool_gib, _ = CASES[name]
    cfg = os.path.join(GOLD, name, "config.json")
    with control.Experiment(cfg) as exp:
        exp.set("workload.window_s", window)
        exp.capture(str(tmp_path / "cpu"))
        steps_planned = sum(1 for _ in open(tmp_path / "cpu" / "steps.csv")) - 1
    with control.Experiment(cfg) as exp:
        exp.set("workload.window_s", window)
        exp.attach_gpu([0], pool_gib << 30, gpu.LIB_PATH)
        exp.capture(str(tmp_path / "gpu"))
        m = {k: exp.metric(k) for k in ["gpu.steps", "gpu.decode_tokens", "gpu.prefill_tokens",
                                        "gpu.swap_out_bytes", "gpu.instance_starts", "gpu.kernel_launches"]}
    assert _digests(tmp_path / "gpu") == _digests(tmp_path / "cpu")
    assert steps_planned > 0
    # every planned step ran on the device (a decode step of > 8 requests is split into launches of 8)
    assert m["gpu.steps"] >= steps_planned
    assert m["gpu.decode_tokens"] > 0 and m["gpu.prefill_tokens"] > 0 and m["gpu.kernel_launches"] > 0
    if "evict" in name:
        with open(tmp_path / "gpu" / "events.jsonl") as fh:
            evictions = sum(1 for line in fh if "evict" in line.lower())
        if evictions:
            assert m["gpu.swap_out_bytes"] > 0


def test_fleet_two_nodes_one_device_wall_clock(tmp_path, monkeypatch):
    """C5's fleet path on the one GPU a test box has: two GPU nodes driven as two
    handles on device 0 (attach_gpu devices [0, 0]) from one host event loop, in
    wall-clock mode (completions and emission times are CUDA events). Both nodes
    receive instances through the control plane's placement, every request gets an
    outcome, and the models-per-GPU accounting is filled in."""
    import bench
    monkeypatch.chdir(ROOT)
    monkeypatch.setenv("MESH_GPU_LANES", "4")
    cfg = bench.fleet_scenario(2, 1.0, window=12.0, mem_gb=60.0)  # two 60 GB nodes share one B200
    with control.Experiment(cfg) as exp:
        exp.out_dir(str(tmp_path))
        exp.attach_gpu([0, 0], 24 << 30, gpu.LIB_PATH)
        exp.run()
        m = {k: exp.metric(k) for k in ["gpu_nodes_used", "gpu_instances_max", "gpu_instances_avg", "total_requests",
                                        "slo_compliant_rate", "wall_s", "gpu.steps", "gpu.decode_tokens"]}
    assert m["total_requests"] > 0 and m["gpu.steps"] > 0 and m["gpu.decode_tokens"] > 0
    assert m["gpu_nodes_used"] == 2 and m["gpu_instances_max"] >= 2
    assert 12.0 <= m["wall_s"] < 60.0
    assert 0.0 < m["slo_compliant_rate"] <= 1.0
