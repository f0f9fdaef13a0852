"""Decision parity of the C++ control plane (libllmmesh.so) with the reference.

For every scenario under tests/golden/ctrl the reference simulator's artifacts
were digested by tests/golden/make_ctrl_golden.py. Our control plane must
reproduce them byte for byte: the event log (order and %.9f times), request
outcomes, SLO summary, TTFT CDF, the ScaleOp transcript (every KV grow/shrink,
model load/unload with its from/to bytes and execution window), every launched
step plan, and the cluster state hash.
"""
import hashlib
import json
import os

import pytest

from paper_2507_00507_b200 import build, control

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "ctrl")
SCENARIOS = sorted(d for d in os.listdir(GOLD) if os.path.exists(os.path.join(GOLD, d, "golden.json")))


@pytest.fixture(scope="module")
def lib():
    build.build_control()
    return control.load()


def sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


@pytest.mark.parametrize("name", SCENARIOS)
def test_artifacts_byte_identical(lib, name, tmp_path, monkeypatch):
    monkeypatch.chdir(ROOT)
    gold = json.load(open(os.path.join(GOLD, name, "golden.json")))
    with control.Experiment(os.path.join(GOLD, name, "config.json"), lib) as exp:
        exp.capture(str(tmp_path))
    for art, digest in gold["artifacts"].items():
        assert sha(tmp_path / art) == digest, f"{name}: {art} differs from the reference"
    with open(tmp_path / "summary.json") as fh:
        assert json.load(fh) == gold["summary"]


def test_reference_defect_reproduced(lib, monkeypatch, tmp_path):
    """The reference throws SimError("ensure_kv_capacity: did not converge") on
    this scenario (eviction ping-pong); the drop-in must fail
    the same way, with LLM_ERR_RUNTIME and the same message."""
    monkeypatch.chdir(ROOT)
    d = os.path.join(GOLD, "c4_defect_pingpong")
    expected = json.load(open(os.path.join(d, "expected_error.json")))
    assert expected["exit_code"] == 3
    with control.Experiment(os.path.join(d, "config.json"), lib) as exp:
        with pytest.raises(control.LlmError) as err:
            exp.capture(str(tmp_path))
    assert err.value.status == control.LLM_ERR_RUNTIME
    assert "ensure_kv_capacity: did not converge" in str(err.value)
    assert "ensure_kv_capacity: did not converge" in expected["stderr"]
