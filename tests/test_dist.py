"""Multi-process path of bench.py on CPU (gloo, world size 2): one rank per
node, max-over-ranks device time, summed tokens (weak scaling)."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_reduction_over_gloo():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "helpers", "dist_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    r = json.loads(line)
    assert r["ws"] == 2
    assert r["wall"] == 2.0          # max over ranks
    assert r["tokens"] == 300.0      # sum over ranks
    assert r["value"] == 150.0
    # C5 fleet placement over the two nodes (cold starts on the node with the most
    # free optimistic budget, cluster.cpp:325-365): both nodes host instances
    f = r["fleet"]
    assert f["gpu_nodes_used"] == 2 and f["gpu_instances_max"] >= 2 and f["total_requests"] > 0
