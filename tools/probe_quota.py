"""Per-SM streaming rate of the decode kernel vs SM quota (device time, not the bench).

For each (model, quota) runs B = 8 decode at context CTX and prints ms/step,
GB/s and GB/s per SM. MESH_GPU_SKIP in the environment
isolates the attention / GEMV phases.
usage: python tools/probe_quota.py 1b:17,148 3b:56,148
"""
import json
import os
import sys

sys.path.insert(0, ".")
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402

CTX = int(os.environ.get("PROBE_CTX", "1024"))
try:  # the driver-written measured copy peak of this pool
    PEAK = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    PEAK = 6549.1
ITERS = int(os.environ.get("PROBE_ITERS", "20"))
B = 8


def run(name: str, quota: int) -> dict:
    s = SHAPES[name]
    with MeshGpu(0, sm_quota=quota, kv_pool_bytes=40 << 30) as g:
        g.create_instance(1, s, seed=1)
        g.kv_resize(1, 0, (B + 2) * (CTX + 64) * s.kv_bytes_per_token)
        for r in range(B):
            g.step(1, prefill=r, prefill_len=CTX)
        tdir = os.environ.get("PROBE_TRACE")
        if tdir:  # CTA 0 phase timeline + per-CTA barrier arrivals of one traced launch
            os.environ["MESH_GPU_TRACE"] = os.path.join(tdir, f"tr_{name}_{quota}_s{os.environ.get('MESH_GPU_SKIP', '0')}.txt")
        ms = g.bench_decode(1, list(range(B)), ITERS)
        os.environ.pop("MESH_GPU_TRACE", None)
    byts = s.weight_bytes_streamed + B * (CTX + 1) * s.kv_bytes_per_token + B * s.d_model * 2
    gbs = byts / ms / 1e6
    return dict(model=name, quota=quota, ms=round(ms, 4), GBps=round(gbs, 1), GBps_per_sm=round(gbs / quota, 2),
                frac=round(gbs / PEAK, 3), skip=os.environ.get("MESH_GPU_SKIP", "0"))


for arg in sys.argv[1:] or ["1b:17,148"]:
    name, qs = arg.split(":")
    for q in qs.split(","):
        print(json.dumps(run(name, int(q))), flush=True)
