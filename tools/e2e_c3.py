"""One C3 e2e run (bench.py's e2e leg) at a load scale, keeping the control
plane's outputs, plus a violation breakdown from requests.csv:
    python tools/e2e_c3.py 8 [out_dir]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)

import bench  # noqa: E402
from paper_2507_00507_b200 import control, gpu  # noqa: E402


def main():
    if os.environ.get("E2E_PRE_NODE"):  # reproduce bench.py: the value leg's node first, same process
        node = bench.Colocated(0)
        node.k = 0
        node.fill()
        node.run(len(bench.MODELS) * bench.BATCH)
        node.run(int(os.environ["E2E_PRE_NODE"]))
        node.g.sync()
        node.g.close()
    k = int(sys.argv[1])
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join("gpurun_out", f"e2e_s{k}")
    os.makedirs(out, exist_ok=True)
    os.environ["MESH_GPU_LANES"] = str(bench.LANES)
    os.environ.setdefault("MESH_GPU_KV_PREALLOC_GB", str(bench.KV_PREALLOC_GB))
    os.environ.setdefault("MESH_GPU_KV_GRANULE_MB", str(bench.KV_GRANULE_MB))
    cfg = os.path.join(bench.C3_DIR, f"s{k}", "config.json")
    with control.Experiment(cfg) as exp:
        for kv in sys.argv[3:]:
            key, val = kv.split("=", 1)
            exp.set(key, json.loads(val) if val[:1] in "0123456789-[{tf" else val)
        exp.out_dir(out)
        exp.attach_gpu([0], bench.E2E_KV_POOL, gpu.LIB_PATH)
        exp.run()
        names = ["wall_s", "slo_compliant_rate", "total_requests", "gpu.steps", "gpu.lane_busy_s",
                 "gpu.host_ms.instance_create", "gpu.host_ms.instance_destroy", "gpu.host_ms.kv_resize",
                 "gpu.host_ms.step_issue", "gpu.host_ms.step_wait", "gpu.instance_starts", "gpu_instances_avg",
                 "gpu_instances_max", "gpu.kv_reclaims", "gpu.host_ms.vmm", "gpu.vmm_calls", "gpu.vmm_unmaps",
                 "gpu.dp_ms.instance_create", "gpu.dp_ms.instance_destroy", "gpu.dp_ms.kv_resize", "gpu.dp_ms.step",
                 "gpu.weight_cache_hits", "gpu.migrations", "evictions", "gpu_models_avg", "gpu_models_max"]
        m = {n: exp.metric(n) for n in names}
    rows = list(csv.DictReader(open(os.path.join(out, "requests.csv"))))
    by = {}
    for r in rows:
        key = (r.get("model_id") or r.get("model"), r["outcome"])
        by[key] = by.get(key, 0) + 1
    m["outcomes"] = {f"{a}:{b}": n for (a, b), n in sorted(by.items())}
    ttft = sorted(float(r["ttft_s"]) for r in rows if r.get("ttft_s") not in (None, "", "-1"))
    if ttft:
        m["ttft_p50_p90_p99"] = [ttft[len(ttft) // 2], ttft[int(0.9 * len(ttft))], ttft[int(0.99 * len(ttft)) - 1]]
    print(json.dumps(m))


if __name__ == "__main__":
    main()
