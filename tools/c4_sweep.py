"""C4 variants (hot / cold rates, node memory) through the GPU-attached control plane in
wall-clock mode: which settings make ensure_kv_capacity evict (and the data plane swap)."""
import json, os, sys, tempfile
sys.path.insert(0, "scenarios"); sys.path.insert(0, ".")
os.environ["MESH_GPU_LANES"] = "8"
os.environ["MESH_GPU_SWAP_POOL_MB"] = "4096"
import make_scenarios as ms
from paper_2507_00507_b200 import control, gpu
for hot, cold, mem in [(6.0, 1.0, 44.0), (8.0, 2.0, 44.0), (4.0, 1.0, 42.0)]:
    d = tempfile.mkdtemp()
    ms.make_c4(d, hot, cold, mem)
    cfg = os.path.join(d, "config.json")
    c = json.load(open(cfg)); c["workload"]["trace"] = os.path.join(d, "trace.csv"); c["workload"]["lengths"] = os.path.join(d, "lengths.csv"); json.dump(c, open(cfg, "w"))
    try:
        with control.Experiment(cfg) as exp:
            exp.out_dir(d); exp.attach_gpu([0], 48 << 30, gpu.LIB_PATH); exp.run()
            print(hot, cold, mem, {k: round(exp.metric(k), 3) for k in ["slo_compliant_rate", "evictions", "gpu.swap_out_bytes", "gpu.swap_in_bytes", "total_requests", "wall_s", "pingpong_drops"]}, flush=True)
    except Exception as e:
        print(hot, cold, mem, "ERR", e, flush=True)
