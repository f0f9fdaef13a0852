"""Runs a C2 scenario through llmmesh.h with the GPU attached (debug helper)."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_00507_b200 import control, gpu
cfg = sys.argv[1] if len(sys.argv) > 1 else "scenarios/c2_saturated/config.json"
window = float(sys.argv[2]) if len(sys.argv) > 2 else None
with control.Experiment(cfg) as exp:
    if window:
        exp.set("workload.window_s", window)
    exp.out_dir(tempfile.mkdtemp(prefix="mesh_e2e_"))
    exp.attach_gpu([0], 48 << 30, gpu.LIB_PATH)
    t0 = time.time()
    try:
        exp.run()
        keys = ["gpu.steps", "gpu.decode_tokens", "gpu.prefill_tokens", "slo_compliant_rate", "gpu.device_ms",
                "gpu.instance_starts", "gpu.host_ms.instance_create", "gpu.host_ms.instance_destroy",
                "gpu.host_ms.kv_resize", "gpu.host_ms.step_issue", "gpu.host_ms.step_wait", "gpu.vmm_calls",
                "gpu.host_ms.vmm", "gpu.kv_reclaims", "gpu.weight_cache_hits"]
        print("ok", time.time() - t0, {k: exp.metric(k) for k in keys})
    except Exception as e:
        print("FAIL after", time.time() - t0, e)
