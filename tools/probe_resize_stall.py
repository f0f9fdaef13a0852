"""Does a KV grow / shrink stall the co-located lanes?  Eight C3 instances keep 4 decode
steps queued each; then one instance's KV is grown by GROW_GB (new granules: cuMemMap +
cuMemSetAccess) or shrunk back.  Reports the call's host time and how many of the queued
steps (issued before the call, ~40 ms of work per lane) had completed when it returned:
all of them means the call drained the device.
usage: python tools/probe_resize_stall.py [grow_gb]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402


def main():
    grow_gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    ctx = 512
    g = MeshGpu(0, kv_pool_bytes=bench.KV_POOL, lanes=8)
    shapes = [SHAPES[m] for m in bench.MODELS]
    rids, kv = [], []
    for iid, (m, s) in enumerate(zip(bench.MODELS, shapes)):
        g.create_instance(iid, s, seed=1000 + bench.MODELS.index(m))
        kv.append(8 * (ctx + 200) * s.kv_bytes_per_token)
        g.kv_resize(iid, 0, kv[-1])
        rr = [iid * 100 + b for b in range(8)]
        for r in rr:
            g.step(iid, prefill=r, prefill_len=ctx)
        rids.append(rr)
    g.sync()
    out = []
    for trial, (what, target) in enumerate([("grow", kv[0] + int(grow_gb * 2**30)), ("shrink", kv[0]),
                                            ("grow", kv[0] + int(grow_gb * 2**30)), ("shrink", kv[0])]):
        q = []
        for k in range(4):
            for iid in range(8):
                q.append(g.step_async(iid, decode=rids[iid]))
        time.sleep(0.002)
        before = sum(g.done(t) for t in q)
        t0 = time.perf_counter()
        g.kv_resize(0, kv[0] if what == "grow" else kv[0] + int(grow_gb * 2**30), target)
        dt = (time.perf_counter() - t0) * 1e3
        after = sum(g.done(t) for t in q)
        st = g.stats()
        out.append({"op": what, "call_ms": round(dt, 3), "queued": len(q), "done_before": before, "done_after": after,
                    "vmm_calls": st.get("vmm_calls"), "vmm_unmaps": st.get("vmm_unmaps")})
        for t in q:
            g.wait(t)
    g.close()
    print(json.dumps({"grow_gb": grow_gb, "trials": out}))


if __name__ == "__main__":
    main()
