"""Does co-location slow each lane down?  The C3 node's eight instances (bench.MODELS,
batch 8, contexts ~CTX) on eight lanes: each instance's decode step time alone (the
other lanes idle), then all eight stepping concurrently; per-lane step time from the
host-observed completion of each lane's last step (steps are ms long, queued ahead).
Prints one JSON object: per instance alone/concurrent ms and GB/s, and the node's
aggregate decode GB/s in the concurrent run.
usage: python tools/probe_concurrency.py [steps] [ctx]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    g = MeshGpu(0, kv_pool_bytes=bench.KV_POOL, lanes=8)
    shapes = [SHAPES[m] for m in bench.MODELS]
    rids = []
    for iid, (m, s) in enumerate(zip(bench.MODELS, shapes)):
        g.create_instance(iid, s, seed=1000 + bench.MODELS.index(m))
        g.kv_resize(iid, 0, 8 * (ctx + 2 * steps + 64) * s.kv_bytes_per_token)
        rr = [iid * 100 + b for b in range(8)]
        for r in rr:
            g.step(iid, prefill=r, prefill_len=ctx)
        rids.append(rr)
    g.sync()
    nbytes = []
    for iid, s in enumerate(shapes):
        nbytes.append(s.weight_bytes_streamed + 8 * (ctx + steps) * s.kv_bytes_per_token)
    out = {"steps": steps, "ctx": ctx, "models": bench.MODELS, "lanes": [g.instance_lane(i) for i in range(8)]}
    alone = []
    for iid in range(8):
        g.sync()
        t0 = time.perf_counter()
        t = [g.step_async(iid, decode=rids[iid]) for _ in range(steps)]
        g.wait(t[-1])
        alone.append((time.perf_counter() - t0) * 1e3 / steps)
    g.sync()
    t0 = time.perf_counter()
    last = [None] * 8
    for k in range(steps):
        for iid in range(8):
            last[iid] = g.step_async(iid, decode=rids[iid])
    fin = [None] * 8
    while any(f is None for f in fin):
        for iid in range(8):
            if fin[iid] is None and g.done(last[iid]):
                fin[iid] = time.perf_counter()
        time.sleep(0.0002)
    span = max(fin) - t0
    conc = [(f - t0) * 1e3 / steps for f in fin]
    out["alone_ms"] = [round(x, 3) for x in alone]
    out["concurrent_ms"] = [round(x, 3) for x in conc]
    out["slowdown"] = [round(c / a, 3) for a, c in zip(alone, conc)]
    out["alone_GBs"] = [round(b / a / 1e6, 1) for b, a in zip(nbytes, alone)]
    out["node_GBs_concurrent"] = round(sum(nbytes) * steps / span / 1e9, 1)
    out["node_frac"] = round(out["node_GBs_concurrent"] / 6456.5, 3)
    g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
