"""KV-move bandwidths of the data plane (swap vs measured pinned-host
bandwidth, migration vs peer copy, compaction vs HBM), one GPU:

  swap_out   bytes of one request's blocks / (host-observed time from the call to
             swap_state == parked), gather kernel -> host-mapped pinned memory
  swap_in    bytes / (swap_in call .. sync), scatter kernel from pinned memory
  migrate    bytes / (migrate call .. sync), copy kernel between two handles of
             one device (HBM -> HBM; across devices the same kernel loads over NVLink)
  pinned     torch pinned-host <-> device copies of the same size (copy engine peak)

Writes one JSON object to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402


def pinned_gbs(nbytes):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name] = 5 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "7b"
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    shape = SHAPES[name].replace(n_layers=int(os.environ.get("PROBE_LAYERS", SHAPES[name].n_layers)))
    C = shape.kv_bytes_per_token
    res = {"model": name, "layers": shape.n_layers, "tokens": L, "kv_bytes_per_token": C}
    g = MeshGpu(0, kv_pool_bytes=16 << 30, prompt_seed=1, swap_pool_mb=4096, lanes=2)
    g2 = MeshGpu(0, kv_pool_bytes=16 << 30, prompt_seed=1)
    try:
        g.create_instance(1, shape, seed=1)
        g2.create_instance(1, shape, seed=1)
        g.kv_resize(1, 0, 4 * (L + 64) * C)
        g2.kv_resize(1, 0, 4 * (L + 64) * C)
        swap_out, swap_in, mig = [], [], []
        for it in range(4):
            rid = 100 + it
            g.step(1, prefill=rid, prefill_len=L)
            g.sync()
            _, blocks = g.request_info(1, rid)
            nbytes = len(blocks) * 16 * C
            t0 = time.perf_counter()
            g.swap_out(1, rid)
            t_call = time.perf_counter() - t0
            while g.swap_state(rid) != "parked":
                pass
            t1 = time.perf_counter()
            swap_out.append((nbytes / (t1 - t0) / 1e9, t_call * 1e3))
            t0 = time.perf_counter()
            g.swap_in(1, rid)
            g.sync()
            t1 = time.perf_counter()
            swap_in.append(nbytes / (t1 - t0) / 1e9)
            t0 = time.perf_counter()
            g.migrate_to(1, g2, 1, rid)
            g2.sync()
            t1 = time.perf_counter()
            mig.append(nbytes / (t1 - t0) / 1e9)
            g2.request_free(1, rid)
        res["request_bytes"] = nbytes
        res["swap_out_gbs"] = max(x[0] for x in swap_out[1:])
        res["swap_out_call_ms"] = min(x[1] for x in swap_out[1:])
        res["swap_in_gbs"] = max(swap_in[1:])
        res["migrate_same_device_gbs"] = max(mig[1:])
        res["pinned_copy_engine_gbs"] = pinned_gbs(nbytes)
        res["note"] = ("host-observed wall times (call .. completion poll / sync); swap_out_call_ms is the time "
                       "the swap_out call itself holds the host (no device wait)")
    finally:
        g.close()
        g2.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
