"""Measured B200 cost tables (the mesh_gpu_profile role of 8(b)).

Runs the data plane's own kernels over the reference's sample grid (powers of
two plus the endpoints, proj/src/perfmodel.cpp:34-53) and writes the reference
CSV form `kind,batch,len,seconds` (proj/src/perfmodel.cpp:156-210):

  prefill,1,L,s    device time of one prefill step of L tokens (median of 3)
  decode,B,L,s     device time of one decode step of B requests at context L
                   (mesh_gpu_bench_decode: back-to-back launches, CUDA events)

plus the CostParams the reference reads from `perf.gpu.*`
(proj/src/config.cpp:36-46), fitted to its formulas
(scale_latency = min(from, to) / rate, cold_start = param_bytes / load_bw,
proj/src/perfmodel.cpp:107-119):

  scale_up_gbps      min(from,to) / wall time of a 1 -> 2 GiB KV grow (VMM map)
  scale_down_gbps    min(from,to) / wall time of a 2 -> 1 GiB KV shrink after
                     ~1.8 GiB of requests with every other one freed (batched
                     block-copy compaction moves the live blocks above 1 GiB)
  compaction_gbps    (read + write) bytes moved / that wall time
  load_gbps          weight bytes / wall time of instance_create (device init)
  min_scale_latency_s  wall time of a 0 -> 64 MiB grow
  unload_latency_s   wall time of instance_destroy

usage: python tools/measure_tables.py [--out DIR] [size classes ...]   (on a B200)
Writes <sc>_gpu_b200.csv and b200_cost_params.json into DIR
(default paper_2507_00507_b200/tables/).
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_00507_b200 import tables  # noqa: E402
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu  # noqa: E402

GIB = 1 << 30


def measure(sc: str, params: dict) -> list:
    s = SHAPES[sc]
    C = s.kv_bytes_per_token
    rows = []
    with MeshGpu(0, kv_pool_bytes=64 * GIB, lanes=1) as g:
        t0 = time.perf_counter()
        g.create_instance(1, s, seed=11)
        load_s = time.perf_counter() - t0
        wbytes = s.weight_bytes_streamed
        params.setdefault("load", []).append(wbytes / load_s / 1e9)
        target = 9 * (s.max_seq_len + 32) * C
        g.kv_resize(1, 0, target)
        rid = [0]

        def fresh():
            rid[0] += 1
            return rid[0]

        for L in tables.grid(s.max_seq_len):
            ts = []
            for _ in range(3):
                r = fresh()
                g.step(1, prefill=r, prefill_len=L)
                ts.append(g.stats()["last_step_ms"] / 1e3)
                g.request_free(1, r)
            rows.append(("prefill", 1, L, statistics.median(ts)))
        for L in tables.grid(s.max_seq_len):
            rids = [fresh() for _ in range(tables.MAX_BATCH)]
            for r in rids:
                g.step(1, prefill=r, prefill_len=L)
            for b in tables.grid(tables.MAX_BATCH):
                ms = g.bench_decode(1, rids[:b], 10)
                rows.append(("decode", b, L, ms / 1e3))
            for r in rids:
                g.request_free(1, r)
        # KV scale ops at the reference's byte granularity
        g.kv_resize(1, target, 0)
        g.sync()
        t0 = time.perf_counter()
        g.kv_resize(1, 0, 64 << 20)
        g.sync()
        params.setdefault("min_scale", []).append(time.perf_counter() - t0)
        g.kv_resize(1, 64 << 20, GIB)
        g.sync()
        t0 = time.perf_counter()
        g.kv_resize(1, GIB, 2 * GIB)
        g.sync()
        params.setdefault("up", []).append(GIB / (time.perf_counter() - t0) / 1e9)
        # compaction: fill ~1.8 GiB with requests, free every other one, shrink to 1 GiB
        L = max(16, min(s.max_seq_len, (64 << 20) // C))
        live = []
        for i in range(int(1.8 * GIB) // (L * C)):
            r = fresh()
            g.step(1, prefill=r, prefill_len=L)
            live.append(r)
        for r in live[::2]:
            g.request_free(1, r)
        g.sync()
        moved0 = g.stats()["bytes_moved"]
        t0 = time.perf_counter()
        g.kv_resize(1, 2 * GIB, GIB)
        g.sync()
        dt = time.perf_counter() - t0
        params.setdefault("down", []).append(GIB / dt / 1e9)
        params.setdefault("compaction", []).append((g.stats()["bytes_moved"] - moved0) / dt / 1e9)
        t0 = time.perf_counter()
        g.destroy_instance(1)
        params.setdefault("unload", []).append(time.perf_counter() - t0)
    return rows


def main():
    args = sys.argv[1:]
    out = tables.TABLE_DIR
    if args[:1] == ["--out"]:
        out, args = args[1], args[2:]
    classes = args or ["1b", "3b", "7b", "13b"]
    params = {}
    for sc in classes:
        rows = measure(sc, params)
        path = tables.write_table(os.path.join(out, os.path.basename(tables.measured_table_path(sc))), rows)
        print(sc, "->", os.path.relpath(path, ROOT), f"{len(rows)} rows", flush=True)
    cost = {
        "scale_up_gbps": statistics.median(params["up"]),
        "scale_down_gbps": statistics.median(params["down"]),
        "load_gbps": statistics.median(params["load"]),
        "min_scale_latency_s": statistics.median(params["min_scale"]),
        "unload_latency_s": statistics.median(params["unload"]),
        "compaction_gbps": statistics.median(params["compaction"]),
        "how": "tools/measure_tables.py on one B200 (wall time of the mesh_gpu C ABI call + stream drain)",
    }
    with open(os.path.join(out, "b200_cost_params.json"), "w") as fh:
        json.dump(cost, fh, indent=1)
    print(json.dumps(cost))


if __name__ == "__main__":
    main()
