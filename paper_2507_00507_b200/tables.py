"""Step-latency tables for the cost seam (reference CSV form `kind,batch,len,seconds`,
proj/src/perfmodel.cpp:156-210) on the reference's sample grid: powers of two
plus the endpoints (L_max, B_max).

  *_gpu_model.csv   analytic B200 roofline model (bytes / measured HBM
                    bandwidth for decode, flops / measured bf16 peak for
                    prefill, plus a fixed launch floor). Deterministic, used
                    by the parity scenarios.
  *_gpu_b200.csv    measured on a B200 by tools/measure_tables.py (the
                    mesh_gpu_profile role of SURVEY 8(b)/8(f)-1).
"""
from __future__ import annotations

import os

from .gpu import SHAPES

_HERE = os.path.dirname(os.path.abspath(__file__))
TABLE_DIR = os.path.join(_HERE, "tables")

HBM_GBPS = 6539.2          # MEASURED_PEAKS.json hbm_gbs
BF16_TFLOPS = 1388.5       # MEASURED_PEAKS.json bf16_tflops_sustained
DECODE_FLOOR_S = 40e-6
PREFILL_FLOOR_S = 120e-6
MAX_BATCH = 8              # the decode kernel's mma n-dimension


def grid(top: int) -> list[int]:
    g, x = [], 1
    while x < top:
        g.append(x)
        x *= 2
    g.append(top)
    return g


def decode_bytes(shape, batch: int, avg_len: int) -> float:
    c = shape.kv_bytes_per_token
    return shape.weight_bytes_streamed + batch * avg_len * c + batch * c + batch * shape.d_model * 2


def prefill_flops(shape, length: int) -> float:
    return (2.0 * length * shape.p_body + 2.0 * shape.vocab * shape.d_model +
            2.0 * shape.n_layers * shape.n_heads * shape.d_head * length * (length + 1))


def model_rows(size_class: str):
    s = SHAPES[size_class]
    rows = []
    for length in grid(s.max_seq_len):
        rows.append(("prefill", 1, length, PREFILL_FLOOR_S + prefill_flops(s, length) / (BF16_TFLOPS * 1e12)))
    for b in grid(MAX_BATCH):
        for length in grid(s.max_seq_len):
            rows.append(("decode", b, length, DECODE_FLOOR_S + decode_bytes(s, b, length) / (HBM_GBPS * 1e9)))
    return rows


def write_table(path: str, rows) -> str:
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        fh.write("kind,batch,len,seconds\n")
        for kind, b, length, sec in rows:
            fh.write(f"{kind},{b},{length},{sec:.12g}\n")
    return path


def model_table_path(size_class: str) -> str:
    return os.path.join(TABLE_DIR, f"{size_class}_gpu_model.csv")


def measured_table_path(size_class: str) -> str:
    return os.path.join(TABLE_DIR, f"{size_class}_gpu_b200.csv")


def measured_cost_params() -> dict:
    """perf.gpu.* (proj/src/config.cpp:36-46) measured by tools/measure_tables.py."""
    import json
    with open(os.path.join(TABLE_DIR, "b200_cost_params.json")) as fh:
        p = json.load(fh)
    return {k: p[k] for k in ("scale_up_gbps", "scale_down_gbps", "load_gbps", "min_scale_latency_s",
                              "unload_latency_s")}


def write_model_tables() -> None:
    for sc in ("1b", "3b", "7b", "13b"):
        write_table(model_table_path(sc), model_rows(sc))


if __name__ == "__main__":
    write_model_tables()
