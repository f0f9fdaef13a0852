"""Writes tests/golden/block_tables.json: the block tables of every resident
request after each op of oracle/block_table.py's scripted grow / shrink / free /
swap sequence, with KV targets from the reference's m_require + watermark rule
(proj/src/memory.cpp:19-36). Run from the repo root:
    python tests/golden/make_block_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import block_table as bt  # noqa: E402
from paper_2507_00507_b200.gpu import SHAPES  # noqa: E402

SHAPE = SHAPES["tiny"].replace(max_seq_len=1024)


def main():
    C = SHAPE.kv_bytes_per_token
    ops = bt.script()
    snaps = bt.run(C, ops)
    out = {"shape": "tiny", "max_seq_len": SHAPE.max_seq_len, "kv_bytes_per_token": C,
           "avg_output": bt.AVG_OUT, "min_total_len": bt.MIN_TOTAL, "watermark_pct": bt.WATERMARK,
           "ops": [list(o) for o in ops], "snapshots": snaps}
    with open(os.path.join(ROOT, "tests", "golden", "block_tables.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
