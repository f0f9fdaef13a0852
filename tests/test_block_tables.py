"""CPU side of the block-table golden (tests/golden/block_tables.json): the
restated policy (oracle/block_table.py) reproduces the committed golden, and its
byte targets follow the reference's own known answers for m_require and the
watermark (proj/tests/test_memory.cpp:31-75). The GPU side is
tests/test_gpu_swap_migrate.py::test_block_tables_match_golden."""
import json
import os

from oracle import block_table as bt

KiB, GiB, GB = 1024, 1 << 30, 10**9
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "block_tables.json")


def test_m_require_known_answers():
    C = 512 * KiB  # the reference's 7b model: avg_output 120 (fixed), min_total_len 4096
    assert bt.m_require([(100, 50), (200, 10)], C, 120.0, 4096) == 2 * GiB
    assert bt.m_require([], C, 120.0, 4096) == 512 * KiB * 4096
    assert bt.m_require([(3000, 2000)], C, 120.0, 4096) == 512 * KiB * 5000


def test_watermark_known_answers():
    assert bt.watermark_decide(10 * GB, 11 * GB, 20.0) == ("up", int(13.2 * GB))
    assert bt.watermark_decide(16 * GB, 10 * GB, 20.0) == ("down", 12 * GB)
    assert bt.watermark_decide(13 * GB, 10 * GB, 20.0)[0] == "hold"


def test_policy_reproduces_golden():
    with open(GOLDEN) as fh:
        gold = json.load(fh)
    ops = [tuple(o) for o in gold["ops"]]
    assert json.loads(json.dumps([list(o) for o in bt.script()])) == gold["ops"]
    assert bt.run(gold["kv_bytes_per_token"], ops) == gold["snapshots"]


def test_golden_exercises_grow_shrink_compaction_and_resume():
    with open(GOLDEN) as fh:
        gold = json.load(fh)
    caps = [s["cap"] for s in gold["snapshots"]]
    assert any(b < a for a, b in zip(caps, caps[1:])), "no shrink"
    assert any(b > a for a, b in zip(caps, caps[1:])), "no grow"
    kinds = {o[0] for o in gold["ops"]}
    assert {"admit", "prefill", "decode", "free", "swap_out", "shrink"} <= kinds
    # some block moved by compaction: a request's block list changed without an allocation
    moved = False
    for (op, a, b) in zip(gold["ops"][1:], gold["snapshots"], gold["snapshots"][1:]):
        for rid, blocks in b["blocks"].items():
            old = a["blocks"].get(rid)
            if old and len(old) == len(blocks) and old != blocks:
                moved = True
    assert moved, "no compaction move"
