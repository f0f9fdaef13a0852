"""GPU: the KV pool's block tables against the committed golden, the
asynchronous preemption swap (pinned host space, event-gated resume) and live
KV migration, through the mesh_gpu C ABI.

  * block tables: after every op of oracle/block_table.py's scripted
    grow / shrink / free / swap / resume sequence (KV targets from the
    reference's m_require + watermark rule, proj/src/memory.cpp:19-36), every
    resident request's block ids and the instance's capacity equal
    tests/golden/block_tables.json exactly;
  * swap: swap_out returns while the request's decode steps are still queued;
    the parked history completes as they retire; resume (re-prefill of
    ctx + 1 tokens, or an explicit swap_in prefetch followed by plain decode)
    continues the request with logits within the oracle tolerance
    (tests/test_gpu_parity.py), on the same or on another handle;
  * migration: between two handles of one device (the two-handle case of the
    per-device launch configuration) and, when a second GPU exists, across
    devices over peer access.
"""
import json
import os

import numpy as np
import pytest

from oracle import block_table as bt
from oracle import llama_oracle as ora
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu, lib
from test_gpu_parity import SEED_PROMPT, _check

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "block_tables.json")


def _prompt(rid, n, vocab):
    return [ora.prompt_token(SEED_PROMPT, rid, i, vocab) for i in range(n)]


def test_block_tables_match_golden():
    with open(GOLDEN) as fh:
        gold = json.load(fh)
    shape = SHAPES[gold["shape"]].replace(max_seq_len=gold["max_seq_len"])
    C = shape.kv_bytes_per_token
    assert C == gold["kv_bytes_per_token"]
    with MeshGpu(0, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT) as g:
        g.create_instance(1, shape, seed=3)
        target = 0
        for i, (op, snap) in enumerate(zip(gold["ops"], gold["snapshots"])):
            kind = op[0]
            if kind == "free":
                g.request_free(1, op[1])
            if kind in ("admit", "free", "shrink"):
                req = bt.m_require([tuple(x) for x in op[2]], C, gold["avg_output"], gold["min_total_len"])
                act, rec = bt.watermark_decide(target, req, gold["watermark_pct"])
                if act != "hold":
                    g.kv_resize(1, target, rec)
                    target = rec
            elif kind == "prefill":
                g.step(1, prefill=op[1], prefill_len=op[2])
            elif kind == "decode":
                g.step(1, decode=op[1])
            elif kind == "swap_out":
                g.swap_out(1, op[1])
                g.sync()
            kv = g.instance_kv(1)
            assert kv["capacity_blocks"] == snap["cap"], f"op {i} {op[:2]}: capacity"
            for rid, blocks in snap["blocks"].items():
                _, got = g.request_info(1, int(rid))
                assert got == blocks, f"op {i} {op[:2]}: request {rid} blocks {got} != {blocks}"


def _prefill_and_decode(g, iid, model, rid, n, steps, vocab):
    """Prefill + `steps` decodes, every logit checked; returns (oracle seq, last token)."""
    seq = model.new_seq()
    ol = None
    for t in _prompt(rid, n, vocab):
        _, ol = seq.feed(t)
    toks, lg = g.step(iid, prefill=rid, prefill_len=n, vocab=vocab, with_logits=True)
    _check(lg[0], toks[0], ol, f"prefill r{rid}")
    last = toks[0]
    for k in range(steps):
        toks, lg = g.step(iid, decode=[rid], vocab=vocab, with_logits=True)
        _, ol = seq.feed(last)
        _check(lg[0], toks[0], ol, f"decode {k} r{rid}")
        last = toks[0]
    return seq, last


def test_swap_out_is_async_and_history_completes():
    shape = SHAPES["tiny"]
    model = ora.Oracle(shape, 5)
    with MeshGpu(0, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT, swap_pool_mb=64) as g:
        g.capture_logits(True)
        g.create_instance(1, shape, seed=5)
        g.kv_resize(1, 0, 64 * 16 * shape.kv_bytes_per_token)
        seq, last = _prefill_and_decode(g, 1, model, 0, 37, 2, shape.vocab)
        g.capture_logits(False)
        # three decode steps queued, then the swap: nothing waits for them
        tickets = [g.step_async(1, decode=[0]) for _ in range(3)]
        g.swap_out(1, 0)
        assert g.swap_state(0) in ("copying", "parked")
        with pytest.raises(Exception):
            g.request_info(1, 0)  # no longer resident
        emitted = [g.wait(t)[0] for t in tickets]
        g.sync()
        assert g.swap_state(0) == "parked"
        hist = g.request_tokens(1, 0)  # resolved through the parked entry
        assert hist[-3:] == emitted and len(hist) == 37 + 1 + 2 + 3
        for t in [last] + emitted[:-1]:
            seq.feed(t)
        # resume: the re-prefill of I + generated tokens feeds one token on the parked KV
        g.capture_logits(True)
        n = len(hist)
        sw0 = g.stats()["swap_in_bytes"]
        toks, lg = g.step(1, prefill=0, prefill_len=n, vocab=shape.vocab, with_logits=True)
        _, ol = seq.feed(emitted[-1])
        _check(lg[0], toks[0], ol, "resume")
        assert g.stats()["swap_in_bytes"] > sw0
        assert g.swap_state(0) == "none"
        ctx, _ = g.request_info(1, 0)
        assert ctx == n


def test_swap_in_prefetch_then_plain_decode():
    shape = SHAPES["tiny128"]
    model = ora.Oracle(shape, 6)
    with MeshGpu(0, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT) as g:
        g.capture_logits(True)
        g.create_instance(1, shape, seed=6)
        g.kv_resize(1, 0, 64 * 16 * shape.kv_bytes_per_token)
        seq, last = _prefill_and_decode(g, 1, model, 7, 45, 3, shape.vocab)
        live0 = g.instance_kv(1)["live_blocks"]
        g.swap_out(1, 7)
        g.swap_in(1, 7)  # event-gated on the gather, scatter on the side stream; the lane waits by event
        ctx, blocks = g.request_info(1, 7)
        assert ctx == 45 + 3 and len(blocks) == (ctx + 15) // 16
        for k in range(4):  # no prefill: the restored KV and last token feed plain decode steps
            toks, lg = g.step(1, decode=[7], vocab=shape.vocab, with_logits=True)
            _, ol = seq.feed(last)
            _check(lg[0], toks[0], ol, f"decode after swap_in {k}")
            last = toks[0]
        g.request_free(1, 7)
        g.sync()
        g.step(1, prefill=8, prefill_len=5)  # reaps the swapped-out blocks
        assert g.instance_kv(1)["live_blocks"] == 1 and live0 > 1


def test_resume_on_another_handle():
    """Parked requests are process-wide: one evicted on one handle resumes on another."""
    shape = SHAPES["tiny"]
    model = ora.Oracle(shape, 5)
    g1 = MeshGpu(0, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT)
    g2 = MeshGpu(0, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT)
    try:
        for g in (g1, g2):
            g.capture_logits(True)
            g.create_instance(1, shape, seed=5)
            g.kv_resize(1, 0, 64 * 16 * shape.kv_bytes_per_token)
        seq, last = _prefill_and_decode(g1, 1, model, 3, 29, 2, shape.vocab)
        g1.swap_out(1, 3)
        n = 29 + 1 + 2
        toks, lg = g2.step(1, prefill=3, prefill_len=n, vocab=shape.vocab, with_logits=True)
        _, ol = seq.feed(last)
        _check(lg[0], toks[0], ol, "resume on handle 2")
        assert g2.request_info(1, 3)[0] == n
    finally:
        g1.close()
        g2.close()


def _migrate_case(dev_src, dev_dst):
    shape = SHAPES["tiny128"]
    model = ora.Oracle(shape, 9)
    g1 = MeshGpu(dev_src, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT)
    g2 = MeshGpu(dev_dst, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT)
    try:
        for g in (g1, g2):
            g.capture_logits(True)
            g.create_instance(1, shape, seed=9)
            g.kv_resize(1, 0, 64 * 16 * shape.kv_bytes_per_token)
        seq, last = _prefill_and_decode(g1, 1, model, 11, 70, 2, shape.vocab)
        _prefill_and_decode(g1, 1, ora.Oracle(shape, 9), 12, 20, 0, shape.vocab)  # a neighbour that stays
        hist = g1.request_tokens(1, 11)
        mb0 = g2.stats()["migrate_bytes"]
        g1.migrate_to(1, g2, 1, 11)
        assert g2.stats()["migrate_bytes"] > mb0
        assert g2.request_tokens(1, 11) == hist
        for k in range(3):
            toks, lg = g2.step(1, decode=[11], vocab=shape.vocab, with_logits=True)
            _, ol = seq.feed(last)
            _check(lg[0], toks[0], ol, f"decode after migration {k} ({dev_src}->{dev_dst})")
            last = toks[0]
        # the source's blocks come back once the copy read them (reaped at its next step)
        g2.sync()
        g1.step(1, decode=[12])
        assert g1.instance_kv(1)["live_blocks"] == 2  # request 12: 20 + 1 tokens
    finally:
        g1.close()
        g2.close()


def test_migrate_between_two_handles_one_device():
    _migrate_case(0, 0)


def test_migrate_across_devices():
    if lib().mesh_gpu_device_count() < 2:
        pytest.skip("one GPU visible: the cross-device (NVLink P2P) migration needs two")
    _migrate_case(0, 1)
    _migrate_case(1, 0)
