"""GPU parity: the sm_100a data plane (through the mesh_gpu C ABI) against the
CPU numeric oracle (oracle/llama_ref.c) on identical generated weights.

Tolerance (bf16 weights/activations/KV, fp32 accumulation on both sides, the
GPU summing in a different order): per-step logits relative L2 <= 2e-2 and
max |diff| <= 0.05 * max|logit|; the greedy token must agree whenever the
oracle's top-2 logit gap is >= 0.02 (else the oracle follows the GPU token so
the trajectories stay aligned — SURVEY 7.3-1).
"""
import numpy as np
import pytest

from oracle import llama_oracle as ora
from paper_2507_00507_b200.gpu import SHAPES, MeshGpuError, T_LM, T_WDOWN, T_WGATE, T_WK, T_WO, T_WQ, T_WUP, T_WV, MeshGpu

pytestmark = pytest.mark.gpu

REL_L2 = 2e-2
GAP = 0.02
SEED_PROMPT = 1234


def _rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12))


def _check(gpu_logits, gpu_tok, ora_logits, where):
    rl = _rel_l2(gpu_logits, ora_logits)
    assert rl <= REL_L2, f"{where}: logits rel-L2 {rl:.4g}"
    mx = float(np.max(np.abs(ora_logits)))
    assert float(np.max(np.abs(gpu_logits - ora_logits))) <= 0.05 * mx + 1e-3, where
    top = np.argsort(ora_logits)[::-1]
    gap = float(ora_logits[top[0]] - ora_logits[top[1]])
    if gap >= GAP:
        assert gpu_tok == int(top[0]), f"{where}: token {gpu_tok} vs oracle {int(top[0])} (gap {gap:.3f})"


@pytest.fixture(scope="module")
def gpu():
    g = MeshGpu(0, kv_pool_bytes=8 << 30, prompt_seed=SEED_PROMPT)
    g.capture_logits(True)
    yield g
    g.close()


def _oracle_prefill(model, rid, n):
    seq = model.new_seq()
    toks = [ora.prompt_token(SEED_PROMPT, rid, i, model.shape.vocab) for i in range(n)]
    logits = None
    for t in toks:
        _, logits = seq.feed(t)
    return seq, logits


@pytest.mark.parametrize("name", ["tiny", "tiny128"])
def test_generator_weights_bit_exact(gpu, name):
    shape = SHAPES[name]
    iid = 100 + len(name)
    gpu.create_instance(iid, shape, seed=77)
    try:
        d, ff = shape.d_model, shape.d_ff
        checks = [(T_WQ, 1, 5, d), (T_WK, 0, shape.n_kv_heads * shape.d_head - 3, d), (T_WV, 1, 2, d), (T_WO, 0, 7, d),
                  (T_WGATE, 1, 9, d), (T_WUP, 0, ff - 1, d), (T_WDOWN, 1, d - 2, ff)]
        if not shape.tied:
            checks.append((T_LM, 0, shape.vocab - 5, d))
        for tensor, layer, row, k in checks:
            got = gpu.read_weight(iid, tensor, layer, row, k)
            want = np.array([ora.weight(77, tensor, layer, row * k + c) for c in range(k)], dtype=np.float32)
            assert np.array_equal(got, want), (tensor, layer, row)
    finally:
        gpu.destroy_instance(iid)


@pytest.mark.parametrize("name", ["tiny", "tiny128"])
def test_prefill_then_decode_matches_oracle(gpu, name):
    shape = SHAPES[name]
    iid = 200 + len(name)
    gpu.create_instance(iid, shape, seed=11)
    gpu.kv_resize(iid, 0, 4 << 20)
    model = ora.Oracle(shape, 11)
    try:
        rid = 7
        n = 37
        toks, lg = gpu.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
        seq, ol = _oracle_prefill(model, rid, n)
        _check(lg[0], toks[0], ol, f"{name} prefill")
        tok = toks[0]
        for step in range(24):  # crosses the 16-token block boundaries at 48
            toks, lg = gpu.step(iid, decode=[rid], vocab=shape.vocab, with_logits=True)
            _, ol = seq.feed(tok)
            _check(lg[0], toks[0], ol, f"{name} decode {step}")
            tok = toks[0]
        ctx, blocks = gpu.request_info(iid, rid)
        assert ctx == n + 24 and len(blocks) == (ctx + 15) // 16
        assert len(gpu.request_tokens(iid, rid)) == n + 25
    finally:
        gpu.destroy_instance(iid)


def test_ragged_batch_decode(gpu):
    shape = SHAPES["tiny"]
    iid = 300
    gpu.create_instance(iid, shape, seed=5)
    gpu.kv_resize(iid, 0, 8 << 20)
    model = ora.Oracle(shape, 5)
    try:
        lens = [1, 15, 16, 17, 31, 32, 60, 100]
        seqs, last = {}, {}
        for rid, n in zip(range(8), lens):
            toks, lg = gpu.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
            seqs[rid], ol = _oracle_prefill(model, rid, n)
            _check(lg[0], toks[0], ol, f"prefill r{rid}")
            last[rid] = toks[0]
        order = [3, 0, 7, 1, 6, 2, 5, 4]  # admission order is arbitrary
        for step in range(6):
            toks, lg = gpu.step(iid, decode=order, vocab=shape.vocab, with_logits=True)
            for i, rid in enumerate(order):
                _, ol = seqs[rid].feed(last[rid])
                _check(lg[i], toks[i], ol, f"batch step {step} r{rid}")
                last[rid] = toks[i]
        # smaller batches reuse the same requests
        toks, lg = gpu.step(iid, decode=[6, 2], vocab=shape.vocab, with_logits=True)
        for i, rid in enumerate([6, 2]):
            _, ol = seqs[rid].feed(last[rid])
            _check(lg[i], toks[i], ol, f"sub-batch r{rid}")
    finally:
        gpu.destroy_instance(iid)


def test_kv_shrink_compacts_and_preserves_outputs(gpu):
    shape = SHAPES["tiny"]
    iid = 400
    C = shape.kv_bytes_per_token
    gpu.create_instance(iid, shape, seed=9)
    gpu.kv_resize(iid, 0, 400 * C)
    model = ora.Oracle(shape, 9)
    try:
        last, seqs = {}, {}
        for rid, n in [(0, 100), (1, 90), (2, 80)]:
            toks, _ = gpu.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
            seqs[rid], _ = _oracle_prefill(model, rid, n)
            last[rid] = toks[0]
        gpu.request_free(iid, 0)  # frees the low blocks -> request 2's blocks sit high
        before = gpu.instance_kv(iid)
        _, blocks2 = gpu.request_info(iid, 2)
        assert max(blocks2) >= 12
        gpu.kv_resize(iid, 400 * C, 120 * C)
        after = gpu.instance_kv(iid)
        assert after["capacity_blocks"] < before["capacity_blocks"]
        assert after["mapped"] <= before["mapped"]
        _, blocks2b = gpu.request_info(iid, 2)
        assert max(blocks2b) < after["capacity_blocks"]
        assert gpu.stats()["blocks_moved"] > 0
        toks, lg = gpu.step(iid, decode=[1, 2], vocab=shape.vocab, with_logits=True)
        for i, rid in enumerate([1, 2]):
            _, ol = seqs[rid].feed(last[rid])
            _check(lg[i], toks[i], ol, f"post-compaction r{rid}")
    finally:
        gpu.destroy_instance(iid)


def test_swap_out_and_resume(gpu):
    shape = SHAPES["tiny"]
    iid = 500
    gpu.create_instance(iid, shape, seed=21)
    gpu.kv_resize(iid, 0, 4 << 20)
    model = ora.Oracle(shape, 21)
    try:
        rid, n = 42, 50
        toks, _ = gpu.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
        seq, _ = _oracle_prefill(model, rid, n)
        last = toks[0]
        for _ in range(5):
            toks, _ = gpu.step(iid, decode=[rid], vocab=shape.vocab, with_logits=True)
            seq.feed(last)
            last = toks[0]
        gpu.swap_out(iid, rid)
        assert gpu.stats()["swap_out_bytes"] > 0
        # re-admission: the control plane plans a prefill of I + O tokens (compute.cpp:112)
        history = n + 5 + 1
        toks, lg = gpu.step(iid, prefill=rid, prefill_len=history, vocab=shape.vocab, with_logits=True)
        _, ol = seq.feed(last)
        _check(lg[0], toks[0], ol, "resume after swap")
        assert gpu.stats()["swap_in_bytes"] > 0
    finally:
        gpu.destroy_instance(iid)


def test_migrate_between_instances(gpu):
    shape = SHAPES["tiny"]
    gpu.create_instance(600, shape, seed=3)
    gpu.create_instance(601, shape, seed=3)
    gpu.kv_resize(600, 0, 4 << 20)
    gpu.kv_resize(601, 0, 4 << 20)
    model = ora.Oracle(shape, 3)
    try:
        rid, n = 9, 33
        toks, _ = gpu.step(600, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
        seq, _ = _oracle_prefill(model, rid, n)
        last = toks[0]
        gpu.migrate_to(600, gpu, 601, rid)
        assert gpu.stats()["migrate_bytes"] > 0
        toks, lg = gpu.step(601, decode=[rid], vocab=shape.vocab, with_logits=True)
        _, ol = seq.feed(last)
        _check(lg[0], toks[0], ol, "decode after migration")
    finally:
        gpu.destroy_instance(600)
        gpu.destroy_instance(601)


def test_1b_shape_prefill_decode(gpu):
    """The C1 model (TinyLlama-1.1B shape) at reduced context for oracle speed."""
    shape = SHAPES["1b"]
    iid = 700
    gpu.create_instance(iid, shape, seed=1)
    gpu.kv_resize(iid, 0, 64 * 1024 * shape.kv_bytes_per_token // 16)
    model = ora.Oracle(shape, 1)
    try:
        rid, n = 3, 24
        toks, lg = gpu.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
        seq, ol = _oracle_prefill(model, rid, n)
        _check(lg[0], toks[0], ol, "1b prefill")
        last = toks[0]
        for step in range(3):
            toks, lg = gpu.step(iid, decode=[rid], vocab=shape.vocab, with_logits=True)
            _, ol = seq.feed(last)
            _check(lg[0], toks[0], ol, f"1b decode {step}")
            last = toks[0]
    finally:
        model.close()
        gpu.destroy_instance(iid)


@pytest.mark.parametrize("bn,cluster", [("64", ""), ("128", ""), ("256", ""), ("256", "1"), ("128", "2")])
def test_long_prefill_every_tile_width(gpu, bn, cluster, monkeypatch):
    """tcgen05 prefill GEMMs at every token-tile width and token-tile multicast
    cluster size (default: 4 where the weight-tile count allows, else 2), with
    several token tiles and a ragged last tile (700 = 2x256 + 188), then
    decode over the whole KV."""
    monkeypatch.setenv("MESH_PREFILL_BN", bn)
    if cluster:
        monkeypatch.setenv("MESH_PREFILL_CLUSTER", cluster)
    shape = SHAPES["tiny128"]
    iid = 800 + int(bn) + 1000 * int(cluster or 0)
    gpu.create_instance(iid, shape, seed=21)
    gpu.kv_resize(iid, 0, 1024 * shape.kv_bytes_per_token)
    model = ora.Oracle(shape, 21)
    try:
        rid, n = 11, 700
        toks, lg = gpu.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
        seq, ol = _oracle_prefill(model, rid, n)
        _check(lg[0], toks[0], ol, f"BN={bn} prefill {n}")
        last = toks[0]
        for step in range(3):
            toks, lg = gpu.step(iid, decode=[rid], vocab=shape.vocab, with_logits=True)
            _, ol = seq.feed(last)
            _check(lg[0], toks[0], ol, f"BN={bn} decode {step}")
            last = toks[0]
    finally:
        model.close()
        gpu.destroy_instance(iid)


def test_lazy_shrink_slack_reclaimed_by_other_grow():
    """Shrink keeps the tail granules mapped (no stall); a grow of another
    instance that needs them past the pool limit reclaims the slack, and the
    shrunk instance's compacted KV still decodes exactly."""
    shape = SHAPES["tiny"]
    C = shape.kv_bytes_per_token  # 1 KiB/token: a 2 MiB granule holds 128 blocks of 16 tokens
    gran = 2 << 20
    with MeshGpu(0, kv_pool_bytes=4 * gran, prompt_seed=SEED_PROMPT, kv_granule_bytes=gran) as g:
        g.capture_logits(True)
        g.create_instance(1, shape, seed=3)
        g.create_instance(2, shape, seed=4)
        model = ora.Oracle(shape, 3)
        g.kv_resize(1, 0, 3000 * C)  # 196 blocks -> 2 granules
        toks, lg = g.step(1, prefill=5, prefill_len=60, vocab=shape.vocab, with_logits=True)
        seq, ol = _oracle_prefill(model, 5, 60)
        _check(lg[0], toks[0], ol, "prefill")
        g.kv_resize(1, 3000 * C, 200 * C)  # 21 blocks -> needs 1 granule, keeps 2 mapped
        assert g.instance_kv(1)["mapped"] == 2 * gran
        g.kv_resize(2, 0, 4000 * C)  # 258 blocks -> 3 granules: 2 + 3 > 4 forces the reclaim
        assert g.instance_kv(1)["mapped"] == gran
        assert g.instance_kv(2)["mapped"] == 3 * gran
        assert g.stats()["kv_mapped_bytes"] == 4 * gran
        last = toks[0]
        for step in range(3):
            toks, lg = g.step(1, decode=[5], vocab=shape.vocab, with_logits=True)
            _, ol = seq.feed(last)
            _check(lg[0], toks[0], ol, f"decode after reclaim {step}")
            last = toks[0]
        assert g.stats()["kv_reclaims"] == 1
        with pytest.raises(MeshGpuError):
            g.kv_resize(2, 4000 * C, 10000 * C)  # 633 blocks -> 5 granules: beyond the pool
        model.close()


def test_concurrent_lanes_match_oracle():
    """Two execution lanes: instances bind to different lanes (own stream, scratch,
    grid barrier, half of the SMs) and their prefill/decode steps run concurrently;
    every step still matches the oracle."""
    with MeshGpu(0, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT, lanes=2) as g:
        g.capture_logits(True)
        shapes = {1: SHAPES["tiny"], 2: SHAPES["tiny128"]}
        models = {}
        for iid, sh in shapes.items():
            g.create_instance(iid, sh, seed=30 + iid)
            g.kv_resize(iid, 0, 256 * sh.kv_bytes_per_token)
            models[iid] = ora.Oracle(sh, 30 + iid)
        lanes = {iid: g.instance_lane(iid) for iid in shapes}
        assert {lanes[1][0], lanes[2][0]} == {0, 1}
        assert all(c > 0 for _, c in lanes.values()) and sum(c for _, c in lanes.values()) <= 148
        seqs, last = {}, {}
        tk = {iid: g.step_async(iid, prefill=9, prefill_len=40 + 13 * iid) for iid in shapes}
        for iid, t in tk.items():
            toks, lg = g.wait(t, shapes[iid].vocab, True)
            seqs[iid], ol = _oracle_prefill(models[iid], 9, 40 + 13 * iid)
            _check(lg[0], toks[0], ol, f"lane prefill {iid}")
            last[iid] = toks[0]
        for step in range(6):
            tk = {iid: g.step_async(iid, decode=[9]) for iid in shapes}
            for iid, t in tk.items():
                toks, lg = g.wait(t, shapes[iid].vocab, True)
                _, ol = seqs[iid].feed(last[iid])
                _check(lg[0], toks[0], ol, f"lane decode {iid} step {step}")
                last[iid] = toks[0]
        for m in models.values():
            m.close()


@pytest.mark.parametrize("quota", [1, 2, 3, 5, 8, 17])
@pytest.mark.parametrize("name", ["tiny", "tiny128"])
def test_decode_schedules_across_sm_quotas(name, quota):
    """Small SM quotas put GEMV phases with >= 4 tiles per CTA on the dynamic
    tile-claim schedule (claim groups of 1..4 tiles, decode.cu claim_tiles),
    larger quotas keep the static round-robin deal; the quotas here mix both
    within one step. Every schedule must give the oracle's logits for a ragged
    batch over several steps (the claim counters rearm at step end)."""
    shape = SHAPES[name]
    model = ora.Oracle(shape, 9)
    with MeshGpu(0, sm_quota=quota, kv_pool_bytes=1 << 30, prompt_seed=SEED_PROMPT) as g:
        g.capture_logits(True)
        g.create_instance(1, shape, seed=9)
        g.kv_resize(1, 0, 8 << 20)
        lens = [3, 16, 29, 40, 7]
        seqs, last = {}, {}
        for rid, n in enumerate(lens):
            toks, lg = g.step(1, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
            seqs[rid], ol = _oracle_prefill(model, rid, n)
            _check(lg[0], toks[0], ol, f"{name}/q{quota} prefill r{rid}")
            last[rid] = toks[0]
        order = [4, 1, 0, 3, 2]
        for step in range(4):
            toks, lg = g.step(1, decode=order, vocab=shape.vocab, with_logits=True)
            for i, rid in enumerate(order):
                _, ol = seqs[rid].feed(last[rid])
                _check(lg[i], toks[i], ol, f"{name}/q{quota} step {step} r{rid}")
                last[rid] = toks[i]
        g.destroy_instance(1)


def test_arena_backed_at_open_needs_no_vmm_calls(monkeypatch):
    """KV arena backed at open (MESH_GPU_KV_PREALLOC_GB): grows, lazy shrinks, slack
    reclaims, destroy and re-create only reassign slots (no cuMemMap / cuMemUnmap,
    which drain the device), and every request still decodes exactly after its
    blocks moved into slots another instance used before."""
    monkeypatch.setenv("MESH_GPU_KV_PREALLOC_GB", "0.0625")  # 64 MiB = the whole pool
    shape = SHAPES["tiny"]
    C = shape.kv_bytes_per_token
    gran = 2 << 20
    with MeshGpu(0, kv_pool_bytes=32 * gran, prompt_seed=SEED_PROMPT, kv_granule_bytes=gran) as g:
        g.capture_logits(True)
        calls0 = g.stats()["vmm_calls"]
        assert calls0 > 0  # the arena was backed at open
        models = {1: ora.Oracle(shape, 3), 2: ora.Oracle(shape, 4)}
        g.create_instance(1, shape, seed=3)
        g.create_instance(2, shape, seed=4)
        g.kv_resize(1, 0, 20000 * C)   # 1,258 blocks: 10 of the 32 slots
        g.kv_resize(2, 0, 20000 * C)
        seqs, last = {}, {}
        for iid, rid, n in [(1, 5, 200), (2, 6, 150)]:
            toks, lg = g.step(iid, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
            seqs[rid], ol = _oracle_prefill(models[iid], rid, n)
            _check(lg[0], toks[0], ol, f"prefill i{iid}")
            last[rid] = toks[0]
        g.kv_resize(1, 20000 * C, 400 * C)  # lazy: keeps its slots
        g.kv_resize(2, 20000 * C, 400 * C)
        g.create_instance(3, shape, seed=3)
        g.kv_resize(3, 0, 60000 * C)  # needs slots beyond the free ones: takes 1's and 2's slack
        assert g.stats()["kv_reclaims"] >= 1
        g.destroy_instance(3)
        g.create_instance(4, shape, seed=4)  # recycled buffers, slots of the destroyed instance
        g.kv_resize(4, 0, 60000 * C)
        for step in range(3):
            for iid, rid in [(1, 5), (2, 6)]:
                toks, lg = g.step(iid, decode=[rid], vocab=shape.vocab, with_logits=True)
                _, ol = seqs[rid].feed(last[rid])
                _check(lg[0], toks[0], ol, f"decode i{iid} step {step}")
                last[rid] = toks[0]
        assert g.stats()["vmm_calls"] == calls0
        for mdl in models.values():
            mdl.close()
