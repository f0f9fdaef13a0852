"""GPU parity at the full widths the configs run: 1.1B, 3B,
7B and 13B layer shapes, two layers each, against the numeric oracle.

The C2-C5 instances are these models; the rest of tests/ checks the kernels
at small shapes plus a short 1.1B case. Here every full-width code path runs:
  * 1.1B  GQA group 8, d_head 64, untied 32k lm_head;
  * 3B    GQA group 3, d_head 128, TIED 128,256-row lm_head with fused argmax,
          rope theta 5e5;
  * 7B    MHA (group 1), d_head 128, d_ff 11008;
  * 13B   MHA, d_model 5120, 40 heads, d_ff 13824.
Each shape: ragged prefills of 1..900 tokens (several tcgen05 token tiles, a
ragged last tile), then 8 ragged batch-8 decode steps at SM quotas 148 / 56 /
17 (the C2/C3 lane quotas), KV shrink compaction, swap to host + resume, and
migration between two instances — all against oracle/llama_np.py (the numpy
statement of oracle/llama_ref.c, pinned to it in tests/test_oracle_np.py).

Tolerance: tests/test_gpu_parity.py's logits bounds (per-step rel-L2 <= 2e-2,
max |diff| <= 0.05 max|logit|). The greedy-token rule is stated against the
step's measured logit noise, since at these widths (|logit| up to ~3) a fixed
0.02 top-2 gap is inside bf16 noise: with rmsd = rms(gpu - oracle) (itself
bounded by the rel-L2 bound), the GPU's token must equal the oracle's argmax
whenever the oracle's top-2 gap >= max(0.02, 5 rmsd) (a flip then needs a
> 3.5-sigma difference of two logit errors), and otherwise must be a token whose
oracle logit is within that margin of the maximum. The oracle then follows the
GPU's token so the trajectories stay aligned.
"""
import copy

import numpy as np
import pytest

from oracle import llama_np as onp
from oracle import llama_oracle as ora
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu
from test_gpu_parity import GAP, REL_L2, SEED_PROMPT, _rel_l2

pytestmark = pytest.mark.gpu

NAMES = ["1b", "3b", "7b", "13b"]
LENS = [300, 17, 64, 129, 900, 1, 33, 250]
QUOTAS = [148, 56, 17]
DECODE_STEPS = 8
WSEED = 41

_cache: dict = {}


def _shape(name):
    return SHAPES[name].replace(n_layers=2)


def _prompt(rid, n, vocab):
    return [ora.prompt_token(SEED_PROMPT, rid, i, vocab) for i in range(n)]


def _check(gpu_logits, gpu_tok, ora_logits, where):
    rl = _rel_l2(gpu_logits, ora_logits)
    assert rl <= REL_L2, f"{where}: logits rel-L2 {rl:.4g}"
    diff = gpu_logits - ora_logits
    mx = float(np.max(np.abs(ora_logits)))
    assert float(np.max(np.abs(diff))) <= 0.05 * mx + 1e-3, where
    margin = max(GAP, 5.0 * float(np.sqrt(np.mean(diff.astype(np.float64) ** 2))))
    top = np.argsort(ora_logits)[::-1]
    gap = float(ora_logits[top[0]] - ora_logits[top[1]])
    if gap >= margin:
        assert gpu_tok == int(top[0]), f"{where}: token {gpu_tok} vs oracle {int(top[0])} (gap {gap:.3f} >= {margin:.3f})"
    else:
        assert float(ora_logits[gpu_tok]) >= float(ora_logits[top[0]]) - margin, f"{where}: token {gpu_tok} off the top"


def _oracle(name):
    """(oracle, {rid: (seq after prefill, logits, token)}) for one shape at a time."""
    if name not in _cache:
        _cache.clear()
        shape = _shape(name)
        m = onp.NpOracle(shape, WSEED)
        pre = {}
        for rid, n in enumerate(LENS):
            seq = m.new_seq()
            tok, lg = m.prefill(seq, _prompt(rid, n, shape.vocab))
            pre[rid] = (seq, lg, tok)
        _cache[name] = (m, pre)
    return _cache[name]


@pytest.fixture(autouse=True)
def poisoned_kv(monkeypatch):
    monkeypatch.setenv("MESH_GPU_POISON", "1")


@pytest.mark.parametrize("quota", QUOTAS)
@pytest.mark.parametrize("name", NAMES)
def test_full_width_prefill_and_ragged_decode(name, quota):
    shape = _shape(name)
    m, pre = _oracle(name)
    g = MeshGpu(0, sm_quota=quota, kv_pool_bytes=2 << 30, prompt_seed=SEED_PROMPT)
    g.capture_logits(True)
    try:
        g.create_instance(1, shape, seed=WSEED)
        g.kv_resize(1, 0, (sum(LENS) + DECODE_STEPS * len(LENS) + 16 * 16) * shape.kv_bytes_per_token)
        seqs, last = {}, {}
        for rid, n in enumerate(LENS):
            toks, lg = g.step(1, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
            seq, olg, otok = pre[rid]
            _check(lg[0], toks[0], olg, f"{name}/q{quota} prefill r{rid} L={n}")
            seqs[rid] = copy.deepcopy(seq)
            last[rid] = toks[0]
        order = [4, 0, 7, 2, 5, 1, 6, 3]  # admission order, not request order
        for step in range(DECODE_STEPS):
            toks, lg = g.step(1, decode=order, vocab=shape.vocab, with_logits=True)
            outs = m.decode([seqs[r] for r in order], [last[r] for r in order])
            for i, rid in enumerate(order):
                _check(lg[i], toks[i], outs[i][1], f"{name}/q{quota} decode {step} r{rid} pos {LENS[rid] + step}")
                last[rid] = toks[i]
        for rid, n in enumerate(LENS):
            ctx, blocks = g.request_info(1, rid)
            assert ctx == n + DECODE_STEPS and len(blocks) == (ctx + 15) // 16
    finally:
        g.close()


@pytest.mark.parametrize("name", NAMES)
def test_full_width_shrink_swap_migrate(name):
    """KV shrink compaction, swap to pinned host + resume, and migration between
    two instances of the same model, each followed by decode against the oracle."""
    shape = _shape(name)
    m, pre = _oracle(name)
    C = shape.kv_bytes_per_token
    g = MeshGpu(0, kv_pool_bytes=2 << 30, prompt_seed=SEED_PROMPT, lanes=2)
    g.capture_logits(True)
    try:
        g.create_instance(1, shape, seed=WSEED)
        g.create_instance(2, shape, seed=WSEED)
        g.kv_resize(1, 0, 2000 * C)
        g.kv_resize(2, 0, 2000 * C)
        rids = [4, 0, 7]  # 900, 300, 250 tokens
        seqs, last = {}, {}
        for rid in rids:
            toks, lg = g.step(1, prefill=rid, prefill_len=LENS[rid], vocab=shape.vocab, with_logits=True)
            _check(lg[0], toks[0], pre[rid][1], f"{name} prefill r{rid}")
            seqs[rid] = copy.deepcopy(pre[rid][0])
            last[rid] = toks[0]

        def decode(inst, rs, what):
            toks, lg = g.step(inst, decode=rs, vocab=shape.vocab, with_logits=True)
            outs = m.decode([seqs[r] for r in rs], [last[r] for r in rs])
            for i, r in enumerate(rs):
                _check(lg[i], toks[i], outs[i][1], f"{name} {what} r{r}")
                last[r] = toks[i]

        # shrink: request 4 (the low 57 blocks) leaves, 0 and 7 sit above the new cap
        g.request_free(1, 4)
        moved0 = g.stats()["blocks_moved"]
        g.kv_resize(1, 2000 * C, (LENS[0] + LENS[7] + 64) * C)
        kv = g.instance_kv(1)
        for rid in (0, 7):
            _, blocks = g.request_info(1, rid)
            assert max(blocks) < kv["capacity_blocks"]
        assert g.stats()["blocks_moved"] > moved0
        for step in range(3):
            decode(1, [0, 7], f"post-compaction {step}")
        # swap request 0 out to pinned host; its re-prefill (I+O tokens) resumes from the parked KV
        n_hist = LENS[0] + 3 + 1
        sw0 = g.stats()["swap_in_bytes"]
        g.swap_out(1, 0)
        toks, lg = g.step(1, prefill=0, prefill_len=n_hist, vocab=shape.vocab, with_logits=True)
        tok, olg = m.decode([seqs[0]], [last[0]])[0]
        _check(lg[0], toks[0], olg, f"{name} resume after swap")
        last[0] = toks[0]
        assert g.stats()["swap_in_bytes"] > sw0
        # migrate request 7 to instance 2 (another lane), decode both there and here
        g.migrate_to(1, g, 2, 7)
        decode(2, [7], "after migration")
        decode(1, [0], "swapped-in request")
    finally:
        g.close()


@pytest.mark.parametrize("pair,splitk", [("0", "0"), ("1", "0"), ("0", "2"), ("1", "4")])
def test_prefill_gemm_variants(pair, splitk, monkeypatch):
    """The single-CTA and CTA-pair (cta_group::2) prefill GEMMs, with and without
    split-K of the down projection (forced factors), at full width: the 3B shape,
    a 300-token and a 900-token prompt (ragged token tiles), then a decode step."""
    monkeypatch.setenv("MESH_PREFILL_2SM", pair)
    monkeypatch.setenv("MESH_PREFILL_SPLITK", splitk)
    name = "3b"
    m, pre = _oracle(name)
    shape = _shape(name)
    g = MeshGpu(0, kv_pool_bytes=2 << 30, prompt_seed=SEED_PROMPT)
    try:
        g.capture_logits(True)
        g.create_instance(1, shape, seed=WSEED)
        g.kv_resize(1, 0, 1400 * shape.kv_bytes_per_token)
        for rid in (0, 4):
            toks, lg = g.step(1, prefill=rid, prefill_len=LENS[rid], vocab=shape.vocab, with_logits=True)
            _check(lg[0], toks[0], pre[rid][1], f"pair={pair} splitk={splitk} prefill r{rid}")
        toks, lg = g.step(1, decode=[0, 4], vocab=shape.vocab, with_logits=True)
        outs = m.decode([copy.deepcopy(pre[r][0]) for r in (0, 4)], [int(tok) for tok in _first_tokens(g, (0, 4))])
        for i, rid in enumerate((0, 4)):
            _check(lg[i], toks[i], outs[i][1], f"pair={pair} splitk={splitk} decode r{rid}")
    finally:
        g.close()


def _first_tokens(g, rids):
    """The token each request's prefill emitted (the GPU's, which the decode consumed)."""
    return [g.request_tokens(1, r)[LENS[r]] for r in rids]
