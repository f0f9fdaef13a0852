"""GPU parity at long, ragged contexts and reduced SM quotas.

With 148 CTAs and short contexts every CTA holds at most one attention stage,
so the multi-stage paths of the decode kernel (a warp accumulating several
stages of a pair, the CTA-level pre-combine in shared memory, the cp.async
final combine, pairs spanning many CTAs, the global-combine fallback for more
than 8 partials) only run at long contexts or small grids. These tests drive
them with prefill lengths up to 400-900 tokens and SM quotas of 148 / 16 / 3,
against the CPU oracle (same tolerance as tests/test_gpu_parity.py).
"""
import numpy as np
import pytest

from oracle import llama_oracle as ora
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu, Shape
from test_gpu_parity import SEED_PROMPT, _check, _oracle_prefill

pytestmark = pytest.mark.gpu

# GQA group 8 at dh 64 is the 1.1B (TinyLlama) layout: only 3 pairs fit the
# shared-memory pre-combine area, so later pairs take the direct/global paths.
EXTRA = {
    "gq8": Shape(2, 512, 8, 1, 64, 512, 512, False, 1024, 10000.0),
    "gq8kv4": Shape(2, 2048, 32, 4, 64, 512, 512, False, 1024, 10000.0),
}
CASES = {
    "tiny": [300, 200, 225, 150, 401, 100],         # dh 64, GQA 2, RT 32 tokens/stage
    "tiny128": [700, 35, 513, 900, 64, 257, 16],    # dh 128, GQA 4, RT 16 tokens/stage
    "gq8": [923, 318, 254, 827, 334, 808, 607, 369],
    "gq8kv4": [923, 318, 254, 827, 334, 808, 607, 369],
}


@pytest.fixture(autouse=True)
def poisoned_kv(monkeypatch):
    """Newly mapped KV memory is NaN-filled (MESH_GPU_POISON), as recycled memory may
    be in production: any read of unwritten KV that can reach an output fails here."""
    monkeypatch.setenv("MESH_GPU_POISON", "1")


@pytest.mark.parametrize("quota", [0, 16, 3])
@pytest.mark.parametrize("name", ["tiny", "tiny128", "gq8", "gq8kv4"])
def test_long_ragged_decode(name, quota):
    shape = EXTRA.get(name) or SHAPES[name]
    lens = CASES[name]
    g = MeshGpu(0, sm_quota=quota, kv_pool_bytes=2 << 30, prompt_seed=SEED_PROMPT)
    g.capture_logits(True)
    model = ora.Oracle(shape, 21)
    try:
        g.create_instance(1, shape, seed=21)
        g.kv_resize(1, 0, (sum(lens) + 16 * 16) * shape.kv_bytes_per_token)
        seqs, last = {}, {}
        for rid, n in enumerate(lens):
            toks, lg = g.step(1, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
            seqs[rid], ol = _oracle_prefill(model, rid, n)
            _check(lg[0], toks[0], ol, f"{name}/q{quota} prefill r{rid} L={n}")
            last[rid] = toks[0]
        order = list(range(len(lens)))[::-1]
        for step in range(3):
            toks, lg = g.step(1, decode=order, vocab=shape.vocab, with_logits=True)
            assert all(0 <= t < shape.vocab for t in toks), toks
            for i, rid in enumerate(order):
                _, ol = seqs[rid].feed(last[rid])
                _check(lg[i], toks[i], ol, f"{name}/q{quota} decode {step} r{rid} pos {lens[rid] + step}")
                last[rid] = toks[i]
    finally:
        g.close()
