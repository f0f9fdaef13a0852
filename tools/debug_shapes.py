"""Debug probe: per-request decode rel-L2 vs the numpy oracle at a full-width
shape, across SM quotas / context lengths (prints a table)."""
import copy, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import llama_np as onp, llama_oracle as ora
from paper_2507_00507_b200.gpu import SHAPES, MeshGpu

name = sys.argv[1]
quotas = [int(x) for x in sys.argv[2].split(",")]
lens = [int(x) for x in sys.argv[3].split(",")]
extra = dict(kv.split("=") for kv in sys.argv[4:])
shape = SHAPES[name].replace(n_layers=int(extra.get("layers", 2)), **({"d_ff": int(extra["ff"])} if "ff" in extra else {}))
m = onp.NpOracle(shape, 41)
pre = {}
for rid, n in enumerate(lens):
    s = m.new_seq()
    pre[rid] = (s, *m.prefill(s, [ora.prompt_token(1234, rid, i, shape.vocab) for i in range(n)]))
for q in quotas:
    g = MeshGpu(0, sm_quota=q, kv_pool_bytes=2 << 30, prompt_seed=1234)
    g.capture_logits(True)
    g.create_instance(1, shape, seed=41)
    g.kv_resize(1, 0, (sum(lens) + 64 * len(lens) + 256) * shape.kv_bytes_per_token)
    seqs, last = {}, {}
    for rid, n in enumerate(lens):
        toks, lg = g.step(1, prefill=rid, prefill_len=n, vocab=shape.vocab, with_logits=True)
        seqs[rid] = copy.deepcopy(pre[rid][0]); last[rid] = toks[0]
    order = list(range(len(lens)))
    for step in range(2):
        toks, lg = g.step(1, decode=order, vocab=shape.vocab, with_logits=True)
        outs = m.decode([seqs[r] for r in order], [last[r] for r in order])
        rls = [float(np.linalg.norm(lg[i] - outs[i][1]) / np.linalg.norm(outs[i][1])) for i in range(len(order))]
        print(f"q={q} step={step} rel-L2 per request: " + " ".join(f"{x:.3g}" for x in rls), flush=True)
        for i, r in enumerate(order):
            last[r] = toks[i]
    g.close()
