"""TEST INFRASTRUCTURE ONLY (never imported by the product path).

Restatement of the data plane's KV block-table policy, the checker for
tests/test_gpu_block_tables.py and the generator of tests/golden/block_tables.json.
The reference has no block tables ("page-level block management" is a non-goal,
proj/SPEC.md:392): it accounts KV in bytes. What it pins, and what this script
drives the pool with, is the byte target of every KV ScaleOp:

  m_require     proj/src/memory.cpp:19-27   ceil(C * max(sum_r I_r + max(gen_r, avg_out), min_total_len))
  watermark     proj/src/memory.cpp:29-36   recommend = scale_bytes_up(m_req); up if cur < m_req,
                                            down if scale_bytes_up(recommend) < cur, else hold
  scale_bytes_up proj/src/types.hpp:30-32   ceil(base * (100 + pct) / 100)

The block policy it restates (paper_2507_00507_b200/csrc/gpu/dataplane.cu):
  * capacity(target) = ceil((target // C) / 16) + 8 blocks (one partial tail
    block per batch column); grow adds blocks [cap, new_cap) to the free set;
  * allocation takes the LOWEST free block id (overcommit cap+1 when empty);
  * a request's blocks are allocated in position order as its context crosses
    each 16-token boundary (prefill: ceil(L / 16) at once);
  * shrink compacts: requests in id order, blocks in position order, every
    block >= new_cap moves to the lowest free id < new_cap;
  * free / swap-out return blocks below the capacity to the free set (swap-out
    once its gather finished: the test synchronises before the next op);
  * resume of a parked request allocates ceil(ctx / 16) blocks, then the
    resume token's block if it starts a new one.
"""
from __future__ import annotations

import math

KV_BLOCK_TOKENS = 16
DEC_MAXB = 8


def scale_bytes_up(base: int, pct: float) -> int:
    return int(math.ceil(float(base) * (100.0 + pct) / 100.0))


def m_require(batch: list[tuple[int, int]], C: int, avg_output: float, min_total_len: int) -> int:
    """batch = [(input_len, tokens_generated)] (memory.cpp:19-27)."""
    total = 0.0
    for i, gen in batch:
        total += i + max(float(gen), avg_output)
    return int(math.ceil(max(total, float(min_total_len)) * float(C)))


def watermark_decide(cur: int, req: int, pct: float) -> tuple[str, int]:
    rec = scale_bytes_up(req, pct)
    if cur < req:
        return "up", rec
    if scale_bytes_up(rec, pct) < cur:
        return "down", rec
    return "hold", rec


class BlockPool:
    def __init__(self, C: int):
        self.C = C
        self.cap = 0
        self.target = 0
        self.free: set[int] = set()
        self.live = 0
        self.reqs: dict[int, dict] = {}   # rid -> {"ctx", "blocks"}
        self.parked: dict[int, int] = {}  # rid -> ctx of the parked KV

    def blocks_for_target(self, t: int) -> int:
        if t <= 0:
            return 0
        tokens = t // self.C
        return (tokens + KV_BLOCK_TOKENS - 1) // KV_BLOCK_TOKENS + DEC_MAXB

    def _alloc(self) -> int:
        if not self.free:
            b = self.cap
            self.cap += 1
            self.live += 1
            return b
        b = min(self.free)
        self.free.remove(b)
        self.live += 1
        return b

    def _release(self, blocks):
        for b in blocks:
            if b < self.cap:
                self.free.add(b)
            self.live -= 1

    def resize(self, to: int) -> None:
        new_cap = self.blocks_for_target(to)
        if new_cap >= self.cap:
            self.free |= set(range(self.cap, new_cap))
            self.cap = new_cap
            self.target = to
            return
        assert self.live <= new_cap, "shrink below live blocks"
        low = sorted(b for b in self.free if b < new_cap)
        for rid in sorted(self.reqs):
            blocks = self.reqs[rid]["blocks"]
            for i, b in enumerate(blocks):
                if b >= new_cap:
                    blocks[i] = low.pop(0)
        self.free = set(low)
        self.cap = new_cap
        self.target = to

    def prefill(self, rid: int, n: int) -> None:
        r = self.reqs.setdefault(rid, {"ctx": 0, "blocks": []})
        if r["ctx"] == 0 and rid in self.parked:  # resume from parked KV: its blocks first
            ctx = self.parked.pop(rid)
            if ctx == n - 1:
                r["blocks"] = [self._alloc() for _ in range((ctx + KV_BLOCK_TOKENS - 1) // KV_BLOCK_TOKENS)]
                r["ctx"] = ctx
        if r["ctx"] == n - 1 and r["ctx"] > 0:
            p0, L = n - 1, 1
        else:
            self._release(r["blocks"])
            r["blocks"] = []
            p0, L = 0, n
        need = (p0 + L + KV_BLOCK_TOKENS - 1) // KV_BLOCK_TOKENS
        while len(r["blocks"]) < need:
            r["blocks"].append(self._alloc())
        r["ctx"] = p0 + L

    def decode(self, rids) -> None:
        for rid in rids:
            r = self.reqs[rid]
            if r["ctx"] % KV_BLOCK_TOKENS == 0:
                r["blocks"].append(self._alloc())
            r["ctx"] += 1

    def free_request(self, rid: int) -> None:
        r = self.reqs.pop(rid)
        self._release(r["blocks"])

    def swap_out(self, rid: int) -> None:
        r = self.reqs.pop(rid)
        self.parked[rid] = r["ctx"]
        self._release(r["blocks"])

    def snapshot(self) -> dict:
        return {"cap": self.cap, "target": self.target,
                "blocks": {str(rid): list(r["blocks"]) for rid, r in sorted(self.reqs.items())}}


# The scripted sequence (shared by the golden generator and the GPU test).
AVG_OUT = 64.0
MIN_TOTAL = 256
WATERMARK = 20.0


def script():
    """[(op, args)]: admissions resize the pool by the reference's watermark rule
    over m_require of the batch, completions shrink it the same way."""
    lens = {0: (300, 40), 1: (50, 20), 2: (700, 30), 3: (100, 60), 4: (33, 10), 5: (420, 25)}
    ops = []
    batch: dict[int, tuple[int, int]] = {}  # rid -> (I, generated)

    def admit(rid):
        batch[rid] = (lens[rid][0], 0)
        ops.append(("admit", rid, sorted(batch.values())))
        ops.append(("prefill", rid, lens[rid][0]))
        batch[rid] = (lens[rid][0], 1)

    def decode(k):
        for _ in range(k):
            rids = sorted(batch)
            ops.append(("decode", rids))
            for r in rids:
                batch[r] = (batch[r][0], batch[r][1] + 1)

    def finish(rid):
        del batch[rid]
        ops.append(("free", rid, sorted(batch.values())))

    admit(0)
    admit(1)
    admit(2)
    decode(20)
    finish(1)
    admit(3)
    decode(17)
    ops.append(("swap_out", 0, None))
    del_0 = batch.pop(0)
    ops.append(("shrink", None, sorted(batch.values())))
    admit(4)
    decode(5)
    finish(2)
    batch[0] = del_0
    ops.append(("admit", 0, sorted(batch.values())))
    ops.append(("prefill", 0, del_0[0] + del_0[1]))  # re-prefill of I + generated: resumes the parked KV
    batch[0] = (del_0[0], del_0[1] + 1)
    admit(5)
    decode(9)
    finish(3)
    finish(4)
    decode(3)
    return ops


def run(C: int, ops=None):
    """Applies the script to a BlockPool; returns the snapshot after every op."""
    pool = BlockPool(C)
    out = []
    for op in ops or script():
        kind = op[0]
        if kind == "free":
            pool.free_request(op[1])
        if kind in ("admit", "free", "shrink"):
            req = m_require(op[2], C, AVG_OUT, MIN_TOTAL)
            act, rec = watermark_decide(pool.target, req, WATERMARK)
            if act != "hold":
                pool.resize(rec)
        elif kind == "prefill":
            pool.prefill(op[1], op[2])
        elif kind == "decode":
            pool.decode(op[1])
        elif kind == "swap_out":
            pool.swap_out(op[1])
        out.append(pool.snapshot())
    return out
