"""TEST INFRASTRUCTURE ONLY — numpy restatement of the CPU numeric oracle
(oracle/llama_ref.c) for the full-width model shapes. Imported by tests/ only;
never by the product package.

oracle/llama_ref.c feeds one token at a time through double-accumulated GEMVs:
exact, but a 900-token prefill of a full-width 13B layer pair takes minutes.
This module states the SAME numerics contract (llama_ref.c header) with the
positions of a prompt, or the requests of a decode batch, as the rows of one
fp32 GEMM (numpy/OpenBLAS), so the parity tests can check the GPU path at the
3B / 7B / 13B widths the configs actually run:

  weights / embeddings / KV cache  bf16 (RNE), from the shared generator
                                   (ora_gen_bf16 == csrc/gpu/model.cuh);
  residual stream h                fp32;
  normed GEMV input                a = bf16(h * gamma), output * rs,
                                   rs = 1 / sqrt(mean(h^2) + eps) (double sum);
  q, k                             rotate-half RoPE in fp32 (table in double);
  attention                        double scores / softmax over bf16 K/V,
                                   output rounded to bf16 before W_o;
  MLP                              bf16(silu(g * rs) * (u * rs)) before W_down;
  logits                           fp32, greedy argmax, ties to the lowest id.

It differs from llama_ref.c only in GEMM accumulation (fp32 BLAS vs double),
which tests/test_oracle_np.py bounds against llama_ref.c (and against the HF
goldens, round_act = 0).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from oracle import llama_oracle as ora

T_EMB, T_WQ, T_WK, T_WV, T_WO, T_WGATE, T_WUP, T_WDOWN, T_LM, T_GATTN, T_GMLP, T_GFINAL = range(12)


def _lib():
    l = ora.lib()
    if not getattr(l, "_np_bound", False):
        l.ora_gen_bf16.restype = None
        l.ora_gen_bf16.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        l.ora_gen_gain.restype = None
        l.ora_gen_gain.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_void_p]
        l._np_bound = True
    return l


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest-even bf16, returned as fp32 (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    u = (u + (np.uint32(0x7FFF) + ((u >> 16) & np.uint32(1)))) & np.uint32(0xFFFF0000)
    return u.view(np.float32)


def gen_matrix(seed: int, tensor: int, layer: int, rows: int, cols: int) -> np.ndarray:
    raw = np.empty(rows * cols, dtype=np.uint16)
    _lib().ora_gen_bf16(seed, tensor, layer, raw.size, raw.ctypes.data)
    return (raw.astype(np.uint32) << 16).view(np.float32).reshape(rows, cols)


def gen_gain(seed: int, tensor: int, layer: int, n: int) -> np.ndarray:
    g = np.empty(n, dtype=np.float32)
    _lib().ora_gen_gain(seed, tensor, layer, n, g.ctypes.data)
    return g


class NpOracle:
    def __init__(self, shape, seed: int, round_act: bool = True, exact: bool = False):
        """exact: accumulate the GEMMs in double like llama_ref.c (slow; the CPU
        tests use it to show the restatement is the same arithmetic)."""
        s = shape
        self.shape, self.seed, self.round_act, self.exact = s, seed, round_act, exact
        d, qd, kd = s.d_model, s.n_heads * s.d_head, s.n_kv_heads * s.d_head
        self.emb = gen_matrix(seed, T_EMB, 0, s.vocab, d)
        self.lm = self.emb if s.tied else gen_matrix(seed, T_LM, 0, s.vocab, d)
        self.gf = gen_gain(seed, T_GFINAL, 0, d)
        self.layers = []
        for l in range(s.n_layers):
            self.layers.append({
                "wqkv": np.concatenate([gen_matrix(seed, T_WQ, l, qd, d), gen_matrix(seed, T_WK, l, kd, d),
                                        gen_matrix(seed, T_WV, l, kd, d)]),
                "wo": gen_matrix(seed, T_WO, l, d, qd),
                "wgu": np.concatenate([gen_matrix(seed, T_WGATE, l, s.d_ff, d), gen_matrix(seed, T_WUP, l, s.d_ff, d)]),
                "wd": gen_matrix(seed, T_WDOWN, l, d, s.d_ff),
                "ga": gen_gain(seed, T_GATTN, l, d),
                "gm": gen_gain(seed, T_GMLP, l, d),
            })
        half = s.d_head // 2
        # libm pow, as llama_ref.c / the device table (numpy's power differs in the last ulp)
        inv = np.array([math.pow(float(np.float32(s.rope_theta)), -2.0 * i / float(s.d_head)) for i in range(half)])
        ang = np.arange(s.max_seq_len, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = np.cos(ang).astype(np.float32)
        self.sin = np.sin(ang).astype(np.float32)

    def new_seq(self) -> "NpSeq":
        return NpSeq(self)

    # ---- pieces (row-batched)
    def _mm(self, a, w):
        if self.exact:
            return (a.astype(np.float64) @ w.T.astype(np.float64)).astype(np.float32)
        return a @ w.T

    def _act(self, x):
        return bf16_round(x) if self.round_act else x.astype(np.float32)

    def _norm(self, h, gamma):
        ss = np.sum(h.astype(np.float64) ** 2, axis=1)
        rs = (1.0 / np.sqrt(ss / h.shape[1] + float(np.float32(self.shape.rms_eps)))).astype(np.float32)
        return self._act(h * gamma[None, :]), rs

    def _rope(self, x, pos):
        """x [R, heads, dh] fp32, pos [R]: rotate-half."""
        half = x.shape[2] // 2
        c = self.cos[pos][:, None, :]
        s = self.sin[pos][:, None, :]
        x1, x2 = x[:, :, :half], x[:, :, half:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=2)

    def forward(self, seqs: list["NpSeq"], tokens: list[list[int]], all_logits: bool = False):
        """Feeds tokens[i] to seqs[i] at its current length; returns, per sequence,
        (greedy next token, logits of its last fed position) — or every position's
        logits when all_logits."""
        s = self.shape
        H, KV, dh = s.n_heads, s.n_kv_heads, s.d_head
        gq = H // KV
        rows, pos, owner = [], [], []
        for i, (q, tk) in enumerate(zip(seqs, tokens)):
            if q.len + len(tk) > s.max_seq_len:
                raise ValueError("sequence full")
            rows += list(tk)
            pos += list(range(q.len, q.len + len(tk)))
            owner += [i] * len(tk)
        pos = np.asarray(pos, dtype=np.int64)
        owner = np.asarray(owner)
        h = self.emb[np.asarray(rows)].copy()
        scale = 1.0 / np.sqrt(float(dh))
        for l, L in enumerate(self.layers):
            a, rs = self._norm(h, L["ga"])
            qkv = self._mm(a, L["wqkv"]) * rs[:, None]
            q = self._rope(qkv[:, : H * dh].reshape(-1, H, dh), pos)
            k = self._rope(qkv[:, H * dh: (H + KV) * dh].reshape(-1, KV, dh), pos)
            v = qkv[:, (H + KV) * dh:].reshape(-1, KV, dh)
            k, v = self._act(k), self._act(v)
            att = np.empty((len(rows), H, dh), dtype=np.float32)
            for i, sq in enumerate(seqs):
                sel = np.nonzero(owner == i)[0]
                if not len(sel):
                    continue
                p0, n = sq.len, len(sel)
                sq.put(l, p0, k[sel], v[sel])
                K, V = sq.k[l][: p0 + n].astype(np.float64), sq.v[l][: p0 + n].astype(np.float64)
                qi = q[sel].astype(np.float64).reshape(n, KV, gq, dh)
                # scores rounded to fp32 like llama_ref.c's sc[] buffer
                sc = np.matmul(qi.transpose(1, 2, 0, 3), K.transpose(1, 2, 0)[:, None])  # [KV, gq, n, T]
                sc = (sc * scale).astype(np.float32).astype(np.float64)
                causal = np.arange(p0 + n)[None, :] > (p0 + np.arange(n))[:, None]
                sc[:, :, causal] = -np.inf
                sc -= sc.max(axis=3, keepdims=True)
                e = np.exp(sc)
                o = np.matmul(e, V.transpose(1, 0, 2)[:, None]) / e.sum(axis=3, keepdims=True)  # [KV, gq, n, dh]
                att[sel] = o.transpose(2, 0, 1, 3).reshape(n, H, dh).astype(np.float32)
            att = self._act(att).reshape(len(rows), H * dh)
            h = h + self._mm(att, L["wo"])
            a, rs = self._norm(h, L["gm"])
            gu = self._mm(a, L["wgu"])
            gt, up = gu[:, : s.d_ff] * rs[:, None], gu[:, s.d_ff:] * rs[:, None]
            # expf as correctly rounded (glibc): exp in double, rounded once to fp32
            e = np.exp(-gt.astype(np.float64)).astype(np.float32)
            act = self._act(gt / (np.float32(1.0) + e) * up)
            h = h + self._mm(act, L["wd"])
        for sq, tk in zip(seqs, tokens):
            sq.len += len(tk)
        if all_logits:
            sel = np.arange(len(rows))
        else:
            sel = np.asarray([np.nonzero(owner == i)[0][-1] for i in range(len(seqs))])
        a, rs = self._norm(h[sel], self.gf)
        logits = self._mm(a, self.lm) * rs[:, None]
        if all_logits:
            return [logits[owner == i] for i in range(len(seqs))]
        return [(int(np.argmax(logits[j])), logits[j]) for j in range(len(seqs))]

    def prefill(self, seq: "NpSeq", tokens: list[int]):
        return self.forward([seq], [tokens])[0]

    def decode(self, seqs: list["NpSeq"], last: list[int]):
        return self.forward(seqs, [[t] for t in last])


class NpSeq:
    def __init__(self, m: NpOracle):
        s = m.shape
        self.len = 0
        self.cap = 0
        self.kvshape = (s.n_kv_heads, s.d_head)
        self.k = [np.zeros((0,) + self.kvshape, np.float32) for _ in range(s.n_layers)]
        self.v = [np.zeros((0,) + self.kvshape, np.float32) for _ in range(s.n_layers)]

    def put(self, layer: int, p0: int, k, v):
        n = p0 + len(k)
        if n > self.k[layer].shape[0]:
            cap = max(n, 2 * self.k[layer].shape[0], 64)
            for arr in (self.k, self.v):
                grown = np.zeros((cap,) + self.kvshape, np.float32)
                grown[: arr[layer].shape[0]] = arr[layer]
                arr[layer] = grown
        self.k[layer][p0:n] = k
        self.v[layer][p0:n] = v
