"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/llama_ref.c (CPU numeric
oracle). Imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg; never by the product package."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libmesh_oracle.so")


class OraShape(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d", C.c_int), ("n_heads", C.c_int), ("n_kv", C.c_int), ("dh", C.c_int),
                ("ff", C.c_int), ("vocab", C.c_int), ("tied", C.c_int), ("max_seq", C.c_int),
                ("rope_theta", C.c_float), ("eps", C.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            from paper_2507_00507_b200 import build
            build.build_oracle()
        l = C.CDLL(LIB_PATH)
        l.ora_create.restype = C.c_void_p
        l.ora_create.argtypes = [C.POINTER(OraShape), C.c_uint64, C.c_int]
        l.ora_free.argtypes = [C.c_void_p]
        l.ora_seq_new.restype = C.c_void_p
        l.ora_seq_new.argtypes = [C.c_void_p]
        l.ora_seq_free.argtypes = [C.c_void_p]
        l.ora_feed.restype = C.c_int
        l.ora_feed.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_float)]
        l.ora_prompt_token.restype = C.c_int
        l.ora_prompt_token.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int]
        l.ora_weight.restype = C.c_float
        l.ora_weight.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_uint64]
        l.ora_threads.restype = C.c_int
        l.ora_feed_batch.restype = C.c_int
        l.ora_feed_batch.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]
        _lib = l
    return _lib


class Oracle:
    def __init__(self, shape, seed: int, round_act: bool = True):
        s = OraShape(shape.n_layers, shape.d_model, shape.n_heads, shape.n_kv_heads, shape.d_head, shape.d_ff,
                     shape.vocab, int(shape.tied), shape.max_seq_len, shape.rope_theta, shape.rms_eps)
        self.shape = shape
        self.h = lib().ora_create(C.byref(s), seed, int(round_act))

    def close(self):
        if self.h:
            lib().ora_free(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def new_seq(self) -> "OracleSeq":
        return OracleSeq(self)


class OracleSeq:
    def __init__(self, m: Oracle):
        self.m = m
        self.h = lib().ora_seq_new(m.h)

    def set_len(self, n: int) -> None:
        """Bench only: declare n tokens of (zero-valued) KV resident without computing
        them; a decode step's cost depends on the context length, not the values."""
        if not 0 <= n < self.m.shape.max_seq_len:
            raise ValueError("context out of range")
        C.cast(C.c_void_p(self.h), C.POINTER(C.c_int))[0] = n

    def feed(self, token: int, want_logits: bool = True):
        buf = np.zeros(self.m.shape.vocab, dtype=np.float32) if want_logits else None
        ptr = buf.ctypes.data_as(C.POINTER(C.c_float)) if want_logits else None
        nxt = lib().ora_feed(self.m.h, self.h, token, ptr)
        return nxt, buf

    def __del__(self):
        if self.h:
            lib().ora_seq_free(self.h)
            self.h = None


def feed_batch(model: Oracle, seqs: list, tokens: list[int]) -> list[int]:
    """Batched CPU decode step (oracle/cpu_decode.c): the bench's CPU baseline, not the checker."""
    n = len(seqs)
    hs = (C.c_void_p * n)(*[q.h for q in seqs])
    tk = (C.c_int * n)(*tokens)
    nx = (C.c_int * n)()
    if lib().ora_feed_batch(model.h, hs, n, tk, nx) != 0:
        raise RuntimeError("ora_feed_batch: sequence full")
    return list(nx)


def prompt_token(seed: int, request: int, pos: int, vocab: int) -> int:
    return lib().ora_prompt_token(seed, request, pos, vocab)


def weight(seed: int, tensor: int, layer: int, index: int) -> float:
    return lib().ora_weight(seed, tensor, layer, index)


def threads() -> int:
    return lib().ora_threads()
