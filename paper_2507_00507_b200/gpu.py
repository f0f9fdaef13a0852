"""ctypes view of the B200 data plane (include/mesh_gpu.h).

Python is only the test/bench harness here: every call goes straight into
libmesh_gpu.so. Loading fails loudly when the library is missing — there is
no fallback implementation.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MESH_GPU_LIB: an alternative build of the same library (A/B experiments under tools/)
LIB_PATH = os.environ.get("MESH_GPU_LIB") or os.path.join(_HERE, "libmesh_gpu.so")

MESH_OK = 0


class MeshGpuError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"mesh_gpu status {status}: {msg}")
        self.status = status


class ModelShape(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_head", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
                ("tied_embeddings", C.c_int32), ("max_seq_len", C.c_int32), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float)]


class GpuCfg(C.Structure):
    _fields_ = [("device", C.c_int32), ("sm_quota", C.c_int32), ("kv_pool_bytes", C.c_int64),
                ("prompt_seed", C.c_uint64), ("kv_granule_bytes", C.c_int64), ("lanes", C.c_int32),
                ("swap_pool_mb", C.c_int32)]


class StepPlan(C.Structure):
    _fields_ = [("is_prefill", C.c_int32), ("prefill_request", C.c_int64), ("prefill_len", C.c_int32),
                ("prefill_input_len", C.c_int32), ("n_decode", C.c_int32),
                ("decode_requests", C.POINTER(C.c_int64))]


class GpuStats(C.Structure):
    _fields_ = [("kv_mapped_bytes", C.c_int64), ("kv_pool_bytes", C.c_int64), ("blocks_moved", C.c_int64),
                ("bytes_moved", C.c_int64), ("swap_out_bytes", C.c_int64), ("swap_in_bytes", C.c_int64),
                ("migrate_bytes", C.c_int64), ("steps", C.c_int64), ("decode_tokens", C.c_int64),
                ("prefill_tokens", C.c_int64), ("last_step_ms", C.c_double), ("last_kernel_ms", C.c_double),
                ("kernel_launches", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("kv_granule_bytes", C.c_int64), ("vmm_calls", C.c_int64), ("vmm_ms", C.c_double),
                ("kv_reclaims", C.c_int64), ("last_step_end_ms", C.c_double),
                ("weight_cache_hits", C.c_int64), ("peer_devices", C.c_int64),
                ("vmm_unmaps", C.c_int64), ("host_ms_create", C.c_double), ("host_ms_destroy", C.c_double),
                ("host_ms_kv_resize", C.c_double), ("host_ms_step", C.c_double)]


@dataclass(frozen=True)
class Shape:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_head: int
    d_ff: int
    vocab: int
    tied: bool = False
    max_seq_len: int = 2048
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5

    def c(self) -> ModelShape:
        return ModelShape(self.n_layers, self.d_model, self.n_heads, self.n_kv_heads, self.d_head, self.d_ff,
                          self.vocab, int(self.tied), self.max_seq_len, self.rope_theta, self.rms_eps)

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.d_head * 2

    @property
    def p_body(self) -> int:
        d, L = self.d_model, self.n_layers
        q = self.n_heads * self.d_head
        kv = self.n_kv_heads * self.d_head
        per_layer = d * q + 2 * d * kv + q * d + 3 * d * self.d_ff + 2 * d
        return L * per_layer + d

    @property
    def weight_bytes_streamed(self) -> int:
        """bf16 bytes a decode step must read: every weight except an untied input embedding."""
        return 2 * (self.p_body + self.vocab * self.d_model)

    def replace(self, **kw) -> "Shape":
        d = self.__dict__.copy()
        d.update(kw)
        return Shape(**d)


# Appendix B of SURVEY.md (Llama family). 3b uses Llama-3.2's true GQA KV size.
SHAPES: dict[str, Shape] = {
    "1b": Shape(22, 2048, 32, 4, 64, 5632, 32000, False, 2048, 10000.0),
    "3b": Shape(28, 3072, 24, 8, 128, 8192, 128256, True, 4096, 500000.0),
    "7b": Shape(32, 4096, 32, 32, 128, 11008, 32000, False, 4096, 10000.0),
    "13b": Shape(40, 5120, 40, 40, 128, 13824, 32000, False, 4096, 10000.0),
    # tiny shapes for CPU-checkable parity tests (same kernels, same code paths)
    "tiny": Shape(2, 256, 4, 2, 64, 512, 512, False, 512, 10000.0),
    "tiny128": Shape(2, 512, 4, 1, 128, 768, 384, True, 1024, 500000.0),
}

# generator tensor ids (csrc/gpu/model.cuh)
T_EMB, T_WQ, T_WK, T_WV, T_WO, T_WGATE, T_WUP, T_WDOWN, T_LM = range(9)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "mesh_gpu_version": (C.c_char_p, []),
        "mesh_gpu_device_count": (C.c_int32, []),
        "mesh_gpu_open": (C.c_int, [P(GpuCfg), P(C.c_void_p)]),
        "mesh_gpu_close": (None, [C.c_void_p]),
        "mesh_gpu_last_error": (C.c_char_p, [C.c_void_p]),
        "mesh_gpu_instance_create": (C.c_int, [C.c_void_p, C.c_int64, P(ModelShape), C.c_uint64]),
        "mesh_gpu_instance_destroy": (C.c_int, [C.c_void_p, C.c_int64]),
        "mesh_gpu_kv_resize": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64]),
        "mesh_gpu_step": (C.c_int, [C.c_void_p, C.c_int64, P(StepPlan), P(C.c_int64)]),
        "mesh_gpu_step_wait": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int32), C.c_int32, P(C.c_int32),
                                         P(C.c_float), C.c_int64]),
        "mesh_gpu_step_done": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int32)]),
        "mesh_gpu_set_capture_logits": (C.c_int, [C.c_void_p, C.c_int32]),
        "mesh_gpu_request_free": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
        "mesh_gpu_swap_out": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
        "mesh_gpu_swap_in": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
        "mesh_gpu_swap_state": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int32)]),
        "mesh_gpu_migrate": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64]),
        "mesh_gpu_request_info": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(C.c_int32), P(C.c_int32),
                                            P(C.c_int32), C.c_int32]),
        "mesh_gpu_request_tokens": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(C.c_int32), C.c_int32,
                                              P(C.c_int32)]),
        "mesh_gpu_instance_kv": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int64), P(C.c_int64), P(C.c_int32),
                                           P(C.c_int32)]),
        "mesh_gpu_instance_lane": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int32), P(C.c_int32)]),
        "mesh_gpu_read_weight": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, P(C.c_float),
                                           C.c_int32]),
        "mesh_gpu_stats_get": (C.c_int, [C.c_void_p, P(GpuStats)]),
        "mesh_gpu_sync": (C.c_int, [C.c_void_p]),
        "mesh_gpu_bench_decode": (C.c_int, [C.c_void_p, C.c_int64, P(StepPlan), C.c_int32, P(C.c_double)]),
        "mesh_gpu_timer_mark": (C.c_int, [C.c_void_p, C.c_int32]),
        "mesh_gpu_timer_elapsed": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, P(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


EXPORTED = ["mesh_gpu_version", "mesh_gpu_device_count", "mesh_gpu_open", "mesh_gpu_close", "mesh_gpu_last_error",
            "mesh_gpu_instance_create", "mesh_gpu_instance_destroy", "mesh_gpu_kv_resize", "mesh_gpu_step",
            "mesh_gpu_step_wait", "mesh_gpu_step_done", "mesh_gpu_set_capture_logits", "mesh_gpu_request_free", "mesh_gpu_swap_out",
            "mesh_gpu_swap_in", "mesh_gpu_swap_state", "mesh_gpu_migrate", "mesh_gpu_request_info", "mesh_gpu_request_tokens", "mesh_gpu_instance_kv",
            "mesh_gpu_read_weight", "mesh_gpu_stats_get", "mesh_gpu_sync", "mesh_gpu_bench_decode",
            "mesh_gpu_instance_lane"]


class MeshGpu:
    """One B200 (one handle of the C ABI)."""

    def __init__(self, device: int = 0, sm_quota: int = 0, kv_pool_bytes: int = 0, prompt_seed: int = 1234,
                 kv_granule_bytes: int = 0, lanes: int = 0, swap_pool_mb: int = 0):
        self._l = lib()
        cfg = GpuCfg(device, sm_quota, kv_pool_bytes, prompt_seed, kv_granule_bytes, lanes, swap_pool_mb)
        h = C.c_void_p()
        st = self._l.mesh_gpu_open(C.byref(cfg), C.byref(h))
        if st != MESH_OK:
            raise MeshGpuError(st, "mesh_gpu_open failed (no sm_100 device?)")
        self.h = h
        self.prompt_seed = prompt_seed

    def _ck(self, st: int) -> None:
        if st != MESH_OK:
            raise MeshGpuError(st, self._l.mesh_gpu_last_error(self.h).decode())

    def close(self) -> None:
        if self.h:
            self._l.mesh_gpu_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def create_instance(self, iid: int, shape: Shape, seed: int) -> None:
        s = shape.c()
        self._ck(self._l.mesh_gpu_instance_create(self.h, iid, C.byref(s), seed))

    def destroy_instance(self, iid: int) -> None:
        self._ck(self._l.mesh_gpu_instance_destroy(self.h, iid))

    def kv_resize(self, iid: int, frm: int, to: int) -> None:
        self._ck(self._l.mesh_gpu_kv_resize(self.h, iid, frm, to))

    def capture_logits(self, on: bool) -> None:
        self._ck(self._l.mesh_gpu_set_capture_logits(self.h, int(on)))

    def step_async(self, iid: int, *, prefill: int | None = None, prefill_len: int = 0, input_len: int = 0,
                   decode: list[int] | None = None) -> int:
        t = C.c_int64()
        if prefill is not None:
            plan = StepPlan(1, prefill, prefill_len, input_len or prefill_len, 0, None)
            self._ck(self._l.mesh_gpu_step(self.h, iid, C.byref(plan), C.byref(t)))
        else:
            arr = (C.c_int64 * len(decode))(*decode)
            plan = StepPlan(0, -1, 0, 0, len(decode), arr)
            self._ck(self._l.mesh_gpu_step(self.h, iid, C.byref(plan), C.byref(t)))
        return t.value

    def wait(self, ticket: int, vocab: int = 0, with_logits: bool = False):
        toks = (C.c_int32 * 8)()
        n = C.c_int32()
        if with_logits:
            buf = np.zeros(8 * vocab, dtype=np.float32)
            self._ck(self._l.mesh_gpu_step_wait(self.h, ticket, toks, 8, C.byref(n),
                                                buf.ctypes.data_as(C.POINTER(C.c_float)), buf.size))
            return list(toks[: n.value]), buf[: n.value * vocab].reshape(n.value, vocab)
        self._ck(self._l.mesh_gpu_step_wait(self.h, ticket, toks, 8, C.byref(n), None, 0))
        return list(toks[: n.value])

    def done(self, ticket: int) -> bool:
        """Non-blocking: has the step finished on the device?"""
        d = C.c_int32()
        self._ck(self._l.mesh_gpu_step_done(self.h, ticket, C.byref(d)))
        return bool(d.value)

    def step(self, iid: int, **kw):
        vocab = kw.pop("vocab", 0)
        with_logits = kw.pop("with_logits", False)
        return self.wait(self.step_async(iid, **kw), vocab, with_logits)

    def request_free(self, iid: int, rid: int) -> None:
        self._ck(self._l.mesh_gpu_request_free(self.h, iid, rid))

    def swap_out(self, iid: int, rid: int) -> None:
        self._ck(self._l.mesh_gpu_swap_out(self.h, iid, rid))

    def swap_in(self, iid: int, rid: int) -> None:
        self._ck(self._l.mesh_gpu_swap_in(self.h, iid, rid))

    SWAP_STATES = {0: "none", 1: "history", 2: "copying", 3: "parked"}

    def swap_state(self, rid: int) -> str:
        st = C.c_int32()
        self._ck(self._l.mesh_gpu_swap_state(self.h, rid, C.byref(st)))
        return self.SWAP_STATES[st.value]

    def migrate_to(self, src_iid: int, dst: "MeshGpu", dst_iid: int, rid: int) -> None:
        self._ck(self._l.mesh_gpu_migrate(self.h, src_iid, dst.h, dst_iid, rid))

    def request_info(self, iid: int, rid: int):
        ctx, nb = C.c_int32(), C.c_int32()
        ids = (C.c_int32 * 1024)()
        self._ck(self._l.mesh_gpu_request_info(self.h, iid, rid, C.byref(ctx), C.byref(nb), ids, 1024))
        return ctx.value, list(ids[: nb.value])

    def request_tokens(self, iid: int, rid: int) -> list[int]:
        buf = (C.c_int32 * 8192)()
        n = C.c_int32()
        self._ck(self._l.mesh_gpu_request_tokens(self.h, iid, rid, buf, 8192, C.byref(n)))
        return list(buf[: n.value])

    def instance_kv(self, iid: int):
        t, m = C.c_int64(), C.c_int64()
        cap, live = C.c_int32(), C.c_int32()
        self._ck(self._l.mesh_gpu_instance_kv(self.h, iid, C.byref(t), C.byref(m), C.byref(cap), C.byref(live)))
        return {"target": t.value, "mapped": m.value, "capacity_blocks": cap.value, "live_blocks": live.value}

    def instance_lane(self, iid: int) -> tuple[int, int]:
        """(lane, lane SM quota) the instance is bound to."""
        lane, ctas = C.c_int32(), C.c_int32()
        self._ck(self._l.mesh_gpu_instance_lane(self.h, iid, C.byref(lane), C.byref(ctas)))
        return lane.value, ctas.value

    def read_weight(self, iid: int, tensor: int, layer: int, row: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.float32)
        self._ck(self._l.mesh_gpu_read_weight(self.h, iid, tensor, layer, row,
                                              out.ctypes.data_as(C.POINTER(C.c_float)), n))
        return out

    def stats(self) -> dict:
        s = GpuStats()
        self._ck(self._l.mesh_gpu_stats_get(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in GpuStats._fields_}

    def sync(self) -> None:
        self._ck(self._l.mesh_gpu_sync(self.h))

    def timer_mark(self, slot: int) -> None:
        """Records a CUDA event on the compute stream (device-side timing)."""
        self._ck(self._l.mesh_gpu_timer_mark(self.h, slot))

    def timer_elapsed(self, a: int, b: int) -> float:
        """Device milliseconds between two marks (waits for mark b)."""
        ms = C.c_double()
        self._ck(self._l.mesh_gpu_timer_elapsed(self.h, a, b, C.byref(ms)))
        return ms.value

    def bench_decode(self, iid: int, rids: list[int], iters: int) -> float:
        arr = (C.c_int64 * len(rids))(*rids)
        plan = StepPlan(0, -1, 0, 0, len(rids), arr)
        ms = C.c_double()
        self._ck(self._l.mesh_gpu_bench_decode(self.h, iid, C.byref(plan), iters, C.byref(ms)))
        return ms.value
