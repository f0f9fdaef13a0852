"""ctypes view of the control plane's C ABI (include/llmmesh.h, libllmmesh.so).

The same binding works for the reference library (oracle/_ref/libllmmesh_ref.so)
because the entry points and status codes are the reference's; only the
B200 extensions (capture, attach_gpu) are absent there.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libllmmesh.so")

LLM_OK, LLM_ERR_ARG, LLM_ERR_CONFIG, LLM_ERR_RUNTIME = 0, 1, 2, 3

EXPORTED = ["llm_version", "llm_experiment_open", "llm_experiment_set", "llm_experiment_set_seed",
            "llm_experiment_set_output_dir", "llm_experiment_run", "llm_experiment_compare",
            "llm_experiment_metric", "llm_experiment_error", "llm_experiment_close", "llm_experiment_capture",
            "llm_experiment_attach_gpu"]


class LlmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"llm status {status}: {msg}")
        self.status = status


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    P = C.POINTER
    sig = {
        "llm_version": (C.c_char_p, []),
        "llm_experiment_open": (C.c_int, [C.c_char_p, P(C.c_void_p)]),
        "llm_experiment_set": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
        "llm_experiment_set_seed": (C.c_int, [C.c_void_p, C.c_uint64]),
        "llm_experiment_set_output_dir": (C.c_int, [C.c_void_p, C.c_char_p]),
        "llm_experiment_run": (C.c_int, [C.c_void_p]),
        "llm_experiment_compare": (C.c_int, [C.c_void_p, C.c_char_p]),
        "llm_experiment_metric": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_double)]),
        "llm_experiment_error": (C.c_char_p, [C.c_void_p]),
        "llm_experiment_close": (None, [C.c_void_p]),
    }
    if hasattr(lib, "llm_experiment_capture"):
        sig["llm_experiment_capture"] = (C.c_int, [C.c_void_p, C.c_char_p])
        sig["llm_experiment_attach_gpu"] = (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_int32), C.c_int32, C.c_int64])
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


class Experiment:
    def __init__(self, config_path: str, lib: C.CDLL | None = None):
        self.lib = lib or load()
        self.h = C.c_void_p()
        st = self.lib.llm_experiment_open(config_path.encode(), C.byref(self.h))
        if st != LLM_OK:
            raise LlmError(st, "open failed")

    def _ck(self, st: int) -> None:
        if st != LLM_OK:
            raise LlmError(st, self.lib.llm_experiment_error(self.h).decode())

    def set(self, key: str, value) -> "Experiment":
        self._ck(self.lib.llm_experiment_set(self.h, key.encode(), str(value).encode()))
        return self

    def seed(self, s: int) -> "Experiment":
        self._ck(self.lib.llm_experiment_set_seed(self.h, s))
        return self

    def out_dir(self, d: str) -> "Experiment":
        self._ck(self.lib.llm_experiment_set_output_dir(self.h, d.encode()))
        return self

    def run(self) -> None:
        self._ck(self.lib.llm_experiment_run(self.h))

    def compare(self, policies: str) -> None:
        self._ck(self.lib.llm_experiment_compare(self.h, policies.encode()))

    def capture(self, d: str) -> None:
        self._ck(self.lib.llm_experiment_capture(self.h, d.encode()))

    def attach_gpu(self, devices=(0,), kv_pool_bytes: int = 0, gpu_lib: str | None = None) -> None:
        from . import gpu
        arr = (C.c_int32 * len(devices))(*devices)
        self._ck(self.lib.llm_experiment_attach_gpu(self.h, (gpu_lib or gpu.LIB_PATH).encode(), arr, len(devices),
                                                    kv_pool_bytes))

    def metric(self, name: str) -> float:
        v = C.c_double()
        self._ck(self.lib.llm_experiment_metric(self.h, name.encode(), C.byref(v)))
        return v.value

    def close(self) -> None:
        if self.h:
            self.lib.llm_experiment_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
