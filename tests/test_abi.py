"""C-ABI boundary checks (CPU): both libraries load without a GPU and export
every function their public header declares; the data plane reports its
absence of devices with a status instead of falling back to the CPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_00507_b200")


def _declared(header: str, prefix: str) -> list[str]:
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def libs():
    from paper_2507_00507_b200 import build

    build.build_gpu()
    build.build_control()
    return {
        "mesh_gpu.h": C.CDLL(os.path.join(PKG, "libmesh_gpu.so")),
        "llmmesh.h": C.CDLL(os.path.join(PKG, "libllmmesh.so")),
    }


@pytest.mark.parametrize("header,prefix", [("mesh_gpu.h", "mesh_gpu_"), ("llmmesh.h", "llm_")])
def test_every_declared_symbol_is_exported(libs, header, prefix):
    names = _declared(header, prefix)
    assert len(names) >= 10, names
    missing = [n for n in names if not hasattr(libs[header], n)]
    assert not missing, f"{header}: not exported: {missing}"


def test_reference_abi_is_a_subset(libs):
    # proj/include/llmmesh.h:17-56: the entry points callers bind
    ref = ["llm_version", "llm_experiment_open", "llm_experiment_set", "llm_experiment_set_seed",
           "llm_experiment_set_output_dir", "llm_experiment_run", "llm_experiment_compare",
           "llm_experiment_metric", "llm_experiment_error", "llm_experiment_close"]
    assert set(ref) <= set(_declared("llmmesh.h", "llm_"))
    for n in ref:
        assert hasattr(libs["llmmesh.h"], n)


def test_status_codes_and_null_handling(libs):
    L = libs["llmmesh.h"]
    L.llm_experiment_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.llm_experiment_metric.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double)]
    L.llm_experiment_error.restype = C.c_char_p
    L.llm_experiment_error.argtypes = [C.c_void_p]
    assert L.llm_experiment_open(None, None) == 1  # LLM_ERR_ARG (capi.cpp:56-60)
    h = C.c_void_p()
    assert L.llm_experiment_open(b"/nonexistent.json", C.byref(h)) == 0  # config read lazily
    L.llm_experiment_run.argtypes = [C.c_void_p]
    assert L.llm_experiment_run(h) == 2  # LLM_ERR_CONFIG for an unreadable config
    assert L.llm_experiment_error(h)
    d = C.c_double()
    assert L.llm_experiment_metric(h, b"no_such_metric", C.byref(d)) == 1
    L.llm_experiment_close.argtypes = [C.c_void_p]
    L.llm_experiment_close(h)


def test_gpu_library_without_device_fails_loudly(libs):
    G = libs["mesh_gpu.h"]
    G.mesh_gpu_device_count.restype = C.c_int32
    if G.mesh_gpu_device_count() > 0:
        pytest.skip("a GPU is present")
    G.mesh_gpu_version.restype = C.c_char_p
    assert G.mesh_gpu_version()
    # no CPU fallback: opening a device that does not exist returns an error status
    cfg = (C.c_byte * 256)()
    h = C.c_void_p()
    G.mesh_gpu_open.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    assert G.mesh_gpu_open(cfg, C.byref(h)) != 0
