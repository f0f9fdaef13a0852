"""B200-native LLM-Mesh token-level co-located inference step.

Native code only: libllmmesh.so (C++20 control plane, reference C ABI
llmmesh.h) and libmesh_gpu.so (sm_100a data plane, mesh_gpu.h). The Python
modules here are thin ctypes views used by tests and bench.py.
"""
