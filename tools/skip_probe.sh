for sk in 0 1 2 3; do MESH_GPU_SKIP=$sk PROBE_ITERS=30 timeout 120 python tools/probe_perf.py 1b 3b 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('skip=$sk', d['model'], round(d['decode_ms'],3))"; done
