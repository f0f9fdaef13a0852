"""Worker for tests/test_dist.py: the bench's cross-rank plumbing (bench.Dist) on
gloo. Each rank plays an independent co-located node (instances shard by
placement): the job's device time is the max over ranks and its
tokens the sum, exactly as bench.py reduces them."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

d = bench.Dist()
assert d.ws == int(os.environ["WORLD_SIZE"]) and d.backend == "gloo"
d.barrier()
dev_s = 1.0 + d.rank          # rank r "took" 1 + r seconds of device time
tokens = 100.0 * (d.rank + 1)  # and emitted 100 (r + 1) tokens
wall = d.reduce(dev_s, "max")
tok = d.reduce(tokens, "sum")
if d.rank == 0:
    print(json.dumps({"ws": d.ws, "wall": wall, "tokens": tok, "value": tok / wall}))
d.close()
