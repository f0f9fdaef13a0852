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
# the fleet leg's choreography (bench.run_ours, ws > 1): rank 0 drives every node
# through the control plane's placement while the other ranks wait; here on the
# virtual clock (no GPU): the C5 fleet scenario over ws nodes
fleet = None
d.barrier()
if d.rank == 0:
    import tempfile

    from paper_2507_00507_b200 import control
    with control.Experiment(bench.fleet_scenario(d.ws, 2 * d.ws)) as exp:
        exp.set("runtime.clock", "virtual")
        exp.out_dir(tempfile.mkdtemp())
        exp.run()
        fleet = {k: exp.metric(k) for k in ["gpu_nodes_used", "gpu_instances_max", "gpu_instances_avg",
                                            "total_requests", "slo_compliant_rate"]}
d.barrier()
if d.rank == 0:
    print(json.dumps({"ws": d.ws, "wall": wall, "tokens": tok, "value": tok / wall, "fleet": fleet}))
d.close()
