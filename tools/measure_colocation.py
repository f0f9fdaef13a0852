"""Co-location speedup of the C3 node (runtime.colocation_speedup): the device
time of the same instance-step sequence (bench.py's closed C3 loop, same seed)
run on ONE execution lane (instances one at a time on all SMs: the reference's
one-iteration-per-node model) over the time on eight lanes (instances stepping
concurrently on their SM quotas).  Prints one JSON object."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.chdir(ROOT)

import bench  # noqa: E402


def span(lanes, steps):
    bench.LANES = lanes
    node = bench.Colocated(0)
    node.k = 0
    node.fill()
    node.run(len(bench.MODELS) * bench.BATCH)
    node.run(5 * len(bench.MODELS))
    node.g.sync()
    node.reset_counters()
    node.g.timer_mark(0)
    node.mark0 = node.clock
    node.run(steps)
    node.g.timer_mark(1)
    node.g.sync()
    ms = node.g.timer_elapsed(0, 1)
    out = {"lanes": lanes, "device_ms": ms, "decode_steps": node.decode_steps, "prefill_steps": node.prefill_steps,
           "tokens": node.tokens_all, "decode_gbs": node.decode_bytes / (ms / 1e3) / 1e9}
    node.g.close()
    return out


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
    one = span(1, steps)
    eight = span(8, steps)
    print(json.dumps({"steps": steps, "serial": one, "colocated": eight,
                      "colocation_speedup": one["device_ms"] / eight["device_ms"]}))


if __name__ == "__main__":
    main()
