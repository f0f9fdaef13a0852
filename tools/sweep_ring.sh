#!/bin/bash
# decode ring-depth / L2 run-ahead sweep (device time per step)
for m in 1b 7b; do
  for cfg in "16 32" "16 0" "12 0" "8 0" "6 0" "4 0" "8 8"; do
    set -- $cfg
    r=$(MESH_GPU_NSTAGE=$1 MESH_GPU_L2_AHEAD=$2 PROBE_ITERS=10 timeout 120 python tools/probe_perf.py $m 2>&1 | tail -1)
    echo "$m nstage=$1 l2=$2 $r"
  done
done
