# Attention A/B on one GPU: a device-side pipeline trace (MESH_PF_ATTN_TRACE) of one 7B
# L=4000 layer, ncu per-launch times of pf_attn at L=1024/4000, and the prefill parity suites.
# usage (on the GPU box): bash tools/attn_meas.sh

MESH_PF_ATTN_TRACE=gpurun_out/pa_trace4.txt timeout 120 python tools/one_prefill.py 7b 4000 1 > /dev/null 2>&1
for L in 1024 4000; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pf_attn --csv --log-file gpurun_out/attn_$L.csv python tools/one_prefill.py 7b $L 4 > /dev/null 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_long.py -x -q > gpurun_out/pt_attn.log 2>&1; tail -3 gpurun_out/pt_attn.log
