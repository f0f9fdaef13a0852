# A/B of the prefill grid cap on the C3 value leg (device time, same box, alternating order).
# usage (on the GPU box): bash tools/ab_prefill_quota.sh
for i in 1 2; do
  timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/abq_off_$i.json 2> /dev/null
  MESH_PREFILL_QUOTA=1 timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/abq_on_$i.json 2> /dev/null
done
for f in gpurun_out/abq_*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f',d['value'],d['roofline']['frac'],d.get('lane_busy'))"; done
