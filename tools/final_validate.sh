# Round-end validation on one GPU: GPU tests, smoke, the default bench line, and the
# ncu launch list of a short bench (per-launch device times; never a bench value).
# usage (on the GPU box): bash tools/final_validate.sh <tag>
tag=${1:-final}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_$tag.log 2>&1; tail -2 gpurun_out/gputest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$tag.log 2>&1; tail -1 gpurun_out/smoke_$tag.log
timeout 2000 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 300 gpurun_out/bench_$tag.json
MESH_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 200 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; wc -l gpurun_out/launches_$tag.csv
