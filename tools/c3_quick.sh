#!/bin/bash
# Quick tiled-path check under gpurun: GPU parity tests, C3 bench (optionally with env overrides), launch list.
# usage: tools/c3_quick.sh <tag> ["ENV=.. ENV2=.."...]
tag=${1:-run}; shift
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for envs in "" "$@"; do
  env $envs timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', d['ms_per_step'], d['phases_us'], d['graph'], d['parity_sample'], d['roofline']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cub|Radix" -c 60 --csv --log-file gpurun_out/launches_c3_$tag.csv python bench.py --config C3 --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3_$tag.csv 2>&1 | head -16
