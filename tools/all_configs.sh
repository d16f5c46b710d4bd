#!/bin/bash
# Bench every BASELINE config once (device-resident timing, no CPU baseline) and a launch list per config.
# usage: tools/all_configs.sh <tag> [configs...]
tag=${1:-run}; shift
cfgs=${@:-C1 C2 C4 C5}
mkdir -p gpurun_out
for c in $cfgs; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${tag}_$c.json 2> gpurun_out/bench_${tag}_$c.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${tag}_$c.json')); print('$c', d['ms_per_step'], d['value'], d['phases_us'], d['graph'], d.get('parity_sample'))" || tail -3 gpurun_out/bench_${tag}_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cub|Radix" -c 80 --csv --log-file gpurun_out/launches_${tag}_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_${tag}_$c.csv 2>&1 | head -8
done
