#!/bin/bash
# Tiled-path check under gpurun: parity of the tiled kernels, C3 bench x2, launch list, optional ncu of k_tile.
# usage: tools/c3_check.sh <tag> [full]
tag=${1:-run}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
  timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_us'], d['graph'], d['parity_sample'], d['roofline']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv --log-file gpurun_out/launches_c3_$tag.csv python bench.py --config C3 --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_c3_$tag.csv 2>&1 | head -12
if [ "$2" = "full" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 2 -c 2 -o gpurun_out/prof_c3_$tag python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
  ls -la gpurun_out/prof_c3_$tag.ncu-rep
fi
