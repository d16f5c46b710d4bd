#!/bin/bash
# Standard GPU-box check (run under gpurun): parity tests, bench, ncu launch list + full profile.
# usage: tools/gpu_round.sh <tag> [pytest -k expr]
tag=${1:-run}; kexpr=${2:-}
mkdir -p gpurun_out
if [ -n "$kexpr" ]; then
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "$kexpr" 2>&1 | tail -5
else
  python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -3 gpurun_out/bench_$tag.err; cat gpurun_out/bench_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 300 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_resolve|k_exit_final" -s 6 -c 4 -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/ncu_$tag.log 2>&1; tail -2 gpurun_out/ncu_$tag.log
