#!/bin/bash
# Round-2 artefacts under gpurun -> gpurun_out/r02/: default bench line (C3 with e2e +
# cpu_baseline), the reference arm, per-config bench lines, ncu launch lists, and
# ncu --set full captures of the main kernels of C3 / C5 / C4 / C2.
# usage: tools/round_r02.sh [tag]
tag=${1:-v1}
o=gpurun_out/r02
mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -x -q > $o/pytest_gpu_${tag}.log 2>&1; tail -2 $o/pytest_gpu_${tag}.log
timeout 900 python bench.py > $o/bench_${tag}.json 2> $o/bench_${tag}.err; tail -1 $o/bench_${tag}.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $o/bench_${tag}_ref.json 2> $o/bench_${tag}_ref.err
for c in C1 C2 C4 C5 F1-1024; do
  timeout 900 python bench.py --config $c > $o/bench_${tag}_$c.json 2> $o/bench_${tag}_$c.err
  python -c "import json; d=json.load(open('$o/bench_${tag}_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e'] and d['e2e']['value'], d['phases_us'])" || tail -3 $o/bench_${tag}_$c.err
done
for c in C3 C2 C4 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cub|Radix" -c 80 --csv --log-file $o/launches_${tag}_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
  echo "== $c"; python tools/launch_summary.py $o/launches_${tag}_$c.csv 2>&1 | head -8
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_finalize" -s 6 -c 3 -o $o/prof_${tag}_C3 python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_csr" -s 6 -c 2 -o $o/prof_${tag}_C5 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_classify_grid" -s 3 -c 1 -o $o/prof_${tag}_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_arcs_grid|k_tile" -s 6 -c 2 -o $o/prof_${tag}_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
timeout 900 python tools/sweep_f1.py > $o/sweep_f1_${tag}.json 2> $o/sweep_f1_${tag}.err
timeout 1200 python tools/bench_f.py $o/f_rows_${tag}.json > $o/f_rows_${tag}.log 2>&1
ls -la $o
