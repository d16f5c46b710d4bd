#!/bin/bash
# Round artefacts without the large ncu reports (gpurun copies back <= 64 MiB):
# bench lines (default with e2e + cpu_baseline, reference arm, every config),
# launch lists, the C3 ncu --set full capture only, the f1 sweep and the f rows.
# usage: tools/round_light.sh <tag>
tag=${1:-v1}
o=gpurun_out/r02
mkdir -p $o
timeout 900 python bench.py > $o/bench_${tag}.json 2> $o/bench_${tag}.err; tail -1 $o/bench_${tag}.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $o/bench_${tag}_ref.json 2> $o/bench_${tag}_ref.err
for c in C1 C2 C4 C5 F1-1024; do
  timeout 900 python bench.py --config $c > $o/bench_${tag}_$c.json 2> $o/bench_${tag}_$c.err
done
for c in C3 C2 C4 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cub|Radix" -c 80 --csv --log-file $o/launches_${tag}_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_finalize" -s 6 -c 3 -o $o/prof_${tag}_C3 python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
timeout 900 python tools/sweep_f1.py > $o/sweep_f1_${tag}.json 2> $o/sweep_f1_${tag}.err
timeout 1200 python tools/bench_f.py $o/f_rows_${tag}.json > $o/f_rows_${tag}.log 2>&1
ls -la $o | tail -30
