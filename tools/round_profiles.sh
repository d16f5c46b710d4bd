#!/bin/bash
# Round artefacts under gpurun: default bench line (C3, with e2e + cpu_baseline), the reference arm,
# per-config bench lines, launch lists, and one ncu --set full capture of the C3 tile kernels.
# usage: tools/round_profiles.sh <tag>
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; cat gpurun_out/bench_${tag}.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${tag}_ref.json 2> gpurun_out/bench_${tag}_ref.err; cat gpurun_out/bench_${tag}_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|cub|Radix" -c 60 --csv --log-file gpurun_out/launches_${tag}_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_${tag}_C3.csv 2>&1 | head -10
bash tools/all_configs.sh ${tag} C1 C2 C4 C5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_resolve|k_finalize" -s 5 -c 4 -o gpurun_out/prof_${tag}_C3 python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
ls -la gpurun_out/prof_${tag}_C3.ncu-rep
