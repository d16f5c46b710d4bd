#!/bin/bash
# C3 bench under several env settings (timing experiments; no tests). usage: tools/c3_env.sh "ENV=.." ...
for envs in "" "$@"; do
  env $envs timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', d['ms_per_step'], 'main', d['phases_us']['main'])"
done
