# timing variants built into build/ (EG_LIB_PATH override), C3 bench lines
for v in "$@"; do
  EG_LIB_PATH=$PWD/build/lib_$v.so timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_us'], d['parity_sample'])"
done
