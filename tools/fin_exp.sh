# timing variants built into build/ (EG_LIB_PATH override): bench lines for the configs in $CFGS
for v in "$@"; do for c in ${CFGS:-C3}; do
  EG_LIB_PATH=$PWD/build/lib_$v.so timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['ms_per_step'], d['phases_us']['boundary'], d['parity_sample'])"
done; done
