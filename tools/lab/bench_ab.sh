# alternate bench.py (DIC leg only) between the main library and lib_$v for v in $VARIANTS (DIC_LIB)
for i in ${ROUNDS:-1 2 3}; do
  python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e --no-config-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('main', round(d['ms_per_step'],3), d['step_ms'])"
  for v in ${VARIANTS:-$VARIANT}; do
    DIC_LIB=$PWD/tools/lab/libs/lib_$v.so python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e --no-config-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), d['step_ms'])"
  done
done
