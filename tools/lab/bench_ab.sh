# alternate bench.py (DIC leg only) between the main library and lib_$VARIANT (DIC_LIB)
for i in 1 2 3; do
  python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('main', round(d['ms_per_step'],3))"
  DIC_LIB=$PWD/tools/lab/libs/lib_$VARIANT.so python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VARIANT', round(d['ms_per_step'],3))"
done
