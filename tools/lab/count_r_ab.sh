# candidates per thread of the TW = 16 row-lane unit (sizes 3-4): probe + DIC step per variant
for v in main R20 R24 R32; do
  if [ $v = main ]; then unset DIC_LIB; else export DIC_LIB=$PWD/tools/lab/libs/lib_$v.so; fi
  echo "== $v"; python tools/lab/count_mid.py 2>&1 | grep "99999" | grep "sorted=True"
  python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e --no-config-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), d['golden_check']['match'])"
done
