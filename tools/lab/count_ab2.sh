# TW = 16 count units: 1,024 threads (main) against 512 (lib_T512), on the mid-size probe and the DIC step
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -3
for v in main T512; do
  if [ $v = main ]; then unset DIC_LIB; else export DIC_LIB=$PWD/tools/lab/libs/lib_$v.so; fi
  echo "== $v"; python tools/lab/count_mid.py 2>&1 | grep "99999"
  for i in 1 2; do python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e --no-config-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), d['golden_check']['match'])"; done
done
