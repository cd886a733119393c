python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -3
for r in 1 2; do
for v in main HEAD; do
  if [ $v = main ]; then unset DIC_LIB; else export DIC_LIB=$PWD/tools/lab/libs/lib_$v.so; fi
  python bench.py --no-cpu-baseline --no-e2e --no-config-sweep --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_microbench']; r=d['roofline']
print('$v', 'dic', round(d['ms_per_step'],2), 'cfg5 ms', round(k['ms'],2), 'frac', round(k['frac'],3), 'hbm ms', round(k['hbm_streaming']['ms'],3), round(k['hbm_streaming']['frac'],3), 'pair us', round(r['avg_launch_ms']*1e3,1), k['golden_check']['match'], d['host_phases_ms'])"
done
done
