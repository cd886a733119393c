python -m pytest tests/test_gpu_engine.py tests/test_gpu_replicated.py -x -q 2>&1 | tail -3
B="python bench.py --no-cpu-baseline --no-kernel-bench --no-e2e --no-config-sweep"
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["ms_per_step"],3), d["golden_check"]["match"], d["host_phases_ms"])'
for i in 1 2; do
  $B 2>/dev/null | python -c "$P" coop
  DIC_CKPT_COOP=0 $B 2>/dev/null | python -c "$P" plain
done
DIC_LIB=$PWD/tools/lab/libs/lib_TIMING.so python tools/lab/commit_phases.py 2>&1 | tail -45
