#!/bin/bash
# A/B: the bench's timed DIC step with nvidia-smi sampling at 100 ms vs 500 ms vs 2000 ms
for ms in 100 500 2000; do
  python bench.py --no-cpu-baseline --no-e2e --no-kernel-bench --steps 5 --clock-ms $ms 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clock-ms', $ms, 'ms_per_step', round(d['ms_per_step'],2), 'samples', d['clocks'].get('samples'))"
done
