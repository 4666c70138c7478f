#!/bin/bash
# Standard quick GPU check: parity tests, one-tile timeline, short bench of both tensor-core kernels.
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/tc2_trace.py 2>&1 | tail -4
for k in single pair mcast2 mcast4; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --tc-kernel $k > gpurun_out/quick_bench_$k.json 2>gpurun_out/quick_bench_$k.err
  python3 -c "import json; d=json.loads(open('gpurun_out/quick_bench_$k.json').read().strip().splitlines()[-1]); print('$k frame_ms', d['value'], 'tc_ms', d['roofline']['kernel_ms_per_frame'], 'guard_ms', d['roofline']['guard_ms_per_frame'], 'frac', d['roofline']['frac'])" || tail -5 gpurun_out/quick_bench_$k.err
done
