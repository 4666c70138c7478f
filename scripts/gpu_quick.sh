#!/bin/bash
# Standard quick GPU check: parity tests, one-tile timeline, short bench.
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/tc_trace.py 2>&1 | grep -E "encoder|L 0|L 1 |L 2 |L 3 |L16|L32|L33"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick_bench.json 2>gpurun_out/quick_bench.err
python3 -c "import json; d=json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1]); print('frame_ms', d['value'], 'tc_ms', d['roofline']['kernel_ms_per_frame'], 'guard_ms', d['roofline']['guard_ms_per_frame'], 'frac', d['roofline']['frac'])" || tail -5 gpurun_out/quick_bench.err
