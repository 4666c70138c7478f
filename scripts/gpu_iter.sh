#!/bin/bash
# One build -> measure iteration on the GPU box: parity tests, the network-kernel tile timeline,
# the guard timeline and a short headline bench (no CPU baseline).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 200 python scripts/tc_trace.py 3 2>&1 | grep -E "^L 0|^L33|MMA|encoder" | tail -6
timeout 200 python scripts/cl_trace.py 2>&1 | head -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/iter_bench.json 2> gpurun_out/iter_bench.err
python3 -c "import json; d=json.loads(open('gpurun_out/iter_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; print('frame_ms', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), 'tc_ms', round(r['kernel_ms_per_frame'],3), 'guard_ms', round(r['guard_ms_per_frame'],3), 'frac', round(r['frac'],4), 'clk', d['clocks'])" || tail -5 gpurun_out/iter_bench.err
