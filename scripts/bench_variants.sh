#!/bin/bash
# Network-kernel time of library variants: bash scripts/bench_variants.sh KERNEL [lib.so ...]
cd "$(dirname "$0")/.."
k=$1; shift
for lib in paper_2308_04669_b200/libnedf_b200.so "$@"; do
  NEDF_LIB=$lib timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --tc-kernel $k 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$k', 'frame', round(d['value'],3), 'tc_ms', round(d['roofline']['kernel_ms_per_frame'],3), 'guard', round(d['roofline']['guard_ms_per_frame'],3), 'clk', d['clocks'])"
done
