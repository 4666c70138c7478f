#!/bin/bash
# A/B timing on one box: alternate library builds (NEDF_LIB=_var/<name>.so, "main" = the in-tree
# library) through the headline bench, R rounds; prints frame / network / guard ms per run.
# usage: scripts/ab.sh R name1 name2 ...
cd "$(dirname "$0")/.."
R=$1; shift
for r in $(seq 1 $R); do
  for v in "$@"; do
    if [ "$v" = main ]; then unset NEDF_LIB; else export NEDF_LIB="_var/$v.so"; fi
    timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value'],3), round(r['kernel_ms_per_frame'],3), round(r['guard_ms_per_frame'],3), d['clocks']['reasons'])" || echo "$v failed"
  done
done
