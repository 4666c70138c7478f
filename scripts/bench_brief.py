#!/usr/bin/env python3
"""One-line digest of a bench.py JSON line: frame, e2e, network, guard, frac, clocks."""
import json
import sys

try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:  # noqa: BLE001
    print("no bench line:", e)
    sys.exit(0)
r = d.get("roofline", {})
e = d.get("e2e") or {}
print(f"frame_ms {d['value']:.3f} e2e {e.get('value', float('nan')):.3f} net_ms {r.get('kernel_ms_per_frame', 0):.3f} "
      f"guard_ms {r.get('guard_ms_per_frame', 0):.3f} frac {r.get('frac', 0):.4f} min {d.get('frame_ms_min', 0):.3f} "
      f"clk {d.get('clocks')}")
