#!/bin/bash
for c in "$@"; do
  out=$(RQ_CTAS_PER_SM=$c timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
  python - "$c" "$out" <<'PY'
import json, sys
d = json.loads(sys.argv[2]); k = d["kernels_ms"]
print(f"ctas/SM {sys.argv[1]}: chunk up {k['qtilde_v:chunks']:.3f} down {k['qtilde_tv:chunks']:.3f} ms  ({100*d['roofline']['frac']:.1f}%)")
PY
done
