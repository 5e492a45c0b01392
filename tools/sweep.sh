#!/bin/bash
# quick parameter sweep of the chunk layout / kernel shape (device-only timing)
for cfg in "$@"; do
  IFS=: read -r S B T <<< "$cfg"
  out=$(RQ_TILE_LEAVES=$S RQ_CHUNK_BYTES=$B RQ_CHUNK_THREADS=$T timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
  python - "$cfg" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2])
    k = d["kernels_ms"]
    print(f"{sys.argv[1]:>16}  {d['value']/1e9:6.2f} Gbeads/s  ms/step {d['ms_per_step']:.3f}  chunk {d['roofline']['achieved']:7.1f} GB/s ({100*d['roofline']['frac']:4.1f}%)  "
          f"up {k['qtilde_v:chunks']:.3f}/{k['qtilde_v:top']:.3f}  down {k['qtilde_tv:chunks']:.3f}/{k['qtilde_tv:top']:.3f}  B/bead {d['bytes_per_bead_per_op']:.1f} chunks {d['plan']['n_chunks']} cta/sm {d['plan'].get('chunk_ctas_per_sm')} smem {d['plan'].get('chunk_smem_bytes')}")
except Exception as e:
    print(sys.argv[1], "FAILED", sys.argv[2][:300])
PY
done
