"""Print the key numbers of bench.py JSON lines (files given on the command line)."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if d.get("impl") == "reference":
            print(f"{f}: reference {d['value'] / 1e6:.1f} M beads/s ({d['cpu_baseline']['cores']} cores)")
            continue
        r, e, z = d["roofline"], d.get("e2e") or {}, d.get("z_ops") or {}
        k = d["kernels_ms"]
        print(f"{f}: value {d['value'] / 1e9:.3f} G {d['unit']}  step {d['ms_per_step']:.4f} ms  frac {r['frac']:.3f} "
              f"(launch {r['launch_ms']:.4f} ms, share {r['share_of_step']:.2f})  clocks {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
        print("   kernels", {a: round(b, 4) for a, b in k.items()})
        if e:
            print(f"   e2e {e['value'] / 1e9:.3f} G ({e['ms_per_step']:.2f} ms)  numpy {e['numpy']['value'] / 1e9:.3f}  "
                  f"numpy_many {e['numpy_many']['value'] / 1e9:.3f}")
        if z:
            print(f"   zf {z['zf']['frac']:.3f} ztu {z['ztu']['frac']:.3f}  parity {(d.get('parity') or {}).get('max_rel')}  "
                  f"setup {d['setup']['seconds'] * 1e3:.1f} ms  batched {(d.get('batched_k100') or {}).get('value')}")
        if d.get("cpu_baseline"):
            print(f"   cpu_baseline {d['cpu_baseline']['value'] / 1e6:.1f} M")
