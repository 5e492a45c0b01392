"""Short view of bench JSON lines: tools/bench_brief.py FILE..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline") or {}
    print(f"{f}: value {d['value']/1e9:.3f} G, {d['ms_per_step']:.4f} ms/step, steps {d['steps']}")
    if r: print(f"   roofline frac {r['frac']:.3f} ach {r['achieved']:.0f} peak {r['peak']} launch_ms {r['launch_ms']:.4f} bytes {r['bytes_per_launch']/1e6:.1f} MB traffic {r.get('traffic')} share {r.get('share_of_step'):.3f}")
    if d.get("kernels_ms"): print("   kernels", {k: round(v, 4) for k, v in d["kernels_ms"].items()})
    e = d.get("e2e") or {}
    if e: print(f"   e2e {e['value']/1e9:.3f} G ({e.get('ms_per_step')}) numpy {((e.get('numpy') or {}).get('value') or 0)/1e9:.3f} many {((e.get('numpy_many') or {}).get('value') or 0)/1e9:.3f}")
    if d.get("z_ops"): print("   z", {k: (round(v['ms'], 4), round(v['frac'], 3)) for k, v in d["z_ops"].items()})
    if d.get("batched_k100"): print("   k100", d["batched_k100"]["ms_per_step"], d["batched_k100"]["value"]/1e9)
    if d.get("setup"): print("   setup", round(d["setup"]["seconds"], 4), "s", round(d["setup"]["beads_per_s"]/1e6, 1), "M beads/s")
    if d.get("parity"): print("   parity", d["parity"]["max_rel"])
    if d.get("cpu_baseline"): print("   cpu", round(d["cpu_baseline"]["value"]/1e6, 1), "M", d["cpu_baseline"]["cores"])
    if d.get("clocks"): print("   clocks", d["clocks"])
