"""One line per bench JSON: value, e2e, ms/step, per-kernel ms per step, rooflines."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    if "value" not in d:
        print(f, d)
        continue
    ks = d.get("kernels", {})
    kern = " ".join(f"{k}={v['ms_per_step']:.3f}" for k, v in ks.items() if v.get("ms_per_step", 0) > 0.02)
    rf = d.get("roofline") or {}
    b1 = d.get("lb_batch1") or {}
    print(f"{f.split('/')[-1]}: {d['value']:.1f} {d['unit']} e2e {(d.get('e2e') or {}).get('value', 0):.1f} "
          f"ms/step {d.get('ms_per_step', 0):.3f} | {kern} | roof {rf.get('kernel')} {rf.get('frac', 0):.3f} "
          f"hbm {rf.get('hbm_achieved_gbs', 0):.0f} | b1 {b1.get('launch_ms', 0):.4f} ms frac {b1.get('frac', 0):.3f} "
          f"| clocks {d.get('clocks')}")
