import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    r = d.get("roofline") or {}
    b1 = d.get("lb_batch1") or {}
    print(f"{f}: value={d['value']:.1f} q/s ms/step={d['ms_per_step']:.3f} e2e={d['e2e']['value']:.1f} "
          f"roof[{r.get('kernel')},{r.get('bound')}] frac={r.get('frac', 0):.3f} ach={r.get('achieved', 0):.1f} "
          f"lb_b1 frac={b1.get('frac', 0):.3f} ms={b1.get('launch_ms', 0):.3f} summ frac={d['summarize']['roofline']['frac']:.3f} clocks={d['clocks']}")
    print("   ", {k: (round(v['ms_per_step'], 3), round(v['share'], 3)) for k, v in d['kernels'].items()})
    print("   ", d['pruning'], "cpu", (d.get('cpu_baseline') or {}).get('value'))
