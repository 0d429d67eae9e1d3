"""One-line summary of bench JSON lines: value, step time, roofline fractions per sweep, clocks."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e)
        continue
    r = d.get("roofline", {})
    sw = r.get("sweeps", {})
    fr = " ".join(f"{k}={v.get('frac')}({v.get('avg_launch_us')}us)" for k, v in sw.items())
    c = d.get("clocks", {})
    e2e = (d.get("e2e") or {}).get("value")
    print(f"{p}: {d.get('value')} {d.get('unit')} ms={d.get('ms_per_step')} frac={r.get('frac')} {fr} "
          f"e2e={e2e} sm={c.get('sm_mhz')} {c.get('reasons')}")
