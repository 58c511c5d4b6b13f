"""Summarise bench JSON lines (tool): python tools/showb2.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e)
        continue
    r = d.get("roofline", {})
    st = r.get("step") or {}
    cls = r.get("classes") or {}
    print(f"{f.split('/')[-1]:48s} {d['value']:>12.1f} {d['ms_per_step']:8.4f}ms e2e={d['e2e']['value']} "
          f"dom={r.get('class')} frac={r.get('frac')} step={st.get('frac')} "
          + " ".join(f"{k}:{v.get('measured_us') or v.get('measured_ms_per_solve')}/{v.get('frac')}" for k, v in cls.items())
          + f" avg_us={r.get('avg_us')}")
