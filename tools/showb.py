"""Print the key numbers of bench JSON lines (tool)."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    r = d.get("roofline") or {}
    print(f.split("/")[-1], d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), "frac", r.get("frac"),
          "ach", r.get("achieved"), "avg_us", r.get("avg_us"), "step_frac", r.get("step_fp64_frac"))
