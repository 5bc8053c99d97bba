import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    r = d.get("roofline") or {}
    print(f, "value %.4g" % d["value"], "ms/step %.4f" % d["ms_per_step"], "roof", r.get("kernel"), r.get("achieved"), r.get("frac"))
    for k, v in (d.get("kernels") or {}).items():
        print("   ", k, {a: round(b, 4) if isinstance(b, float) else b for a, b in v.items()})
