import json, sys
for l in open(sys.argv[1]):
    l = l.strip()
    if l.startswith("=="):
        print(l)
        continue
    try:
        d = json.loads(l)
        print("  ", d["config"], {k: round(v, 2) for k, v in d["by_kind_ms"].items()})
    except Exception:
        print("  ", l[:300])
