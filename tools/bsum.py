"""One-line summary of bench.py JSON lines (per-launch ms and algorithmic fractions)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    steps = [(s["launch"][:24], round(s["ms"], 1), round(s.get("alg_frac") or 0, 2))
             for s in d.get("steps_per_colouring", []) if s["ms"] > 0.5]
    print(f, round(d.get("value", 0), 4), d.get("status"), steps)
