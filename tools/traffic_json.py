"""ncu launch list (gpu__time_duration, dram bytes) of one colouring -> profiles/ncu_traffic.json.

    python tools/traffic_json.py <ncu csv> <template> <precision> <layout> <scale> [--out FILE]

The record is stamped with paper_2009_11665_b200.build.source_hash() of the tree the
capture ran on; bench.py quotes `traffic` only when the stamp equals its own sources.
Per class (as bench.py's roofline classes): DRAM bytes (read + write) of the class over the
colouring divided by the class's profiler records (one per DP step, as bench.py counts
launches: a step may run several kernels — heavy rows, bucket hubs), and per kernel
launch: kernel, ms, DRAM GB, L2 hit rate.  [--steps LOG]: the prof_one.py log, whose first
line lists the plan's steps (the last is the top).
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_11665_b200.build import source_hash  # noqa: E402


def classify(name):
    if "colorize" in name:
        return "color"
    if "bucket" in name or "hist" in name:
        return "hist"
    if "atop_leaf" in name or "top_leaf" in name:
        return "top"
    if "reduce" in name:
        return "reduce"
    return "step"


def main():
    path, tmpl, prec, layout, scale = sys.argv[1:6]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "profiles", "ncu_traffic.json")
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    launches = {}
    for r in csv.DictReader(io.StringIO(txt)):
        d = launches.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"]})
        v = r["Metric Value"].replace(",", "")
        d[r["Metric Name"]] = float(v) if v not in ("", "n/a") else None
    recs = []
    for i in sorted(launches):
        d = launches[i]
        recs.append({"kernel": d["kernel"].split("(")[0], "ms": d.get("gpu__time_duration.sum", 0) / 1e6,
                     "dram_bytes": (d.get("dram__bytes_read.sum") or 0) + (d.get("dram__bytes_write.sum") or 0),
                     "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct")})
    # the last launch of each fused step class with a GENERAL top is the top step (cls 3)
    key = f"{tmpl}/{prec}/{layout}/scale{scale}"
    per = {}
    astep = [r for r in recs if "astep" in r["kernel"] or "step_kernel" in r["kernel"]]
    for r in recs:
        c = classify(r["kernel"])
        if r is (astep[-1] if astep else None) and not any("top_leaf" in x["kernel"] for x in recs):
            c = "top"
        r["cls"] = c
        per.setdefault(c, []).append(r["dram_bytes"])
    # profiler records per class (bench.py's launch count): one per step
    nrec = {c: len(v) for c, v in per.items()}
    if "--steps" in sys.argv:
        import ast
        first = open(sys.argv[sys.argv.index("--steps") + 1]).read().splitlines()[0]
        steps = ast.literal_eval(first)
        nrec["step"] = len(steps) - 1
        nrec["top"] = 1
        nrec["hist"] = 1
    res = json.load(open(out)) if os.path.exists(out) else {}
    res[key] = {"src_hash": source_hash(), "source": os.path.relpath(path, ROOT),
                "per_class_dram_bytes_per_launch": {c: sum(v) / max(nrec.get(c, len(v)), 1) for c, v in per.items()},
                "launches": recs,
                "how": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                       "lts__t_sector_hit_rate.pct --replay-mode application --clock-control none "
                       "(tools/traffic.sh): one colouring of the bench configuration"}
    res.pop("_note", None)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res[key]["per_class_dram_bytes_per_launch"]))


if __name__ == "__main__":
    main()
