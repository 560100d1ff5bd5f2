"""Summarise tools/variant_eval.py JSON lines (one per library variant) as a
k_evaluate-ms table relative to the first line (dev helper)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
base = rows[0]
cases = [k for k in base if k != "lib"]
print("%-22s" % "variant" + "".join("%15s" % c for c in cases))
for r in rows:
    cells = []
    for c in cases:
        if c not in r:
            cells.append("%15s" % "-")
            continue
        d = r[c]["eval_ms"] / base[c]["eval_ms"] - 1
        same = "" if r[c]["est"] == base[c]["est"] else "!"
        cells.append("%9.2f %+4.0f%%%s" % (r[c]["eval_ms"], 100 * d, same))
    print("%-22s" % r["lib"][-22:] + "".join(cells))
