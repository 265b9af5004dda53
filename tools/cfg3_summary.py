"""Summarise the config-3 sweep (tools/sweep_cfg3.sh) into one JSON document."""
import glob
import json
import os
import sys

d = sys.argv[1]
rows = {}
for f in sorted(glob.glob(os.path.join(d, "s*_cp*_*.json"))):
    name = os.path.basename(f)[:-5]
    s, cp, mode = name.split("_")
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    r = rows.setdefault((int(s[1:]), float(cp[2:])), {})
    r[mode] = {"samples_per_s": j["value"], "ms_per_step": j["ms_per_step"],
               "dedupe_factor": j.get("stats", {}).get("dedupe_factor")}
out = []
for (s, cp), r in sorted(rows.items()):
    e = {"samples_per_session": s, "change_prob": cp, **r}
    if "dedup" in r and "kjt" in r:
        e["dedup_speedup"] = r["dedup"]["samples_per_s"] / r["kjt"]["samples_per_s"]
    out.append(e)
print(json.dumps({"workload": "cfg3: B=65536, 26 keys (cfg2 lengths), 26 x 10M x 128 fp32 tables, "
                  "fixed session length S, dedup vs KJT path (dedup + pooled fwd + expand + bwd + SGD)",
                  "rows": out}, indent=1))
