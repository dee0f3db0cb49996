#!/usr/bin/env python
"""profiles/traffic.json from ncu raw CSV exports (--print-units base):
DRAM bytes (read + write) per profiled launch, keyed by config and
"family L=level".  Usage: traffic_json.py ROUND CFG CSV FAMILY:LEVEL [FAMILY:LEVEL ...]
(one FAMILY:LEVEL per profiled launch, in order)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rnd, cfg, path, keys):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    out_path = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for r, key in zip(rows[2:], keys):
        fam, lev = key.split(":")
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
        tj.setdefault(cfg, {})[f"{fam} L={lev}"] = {
            "bytes": int(rd + wr), "kernel": r[h.index("Kernel Name")], "report": os.path.basename(path),
            "round": rnd}
    json.dump(tj, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:])
