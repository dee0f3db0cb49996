#!/usr/bin/env python
"""Write committed profile summaries from ncu reports (read here, no GPU).

    profile_report.py ROUND CONFIG LABEL@REP[:LAUNCH] ...

For each report: profiles/<ROUND>_<LABEL>.txt (key metrics, stall reasons,
hottest source lines) and the per-launch DRAM traffic
(dram__bytes_read.sum + dram__bytes_write.sum) into profiles/traffic.json
under [CONFIG][LABEL], which bench.py reports as roofline.traffic."""
import contextlib
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import ncu_hot  # noqa: E402
import ncu_summary  # noqa: E402


def dram_bytes(rep, launch):
    import csv
    out = subprocess.check_output(["ncu", "-i", rep, "-s", str(launch), "-c", "1", "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(out)))
    h, units, r = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = float(r[h.index(k)].replace(",", ""))
        u = units[h.index(k)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        tot += v * scale
    return int(tot), r[h.index("Kernel Name")]


def main():
    rnd, cfg = sys.argv[1], sys.argv[2]
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in sys.argv[3:]:
        label, rest = spec.split("@", 1)
        rep, launch = (rest.split(":") + ["0"])[:2]
        launch = int(launch)
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            print(f"# {rnd} {cfg} {label}: ncu --set full --clock-control none (launch {launch} of {os.path.basename(rep)})")
            ncu_summary.main(rep, launch)
            print("\nhottest source lines (warp-stall samples):")
            ncu_hot.main(rep, 20, launch)
        by, name = dram_bytes(rep, launch)
        print(f"\nDRAM traffic (read+write) of this launch: {by} bytes", file=buf)
        fn = f"{rnd}_{cfg}_{label}".replace(" ", "_").replace("=", "")
        with open(os.path.join(ROOT, "profiles", fn + ".txt"), "w") as f:
            f.write(buf.getvalue())
        traffic.setdefault(cfg, {})[label] = {"bytes": by, "kernel": name, "report": os.path.basename(rep),
                                              "round": rnd}
        print(label, by, name)
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
