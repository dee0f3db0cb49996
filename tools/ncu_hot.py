#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples from an ncu report (needs
-lineinfo).  Usage: ncu_hot.py REP [N] [launch index]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, top=25, skip=0):
    out = subprocess.check_output(["ncu", "-i", rep, "-s", str(skip), "-c", "1", "--page", "source", "--csv",
                                   "--print-source", "cuda,sass"]).decode(errors="replace")
    rows = list(csv.reader(io.StringIO(out)))
    agg = defaultdict(float)
    text = {}
    fname = ""
    h = None
    cur_line = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if h is None or len(r) < 5:
            continue
        if r[0].strip():
            cur_line = (fname, r[0])
            text[cur_line] = r[1].strip()[:100]
        try:
            w = float(r[h.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        if cur_line:
            agg[cur_line] += w
    tot = sum(agg.values()) or 1
    for k, w in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * w / tot:5.1f}%  {k[0]}:{k[1]:>5}  {text.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
