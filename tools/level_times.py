#!/usr/bin/env python
"""Per-(phase, level) device times of one config (CUDA events around every
launch, library timing).  Usage: level_times.py [config] [N] [steps]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11686_b200 import generators as gen  # noqa: E402
from paper_2502_11686_b200 import ks  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
generic = os.environ.get("KS_GENERIC") == "1"
p = gen.make(cfg, N=N)
s = ks.Smoother(p, generic=generic)
for _ in range(2):
    s.run()
s.check()
s.set_timing(True)
for _ in range(steps):
    s.run()
lt = s.launch_times()
agg = defaultdict(float)
for fam, lev, ms in lt:
    agg[(fam, lev)] += ms / steps
tot = sum(agg.values())
print(f"{cfg} N={p.N}: {tot:.3f} ms/step (sum of launches)")
for (fam, lev), ms in sorted(agg.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if ms > 0.01 * tot / 10:
        print(f"  {fam:8s} L={lev:2d} {ms:8.3f} ms")
