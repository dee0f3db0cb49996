#!/usr/bin/env python
"""Profiling driver: `warm` warm-up runs of one config, then ONE more run
(the one an ncu --launch-skip selects).  Usage: prof_run.py [config] [N] [warm]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11686_b200 import generators as gen  # noqa: E402
from paper_2502_11686_b200 import ks  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
generic = os.environ.get("KS_GENERIC") == "1"
p = gen.make(cfg, N=N)
s = ks.Smoother(p, generic=generic)
for _ in range(warm + 1):
    s.run()
s.check()
torch.cuda.synchronize()
print("ok", cfg, p.N)
