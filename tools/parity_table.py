#!/usr/bin/env python
"""Measured parity errors of the GPU path against the CPU oracle on every
BASELINE.json config at full size (SURVEY §8(c.5) metric: per-step normwise
relative errors), plus the paper's n = 500 size at reduced k.  Prints a
markdown table (committed as profiles/r2_parity_errors.md)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2502_11686_b200 import generators as gen  # noqa: E402
from paper_2502_11686_b200 import ks  # noqa: E402
from tests.dense import rel_cov_err, rel_state_err  # noqa: E402


def glob_err(x, xo):
    return float(np.abs(x - xo).max() / np.abs(xo).max())


rows = []
cases = [("c1", gen.make("c1"), {}), ("c2", gen.make("c2"), {}), ("c3", gen.make("c3"), {}),
         ("c4", gen.make("c4"), {}), ("c5", gen.make("c5"), {}),
         ("c4 (large-n path forced)", gen.make("c4"), {"big": True}),
         ("paper n=m=500, k=6", gen.paper_problem(6, 500, seed=5), {})]
for name, p, kw in cases:
    s = ks.Smoother(p, **kw)
    s.run()
    s.check()
    x, S = s.states.cpu().numpy(), s.cov.cpu().numpy()
    t0 = time.perf_counter()
    xo, So = oracle.smooth(p)
    dt = time.perf_counter() - t0
    rows.append((name, p.N, p.n, p.m_max, rel_state_err(x, xo), rel_cov_err(S, So), glob_err(x, xo), dt))
    print(rows[-1], flush=True)
    del s
    torch.cuda.empty_cache()
print()
print(f"GPU: {torch.cuda.get_device_name(0)}; oracle: plain-C sequential Paige-Saunders + Alg. 1 (1 thread)")
print()
print("| case | N | n | m | e_state (per-step) | e_cov (per-step) | e_state (global) | oracle s |")
print("|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} | {r[4]:.2e} | {r[5]:.2e} | {r[6]:.2e} | {r[7]:.1f} |")
print()
print("Bars (BASELINE.json north_star): e_state <= 1e-9, e_cov <= 1e-8.")
