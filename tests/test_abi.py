"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/ks.h declares, and its host-side sizing logic behaves (no kernels)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def ks():
    from paper_2502_11686_b200 import build, ks as _ks
    build.build()
    _ks.lib()
    return _ks


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("ks_create", "ks_whiten", "ks_factor", "ks_solve", "ks_selinv", "ks_get"):
        assert f in fns


def test_library_exports_every_header_symbol(ks):
    out = subprocess.check_output(["nm", "-D", "--defined-only", ks.LIB_PATH]).decode()
    exported = set(re.findall(r" T (ks_\w+)", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    for f in header_functions():
        getattr(ks.lib(), f)
    assert set(ks.EXPORTS) == set(header_functions())


def test_library_is_sm100a(ks):
    out = subprocess.check_output(["cuobjdump", "--list-elf", ks.LIB_PATH]).decode()
    assert "sm_100a" in out


def _problem(ks, N, n, m, **kw):
    pr = ks.ks_problem()
    pr.nsteps, pr.n, pr.m_max = N, n, m
    pr.F = pr.K = 0x1000
    pr.H = pr.L = pr.o = 0x1000 if m else None
    for k, v in kw.items():
        setattr(pr, k, v)
    return pr


def test_workspace_sizing_host_logic(ks):
    L = ks.lib()
    ws = lambda pr, sh=None: L.ks_workspace_bytes(C.byref(pr), None if sh is None else C.byref(sh))
    a = ws(_problem(ks, 1000, 6, 6, sF=36, sK=36, sH=36, sL=36, so=6))
    b = ws(_problem(ks, 1000, 6, 6, so=6))               # constant model: smaller
    assert a > b > 0
    big = ws(_problem(ks, 1 << 22, 6, 3, so=3, flags=ks.KS_OUTPUTS_BOUND))
    assert 4e9 < big < 2e10                              # ~ (E + R record + X) per step
    assert ws(_problem(ks, 0, 6, 6)) == 0                # bad sizes
    assert ws(_problem(ks, 10, 0, 6)) == 0
    assert ws(_problem(ks, 10, 6, 6, sF=5)) == 0         # stride smaller than a block
    assert ws(_problem(ks, 10, 6, 6, flags=1 << 12)) == 0  # unknown flag
    assert ws(_problem(ks, 10, 6, 6, flags=ks.KS_COV_IS_CHOL)) > 0
    assert ws(_problem(ks, 10, 600, 6)) == 0             # n > KS_MAX_N
    big = ws(_problem(ks, 500, 500, 500, so=500))        # the paper's n = m = 500 size: the large-n path
    assert 1e10 < big < 3e10
    assert ws(_problem(ks, 500, 500, 600, so=600)) == 0  # stage stacks beyond the panel's shared memory
    assert ws(_problem(ks, 100, 6, 6, so=6, flags=ks.KS_BIG_PATH)) > 0
    # multi-GPU: a ks_dist without a communicator (caller-driven exchange)
    def dist(rank, nranks, first, total):
        d = C.c_void_p()
        rc = L.ks_dist_create(C.byref(d), rank, nranks, None, first, total)
        return rc, d
    rc, d = dist(1, 4, 1024, 4096)
    assert rc == ks.KS_OK
    wsd = lambda pr: L.ks_workspace_bytes(C.byref(pr), d)
    assert wsd(_problem(ks, 1024, 6, 3, so=3)) > 0
    assert wsd(_problem(ks, 1000, 6, 3, so=3)) == 0     # shard size must match (power of two, rank order)
    r, n, nc = C.c_int(), C.c_int(), C.c_int()
    assert L.ks_dist_info(d, C.byref(r), C.byref(n), C.byref(nc)) == ks.KS_OK
    assert (r.value, n.value, nc.value) == (1, 4, 0)
    L.ks_dist_destroy(d)
    rc, d2 = dist(1, 4, 1000, 4000)                      # a 1000-step shard: accepted by ks_dist_create ...
    assert rc == ks.KS_OK
    assert L.ks_workspace_bytes(C.byref(_problem(ks, 1000, 6, 3, so=3)), d2) == 0   # ... not by the context
    L.ks_dist_destroy(d2)
    assert dist(4, 4, 0, 4096)[0] == ks.KS_ERR_ARG        # bad rank
    assert dist(0, 4, 4096, 4096)[0] == ks.KS_ERR_ARG     # first step outside the problem


def test_strerror(ks):
    assert ks.strerror(ks.KS_ERR_RANK) == "least-squares matrix rank deficient"
    assert ks.strerror(99) == "unknown"


def test_level_plan_matches_golden(ks):
    """The library's host level plan (the permutation P of SURVEY §8(a) a2)
    against the worked examples of S:195-197 (tests/golden/oddeven_order.json):
    which step is eliminated at which level, and the elimination order
    (by level, ascending steps within a level)."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "oddeven_order.json")))
    for case in g["cases"]:
        N = case["N"]
        nl, lv = ks.level_of_steps(N)
        assert nl == int(np.floor(np.log2(N))) + 1
        order = sorted(range(N), key=lambda j: (lv[j], j))
        assert order == case["order"], (N, order)
        assert [int(lv[j]) for j in order] == case["levels"], N
    # the trailing-ones rule at larger N (odd levels included)
    for N in (5, 6, 7, 100, 1000, 1023, 4097):
        nl, lv = ks.level_of_steps(N)
        for j in range(N):
            t = (j + 1) >> int(lv[j])
            assert ((j + 1) & ((1 << int(lv[j])) - 1)) == 0
            K = N >> int(lv[j])
            assert (t - 1) % 2 == 0 or (t - 1 == K - 1), (N, j)
