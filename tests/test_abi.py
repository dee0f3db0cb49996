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
    assert ws(_problem(ks, 10, 6, 6, flags=64)) == 0     # unknown flag
    assert ws(_problem(ks, 10, 200, 6)) == 0             # n > KS_MAX_N
    sh = ks.ks_shard(); sh.rank, sh.nranks = 1, 4
    assert ws(_problem(ks, 1024, 6, 3, so=3), sh) > 0
    assert ws(_problem(ks, 1000, 6, 3, so=3), sh) == 0   # shard size must be a power of two
    sh.rank = 4
    assert ws(_problem(ks, 1024, 6, 3, so=3), sh) == 0   # bad rank


def test_strerror(ks):
    assert ks.strerror(ks.KS_ERR_RANK) == "least-squares matrix rank deficient"
    assert ks.strerror(99) == "unknown"
