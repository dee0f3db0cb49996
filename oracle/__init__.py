"""ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/libks_oracle.so`` (plain C, ks_oracle.c): a
sequential Paige-Saunders QR smoother with the paper's Algorithm 1 SelInv,
written from PAPER.md.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2502_11686_b200``) and never imports it.

Every function here is pinned in tests/test_oracle.py against something other
than itself (dense lstsq / dense Gram inverse, noise-free recovery, closed
forms, the paper's / SPEC's worked values, scipy's DARE).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ks_oracle.c")
_LIB = os.path.join(_HERE, "libks_oracle.so")

ORA_OK, ORA_ERR_ARG, ORA_ERR_NOT_SPD, ORA_ERR_RANK = 0, 1, 5, 6


class OracleError(RuntimeError):
    def __init__(self, code, step=-1, kind=0):
        super().__init__(f"oracle error {code} at step {step} (kind {kind})")
        self.code, self.step, self.kind = code, step, kind


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32 = C.POINTER(C.c_double), C.c_int64, C.c_int
        pi32, pi64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
        _lib.oracle_whiten.argtypes = [i64, i32, i32, pi32, d, i64, d, i64, d, i64, d, i64, d, i64,
                                       d, i64, d, d, d, d, d, pi64, C.POINTER(C.c_int)]
        _lib.oracle_factor.argtypes = [i64, i32, i32, pi32, d, d, d, d, d, d, d, d, pi64]
        _lib.oracle_solve.argtypes = [i64, i32, d, d, d, d]
        _lib.oracle_selinv.argtypes = [i64, i32, d, d, d, d]
        _lib.oracle_smooth.argtypes = [i64, i32, i32, pi32, d, i64, d, i64, d, i64, d, i64, d, i64,
                                       d, i64, d, d, pi64, C.POINTER(C.c_int)]
        for f in (_lib.oracle_whiten, _lib.oracle_factor, _lib.oracle_solve, _lib.oracle_selinv,
                  _lib.oracle_smooth):
            f.restype = C.c_int
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _inputs(p):
    """Pointer/stride tuple of a generators.Problem-like object."""
    m = np.ascontiguousarray(p.m, np.int32)
    arrs = {}
    for k in ("F", "H", "c", "o", "K", "L"):
        a = getattr(p, k)
        arrs[k] = None if a is None else np.ascontiguousarray(a, np.float64)
    def st(k):
        a = arrs[k]
        return 0 if a is None or a.shape[0] == 1 else int(np.prod(a.shape[1:]))
    args = (p.N, p.n, p.m_max, m.ctypes.data_as(C.POINTER(C.c_int32)),
            _p(arrs["F"]), st("F"), _p(arrs["H"]), st("H"), _p(arrs["c"]), st("c"),
            _p(arrs["o"]), st("o"), _p(arrs["K"]), st("K"), _p(arrs["L"]), st("L"))
    return args, (m, arrs)


def smooth(p, cov: bool = True):
    """Smoothed states [N, n] and (if cov) covariance blocks [N, n, n]."""
    args, keep = _inputs(p)
    x = np.empty((p.N, p.n))
    S = np.empty((p.N, p.n, p.n)) if cov else None
    bs, bk = C.c_int64(-1), C.c_int(0)
    rc = lib().oracle_smooth(*args, _p(x), _p(S), C.byref(bs), C.byref(bk))
    if rc:
        raise OracleError(rc, bs.value, bk.value)
    return (x, S) if cov else x


def whiten(p):
    """Whitened blocks C [N,m_max,n], y [N,m_max], B [N,n,n], D [N,n,n], e [N,n]."""
    args, keep = _inputs(p)
    N, n, mx = p.N, p.n, p.m_max
    C_ = np.zeros((N, max(mx, 0), n)); y = np.zeros((N, max(mx, 0)))
    B = np.zeros((N, n, n)); D = np.zeros((N, n, n)); e = np.zeros((N, n))
    bs, bk = C.c_int64(-1), C.c_int(0)
    rc = lib().oracle_whiten(*args, _p(C_), _p(y), _p(B), _p(D), _p(e), C.byref(bs), C.byref(bk))
    if rc:
        raise OracleError(rc, bs.value, bk.value)
    return dict(C=C_, y=y, B=B, D=D, e=e)


def factor(p, w=None):
    """Block-bidiagonal R (Rd [N,n,n], Ro [N,n,n] = R_{i,i+1}) and z [N,n]."""
    w = whiten(p) if w is None else w
    N, n = p.N, p.n
    m = np.ascontiguousarray(p.m, np.int32)
    Rd = np.zeros((N, n, n)); Ro = np.zeros((N, n, n)); z = np.zeros((N, n))
    bs = C.c_int64(-1)
    rc = lib().oracle_factor(N, n, p.m_max, m.ctypes.data_as(C.POINTER(C.c_int32)),
                             _p(w["C"]), _p(w["y"]), _p(w["B"]), _p(w["D"]), _p(w["e"]),
                             _p(Rd), _p(Ro), _p(z), C.byref(bs))
    if rc:
        raise OracleError(rc, bs.value)
    return Rd, Ro, z


def solve(Rd, Ro, z):
    N, n = z.shape
    x = np.empty((N, n))
    lib().oracle_solve(N, n, _p(np.ascontiguousarray(Rd)), _p(np.ascontiguousarray(Ro)),
                       _p(np.ascontiguousarray(z)), _p(x))
    return x


def selinv(Rd, Ro):
    """Alg. 1: diagonal blocks S_jj [N,n,n] and S_{j,j+1} [N,n,n] (last = 0)."""
    N, n = Rd.shape[0], Rd.shape[1]
    S = np.empty((N, n, n)); X = np.zeros((N, n, n))
    lib().oracle_selinv(N, n, _p(np.ascontiguousarray(Rd)), _p(np.ascontiguousarray(Ro)), _p(S), _p(X))
    return S, X
