"""Thin ctypes binding of libks.so (include/ks.h) -- argument marshalling only.

Every step of the smoother runs in the sm_100a kernels of ``csrc/``; this
module only turns torch tensors into pointers, strides and a CUDA stream.
There is no CPU fallback: if the extension is missing, importing
``lib()`` raises.

Names follow the ABI: ``ks_create``, ``ks_whiten``, ``ks_factor``,
``ks_solve``, ``ks_selinv``, ``ks_get``.  ``Smoother`` bundles one context.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KS_LIB") or os.path.join(_HERE, "libks.so")   # KS_LIB: A/B variants

KS_OK, KS_ERR_ARG, KS_ERR_ORDER, KS_ERR_CUDA, KS_ERR_NCCL, KS_ERR_NOT_SPD, KS_ERR_RANK, \
    KS_ERR_WORKSPACE = range(8)
KS_HOST_INPUTS, KS_OUTPUTS_BOUND, KS_GENERIC_PATH, KS_NO_FUSED_TAIL, KS_COV_IS_CHOL, KS_KEEP_WHITENING, \
    KS_BIG_PATH = 1, 2, 4, 8, 16, 32, 64
FAMILIES = ("whiten", "factor", "solve", "selinv", "boundary", "backward")

EXPORTS = ("ks_workspace_bytes", "ks_create", "ks_whiten", "ks_factor", "ks_solve", "ks_selinv",
           "ks_solve_selinv", "ks_get", "ks_sync_status", "ks_boundary_buffers", "ks_factor_boundary",
           "ks_set_timing", "ks_get_timing", "ks_get_launch_times", "ks_info",
           "ks_peak_fp64_tflops", "ks_strerror", "ks_destroy",
           "ks_dist_unique_id", "ks_dist_create", "ks_dist_info", "ks_dist_destroy",
           "ks_level_of_steps", "ks_update_obs", "ks_get_async", "ks_get_packed")


class KsError(RuntimeError):
    def __init__(self, code: int, what: str = "", step: int = -1, kind: int = 0):
        msg = f"{what}: {strerror(code)} (code {code})"
        if step >= 0:
            msg += f" at step {step}" + (f" (kind {kind})" if kind else "")
        super().__init__(msg)
        self.code, self.step, self.kind = code, step, kind


class ks_problem(C.Structure):
    _fields_ = [("nsteps", C.c_int64), ("n", C.c_int32), ("m_max", C.c_int32),
                ("m", C.c_void_p), ("F", C.c_void_p), ("H", C.c_void_p), ("c", C.c_void_p),
                ("o", C.c_void_p), ("K", C.c_void_p), ("L", C.c_void_p),
                ("sF", C.c_int64), ("sH", C.c_int64), ("sc", C.c_int64), ("so", C.c_int64),
                ("sK", C.c_int64), ("sL", C.c_int64), ("flags", C.c_uint32),
                ("batch", C.c_int64), ("Hev", C.c_void_p), ("sHev", C.c_int64), ("l", C.c_void_p),
                ("nstate", C.c_void_p), ("nstate_min", C.c_int32)]


_lib = None


def lib():
    """Load the in-tree libks.so; fail loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t
        L.ks_workspace_bytes.argtypes = [C.POINTER(ks_problem), vp]
        L.ks_workspace_bytes.restype = sz
        L.ks_create.argtypes = [C.POINTER(vp), C.POINTER(ks_problem), vp, sz, vp, vp, vp, vp]
        L.ks_dist_unique_id.argtypes = [C.c_char_p]
        L.ks_dist_create.argtypes = [C.POINTER(vp), i32, i32, C.c_char_p, i64, i64]
        L.ks_dist_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        L.ks_dist_destroy.argtypes = [vp]
        L.ks_dist_destroy.restype = None
        L.ks_level_of_steps.argtypes = [i64, vp]
        for f in ("ks_whiten", "ks_factor", "ks_solve", "ks_selinv", "ks_solve_selinv",
                  "ks_factor_boundary"):
            getattr(L, f).argtypes = [vp]
        L.ks_get.argtypes = [vp, vp, vp]
        L.ks_get_async.argtypes = [vp, vp, vp]
        L.ks_get_packed.argtypes = [vp, vp, vp, i32]
        L.ks_update_obs.argtypes = [vp, vp]
        L.ks_sync_status.argtypes = [vp, C.POINTER(i64), C.POINTER(i32)]
        L.ks_boundary_buffers.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(sz)]
        L.ks_set_timing.argtypes = [vp, i32]
        L.ks_get_timing.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(i64)]
        L.ks_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.ks_get_launch_times.argtypes = [vp, i64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                          C.POINTER(C.c_float)]
        L.ks_get_launch_times.restype = i64
        L.ks_peak_fp64_tflops.argtypes = [vp]
        L.ks_peak_fp64_tflops.restype = C.c_double
        L.ks_strerror.argtypes = [i32]
        L.ks_strerror.restype = C.c_char_p
        L.ks_destroy.argtypes = [vp]
        L.ks_destroy.restype = None
        for f in EXPORTS:
            if f not in ("ks_workspace_bytes", "ks_strerror", "ks_destroy", "ks_get_launch_times",
                         "ks_peak_fp64_tflops", "ks_dist_destroy"):
                getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def strerror(code: int) -> str:
    try:
        return lib().ks_strerror(code).decode()
    except ImportError:
        return str(code)


def _check(code: int, what: str):
    if code != KS_OK:
        raise KsError(code, what)


def _stride(a: Optional[torch.Tensor]) -> int:
    if a is None or a.shape[0] == 1:
        return 0
    return int(np.prod(a.shape[1:]))


def _as_tensor(a, device, pin=False):
    if a is None:
        return None
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    if device is not None:
        t = t.to(device)
    elif pin and not t.is_pinned():
        t = t.pin_memory()
    return t.contiguous()


class Dist:
    """One rank's ks_dist (include/ks.h): rank r of `nranks` owns the global
    steps [first_global_step, first_global_step + nsteps_global / nranks).
    ``uid`` (128 bytes from ``Dist.unique_id()`` on rank 0, broadcast by the
    caller) makes the library create its own NCCL communicator -- a collective
    call, with this rank's CUDA device current -- and ks_factor then does the
    boundary allgather itself; ``uid=None`` leaves the exchange to the caller
    (ks_boundary_buffers + ks_factor_boundary)."""

    def __init__(self, rank: int, nranks: int, first_global_step: int, nsteps_global: int,
                 uid: Optional[bytes] = None, device=None):
        self.L = lib()
        self.rank, self.nranks = int(rank), int(nranks)
        self.first, self.nglobal = int(first_global_step), int(nsteps_global)
        if uid is not None and len(uid) != 128:
            raise ValueError("uid must be 128 bytes")
        d = C.c_void_p()
        if device is not None:
            with torch.cuda.device(torch.device(device)):
                rc = self.L.ks_dist_create(C.byref(d), self.rank, self.nranks, uid, self.first, self.nglobal)
        else:
            rc = self.L.ks_dist_create(C.byref(d), self.rank, self.nranks, uid, self.first, self.nglobal)
        _check(rc, "ks_dist_create")
        self.ptr = d

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().ks_dist_unique_id(buf), "ks_dist_unique_id")
        return buf.raw

    def info(self):
        r, n, nc = C.c_int(), C.c_int(), C.c_int()
        _check(self.L.ks_dist_info(self.ptr, C.byref(r), C.byref(n), C.byref(nc)), "ks_dist_info")
        return {"rank": r.value, "nranks": n.value, "nccl_nranks": nc.value}

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                self.L.ks_dist_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


class Smoother:
    """One ks_ctx over a problem whose arrays are torch tensors (or numpy).

    ``problem`` is any object with N, n, m_max, m, F, H, K, L, o, c attributes
    (e.g. ``generators.Problem``).  ``host_inputs=True`` keeps the inputs in
    pinned host memory and lets ks_whiten copy them (end-to-end path).
    Time-sharded multi-GPU: ``dist=Dist(...)`` (this rank's shard of the
    global problem; ``problem`` is the local shard), or the shorthand
    ``shard=(rank, nranks)`` for a caller-driven exchange with power-of-two
    shards.  ``chol=True``: K and L hold lower Cholesky factors
    (KS_COV_IS_CHOL).
    """

    def __init__(self, problem, device="cuda", stream: Optional[torch.cuda.Stream] = None,
                 host_inputs: bool = False, bind_outputs: bool = True, cov: bool = True,
                 shard=None, inputs=None, generic: bool = False, fused_tail: bool = True,
                 dist: Optional[Dist] = None, chol: bool = False, batch: int = 1,
                 keep_whitening: bool = False, big: bool = False):
        self.L = lib()
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        p = problem
        self.N, self.n, self.m_max = int(p.N), int(p.n), int(p.m_max)
        tgt = None if host_inputs else self.device
        if inputs is None:
            inputs = {k: _as_tensor(getattr(p, k), tgt, pin=host_inputs)
                      for k in ("F", "H", "K", "L", "o", "c")}
            m = np.ascontiguousarray(p.m, np.int32)
            # all m_i == m_max: pass m = NULL (lets a constant observation model
            # be whitened once, stride 0)
            inputs["m"] = None if bool(np.all(m == p.m_max)) else _as_tensor(m, tgt, pin=host_inputs)
            # the general model: evolution matrix H_i, rows l_i, state dims n_i
            inputs["Hev"] = _as_tensor(getattr(p, "Hev", None), tgt, pin=host_inputs)
            for k in ("l", "nstate"):
                a = getattr(p, k, None)
                inputs[k] = None if a is None else _as_tensor(np.ascontiguousarray(a, np.int32), tgt,
                                                              pin=host_inputs)
        self.inputs = inputs  # keep alive (borrowed by the library)
        for k in ("F", "H", "K", "L", "o", "c", "Hev"):
            t = inputs.get(k)
            assert t is None or t.dtype == torch.float64
        pr = ks_problem()
        pr.nsteps, pr.n, pr.m_max = self.N, self.n, self.m_max
        ptr = lambda t: None if t is None else t.data_ptr()
        pr.m = ptr(inputs["m"])
        pr.F, pr.H, pr.c, pr.o, pr.K, pr.L = (ptr(inputs[k]) for k in ("F", "H", "c", "o", "K", "L"))
        pr.sF, pr.sH, pr.sc, pr.so, pr.sK, pr.sL = (_stride(inputs[k]) for k in ("F", "H", "c", "o", "K", "L"))
        pr.Hev, pr.sHev = ptr(inputs.get("Hev")), _stride(inputs.get("Hev"))
        pr.l, pr.nstate = ptr(inputs.get("l")), ptr(inputs.get("nstate"))
        if inputs.get("nstate") is not None:
            pr.nstate_min = int(inputs["nstate"].min().item())
        pr.flags = (KS_HOST_INPUTS if host_inputs else 0) | (KS_OUTPUTS_BOUND if bind_outputs else 0) | \
            (KS_GENERIC_PATH if generic else 0) | (0 if fused_tail else KS_NO_FUSED_TAIL) | \
            (KS_COV_IS_CHOL if chol else 0) | (KS_KEEP_WHITENING if keep_whitening else 0) | \
            (KS_BIG_PATH if big else 0)
        pr.batch = int(batch)
        self.problem = pr
        if dist is None and shard is not None:
            r, P = int(shard[0]), int(shard[1])
            dist = Dist(r, P, r * self.N, P * self.N)
        self.dist = dist   # keep alive (borrowed by the context)
        dp = dist.ptr if dist is not None else None
        with torch.cuda.device(self.device):
            nbytes = self.L.ks_workspace_bytes(C.byref(pr), dp)
            if nbytes == 0:
                raise KsError(KS_ERR_ARG, "ks_workspace_bytes")
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self.states = self.cov = None
            if bind_outputs:
                self.states = torch.empty((self.N, self.n), dtype=torch.float64, device=self.device)
                if cov:
                    self.cov = torch.empty((self.N, self.n, self.n), dtype=torch.float64, device=self.device)
            ctx = C.c_void_p()
            _check(self.L.ks_create(C.byref(ctx), C.byref(pr), self.workspace.data_ptr(), nbytes,
                                    self.stream.cuda_stream, dp,
                                    None if self.states is None else self.states.data_ptr(),
                                    None if self.cov is None else self.cov.data_ptr()), "ks_create")
        self.ctx = ctx

    def _call(self, fn, what):
        # the library launches on the current device: make this context's current
        with torch.cuda.device(self.device):
            _check(fn(self.ctx), what)

    # --- the ABI calls -------------------------------------------------------
    def whiten(self):
        self._call(self.L.ks_whiten, "ks_whiten")

    def factor(self):
        self._call(self.L.ks_factor, "ks_factor")

    def factor_boundary(self):
        self._call(self.L.ks_factor_boundary, "ks_factor_boundary")

    def boundary_buffers(self):
        s, r, b = C.c_void_p(), C.c_void_p(), C.c_size_t()
        _check(self.L.ks_boundary_buffers(self.ctx, C.byref(s), C.byref(r), C.byref(b)),
               "ks_boundary_buffers")
        return s.value, r.value, b.value

    def boundary_tensors(self):
        """(send, recv) as uint8 views of the workspace: the caller-driven
        boundary allgather is dist.all_gather_into_tensor(recv, send)."""
        s, r, nb = self.boundary_buffers()
        base = self.workspace.data_ptr()
        P = self.dist.nranks
        return (self.workspace[s - base:s - base + nb], self.workspace[r - base:r - base + P * nb])

    def solve(self):
        self._call(self.L.ks_solve, "ks_solve")

    def selinv(self):
        self._call(self.L.ks_selinv, "ks_selinv")

    def solve_selinv(self):
        self._call(self.L.ks_solve_selinv, "ks_solve_selinv")

    def update_obs(self, o):
        """ks_update_obs: new observations (same shape as the problem's o),
        re-whitened in place; continue with factor() and solve()."""
        host = bool(self.problem.flags & KS_HOST_INPUTS)
        t = _as_tensor(o, None if host else self.device, pin=host)
        assert t.dtype == torch.float64 and tuple(t.shape) == tuple(self.inputs["o"].shape)
        self.inputs["o_update"] = t   # keep alive until the enqueued work completes
        self._call(lambda ctx: self.L.ks_update_obs(ctx, t.data_ptr()), "ks_update_obs")

    def get(self, states=None, cov=None, sync: bool = True):
        """Copy results into torch tensors (device or host); sync=False:
        ks_get_async (host copies only enqueued; synchronise the stream)."""
        sp = None if states is None else states.data_ptr()
        cp = None if cov is None else cov.data_ptr()
        fn = self.L.ks_get if sync else self.L.ks_get_async
        _check(fn(self.ctx, sp, cp), "ks_get" if sync else "ks_get_async")
        return states, cov

    def get_packed(self, states=None, cov_packed=None, sync: bool = True):
        """ks_get_packed: covariance blocks as their upper triangles by rows
        (N x n(n+1)/2) into a device tensor or a PINNED host tensor."""
        sp = None if states is None else states.data_ptr()
        cp = None if cov_packed is None else cov_packed.data_ptr()
        _check(self.L.ks_get_packed(self.ctx, sp, cp, 1 if sync else 0), "ks_get_packed")
        return states, cov_packed

    def sync_status(self):
        st, kd = C.c_int64(-1), C.c_int(0)
        rc = self.L.ks_sync_status(self.ctx, C.byref(st), C.byref(kd))
        return rc, st.value, kd.value

    def check(self):
        rc, st, kd = self.sync_status()
        if rc != KS_OK:
            raise KsError(rc, "ks_sync_status", st, kd)

    def set_timing(self, on=True):
        _check(self.L.ks_set_timing(self.ctx, 1 if on else 0), "ks_set_timing")

    def timing(self):
        ms = (C.c_double * len(FAMILIES))()
        cnt = (C.c_int64 * len(FAMILIES))()
        _check(self.L.ks_get_timing(self.ctx, ms, cnt), "ks_get_timing")
        return {f: (ms[i], cnt[i]) for i, f in enumerate(FAMILIES)}

    def launch_times(self):
        """[(family, level, ms)] of every timed launch since set_timing()."""
        n = self.L.ks_get_launch_times(self.ctx, 0, None, None, None)
        if n < 0:
            raise KsError(-n, "ks_get_launch_times")
        fam = (C.c_int32 * max(n, 1))(); lev = (C.c_int32 * max(n, 1))(); ms = (C.c_float * max(n, 1))()
        self.L.ks_get_launch_times(self.ctx, n, fam, lev, ms)
        return [(FAMILIES[fam[i]], lev[i], ms[i]) for i in range(n)]

    def info(self):
        lv, la = C.c_int64(), C.c_int64()
        _check(self.L.ks_info(self.ctx, C.byref(lv), C.byref(la)), "ks_info")
        return {"levels": lv.value, "launches": la.value}

    def run(self, cov: bool = True, fused: bool = True):
        """whiten -> factor -> solve [-> selinv] (enqueue only); with cov and
        fused, the two backward phases run as one ks_solve_selinv sweep."""
        self.whiten()
        self.factor()
        if cov and fused:
            self.solve_selinv()
            return
        self.solve()
        if cov:
            self.selinv()

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.L.ks_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass


def level_of_steps(N: int):
    """(number of levels, elimination level of every step) from the library's
    host level plan (ks_level_of_steps; no GPU needed)."""
    lv = np.zeros(N, np.int32)
    nl = lib().ks_level_of_steps(int(N), lv.ctypes.data)
    if nl < 0:
        raise KsError(-nl, "ks_level_of_steps")
    return nl, lv


def peak_fp64_tflops(stream=None) -> float:
    """Measured DFMA throughput (TFLOP/s) of the current device."""
    st = stream if stream is not None else torch.cuda.current_stream()
    return float(lib().ks_peak_fp64_tflops(st.cuda_stream))


def smooth(problem, cov: bool = True, device="cuda"):
    """Convenience: full pipeline, returns (states, cov) as device tensors."""
    s = Smoother(problem, device=device, cov=cov)
    s.run(cov=cov)
    s.check()
    return s.states, s.cov
