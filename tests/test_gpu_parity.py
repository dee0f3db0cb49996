"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle.

Metric: per-step normwise relative error,
e_state = max_i |x_i - x_i^ora|_inf / |x_i^ora|_inf <= 1e-9 and
e_cov   = max_i |S_ii - S_ii^ora|_max / |S_ii^ora|_max <= 1e-8 (BASELINE.json).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_11686_b200 import generators as gen
from tests.dense import rel_cov_err, rel_state_err

pytestmark = pytest.mark.gpu

TOL_X, TOL_S = 1e-9, 1e-8


def ks():
    from paper_2502_11686_b200 import ks as _ks
    return _ks


def gpu_smooth(p, cov=True, fused=True, **kw):
    s = ks().Smoother(p, cov=cov, **kw)
    s.run(cov=cov, fused=fused)
    s.check()
    x = s.states.cpu().numpy()
    S = s.cov.cpu().numpy() if cov else None
    return x, S, s


def assert_parity(p, cov=True, **kw):
    x, S, s = gpu_smooth(p, cov=cov, **kw)
    xo, So = oracle.smooth(p)
    ex = rel_state_err(x, xo)
    assert ex <= TOL_X, f"{p.name} N={p.N}: state err {ex:.3e}"
    if cov:
        es = rel_cov_err(S, So)
        assert es <= TOL_S, f"{p.name} N={p.N}: cov err {es:.3e}"
        assert np.array_equal(S, np.swapaxes(S, 1, 2))
    return s


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8, 9, 15, 16, 17, 31, 33, 64, 100, 127, 257])
@pytest.mark.parametrize("n", [1, 2, 3, 6, 8])
def test_random_small_all_parities(N, n, generic):
    """Both kernel families: the small-n register path (default for n, m <= 8)
    and the CTA shared-memory path (KS_GENERIC_PATH)."""
    rng = np.random.default_rng(N * 100 + n)
    m = None if N > 1 else n
    p = gen.random_problem(rng, N, n, m=m, m_max=n + 1 if n < 8 else 8)
    if n == 8:
        p.m = np.minimum(p.m, 8)
    if N > 1:
        p.m[-1] = max(p.m[-1], 1)
    assert_parity(p, generic=generic)


@pytest.mark.parametrize("const", [False, True])
@pytest.mark.parametrize("n,mmax", [(4, 9), (8, 3), (9, 1), (12, 12), (13, 20), (17, 17), (24, 5),
                                    (33, 7), (40, 41), (48, 48)])
def test_random_dims(n, mmax, const):
    rng = np.random.default_rng(n * 7 + mmax)
    N = 45
    m = np.full(N, mmax, np.int32) if const else rng.integers(0, mmax + 1, N).astype(np.int32)
    m[0] = max(m[0], n) if mmax >= n else m[0]
    if mmax < n:
        m[:] = mmax
    p = gen.random_problem(rng, N, n, m=m, m_max=mmax, const=const)
    assert_parity(p)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("cfg,N", [("c1", None), ("c2", 2000), ("c3", 2001), ("c4", 301),
                                   ("c5", 1 << 16), ("c5", 12345)])
def test_configs_reduced(cfg, N, generic):
    assert_parity(gen.make(cfg, N=N), generic=generic)


# Odd levels >= 1 above the fused tail (K > 128): K/2 % 64 != 0 runs the last
# column in its own thread beside the last pair (split_odd: N = 1550 -> K_1 =
# 775, N = 6300 -> K_2 = 1575, N = 12345 -> K_3 = 1543), K/2 % 64 == 0 keeps
# both in one thread (N = 258 -> K_1 = 129, N = 33282 -> K_1 = 16641 = 2*8320+1).
@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c2", "c3", "c5"])
@pytest.mark.parametrize("N", [1550, 6300, 258, 33282])
def test_odd_levels_split_and_serial(cfg, N):
    assert_parity(gen.make(cfg, N=N))


@pytest.mark.parametrize("n", [6, 48])
def test_paper_benchmark_class(n):
    """The paper's own problem class."""
    assert_parity(gen.paper_problem(1000 if n == 6 else 200, n, seed=n))


def test_nc_variant_states_only():
    p = gen.make("c2", N=999)
    x, _, s = gpu_smooth(p, cov=False)
    assert rel_state_err(x, oracle.smooth(p, cov=False)) <= TOL_X


def test_noise_free_recovery():
    p = gen.make("c2", N=3000, noise_free=True)
    x, _, _ = gpu_smooth(p, cov=False)
    assert rel_state_err(x, p.x_true) <= 1e-9


@pytest.mark.parametrize("generic", [False, True])
def test_determinism_bitwise(generic):
    p = gen.make("c3", N=5000)
    x1, S1, _ = gpu_smooth(p, generic=generic)
    x2, S2, _ = gpu_smooth(p, generic=generic)
    assert np.array_equal(x1, x2) and np.array_equal(S1, S2)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("case", ["c2", "c3", "c5", "r1", "r2", "r5", "r7", "r8"])
def test_fused_backward_matches_separate(case, generic):
    """ks_solve_selinv (one sweep) gives the same bits as ks_solve + ks_selinv."""
    if case.startswith("r"):
        n = int(case[1:])
        rng = np.random.default_rng(50 + n)
        p = gen.random_problem(rng, 777, n, m_max=min(n + 1, 8))
        p.m = np.minimum(p.m, p.m_max)
    else:
        p = gen.make(case, N=4097 if case != "c5" else 12345)
    x1, S1, _ = gpu_smooth(p, fused=True, generic=generic)
    x2, S2, _ = gpu_smooth(p, fused=False, generic=generic)
    assert np.array_equal(x1, x2) and np.array_equal(S1, S2)
    xo, So = oracle.smooth(p)
    assert rel_state_err(x1, xo) <= TOL_X and rel_cov_err(S1, So) <= TOL_S


@pytest.mark.parametrize("case", [("c5", 12345), ("c5", 1 << 14), ("c2", 5000), ("c3", 777), ("c1", None),
                                  ("r1", 300), ("r3", 129), ("r7", 1000), ("r8", 500)])
def test_fused_tail_matches_level_launches(case):
    """The recursion tail in one on-chip kernel gives the same bits as one
    launch per level (KS_NO_FUSED_TAIL)."""
    name, N = case
    if name.startswith("r"):
        n = int(name[1:])
        rng = np.random.default_rng(7 * n + N)
        p = gen.random_problem(rng, N, n, m_max=min(n + 1, 8))
        p.m = np.minimum(p.m, p.m_max)
    else:
        p = gen.make(name, N=N)
    x1, S1, s1 = gpu_smooth(p)
    x2, S2, _ = gpu_smooth(p, fused_tail=False)
    assert np.array_equal(x1, x2) and np.array_equal(S1, S2)


def test_small_and_generic_paths_agree():
    p = gen.make("c2", N=4097)
    x1, S1, _ = gpu_smooth(p)
    x2, S2, _ = gpu_smooth(p, generic=True)
    assert rel_state_err(x1, x2) <= 1e-12 and rel_cov_err(S1, S2) <= 1e-12


def test_host_inputs_and_get():
    """KS_HOST_INPUTS (pinned host inputs, H2D inside ks_whiten) and ks_get
    into host and device buffers give the same bits as device inputs."""
    p = gen.make("c2", N=1500)
    x1, S1, _ = gpu_smooth(p)
    s = ks().Smoother(p, host_inputs=True, bind_outputs=False)
    s.run()
    xs = torch.empty((p.N, p.n), dtype=torch.float64).pin_memory()
    Ss = torch.empty((p.N, p.n, p.n), dtype=torch.float64).pin_memory()
    s.get(xs, Ss)
    s.check()
    assert np.array_equal(xs.numpy(), x1) and np.array_equal(Ss.numpy(), S1)
    xd = torch.empty((p.N, p.n), dtype=torch.float64, device="cuda")
    s.get(xd, None)
    assert np.array_equal(xd.cpu().numpy(), x1)
    # ks_get_async: enqueued only; equal once the stream is synchronised
    xa = torch.zeros((p.N, p.n), dtype=torch.float64).pin_memory()
    Sa = torch.zeros((p.N, p.n, p.n), dtype=torch.float64).pin_memory()
    s.get(xa, Sa, sync=False)
    s.stream.synchronize()
    assert np.array_equal(xa.numpy(), x1) and np.array_equal(Sa.numpy(), S1)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c2", "c4", "c1", "c5"])
def test_get_packed(case):
    """ks_get_packed: the upper triangles by rows of the covariance blocks
    equal the full blocks' (bitwise), into device memory, pinned host memory
    (written by the kernel over PCIe; c5 at N = 2^20: 22 M doubles) and
    asynchronously; pageable host memory and a missing ks_selinv are
    rejected."""
    p = gen.make(case, N={"c2": 1500, "c4": 45, "c1": 7, "c5": 1 << 20}[case])
    x1, S1, _ = gpu_smooth(p)
    n = p.n
    iu = np.triu_indices(n)
    want = S1[:, iu[0], iu[1]]
    s = ks().Smoother(p, host_inputs=True, bind_outputs=False)
    s.run()
    Pk = n * (n + 1) // 2
    dev = torch.full((p.N, Pk), np.nan, dtype=torch.float64, device="cuda")
    xd = torch.empty((p.N, n), dtype=torch.float64, device="cuda")
    s.get_packed(xd, dev)
    assert np.array_equal(dev.cpu().numpy(), want) and np.array_equal(xd.cpu().numpy(), x1)
    hp = torch.full((p.N, Pk), np.nan, dtype=torch.float64).pin_memory()
    xh = torch.empty((p.N, n), dtype=torch.float64).pin_memory()
    s.get_packed(xh, hp)
    assert np.array_equal(hp.numpy(), want) and np.array_equal(xh.numpy(), x1)
    ha = torch.full((p.N, Pk), np.nan, dtype=torch.float64).pin_memory()
    s.get_packed(None, ha, sync=False)
    s.stream.synchronize()
    assert np.array_equal(ha.numpy(), want)
    with pytest.raises(ks().KsError):
        s.get_packed(None, torch.empty((p.N, Pk), dtype=torch.float64))   # pageable
    s2 = ks().Smoother(p)
    s2.whiten(); s2.factor(); s2.solve()
    with pytest.raises(ks().KsError):
        s2.get_packed(None, dev)


@pytest.mark.parametrize("eps", [1e-3, 1e-6])
def test_cta_panel_gram_guard(eps):
    """The CTA path's Gram-downdated Householder panel (DESIGN reading R28):
    observation and evolution matrices whose odd columns nearly repeat the
    even ones (relative difference eps) make the stacked block columns of
    every stage-1 panel nearly pairwise dependent, so the downdated norms
    cancel and the accuracy guard recomputes the Gram exactly (counted in
    the profiling build; tools/micro/qr_bench.cu checks the same at the QR
    level).  The smoothed results still match the oracle."""
    p = gen.make("c4", N=45)
    rng = np.random.default_rng(7)
    for A in (p.H, p.F):
        A[..., 1::2] = A[..., 0::2] + eps * rng.standard_normal(A[..., 0::2].shape)
    assert_parity(p, generic=True)


@pytest.mark.parametrize("case", [("c2", 3001), ("c1", 1000), ("c3", 777), ("c5", 40000)])
def test_split_levels_match_one_thread_form(case, monkeypatch):
    """Levels with at most one 64-pair CTA per SM run three threads per pair
    (stage 1 + pass B, stage 3, pass A + post); KS_NO_SPLIT_LEVELS forces the
    one-thread-per-pair kernels (split odd levels included).  Bitwise equal."""
    cfg, N = case
    p = gen.make(cfg, N=N)
    x1, S1, _ = gpu_smooth(p)
    monkeypatch.setenv("KS_NO_SPLIT_LEVELS", "1")
    x2, S2, _ = gpu_smooth(p)
    assert np.array_equal(x1, x2) and np.array_equal(S1, S2)


def test_level_count():
    for N in (1, 2, 3, 7, 8, 9, 1000, 4096):
        s = ks().Smoother(gen.make("c1", N=max(N, 2)) if N > 1 else gen.random_problem(
            np.random.default_rng(0), 1, 2, m=2))
        assert s.info()["levels"] == int(np.floor(np.log2(s.N))) + 1


def test_error_not_spd():
    rng = np.random.default_rng(9)
    p = gen.random_problem(rng, 20, 3, m=3)
    p.K[7] = -np.eye(3)
    s = ks().Smoother(p)
    s.run()
    rc, step, kind = s.sync_status()
    assert rc == ks().KS_ERR_NOT_SPD and step == 7 and kind == 1
    p = gen.random_problem(rng, 20, 3, m=3)
    p.L[11] = np.diag([1.0, 1.0, -2.0])
    s = ks().Smoother(p)
    s.run()
    rc, step, kind = s.sync_status()
    assert rc == ks().KS_ERR_NOT_SPD and step == 11 and kind == 2


def test_error_rank():
    rng = np.random.default_rng(10)
    p = gen.random_problem(rng, 16, 2, m=0)
    s = ks().Smoother(p)
    s.run()
    rc, _, _ = s.sync_status()
    assert rc == ks().KS_ERR_RANK


def test_error_order_and_args():
    p = gen.make("c1", N=64)
    s = ks().Smoother(p)
    with pytest.raises(ks().KsError) as ei:
        s.factor()
    assert ei.value.code == ks().KS_ERR_ORDER
    s.whiten()
    with pytest.raises(ks().KsError):
        s.solve()
    with pytest.raises(ks().KsError):
        s.get(torch.empty((64, 2), dtype=torch.float64, device="cuda"))


def _virtual_shards(p, P, cov=True, generic=False, fused=False):
    """The time-sharded multi-GPU algorithm with P ranks emulated on one GPU:
    each rank's local levels run in its own context; the allgather is a
    device copy into every rank's receive buffer (no rank waits on another)."""
    from paper_2502_11686_b200 import dist as kdist
    parts = [ks().Smoother(kdist.pad_shard(p, r, P), shard=(r, P, None), generic=generic)
             for r in range(P)]
    for s in parts:
        s.whiten()
        s.factor()
    views = [s.boundary_tensors() for s in parts]
    gathered = torch.cat([snd for snd, _ in views])
    for s, (_, rcv) in zip(parts, views):
        rcv.copy_(gathered)
        s.factor_boundary()
        if cov and fused:
            s.solve_selinv()
            continue
        s.solve()
        if cov:
            s.selinv()
    for s in parts:
        s.check()
    x = np.concatenate([s.states.cpu().numpy() for s in parts])
    S = np.concatenate([s.cov.cpu().numpy() for s in parts]) if cov else None
    # padded shards (N not P x a power of two, reading R29): the decoupled
    # steps come out as u = 0, S = I exactly; the real steps are the first N
    assert np.array_equal(x[p.N:], np.zeros_like(x[p.N:]))
    if cov:
        assert np.abs(S[p.N:] - np.eye(p.n)).max(initial=0.0) <= 1e-15
        S = S[:p.N]
    x = x[:p.N]
    _virtual_shards.launches = [s.info()["launches"] for s in parts]
    return x, S


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("cfg,N,P", [("c5", 1 << 12, 2), ("c5", 1 << 12, 4), ("c5", 1 << 12, 8),
                                     ("c2", 1 << 11, 2), ("c3", 1 << 11, 8), ("c1", 1 << 10, 4),
                                     ("c2", 3 * 256, 3), ("c4", 64, 2),
                                     # any N (padded shards, reading R29)
                                     ("c2", 1000, 3), ("c1", 1000, 8), ("c3", 777, 4),
                                     ("c5", 5000, 8), ("c4", 100, 3)])
def test_virtual_shards_match_oracle(cfg, N, P, generic):
    p = gen.make(cfg, N=N)
    x, S = _virtual_shards(p, P, generic=generic)
    xf, Sf = _virtual_shards(p, P, generic=generic, fused=True)
    assert np.array_equal(x, xf) and np.array_equal(S, Sf)
    xo, So = oracle.smooth(p)
    assert rel_state_err(x, xo) <= TOL_X
    assert rel_cov_err(S, So) <= TOL_S
    x1, S1, _ = gpu_smooth(p, generic=generic)
    if (N // P) & (N // P - 1) == 0 and P & (P - 1) == 0:
        # power-of-two shards: the single-GPU elimination order.  The small
        # path runs the boundary system on the same per-column routines as
        # one GPU (SURVEY §8(e) invariant, T3): bitwise equal.  The generic
        # path's boundary kernels differ in rounding only.
        if generic:
            assert rel_state_err(x, x1) <= 1e-12 and rel_cov_err(S, S1) <= 1e-12
        else:
            assert np.array_equal(x, x1) and np.array_equal(S, S1)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_configs_full_size(cfg):
    """BASELINE.json configs at full size, every output compared."""
    assert_parity(gen.make(cfg))


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("cfg,N", [("c2", 1500), ("c3", 777), ("c5", 4096), ("c4", 65)])
def test_cov_is_chol(cfg, N, generic):
    """KS_COV_IS_CHOL: K and L given as lower Cholesky factors (north_star's
    "whitening factors K_i, L_i"; any V with V^T V = K^-1 whitens)
    give the covariance path's results."""
    if generic is False and cfg == "c4":
        pytest.skip("n = 48 runs on the CTA path only")
    p = gen.make(cfg, N=N)
    x1, S1, _ = gpu_smooth(p, generic=generic)
    q = gen.make(cfg, N=N)
    q.K = np.linalg.cholesky(q.K)
    q.L = np.linalg.cholesky(q.L)
    q.K = np.tril(q.K) + np.triu(np.full_like(q.K, np.nan), 1)   # only the lower triangle is read
    q.L = np.tril(q.L) + np.triu(np.full_like(q.L, np.nan), 1)
    x2, S2, _ = gpu_smooth(q, generic=generic, chol=True)
    assert rel_state_err(x2, x1) <= 1e-12 and rel_cov_err(S2, S1) <= 1e-12
    xo, So = oracle.smooth(p)
    assert rel_state_err(x2, xo) <= TOL_X and rel_cov_err(S2, So) <= TOL_S


def test_cov_is_chol_zero_diagonal():
    rng = np.random.default_rng(4)
    p = gen.random_problem(rng, 20, 3, m=3)
    p.K = np.linalg.cholesky(p.K)
    p.L = np.linalg.cholesky(p.L)
    p.K[5, 1, 1] = 0.0
    s = ks().Smoother(p, chol=True)
    s.run()
    rc, step, kind = s.sync_status()
    assert rc == ks().KS_ERR_NOT_SPD and step == 5 and kind == 1


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("scale", [1e-40, 1e-20, 1.0, 1e20, 1e40])
def test_scale_sweep(scale, generic):
    """Scaling K and L by s^2 and o by s scales the whitened system by 1/s
    and leaves the states scaled by s and the covariances by s^2: every
    output must still match the oracle (the small path's empty-row prior
    2^-600 is far below the data across this range)."""
    rng = np.random.default_rng(11)
    p = gen.random_problem(rng, 300, 4, m_max=5)
    p.K = p.K * scale ** 2
    p.L = p.L * scale ** 2
    p.o = p.o * scale
    if p.c is not None:
        p.c = p.c * scale
    x, S, _ = gpu_smooth(p, generic=generic)
    xo, So = oracle.smooth(p)
    assert rel_state_err(x, xo) <= TOL_X and rel_cov_err(S, So) <= TOL_S


def test_scale_out_of_range_rejected():
    """Outside the small path's exponent range (whitened block norms beyond
    [1e-80, 1e60]) the problem is rejected, not solved inaccurately."""
    rng = np.random.default_rng(12)
    for scale in (1e-70, 1e90):
        p = gen.random_problem(rng, 64, 3, m=3)
        p.K = p.K * scale ** 2
        p.L = p.L * scale ** 2
        p.o = p.o * scale
        s = ks().Smoother(p)
        s.run()
        rc, step, kind = s.sync_status()
        assert rc == ks().KS_ERR_ARG and kind == 3, (scale, rc)
        x, S, _ = gpu_smooth(p, generic=True)    # the CTA path has no such limit
        xo, So = oracle.smooth(p)
        assert rel_state_err(x, xo) <= TOL_X and rel_cov_err(S, So) <= TOL_S


# ---- batched independent problems, repeated solves ----

def _batch_cases(case):
    if case == "random":
        rng = np.random.default_rng(21)
        return [gen.random_problem(rng, 100, 3, m_max=4) for _ in range(8)]
    if case == "c5":
        p = gen.make("c5", N=1 << 16)
        return [p.slice(b << 12, (b + 1) << 12) for b in range(16)]
    if case == "c1":
        p = gen.make("c1")
        return [p.slice(b * 100, (b + 1) * 100) for b in range(10)]
    if case == "c1_singletons":
        p = gen.make("c1", N=64)
        return [p.slice(b, b + 1) for b in range(64)]
    if case == "c4":
        p = gen.make("c4", N=96)
        return [p.slice(b * 24, (b + 1) * 24) for b in range(4)]
    raise ValueError(case)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("case", ["random", "c5", "c1", "c1_singletons", "c4"])
def test_batched_problems(case, generic):
    """ks_problem.batch = B: one context over B independent problems laid end
    to end; every problem's outputs match the oracle run on that problem
    alone (whose first step has no evolution row)."""
    if case == "c4" and not generic:
        pytest.skip("n = 48 runs on the CTA path only")
    parts = _batch_cases(case)
    p = gen.Problem.concat(parts)
    s = ks().Smoother(p, batch=len(parts), generic=generic)
    s.run()
    s.check()
    x, S = s.states.cpu().numpy(), s.cov.cpu().numpy()
    Nb = parts[0].N
    for b, q in enumerate(parts):
        xo, So = oracle.smooth(q)
        xb, Sb = x[b * Nb:(b + 1) * Nb], S[b * Nb:(b + 1) * Nb]
        assert rel_state_err(xb, xo) <= TOL_X, (b, rel_state_err(xb, xo))
        assert rel_cov_err(Sb, So) <= TOL_S, (b, rel_cov_err(Sb, So))


def test_batched_bad_args():
    p = gen.make("c1", N=100)
    with pytest.raises(ks().KsError):
        ks().Smoother(p, batch=7)        # 100 % 7 != 0


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("cfg,N", [("c2", 2000), ("c3", 1777), ("c5", 1 << 14), ("c4", 41)])
def test_update_obs(cfg, N, host, generic):
    """ks_update_obs: new observations re-whitened in place (the model's
    whitening kept), then factor + solve; the states equal a fresh run on the
    new observations and the earlier covariances stay valid (they do not
    depend on o)."""
    if cfg == "c4" and not generic:
        pytest.skip("n = 48 runs on the CTA path only")
    p = gen.make(cfg, N=N)
    q = gen.make(cfg, N=N)
    rng = np.random.default_rng(5)
    q.o = q.o + rng.standard_normal(q.o.shape) * (np.abs(q.o).max() * 0.1 + 1.0)
    q.o[np.arange(q.m_max)[None, :] >= q.m[:, None]] = 0.0
    s = ks().Smoother(p, keep_whitening=True, host_inputs=host, bind_outputs=not host, generic=generic)
    s.run()
    s.check()
    x1 = torch.empty((N, p.n), dtype=torch.float64)
    S1 = torch.empty((N, p.n, p.n), dtype=torch.float64)
    s.get(x1, S1)
    s.update_obs(q.o)
    s.factor()
    s.solve()
    s.check()
    x2 = torch.empty((N, p.n), dtype=torch.float64)
    S2 = torch.empty((N, p.n, p.n), dtype=torch.float64)
    s.get(x2, S2)
    xf, Sf, _ = gpu_smooth(q, generic=generic)
    assert rel_state_err(x2.numpy(), xf) <= 1e-12
    assert np.array_equal(S2.numpy(), S1.numpy())
    assert rel_cov_err(S2.numpy(), Sf) <= 1e-12
    xo = oracle.smooth(q, cov=False)
    assert rel_state_err(x2.numpy(), xo) <= TOL_X


def test_update_obs_needs_kept_whitening():
    p = gen.make("c2", N=500)
    s = ks().Smoother(p)
    s.run()
    with pytest.raises(ks().KsError) as ei:
        s.update_obs(p.o)
    assert ei.value.code == ks().KS_ERR_ARG


# ---- the general model ----

def _general_parity(p, generic, noise_free=False):
    from oracle import general as og
    s = ks().Smoother(p, generic=generic)
    s.run()
    s.check()
    x, S = s.states.cpu().numpy(), s.cov.cpu().numpy()
    ns = p.nstate if p.nstate is not None else np.full(p.N, p.n)
    xo, So = og.smooth_general(p)
    mask_x = np.arange(p.n)[None, :] < ns[:, None]
    mask_S = mask_x[:, :, None] & mask_x[:, None, :]
    assert rel_state_err(np.where(mask_x, x, 0.0), xo) <= TOL_X
    assert rel_cov_err(np.where(mask_S, S, 0.0), So) <= TOL_S
    # the embedding's padding components: pinned to 0, uncorrelated with the state
    pad = ~mask_x
    assert np.abs(x[pad]).max(initial=0.0) <= 1e-12 * np.abs(xo).max()
    cross = mask_x[:, :, None] & pad[:, None, :]
    assert np.abs(S[cross]).max(initial=0.0) <= 1e-12 * np.abs(So).max()
    if noise_free:
        assert rel_state_err(np.where(mask_x, x, 0.0), p.x_true) <= 1e-9
    return s


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("n,nmin,mmax,N", [(2, 1, 2, 257), (4, 1, 4, 300), (4, 2, 3, 1000), (6, 4, 4, 513),
                                           (8, 8, 8, 129), (6, 2, 6, 200), (12, 5, 12, 150)])
def test_general_model(n, nmin, mmax, N, generic):
    """Per-step state dimensions n_i and rectangular evolution H_i (l_i x n_i,
    l_i != n_i) against the general-model oracle; the small path takes the
    problems whose padded observation blocks fit (m_max + n - min n_i <= 8)."""
    rng = np.random.default_rng(1000 * n + 10 * nmin + mmax)
    p = gen.general_problem(rng, N, n, m_max=mmax, nmin=nmin)
    s = _general_parity(p, generic)
    if not generic:
        assert s.problem.n == n


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("n,nmin,N,P", [(4, 1, 512, 4), (6, 3, 300, 2), (3, 1, 1000, 8)])
def test_general_model_virtual_shards(n, nmin, N, P, generic):
    """Per-step n_i and rectangular H_i on time shards (power-of-two and
    padded): every rank's first F_i has its ignored columns zeroed by
    dist.pad_shard (the library cannot mask them there, include/ks.h); the
    gathered shards match the general-model oracle."""
    from oracle import general as og
    rng = np.random.default_rng(300 + n + N)
    p = gen.general_problem(rng, N, n, m_max=n, nmin=nmin)
    x, S = _virtual_shards(p, P, generic=generic)
    xo, So = og.smooth_general(p)
    mask_x = np.arange(p.n)[None, :] < p.nstate[:, None]
    mask_S = mask_x[:, :, None] & mask_x[:, None, :]
    assert rel_state_err(np.where(mask_x, x, 0.0), xo) <= TOL_X
    assert rel_cov_err(np.where(mask_S, S, 0.0), So) <= TOL_S


@pytest.mark.parametrize("generic", [False, True])
def test_general_model_noise_free(generic):
    rng = np.random.default_rng(77)
    p = gen.general_problem(rng, 2000, 4, m_max=4, nmin=2, noise_free=True)
    _general_parity(p, generic, noise_free=True)


@pytest.mark.parametrize("generic", [False, True])
def test_general_rectangular_only(generic):
    """Uniform n_i = n, l_i in [1, n] with a per-step H_i; and a constant
    non-identity H (stride 0, the constant-model path)."""
    rng = np.random.default_rng(5)
    p = gen.general_problem(rng, 700, 5, m_max=5, nmin=5)
    p.nstate = None
    _general_parity(p, generic)
    q = gen.make("c2", N=999)
    q.Hev = (np.eye(6) + 0.3 * rng.standard_normal((6, 6)))[None]
    _general_parity(q, generic)


def test_general_with_batch_and_host_inputs():
    rng = np.random.default_rng(9)
    parts = [gen.general_problem(rng, 64, 3, m_max=3, nmin=1) for _ in range(4)]
    from oracle import general as og
    p = gen.Problem.concat(parts)
    s = ks().Smoother(p, batch=4, host_inputs=True, bind_outputs=False)
    s.run()
    xs = torch.empty((p.N, p.n), dtype=torch.float64)
    Ss = torch.empty((p.N, p.n, p.n), dtype=torch.float64)
    s.get(xs, Ss)
    s.check()
    for b, q in enumerate(parts):
        xo, So = og.smooth_general(q)
        ns = q.nstate
        m = np.arange(p.n)[None, :] < ns[:, None]
        xb = np.where(m, xs.numpy()[b * 64:(b + 1) * 64], 0.0)
        Sb = np.where(m[:, :, None] & m[:, None, :], Ss.numpy()[b * 64:(b + 1) * 64], 0.0)
        assert rel_state_err(xb, xo) <= TOL_X and rel_cov_err(Sb, So) <= TOL_S


# ---- the large-n path (n = m = 500) ----

@pytest.mark.parametrize("n,N,mmax,const", [(2, 1, 2, False), (3, 2, 4, False), (3, 5, 1, False), (6, 8, 6, True),
                                            (6, 17, 7, False), (9, 33, 9, False), (17, 64, 17, True),
                                            (5, 100, 2, False), (20, 21, 25, False)])
def test_big_path_small_n(n, N, mmax, const):
    """The large-n path's batched kernels forced at small n (KS_BIG_PATH) --
    every level shape, odd levels, ragged m_i -- against the oracle."""
    rng = np.random.default_rng(31 * n + N)
    m = n if N == 1 else (mmax if const else None)
    p = gen.random_problem(rng, N, n, m=m, m_max=mmax, const=const)
    p.m = np.minimum(p.m, mmax).astype(np.int32)
    if N > 1 and mmax < n:
        p.m[:] = mmax
    assert_parity(p, big=True)


@pytest.mark.parametrize("cfg,N", [("c4", 65), ("c2", 300), ("c3", 257), ("c5", 1000)])
def test_big_path_configs(cfg, N):
    assert_parity(gen.make(cfg, N=N), big=True)
    x1, S1, _ = gpu_smooth(gen.make(cfg, N=N), big=True)
    x2, S2, _ = gpu_smooth(gen.make(cfg, N=N))
    assert rel_state_err(x1, x2) <= 1e-11 and rel_cov_err(S1, S2) <= 1e-11


@pytest.mark.parametrize("n,N", [(72, 20), (128, 9), (200, 5)])
def test_big_path_large_n(n, N):
    """n beyond the CTA path's shared memory: the default path is the large-n one."""
    assert_parity(gen.paper_problem(N, n, seed=n))
    assert_parity(gen.random_problem(np.random.default_rng(n), N, n, m=n))


def test_big_path_batch_and_nc():
    parts = [gen.paper_problem(12, 80, seed=s) for s in range(3)]
    p = gen.Problem.concat(parts)
    s = ks().Smoother(p, batch=3)
    s.run()
    s.check()
    x, S = s.states.cpu().numpy(), s.cov.cpu().numpy()
    for b, q in enumerate(parts):
        xo, So = oracle.smooth(q)
        assert rel_state_err(x[b * 12:(b + 1) * 12], xo) <= TOL_X
        assert rel_cov_err(S[b * 12:(b + 1) * 12], So) <= TOL_S
    q = gen.paper_problem(40, 72, seed=1)
    x, _, _ = gpu_smooth(q, cov=False)
    assert rel_state_err(x, oracle.smooth(q, cov=False)) <= TOL_X


@pytest.mark.slow
def test_big_path_n500():
    """The paper's n = m = 500 size at reduced k (the oracle is plain C,
    about 46 n^3 flops per step)."""
    assert_parity(gen.paper_problem(6, 500, seed=5))


@pytest.mark.parametrize("cfg,N,P", [("c5", 1 << 14, 4), ("c5", 1 << 16, 8), ("c2", 1 << 12, 2)])
def test_sharded_launch_count(cfg, N, P):
    """A sharded rank runs the single-GPU plan of its N/P steps (fused tail
    and subtree pass included) plus three launches for the boundary system
    (re-tiling the gathered entries, its factor tail, its backward tail)."""
    p = gen.make(cfg, N=N)
    _virtual_shards(p, P, fused=True)
    q = gen.make(cfg, N=N // P)
    s = ks().Smoother(q)
    s.run()
    s.check()
    one = s.info()["launches"]
    assert all(l == one + 3 for l in _virtual_shards.launches), (one, _virtual_shards.launches)


def test_big_path_chol_and_host_inputs():
    """The large-n path with Cholesky-factor inputs (KS_COV_IS_CHOL) and with
    pinned host inputs (KS_HOST_INPUTS, ks_get into host buffers)."""
    rng = np.random.default_rng(17)
    p = gen.random_problem(rng, 40, 70, m=70)
    xo, So = oracle.smooth(p)
    q = gen.random_problem(np.random.default_rng(17), 40, 70, m=70)
    q.K = np.linalg.cholesky(q.K)
    q.L = np.linalg.cholesky(q.L)
    x, S, _ = gpu_smooth(q, chol=True)
    assert rel_state_err(x, xo) <= TOL_X and rel_cov_err(S, So) <= TOL_S
    s = ks().Smoother(p, host_inputs=True, bind_outputs=False)
    s.run()
    xs = torch.empty((p.N, p.n), dtype=torch.float64)
    Ss = torch.empty((p.N, p.n, p.n), dtype=torch.float64)
    s.get(xs, Ss)
    s.check()
    assert rel_state_err(xs.numpy(), xo) <= TOL_X and rel_cov_err(Ss.numpy(), So) <= TOL_S


def test_big_path_errors():
    """Non-SPD covariance and rank deficiency are reported on the large-n path."""
    rng = np.random.default_rng(18)
    p = gen.random_problem(rng, 12, 66, m=66)
    p.K[5] = -np.eye(66)
    s = ks().Smoother(p)
    s.run()
    rc, step, kind = s.sync_status()
    assert rc == ks().KS_ERR_NOT_SPD and step == 5 and kind == 1
    p = gen.random_problem(rng, 12, 66, m=0)
    s = ks().Smoother(p)
    s.run()
    assert s.sync_status()[0] == ks().KS_ERR_RANK


@pytest.mark.parametrize("n,N,P", [(3, 1 << 10, 4), (5, 1 << 11, 2), (7, 1 << 10, 8)])
def test_virtual_shards_odd_n(n, N, P):
    """Odd state dimensions on sharded ranks (the small path's non-TMA
    backward and the AoS boundary entry of an odd n)."""
    rng = np.random.default_rng(60 + n)
    p = gen.random_problem(rng, N, n, m_max=min(n + 1, 8))
    p.m = np.minimum(p.m, p.m_max).astype(np.int32)
    x, S = _virtual_shards(p, P, fused=True)
    xo, So = oracle.smooth(p)
    assert rel_state_err(x, xo) <= TOL_X and rel_cov_err(S, So) <= TOL_S
    x1, S1, _ = gpu_smooth(p)
    assert np.array_equal(x, x1) and np.array_equal(S, S1)


@pytest.mark.parametrize("n,N", [(12, 1500), (24, 700), (40, 301)])
def test_cta_path_larger_N(n, N):
    """The CTA path (n > 8) at larger N: many levels, odd levels, split last columns."""
    rng = np.random.default_rng(70 + n)
    p = gen.random_problem(rng, N, n, m=n)
    # a stable evolution (random_problem's 0.9 Q + 0.2 E has spectral radius
    # > 1 at n >= 12: over 1500 steps the states would span 1e0..1e69 and the
    # per-step relative metric would measure the conditioning, not the method)
    p.F = 0.97 * gen.haar_orthogonal(rng, N, n)
    p.x, p.o = gen.simulate(rng, p.F, p.K, p.H, p.L, p.m, c=p.c)
    assert_parity(p)
