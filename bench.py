#!/usr/bin/env python
"""Benchmark: smoothed steps/s of the Odd-Even Kalman smoother (states +
covariances, fp64) on BASELINE.json config 5 (k = 2^22 steps, n = 6, m = 3,
constant-velocity model), time-sharded over N GPUs (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ks|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = ks_whiten + ks_factor (on N > 1 the local levels, the library's
NCCL allgather of the boundary columns and the boundary system) +
ks_solve_selinv (solve + SelInv in one backward sweep) with inputs resident in HBM (outputs bound
to caller buffers, so ks_get is free).  The working set (~11 GB) is far
larger than L2 (126 MB), so no L2 flush is needed between steps.

Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU oracle
(the reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "smoothed steps/s (states+covariances, fp64)"
UNIT = "steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ks", choices=["ks", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--N", type=int, default=None, help="override the config's step count")
    ap.add_argument("--cpu-sample", type=int, default=1 << 20,
                    help="steps of the workload the oracle cpu_baseline runs (3 passes of ~2.5 s)")
    ap.add_argument("--ref-sample", type=int, default=1 << 18,
                    help="steps per --impl reference step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling runs: no e2e / cpu baseline")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    ap.add_argument("--no-per-config", action="store_true", help="skip the c1-c4 per_config block")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "host"],
                    help="N > 1: the library's NCCL allgather (default), or -- a validation mode for "
                         "boxes with fewer GPUs than ranks -- the caller-driven exchange staged through "
                         "host memory over gloo (ranks may share a GPU; eager, not a multi-GPU number)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_desc(cfg, N):
    d = {"c1": "k=1000, n=2, m=2 rotation model", "c2": "k=1e5, n=m=6 random SPD noise",
         "c3": "k=1e5, n=6, m_i in {0,2,6}", "c4": "k=2e4, n=m=48",
         "c5": "k=2^22, n=6, m=3 constant-velocity 3-D model"}[cfg]
    return f"BASELINE.json config {cfg[1]} ({d}), N={N}"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.count(",") >= 8]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def roofline(launches, N, n, m, strides, p64_tf, cfg="c5"):
    """Dominant launch (largest total time in the timed region) vs its roofline."""
    from paper_2502_11686_b200 import model
    groups = {}
    for fam, lev, ms in launches:
        groups.setdefault((fam, lev), []).append(ms)
    (fam, lev), mss = max(groups.items(), key=lambda kv: sum(kv[1]))
    avg_s = sum(mss) / len(mss) / 1e3
    by, fl, units = model.launch_cost(fam, lev, N, n, m, strides)
    bw, bw_src = peaks()
    t_hbm, t_fp = by / (bw * 1e9), fl / (p64_tf * 1e12)
    total = sum(sum(v) for v in groups.values())
    share = sum(mss) / total
    if t_hbm >= t_fp:
        ach = by / avg_s / 1e9
        r = {"bound": "hbm", "achieved": ach, "peak": bw, "unit": "GB/s", "frac": ach / bw,
             "peak_source": bw_src}
    else:
        ach = fl / avg_s / 1e12
        r = {"bound": "alu", "achieved": ach, "peak": p64_tf, "unit": "TFLOP/s", "frac": ach / p64_tf,
             "peak_source": "measured fp64 DFMA peak (ks_peak_fp64_tflops, this run)"}
    traffic, tsrc, kname = None, None, f"{fam} launch L={lev}"
    try:   # DRAM bytes of this launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        rec = tj.get(cfg, {}).get(f"{fam} L={lev}")
        if rec:
            traffic, tsrc = rec["bytes"], f"profiles/traffic.json <- {rec['round']} ncu --set full ({rec['report']})"
            kname = f"{rec['kernel']} L={lev}"
    except Exception:
        pass
    r.update({"traffic": traffic, "traffic_source": tsrc, "kernel": kname,
              "launch_ms": avg_s * 1e3,
              "share_of_step": share, "algorithmic_bytes": by, "algorithmic_flops": fl,
              "units": units,
              "other_roof_frac": (fl / avg_s / 1e12 / p64_tf) if r["bound"] == "hbm"
              else (by / avg_s / 1e9 / bw)})
    return r


def run_reference(a, world, rank):
    if rank != 0:
        return 0
    import oracle
    from paper_2502_11686_b200 import generators as gen
    N = a.N or gen.CONFIGS[a.config]["N"]
    S = min(a.ref_sample, N)
    p = gen.make(a.config, N=S)
    oracle.build()
    for _ in range(a.warmup):
        oracle.smooth(p)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        oracle.smooth(p)
    dt = (time.perf_counter() - t0) / a.steps
    v = S / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "resources_used": {"gpus": 0, "host_cores": 1},
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(a.config, N), "parallelism": "1 host core"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {S} steps of the workload per step (plain-C "
                                       f"sequential Paige-Saunders + Alg. 1, oracle/)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def relaunch(a):
    """`--gpus N > 1` without a launcher: re-exec through torch.distributed.run
    with one rank per GPU (the driver's own launch line)."""
    import socket
    have = torch.cuda.device_count()
    if have < a.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {a.gpus} but only {have} CUDA device(s) visible",
                          "n_gpus": a.gpus}), flush=True)
        return 1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def timed_graph(run, stream, steps, warmup):
    """CUDA-graph capture of one step, then `steps` replays timed with CUDA
    events on the launching stream (ms per step)."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        run()
    for _ in range(max(warmup, 1)):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, g


def per_config(dev, stream, p64, steps=10):
    """c1-c4 at full size in the same run (parity cases; c5 is the headline):
    ms/step and steps/s with and without covariances (NC), and
    the step against its algorithmic roofline (model.step_totals)."""
    from paper_2502_11686_b200 import generators as gen
    from paper_2502_11686_b200 import ks, model
    bw = peaks()[0]
    out = {}
    for cfg in ("c1", "c2", "c3", "c4", "paper_n500"):
        # paper_n500: the paper's third size: k = 500
        # steps, n = m = 500, its benchmark class (fixed orthonormal F and G,
        # K = L = I, random o) -- the large-n path
        p = gen.paper_problem(500, 500, seed=0) if cfg == "paper_n500" else gen.make(cfg)
        strides = {"C": int(p.H.shape[0] > 1 or p.L.shape[0] > 1 or not bool((p.m == p.m_max).all())),
                   "E": int(p.F.shape[0] > 1 or p.K.shape[0] > 1 or p.c is not None)}
        res = {"N": p.N, "n": p.n, "m": p.m_max}
        for variant, cov in (("states+cov", True), ("states_nc", False)):
            sm = ks.Smoother(p, device=dev, stream=stream, cov=cov)
            for _ in range(3):
                sm.run(cov=cov)
            sm.check()
            l0 = sm.info()["launches"]
            sm.run(cov=cov)
            nl = sm.info()["launches"] - l0
            ms, g = timed_graph(lambda: sm.run(cov=cov), stream, steps if p.n <= 64 else 3, 3 if p.n <= 64 else 1)
            sm.check()
            sb, sf = model.step_totals(p.N, p.n, p.m_max, strides, cov=cov)
            t_h, t_f = sb / (bw * 1e9), sf / (p64 * 1e12)
            res[variant] = {"ms_per_step": ms, "steps_per_s": p.N / (ms / 1e3), "gpu_launches": nl,
                            "algorithmic_bytes": sb, "algorithmic_flops": sf,
                            "bound": "hbm" if t_h >= t_f else "fp64",
                            "roofline_frac": max(t_h, t_f) / (ms / 1e3),
                            "hbm_frac": t_h / (ms / 1e3), "fp64_frac": t_f / (ms / 1e3)}
            del g, sm
            torch.cuda.empty_cache()
        out[cfg] = res
    out["_note"] = ("CUDA-graph replay, inputs resident, 1 GPU; roofline_frac = max(bytes/HBM peak, "
                    "flops/FP64 peak) / step time with the level-synchronous algorithmic totals of "
                    "paper_2502_11686_b200/model.py (c3 counted at m = m_max, an upper bound)")
    return out


def main():
    a = parse()
    world, rank, local = dist_env()
    if a.impl == "reference":
        return run_reference(a, world, rank)
    if world == 1 and a.gpus > 1:
        return relaunch(a)
    if world != a.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {a.gpus}")
    from paper_2502_11686_b200 import generators as gen
    from paper_2502_11686_b200 import ks, model
    from paper_2502_11686_b200 import dist as kdist
    assert torch.cuda.is_available(), "bench needs a GPU (there is no CPU fallback)"
    host_x = world > 1 and a.exchange == "host"
    local = local % torch.cuda.device_count() if host_x else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    P = world
    nccl = None
    if P > 1:
        if host_x:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    p = gen.make(a.config, N=a.N)
    N = p.N
    # rank r owns steps [r*M, (r+1)*M), M a power of two (N not P x a power
    # of two: decoupled padding steps at the global end, R29)
    M, _ = kdist.shard_plan(N, P)
    lo = rank * M
    local_p = kdist.pad_shard(p, rank, P) if P > 1 else p
    strides = {"C": int(local_p.H.shape[0] > 1 or local_p.L.shape[0] > 1),
               "E": int(local_p.F.shape[0] > 1 or local_p.K.shape[0] > 1 or local_p.c is not None)}
    # every library call goes to one side stream (CUDA graphs cannot capture
    # the legacy default stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    p64 = ks.peak_fp64_tflops(stream)

    kd = None
    if host_x:   # no communicator: ks_factor stops after the local levels
        kd = ks.Dist(rank, P, lo, P * M)
    elif P > 1:
        # the library's own NCCL communicator (ks_dist_*): rank 0's unique id
        # travels over the torch process group; ks_factor then allgathers the
        # boundary columns itself, on the context's stream
        obj = [ks.Dist.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        kd = ks.Dist(rank, P, lo, P * M, uid=obj[0], device=dev)
        nccl = kd.info()
        v = torch.cuda.nccl.version()
        nccl["torch_nccl_version"] = ".".join(map(str, v)) if isinstance(v, (tuple, list)) else str(v)
        print(f"[rank {rank}] ks_dist: NCCL communicator with {nccl['nccl_nranks']} ranks", file=sys.stderr,
              flush=True)

    sm = ks.Smoother(local_p, device=dev, stream=stream, dist=kd)

    def step(s, get=None):
        s.whiten()
        s.factor()          # P > 1: local levels, NCCL boundary allgather, boundary system
        if host_x:          # validation mode: the boundary allgather through host memory (gloo)
            snd, rcv = s.boundary_tensors()
            sh = snd.cpu()
            rh = torch.empty(P * sh.numel(), dtype=torch.uint8)
            kdist.exchange_boundary(sh, rh)
            rcv.copy_(rh.to(dev))
            s.factor_boundary()
        s.solve_selinv()
        if get is not None:
            s.get(*get)

    for _ in range(max(a.warmup, 1)):
        step(sm)
    sm.check()
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()

    # (1) per-launch device times (library events around every launch): the
    # phase split and the roofline's dominant launch
    sm.set_timing(True)
    l0 = sm.info()["launches"]
    for _ in range(a.steps):
        step(sm)
    launches = sm.launch_times()
    n_launch = (sm.info()["launches"] - l0) // a.steps
    fam_ms = {}
    for fam, lev, t in launches:
        fam_ms[fam] = fam_ms.get(fam, 0.0) + t / a.steps
    sm.set_timing(False)
    sm.check()

    # (2) the headline: K steps as CUDA-graph replays (one graph = one step's
    # launches, the NCCL allgather included on N > 1), or eagerly with
    # --no-graph; CUDA events on the launching stream, max over ranks
    graph = None
    if not (a.no_graph or host_x):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step(sm)
        for _ in range(max(a.warmup, 1)):
            graph.replay()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else (lambda: step(sm))
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.steps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    # spread: the same K steps again, one event pair per step (not the headline)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    evs[0].record(stream)
    for k in range(a.steps):
        run()
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    per = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(a.steps))
    spread = {"min": per[0], "median": per[len(per) // 2], "max": per[-1]}
    eager_ms = None
    if graph is not None:   # the eager (launch-by-launch) mode beside the graph replay
        for _ in range(2):
            step(sm)
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(a.steps):
            step(sm)
        eb.record(stream)
        torch.cuda.synchronize()
        eager_ms = ea.elapsed_time(eb) / a.steps
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / a.steps
    if P > 1:
        ms = kdist.max_over_ranks(ms, None if host_x else dev)
    sm.check()
    value = N / (ms / 1e3)
    rl = roofline(launches, M, p.n, p.m_max, strides, p64, a.config if P == 1 and a.N is None else "")
    sb, sf = model.step_totals(M, p.n, p.m_max, strides)
    bw = peaks()[0]
    step_rl = {"algorithmic_bytes": sb, "algorithmic_flops": sf,
               "hbm_frac": sb / (ms / 1e3) / 1e9 / bw, "fp64_frac": sf / (ms / 1e3) / 1e12 / p64}

    e2e = None
    timing = "CUDA-graph replay of the whole step" if graph is not None else "eager launches"
    if not (a.no_e2e or a.quick):
        graph = None
        del sm
        torch.cuda.empty_cache()
        # End to end through the public API: pinned host inputs (KS_HOST_INPUTS:
        # ks_whiten copies them in), results copied to pinned host buffers.
        # One GPU: two contexts on two streams take alternate steps (a stream
        # of problems), so the device-to-host copy of one step (ks_get_async)
        # overlaps the next step's input copy and compute; the copies are
        # full-duplex PCIe DMA.  N > 1: one context per rank, sequential.
        nctx = 2 if P == 1 else 1
        streams = [stream] + [torch.cuda.Stream(dev) for _ in range(nctx - 1)]
        ctxs = [ks.Smoother(local_p, device=dev, stream=st, host_inputs=True, bind_outputs=False, dist=kd)
                for st in streams]
        h2d = sum(t.numel() * t.element_size() for t in ctxs[0].inputs.values() if t is not None)
        ke = max(2, min(a.steps, 6))
        pk = p.n * (p.n + 1) // 2

        def run_e2e(packed):
            # packed: ks_get_packed (S_ii symmetric: its upper triangle by
            # rows, n(n+1)/2 of the n^2 doubles, written straight into pinned
            # host memory); else ks_get_async of the full n x n blocks
            outs = [(torch.empty((M, p.n), dtype=torch.float64).pin_memory(),
                     torch.empty((M, pk) if packed else (M, p.n, p.n), dtype=torch.float64).pin_memory())
                    for _ in range(nctx)]
            d2h = outs[0][0].numel() * 8 + outs[0][1].numel() * 8

            def e2e_step(k):
                c = ctxs[k % nctx]
                with torch.cuda.stream(streams[k % nctx]):
                    c.whiten()
                    c.factor()
                    if host_x:
                        snd, rcv = c.boundary_tensors()
                        sh = snd.cpu()
                        rh = torch.empty(P * sh.numel(), dtype=torch.uint8)
                        kdist.exchange_boundary(sh, rh)
                        rcv.copy_(rh.to(dev))
                        c.factor_boundary()
                    c.solve_selinv()
                    if packed:
                        c.get_packed(*outs[k % nctx], sync=False)
                    else:
                        c.get(*outs[k % nctx], sync=False)

            for k in range(max(a.warmup, 1) * nctx):
                e2e_step(k)
            torch.cuda.synchronize()
            for c in ctxs:
                c.check()
            if P > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for st in streams[1:]:
                st.wait_event(e0)
            for k in range(ke):
                e2e_step(k)
            ends = []
            for st in streams:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(st)
                ends.append(ev)
            torch.cuda.synchronize()
            mse = max(e0.elapsed_time(ev) for ev in ends) / ke
            if P > 1:
                mse = kdist.max_over_ranks(mse, None if host_x else dev)
            return {"value": N / (mse / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d * P),
                    "d2h_bytes_per_step": int(d2h * P), "ms_per_step": mse, "steps": ke,
                    "path": "ks_create(KS_HOST_INPUTS) pinned host inputs -> whiten(H2D) .. solve_selinv -> " +
                            ("ks_get_packed(pinned host states, covariance upper triangles n(n+1)/2 per step)"
                             if packed else "ks_get_async(pinned host states, full n x n covariances)") +
                            (f"; {nctx} contexts on {nctx} streams take alternate steps (copies overlap the "
                             f"other context's work)" if nctx > 1 else "")}

        e2e = run_e2e(True)
        e2e["full_cov"] = run_e2e(False)
        del ctxs
        torch.cuda.empty_cache()

    cpu = None
    cfgs = None
    if rank == 0 and P == 1 and not (a.no_cpu_baseline or a.quick):
        import oracle
        S = min(a.cpu_sample, N)
        q = p.slice(0, S) if S < N else p
        oracle.build()
        # median of 3 passes (1 pass when a pass exceeds 10 s)
        dts = []
        for _ in range(3):
            t0 = time.perf_counter()
            oracle.smooth(q)
            dts.append(time.perf_counter() - t0)
            if dts[0] > 10.0:
                break
        dt = statistics.median(dts)
        cpu = {"value": S / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {S} of the {N} steps, median of {len(dts)} passes of the plain-C sequential "
                         f"Paige-Saunders + Alg. 1 oracle ({', '.join(f'{x:.2f}' for x in dts)} s, 1 thread)",
               "host_cpu": _cpu_model(), "nproc": os.cpu_count()}
    if rank == 0 and P == 1 and not (a.quick or a.no_per_config):
        cfgs = per_config(dev, stream, p64)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": P, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": f"synthetic: generators.make('{a.config}') (seeded, BASELINE.json recipe)",
                "config": {"workload": workload_desc(a.config, N), "N": N, "n": p.n, "m": p.m_max,
                           "parallelism": f"time-shard x{P} (NCCL allgather of the boundary columns)"
                           if P > 1 else "1 GPU",
                           "l2": "working set (~11 GB at c5) >> 126 MB L2; no flush",
                           **({"shard_steps": M, "padding_steps": P * M - N} if P > 1 else {})},
                "roofline": rl, "step_roofline": step_rl, "cpu_baseline": cpu, "e2e": e2e,
                "timing": timing, "ms_per_step_spread": spread, "eager_ms_per_step": eager_ms,
                "gpu_launches": int(n_launch), "clocks": clocks,
                "phases_ms": fam_ms, "fp64_peak_tflops": p64, "nccl": nccl,
                "exchange": ("host-staged gloo allgather, ranks sharing %d GPU(s): a validation run of "
                             "the multi-rank path, not a multi-GPU measurement" % torch.cuda.device_count())
                if host_x else ("library NCCL allgather" if P > 1 else None),
                "per_config": cfgs}
        print(json.dumps(line), flush=True)
    if P > 1:
        dist.barrier()
        del kd
        dist.destroy_process_group()
    return 0


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


if __name__ == "__main__":
    sys.exit(main())
