"""Benchmark: voxel-ADMM-iterations/s (fp64) of the outer iteration.

Default workload (N=1): SURVEY §8(d) config 2 inputs at the metric's 256^3 —
3D two-phase neo-Hookean laminate (Mooney-Rivlin, mu in {1, 0.05},
kappa = 9.8 mu, layers normal to x_1), fully strain-controlled
<F> = diag(0.95, 1, 1), F perturbed once by 1e-4 N(0,1) (seed 0),
RatioToDual(0.3) local policy, default SolverParams.  A step is one ADMM
outer iteration of solver.solve (local step, projection, multiplier ascent,
residuals, penalty update); the exit tolerances are set to 1e-300 so that
exactly W warm-up iterations (from init_state), then K timed ones, run.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--grid 256] [--workload mr|lce]
                  [--impl ours|reference]

Under torchrun (N > 1) the same n^3 grid is split into N slabs along axis
0, one per GPU (solve(..., comm=TorchComm)): the total work is
fixed, so every line says "scaling": "strong"; the timed region is
bracketed by a barrier + synchronize and the max over ranks is reported.
``--grid 512`` is SURVEY config 4 (512^3 over 1/2/4/8 GPUs); ``--workload lce``
is config 3 (add ``--grid 512`` / ``--grid 1024`` under torchrun for config 5).
``--impl reference`` times the CPU restatement of the reference (oracle/,
the "port") on the host cores over the same window.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_ALG_MR3 = 952.0  # algorithmic bytes per voxel-iteration, 3D MR
WORD = 8.0
# FP64 operations (FMA = 2) of one accepted Armijo sweep of the 3D MR descent
# (trial point, det, objective, cofactor gradient, |g|^2)
F_SWEEP_MR3 = 170.0


def fp64_peak_tflops():
    """FP64 (non-tensor) peak: the DFMA microbenchmark measured on this pool's
    B200s (profiles/fp64_peak.json, tools/microbench/fp64_peak.cu), else the
    nominal 148 SMs x 64 DFMA/clk x 2 x max SM clock.  Returns (TF/s, source)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["fp64_dfma_tflops"]), \
                "measured DFMA microbenchmark (profiles/fp64_peak.json)"
    except Exception:
        pass
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except Exception:
        pass
    return 148 * 64 * 2 * mhz * 1e6 / 1e12, "nominal 148 SM x 64 DFMA/clk x 2 x sm_max_mhz"


def laminate(n, dim=3):
    """Config-2 inputs: phase = (x_1 + L)/(2L) < 0.5, composite_moduli(1, 20, 9.8)."""
    L = 0.5
    h = 2 * L / n
    x = -L + h * np.arange(n)
    chi = ((x + L) / (2 * L) < 0.5).astype(float)
    chi = np.broadcast_to(chi.reshape((n,) + (1,) * (dim - 1)), (n,) * dim).ravel()
    mu = 1.0 + (1.0 / 20.0 - 1.0) * chi
    return mu, 9.8 * mu


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def wait_ready(self, timeout=3.0):
        """Block until nvidia-smi delivers its first sample (its start-up takes
        longer than a short timed region), then drop the pre-region samples."""
        t_end = time.perf_counter() + timeout
        while self.proc is not None and not self.rows and time.perf_counter() < t_end:
            time.sleep(0.005)
        self.rows = []

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def stage_bytes(n, dim=3, nl=None):
    """Minimal DRAM bytes per launch of each pipeline stage of OUR dataflow
    (each input read once, each output written once; stencil halos and
    padding not counted); nl = planes of this rank's slab."""
    M = (nl if nl is not None else n) * n ** (dim - 1)
    nh = n // 2 + 1
    D = dim * dim
    spec = dim * (M // n) * nh * 16.0  # d-component half spectrum
    w = WORD * M
    return {
        # standalone local chunk, grad_u implicit: read u, F, lam, mu, kappa; write F
        "local": (dim + 2 * D + 2 + D) * w,
        "row_fwd": D * w + spec,                         # read T = F - lam/rho; write spectrum
        "col_fwd": 2 * spec,
        "col_solve": 2 * spec,
        "col_inv": 2 * spec,
        "plane": 2 * spec,                               # B + C + D in one pass (L2-resident planes)
        "row_inv": spec + dim * w,                       # read spectrum, write u_tilde
        # residual pass: read u_new, u_old (or G_old), F
        "grad": (2 * dim + D) * w,
        # fused ascent + first chunk: read u, F, lam, mu, kappa; write lam, F, T
        "fused": (dim + 2 * D + 2 + 3 * D) * w,
    }


def perturbation(n, planes, dim=3):
    """1e-4 N(0,1) perturbation of F, seeded per axis-0 plane (plane i from
    default_rng([0, i])), so every rank of a slab split generates exactly
    its own planes of the same global field."""
    out = np.empty((len(planes),) + (n,) * (dim - 1) + (dim, dim))
    for k, i in enumerate(planes):
        out[k] = np.random.default_rng([0, int(i)]).standard_normal(out.shape[1:])
    out *= 1e-4
    return out


def setup_problem(mm, n, comm=None):
    """Config-2 inputs at n^3; with a communicator, this rank's slab."""
    dim = 3
    grid = mm.Grid(dim, n, 0.5)
    mu, kap = laminate(n, dim)
    planes = range(n)
    if comm is not None:
        from paper_2010_06697_b200.slab import local_planes, local_points
        pts = local_points(grid, comm)
        mu, kap = mu[pts].copy(), kap[pts].copy()
        sl = local_planes(grid, comm)
        planes = range(sl.start, sl.stop)
    model = mm.MooneyRivlin(mu, kap, dim=dim, mu_rep=1.0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    params = mm.SolverParams()
    st = mm.solver.init_state(grid, model, bc, params, comm=comm)
    st.F = st.F + perturbation(n, planes, dim)
    return grid, model, bc, params, st


def _stage_report(stage_ms, stage_launch, sb):
    per_stage = {}
    for s_name, ms in stage_ms.items():
        nl = stage_launch.get(s_name, 0)
        if nl and s_name in sb:
            avg = ms / nl
            per_stage[s_name] = {"ms_total": round(ms, 4), "launches": nl,
                                 "ms_per_launch": round(avg, 5),
                                 "GBps": round(sb[s_name] / (avg / 1e3) / 1e9, 1)}
    return per_stage


def run_ours(args, rank, world, dist):
    """The MR workload (SURVEY 8(d) config 2 inputs) at n^3 on N GPUs: N = 1
    one context; N > 1 the same n^3 problem split into N slabs along axis 0
    (solve(..., comm=TorchComm): NCCL on the library stream, transposes as
    NVLink peer stores) -- total work fixed, so "strong" scaling at every N."""
    import torch

    import paper_2010_06697_b200 as mm

    dev = bench_device()
    torch.cuda.set_device(dev)
    n = args.n
    M = n ** 3
    comm = None
    exchange = None
    if world > 1:
        from paper_2010_06697_b200.slab import TorchComm
        exchange = args.exchange
        comm = TorchComm(dist, dev, exchange=exchange)
    grid, model, bc, _, st = setup_problem(mm, n, comm)
    pol = mm.RatioToDual(0.3)
    # default SolverParams except the stopping tolerances, so that exactly the
    # requested number of outer iterations runs (they only gate the exit test)
    params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=args.warmup)
    mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False, comm=comm)
    eng = st._engine
    ctx = eng.ctx
    # the CPU baseline continues from this state (iterations W+1, W+2: the
    # first iterations of the GPU's timed window); grad_u is implicit on the
    # device (u_mean + D u_tilde), so the host rebuilds it instead of reading it
    cpu_start = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_start = dict(F=np.array(st.F), lam=np.array(st.lam), u_tilde=np.array(st.u_tilde),
                         u_mean=np.array(st.u_mean), rho=st.rho, r_d_prev=st.r_d_prev,
                         outer_iter=st.outer_iter)
    # device-resident timed loop: results stay in HBM (no write-back of F and
    # lam into the arrays setup_problem handed in; that D2H is part of e2e)
    st.detach_caller_arrays()
    ctx.synchronize()
    ctx.profile_enable(False)
    ctx.profile_read(reset=True)  # launch counts are kept with profiling off
    sampler = ClockSampler(dev)
    sampler.start()
    sampler.wait_ready()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    # the library runs on its own stream; bracket it from the torch stream with
    # full synchronisation on both sides (solve() ends in a host sync)
    t0.record()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    it0 = st.outer_iter
    ps0 = eng.point_sweeps
    params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=args.steps)
    mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False, comm=comm)
    hist = st.history[-args.steps:]
    assert st.outer_iter - it0 == args.steps
    ctx.synchronize()
    w1 = time.perf_counter()
    t1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_total = max(t0.elapsed_time(t1), (w1 - w0) * 1e3)
    _, launches_timed = ctx.profile_read(reset=True)
    if dist is not None:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    sweeps = st.total_sweeps
    point_sweeps = eng.point_sweeps - ps0

    # ---- per-stage device times: a SEPARATE profiled pass (the next K
    # iterations of the same trajectory, CUDA events around every stage on
    # the library's stream), so the timed region above carries no event
    # instrumentation
    ctx.profile_enable(True)
    ps1 = eng.point_sweeps
    mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False, comm=comm)
    ctx.synchronize()
    ctx.profile_enable(False)
    stage_ms, stage_launch = ctx.profile_read(reset=True)
    prof_point_sweeps = eng.point_sweeps - ps1

    # ---- e2e through the public API with host buffers: solve() on a host
    # state (fresh engine: H2D of F, grad_u, lam, moduli), K iterations, then
    # read F, grad_u, lam, u_tilde back to the host.
    host = dict(F=st.F.copy(), grad_u=st.grad_u.copy(), lam=st.lam.copy(),
                u_tilde=st.u_tilde.copy(), u_mean=st.u_mean.copy())
    pinned = {}
    for k in ("F", "grad_u", "lam"):
        t = torch.empty(host[k].shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = host[k]
        pinned[k] = t
    rho, r_d_prev, oi = st.rho, st.r_d_prev, st.outer_iter
    m_loc = eng.npts
    del st, eng, ctx
    import gc
    gc.collect()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0 = time.perf_counter()
    hs = mm.ADMMState(u_mean=host["u_mean"], u_tilde=host["u_tilde"],
                      grad_u=pinned["grad_u"].numpy(), F=pinned["F"].numpy(),
                      lam=pinned["lam"].numpy(), internal={}, rho=rho, outer_iter=oi,
                      r_d_prev=r_d_prev)
    p_e2e = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=args.steps)
    hs, _ = mm.solve(grid, model, bc, p_e2e, policy=pol, state=hs, raise_on_max=False, comm=comm)
    outs = [hs.F, hs.grad_u, hs.lam, hs.u_tilde]
    hs._engine.ctx.synchronize()
    e1 = time.perf_counter()
    e2e_ms = (e1 - e0) * 1e3
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = sum(pinned[k].numel() * 8 for k in pinned) + host["u_tilde"].nbytes + 2 * m_loc * 8
    d2h = sum(o.nbytes for o in outs)

    value = M * args.steps / (ms_total / 1e3)
    e2e_value = M * args.steps / (e2e_ms / 1e3)
    peak, peak_kind = measured_peak()
    per_stage = _stage_report(stage_ms, stage_launch, stage_bytes(n, nl=m_loc // (n * n)))
    dom = max(per_stage, key=lambda k: per_stage[k]["ms_total"]) if per_stage else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(dom) if world == 1 else None
    except Exception:
        pass
    roof = None
    if dom:
        ach = per_stage[dom]["GBps"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs"
                if peak_kind == "measured" else "fallback B200_PROFILING.md",
                "timing": "average launch duration from CUDA events on the library stream in "
                          "the profiled pass (iterations after the timed window)"
                          + ("; rank 0" if world > 1 else "")}
    it_ms = ms_total / args.steps
    # aggregate HBM bandwidth of the N GPUs against N x the per-GPU peak
    roof_it = {"bound": "hbm", "B_alg_per_voxel": B_ALG_MR3,
               "achieved": round(B_ALG_MR3 * M / (it_ms / 1e3) / 1e9, 1), "peak": peak * world,
               "unit": "GB/s",
               "frac": round(B_ALG_MR3 * M / (it_ms / 1e3) / 1e9 / (peak * world), 4)}
    local_ms = sum(stage_ms.get(k, 0.0) for k in ("local", "fused"))
    local_fp64 = None
    if local_ms > 0 and prof_point_sweeps > 0:
        tf = prof_point_sweeps * F_SWEEP_MR3 / (local_ms / 1e3) / 1e12
        pk, pk_src = fp64_peak_tflops()
        local_fp64 = {"bound": "fp64", "stages": ["local", "fused"],
                      "point_sweeps_per_voxel_iter": round(point_sweeps / (m_loc * args.steps), 3),
                      "flop_per_sweep": F_SWEEP_MR3, "achieved": round(tf, 2), "peak": round(pk, 1),
                      "unit": "TFLOP/s", "frac": round(tf / pk, 4),
                      "peak_source": pk_src}
    par = "single GPU" if world == 1 else f"slab x{world} ({exchange} transposes)"
    line = {
        "metric": "voxel-ADMM-iterations/sec (fp64)",
        "value": value,
        "unit": "voxel-iter/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": it_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (config-2 laminate inputs, seeded per plane)",
        "config": {"workload": f"3D neo-Hookean laminate {n}^3 (SURVEY 8(d) config 2 inputs at "
                               f"the metric's {n}^3), the whole grid on {world} GPU(s)",
                   "grid": n, "material": "MooneyRivlin mu in {1, 0.05}, kappa = 9.8 mu",
                   "bc": "strain diag(0.95,1,1)", "policy": "RatioToDual(0.3)",
                   "steps_are": f"outer iterations {args.warmup + 1}..{args.warmup + args.steps}"
                                f" from init_state",
                   "l2": f"inputs larger than L2 (state {32 * 8 * M / world / 1e9:.2f} GB per GPU)",
                   "parallelism": par},
        "local_sweeps_total": int(sweeps),
        "residuals_last": {"r_p": hist[-1].r_p, "r_d": hist[-1].r_d, "r_l": hist[-1].r_l,
                           "rho": hist[-1].rho},
        "stages": per_stage,
        "stages_pass": f"profiled pass, outer iterations {args.warmup + args.steps + 1}.."
                       f"{args.warmup + 2 * args.steps} (not the timed region)"
                       + ("; rank 0's slab" if world > 1 else ""),
        "roofline": roof,
        "roofline_iteration": roof_it,
        "roofline_local_fp64": local_fp64,
        "gpu_launches": int(sum(launches_timed.values())),
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "voxel-iter/s", "h2d_bytes_per_step": h2d / args.steps,
                "d2h_bytes_per_step": d2h / args.steps,
                "how": "solve(max_outer=K) on a host (pinned) state: engine creation (device "
                       "memory from the process's stream-ordered pool, warm after the timed "
                       "run), H2D of F, grad_u, lam, u_tilde, moduli, K iterations, D2H of F "
                       "and lam back into the caller's (pinned) arrays, as the reference "
                       "updates both in place, and of grad_u, u_tilde into fresh host arrays; "
                       "wall clock" + ("; per rank, its slab; max over ranks" if world > 1
                                       else "")},
    }
    if cpu_start is not None:
        line["cpu_baseline"] = cpu_baseline(n, args.cpu_steps, cpu_start)
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_lce(args, rank, world, dist):
    """polydomain LCE, generate_polydomain_n0(grid, 0.25,
    seed=1), LiquidCrystalElastomer(mu=1, r=2, alpha=0.1, frank_kappa=1e-4),
    MacroBC.stress(0), max_local = 2000, RatioToDual(0.3).  A step is one outer
    iteration; the local Newton step is FP64-bound (the HBM
    fraction is not meaningful here), so the line reports FP64 work as
    voxel-sweeps/s beside the metric."""
    import torch

    import paper_2010_06697_b200 as mm

    dev = bench_device()
    torch.cuda.set_device(dev)
    n = args.n
    M = n ** 3
    grid = mm.Grid(3, n, 0.5)
    n0 = mm.generate_polydomain_n0(grid, 0.25, seed=1)
    kw = dict(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, dim=3)
    model = mm.LiquidCrystalElastomer(n0=n0, **kw)
    bc = mm.MacroBC.stress(np.zeros((3, 3)))
    pol = mm.RatioToDual(0.3)
    p_w = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=args.warmup)
    st, _ = mm.solve(grid, model, bc, p_w, policy=pol, raise_on_max=False)
    eng = st._engine
    ctx = eng.ctx
    st.detach_caller_arrays()
    ctx.synchronize()
    ctx.profile_enable(False)
    ctx.profile_read(reset=True)
    sampler = ClockSampler(dev)
    sampler.start()
    sampler.wait_ready()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ps0 = eng.point_sweeps
    sw0 = st.total_sweeps
    p_k = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=args.steps)
    mm.solve(grid, model, bc, p_k, policy=pol, state=st, raise_on_max=False)
    ctx.synchronize()
    w1 = time.perf_counter()
    t1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_total = max(t0.elapsed_time(t1), (w1 - w0) * 1e3)
    _, launches = ctx.profile_read(reset=True)
    point_sweeps = eng.point_sweeps - ps0
    value = M * args.steps / (ms_total / 1e3)
    line = {
        "metric": "voxel-ADMM-iterations/sec (fp64)", "value": value, "unit": "voxel-iter/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-3 polydomain director, seed 1)",
        "config": {"workload": f"3D polydomain liquid-crystal elastomer {n}^3 (SURVEY 8(d) "
                               "config 3)", "grid": n,
                   "material": "LCE mu=1 r=2 alpha=0.1 frank_kappa=1e-4, polydomain n0 "
                               "(correlation 0.25, seed 1)",
                   "bc": "stress 0", "policy": "RatioToDual(0.3), max_local 2000",
                   "steps_are": f"outer iterations {args.warmup + 1}..{args.warmup + args.steps}",
                   "l2": "inputs larger than L2"},
        "local_sweeps_total": int(st.total_sweeps - sw0),
        "point_sweeps_per_voxel_iter": round(point_sweeps / (M * args.steps), 1),
        "voxel_sweeps_per_s": point_sweeps / (ms_total / 1e3),
        "gpu_launches": int(sum(launches.values())),
        "clocks": clocks,
        "e2e": {"value": None, "unit": "voxel-iter/s", "h2d_bytes_per_step": None,
                "d2h_bytes_per_step": None,
                "how": "not measured for the LCE workload (device time dominates: seconds per "
                       "iteration against ~10 GB of state)"},
    }
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        cores = len(os.sched_getaffinity(0))
        oracle.set_threads(cores)
        oracle.set_fft("scipy", cores)
        cn = 24
        on0 = oracle.polydomain_n0(3, cn, 0.5, 0.25, seed=1)
        om = oracle.LCE(n0=on0, **kw)
        op = oracle.Params()
        ost = oracle.init_state(3, cn, om, np.zeros((3, 3), bool), np.zeros((3, 3)), op)
        z = (np.zeros((3, 3), bool), np.zeros((3, 3)))
        # iteration 1 runs at the RatioToDual start tolerance (1.0); the timed
        # iterations 2..3 are in the capped-Newton regime of the GPU's window
        oracle.outer_iteration(3, cn, 0.5, om, ost, op, *z, oracle.RatioToDual(0.3))
        t0c = time.perf_counter()
        for _ in range(2):
            oracle.outer_iteration(3, cn, 0.5, om, ost, op, *z, oracle.RatioToDual(0.3))
        dtc = time.perf_counter() - t0c
        line["cpu_baseline"] = {
            "value": 2 * cn ** 3 / dtc, "unit": "voxel-iter/s", "cores": cores, "kind": "port",
            "sample": f"oracle port (C LCE Newton kernels on {cores} threads), the same material "
                      f"on a {cn}^3 polydomain grid, outer iterations 2..3, {dtc:.1f} s (the "
                      f"full {n}^3 iteration is ~45 min of CPU time, SURVEY 8(d))"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_device():
    """CUDA device of this rank: LOCAL_RANK, or MM_BENCH_DEVICE when set."""
    return int(os.environ.get("MM_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def _oracle_setup(n):
    import oracle

    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    # the reference's transforms: scipy.fft with workers = the host cores
    # (grid.py:213-220 with set_workers(available_cores()))
    oracle.set_fft("scipy", cores)
    mu, kap = laminate(n, 3)
    om = oracle.MR(mu, kap, dim=3, mu_rep=1.0)
    mask = np.ones((3, 3), bool)
    val = np.diag([0.95, 1.0, 1.0])
    return oracle, cores, om, mask, val


def cpu_baseline(n, steps, start):
    """Oracle port on the host cores, bounded sample of the same workload:
    outer iterations W+1 .. W+steps of the same trajectory, continued from the
    GPU's state after its W warm-up iterations (the first iterations of the
    GPU's timed window), so the sample needs no CPU warm-up."""
    oracle, cores, om, mask, val = _oracle_setup(n)
    params = oracle.Params()
    st = oracle.init_state(3, n, om, mask, val, params)
    st.F = np.array(start["F"])
    st.lam = np.array(start["lam"])
    st.u_tilde = np.array(start["u_tilde"])
    st.u_mean = np.array(start["u_mean"])
    st.grad_u = oracle.core.stencil_grad(3, n, 0.5, st.u_tilde) + st.u_mean
    st.rho, st.r_d_prev, st.outer_iter = start["rho"], start["r_d_prev"], start["outer_iter"]
    sym = oracle.symbols(3, n, 0.5)
    pol = oracle.RatioToDual(0.3)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.outer_iteration(3, n, 0.5, om, st, params, mask, val, pol, sym=sym)
    dt = time.perf_counter() - t0
    i0 = start["outer_iter"]
    return {"value": n ** 3 * steps / dt, "unit": "voxel-iter/s", "cores": cores, "kind": "port",
            "sample": f"oracle port (C local kernels on {cores} threads + scipy.fft with "
                      f"{cores} workers, numpy einsum), same laminate at {n}^3, outer "
                      f"iterations {i0 + 1}..{i0 + steps} (the first {steps} of the GPU's "
                      f"timed window, continued from its warm-up state), {dt:.1f} s"}


def run_reference(args, rank):
    if rank != 0:
        return
    n = args.n
    oracle, cores, om, mask, val = _oracle_setup(n)
    params = oracle.Params()
    st = oracle.init_state(3, n, om, mask, val, params)
    st.F = st.F + perturbation(n, range(n))
    sym = oracle.symbols(3, n, 0.5)
    pol = oracle.RatioToDual(0.3)
    for _ in range(args.warmup):
        oracle.outer_iteration(3, n, 0.5, om, st, params, mask, val, pol, sym=sym)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.outer_iteration(3, n, 0.5, om, st, params, mask, val, pol, sym=sym)
    dt = time.perf_counter() - t0
    v = n ** 3 * args.steps / dt
    sample = (f"oracle port (C local kernels on {cores} threads + scipy.fft with {cores} workers, "
              f"numpy einsum) of the same laminate workload at {n}^3, outer iterations "
              f"{args.warmup + 1}..{args.warmup + args.steps} (the GPU arm's timed window)")
    print(json.dumps({
        "impl": "reference", "metric": "voxel-ADMM-iterations/sec (fp64)", "value": v,
        "unit": "voxel-iter/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-2 laminate inputs, seeded per plane)",
        "config": {"workload": f"3D neo-Hookean laminate {n}^3 (SURVEY 8(d) config 2 inputs at "
                               f"the metric's {n}^3), same as the GPU arm", "grid": n,
                   "same_config": True,
                   "steps_are": f"outer iterations {args.warmup + 1}..{args.warmup + args.steps}"
                                f" from init_state"},
        "cpu_baseline": {"value": v, "unit": "voxel-iter/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "voxel-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--grid", dest="n", type=int, default=256,
                    help="n of the n^3 grid (not --n: torchrun would claim it)")
    ap.add_argument("--workload", default="mr", choices=["mr", "lce"],
                    help="mr: SURVEY 8(d) config 2 inputs (headline); lce: config 3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="push", choices=["push", "collective"],
                    help="N>1 slab transposes: peer stores fused into the FFT kernels, or "
                         "NCCL all-to-all")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else max(args.warmup, 1)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        backend = "nccl" if args.impl == "ours" else "gloo"
        # MM_BENCH_BACKEND / MM_BENCH_DEVICE: exercise the N > 1 path with all
        # ranks on one GPU (gloo; NCCL refuses two ranks per device)
        backend = os.environ.get("MM_BENCH_BACKEND", backend)
        if args.impl == "ours":
            torch.cuda.set_device(bench_device())
        tdist.init_process_group(backend=backend)
        dist = tdist
    try:
        if args.impl == "reference":
            run_reference(args, rank)
        else:
            if args.workload == "lce":
                run_lce(args, rank, world, dist)
            else:
                run_ours(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
