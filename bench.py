"""bench.py — B200 benchmark of the matrix-free Stokes hot path (arXiv:1604.07994).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg3] [--n N] [--form mod] [--krylov M]

One JSON line (rank 0).  A *step* is one pass of the whole hot path
over the workload: assemble (coarse coefficients, classification, constant and
explicit stencils, coarse inverse) -> load vector -> one operator apply ->
solve of K x = b to relative residual 1e-8 from x = 0 (GMRES(M) right-
preconditioned by one V_var(3,3) cycle for the unresolved inclusions of cfg3-cfg5,
DESIGN R23; plain V-cycles for cfg1/cfg2).

* Default workload: BASELINE.json configs[2] (cfg3, n = 256, 67.9 M DoF): the
  metric's configs quote no size, so the largest config that BASELINE.json puts on
  one GPU is the N = 1 workload (cfg4 / cfg5 are specified on 8 GPUs).
* metric / unit: BASELINE.json's metric; `value` = device-timed seconds per step
  per DoF (DoF = 4 (n+1)^3), inputs resident in HBM, L2 flushed between
  steps; lower is better.  `apply` reports the operator-apply GDoF/s and HBM GB/s
  (separate loop, L2 flushed before every apply; 65 algorithmic B per vertex,
  SURVEY §8(d)).
* e2e: the same step through the public API from pinned host buffers: element
  classes and forcing copied in, and the solution (4 fields, canonical layout)
  copied back out, every step.
* roofline: the kernel with the largest summed device time in the step (CUDA
  events around every launch on the solver stream) against the measured HBM copy
  bandwidth in MEASURED_PEAKS.json, with SURVEY §8(d)'s algorithmic bytes per
  vertex (apply 65; a velocity colour pass 40 = half of the 80 B two-colour
  sweep; pressure passes 48 / 24; residual 97).
* cpu_baseline: the oracle (oracle/, test infrastructure) timed on this host: its
  C element-loop apply on the full grid (all threads) and on a slab with one
  thread; the solve extrapolated by the oracle multigrid's cost in operator
  applications (its Uzawa step does 9 element-loop products) times the measured
  GMRES iteration / V-cycle count -- labelled "extrapolated".  `--impl reference`
  times the same oracle apply as the reference arm.
* --gpus N > 1 (torchrun) shards the grid in z-slabs over N ranks (NCCL halo
  exchange and allreduce; total work fixed: "strong" scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Stokes operator apply GDoF/s and HBM GB/s vs peak; MG solve s/DoF at 1/2/4/8 GPUs"
RTOL = 1e-8
CFG_INDEX = {"cfg1": 0, "cfg2": 1, "cfg3": 2, "cfg4": 3, "cfg5": 4, "cols": None}
# algorithmic bytes per owned vertex of each profiled op
OP_BYTES = {"apply": 65, "residual": 97, "vel_pass": 40, "p_pass1": 48, "p_pass2": 24, "fwd_sweep": 80}
# iterations our solver needs at rtol 1e-8 (profiles/r02_convergence_probe_gmres.log), for the
# reference arm's extrapolation of the oracle solve (the oracle cannot run it in minutes)
REF_ITS = {"cfg1": 11, "cfg2": 13, "cfg3": 31, "cfg4": 100, "cfg5": 59, "cols": 13}
DEFAULT_KRYLOV = {"cfg1": 0, "cfg2": 0, "cfg3": 12, "cfg4": 100, "cfg5": 30, "cols": 0}
# cfg3: measured best (profiles/r02_bench_cfg3_krylov*.json); cfg5: 30 (12 doubles the iterations);
# cfg4: the plain V-cycle diverges (rho ~ 7 at n = 256) and GMRES(30) stagnates at 5e-4 --
# GMRES(100) converges in 100 iterations (profiles/r02_cfg4_n256_probe.log)


def workload_name(name):
    i = CFG_INDEX[name]
    return (f"{name} (BASELINE configs[{i}])" if i is not None else
            f"{name} (SURVEY NEXT-1: the paper's viscosity columns, free slip, P:772-774 / P:1307)")


def oracle_applies_per_cycle(n, n_coarse=4, nu=3, nu_inc=2):
    """Cost of one V_var cycle of the oracle multigrid in full-grid element-loop
    products: its Uzawa step does 9 (f - B^T p, 4 colour passes of A u, B u, C p, two
    C sweeps), plus one residual per level; level l costs (n_l / n)^3."""
    tot, m, l = 0.0, n, 0
    while m > n_coarse:
        tot += (2 * (nu + nu_inc * l) * 9 + 1) * (m / n) ** 3
        m //= 2
        l += 1
    return tot


FORM_IDX = {"mod": 0, "sym": 1, "grad": 2}
OP_IDX = {"apply": 0, "residual": 1, "vel_pass": 2, "p_pass1": 3, "p_pass2": 4}


def ncu_traffic(kname):
    """DRAM bytes per launch of kernel `kname` from the committed ncu summary, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            mb = json.load(f)["dram_MB_per_launch"].get(kname)
        return None if mb is None else int(mb * 1e6)
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    # one sampler process for the whole run, started before the warm-up (its NVML start-up
    # stalled the first timed step by some 100 ms on some boxes when started right before
    # it); only the samples stamped inside the timed region are kept
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,timestamp")

    def __init__(self, dev):
        self.dev = dev
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.t0 = None

    def mark(self):
        """The timed region starts now."""
        import datetime
        self.t0 = datetime.datetime.now()

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if self.t0 is not None:
            import datetime
            inside = []
            for r in rows:
                try:
                    if datetime.datetime.strptime(r[9], "%Y/%m/%d %H:%M:%S.%f") >= self.t0:
                        inside.append(r)
                except (ValueError, IndexError):
                    inside.append(r)
            rows = inside or rows
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in rows for q in range(4) if r[5 + q].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend)
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def slab_inputs(cfg, ctx):
    """This rank's element classes, forcing, apply input (host numpy)."""
    cz0, cz1 = ctx.cube_range()
    lay = ctx.layout(0)
    N1 = cfg.n + 1
    v0, v1 = lay.z0 * N1 * N1, (lay.z0 + lay.nz_local) * N1 * N1
    cls, fcls = synth.element_classes(cfg, cz0, cz1)
    f = synth.nodal_forcing(cfg, v0, v1) if cfg.forcing == "nodal" else None
    x = synth.apply_input(cfg, v0, v1)
    return cls, fcls, f, x


# ------------------------------------------------------------------------------
# the oracle on the host (reference arm and cpu_baseline): bounded samples
# ------------------------------------------------------------------------------
def _omp_threads(n):
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


def oracle_apply_sample(cfg, form, reps=1, log=None, slab_planes=8):
    """Time the oracle's C element-loop apply (oracle/c/oracle.c) on the full grid with
    all host threads (median of `reps`) and on a slab of `slab_planes` vertex planes
    with one thread.  Returns dict(t_all, threads, gdof_all, gdof_one, t_inputs)."""
    from oracle import capi
    t0 = time.time()
    cls, _ = synth.element_classes(cfg)
    x = synth.apply_input(cfg)
    t_in = time.time() - t0
    capi.lib()
    nthr = os.cpu_count() or 1
    _omp_threads(nthr)
    threads = capi.num_threads()
    ts = []
    for r in range(reps):
        t1 = time.time()
        capi.apply_slab(cfg.n, form, 1.0 / 12.0, cfg.faces, cls, cfg.class_mu, x)
        ts.append(time.time() - t1)
        if log:
            log(f"oracle apply {r}: {ts[-1]:.2f} s ({threads} threads)")
    t_all = float(np.median(ts))
    kv = min(slab_planes, cfg.n + 1)
    _omp_threads(1)
    t1 = time.time()
    capi.apply_slab(cfg.n, form, 1.0 / 12.0, cfg.faces, cls, cfg.class_mu, x, kv0=0, kv1=kv)
    t_one = time.time() - t1
    _omp_threads(nthr)
    dofs_slab = 4 * (cfg.n + 1) ** 2 * kv
    return {"t_all": t_all, "threads": threads, "gdof_all": cfg.dofs / t_all / 1e9,
            "gdof_one": dofs_slab / t_one / 1e9, "t_one_slab": t_one, "slab_planes": kv, "t_inputs": t_in,
            "samples": ts}


def oracle_solve_measured(name="cfg1", n=16):
    """A full oracle solve, timed: the assembled-matrix oracle multigrid (oracle/mg.py,
    scipy, one host thread for the products) on `name` at n to rtol 1e-8 from x = 0 --
    the size the oracle finishes in seconds (SURVEY 8(d) "oracle beside it")."""
    from oracle import fem, mg
    cfg = synth.get_config(name, n=n)
    cls, fcls = synth.element_classes(cfg)
    t0 = time.time()
    H = mg.Hierarchy(n, cls, cfg.class_mu, cfg.faces, "mod")
    pr = H.levels[0].prob
    b = (pr.load_nodal(synth.nodal_forcing(cfg)) if cfg.forcing == "nodal"
         else pr.load_element(fem.element_force(n, fcls, cfg.force_table)))
    t1 = time.time()
    _, hist = H.solve(b, rtol=RTOL, max_cycles=200)
    t2 = time.time()
    return {"workload": f"{name} n={n}", "dofs": cfg.dofs, "cycles": len(hist) - 1,
            "setup_s": round(t1 - t0, 3), "solve_s": round(t2 - t1, 3),
            "s_per_dof": (t2 - t1) / cfg.dofs, "rel_res": hist[-1]}


def oracle_solve_extrapolated(cfg, t_apply, its, krylov):
    """s/DoF of the oracle multigrid solve: `its` V_var cycles (plus one apply per
    GMRES iteration and the residuals) at the measured time per full-grid apply."""
    per = oracle_applies_per_cycle(cfg.n)
    applies = its * (per + (1 if krylov else 1)) + 2
    return t_apply * applies / cfg.dofs, applies


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return 0
    log = lambda s_: print(s_, file=sys.stderr, flush=True)
    kry = args.krylov if args.krylov is not None else DEFAULT_KRYLOV[cfg.name]
    smp = oracle_apply_sample(cfg, args.form, reps=args.warmup + args.steps, log=log)
    tt = smp["samples"][args.warmup:] or smp["samples"]
    t_apply = float(np.median(tt))
    its = REF_ITS.get(cfg.name, 30)
    value, applies = oracle_solve_extrapolated(cfg, t_apply, its, kry)
    sample = (f"per step one oracle apply (plain C element loop, {smp['threads']} host threads) on the full "
              f"{cfg.name} n={cfg.n} grid ({t_apply:.2f} s); the solve is extrapolated as {applies:.0f} "
              f"full-grid element-loop products = {its} preconditioner cycles of the oracle multigrid "
              f"({oracle_applies_per_cycle(cfg.n):.1f} products per V_var(3,3) cycle) -- the iteration count "
              f"our solver measured at this config")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/DoF", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * cfg.dofs * 1e3,
            "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_name(cfg.name), "n": cfg.n,
                       "dofs": cfg.dofs, "form": args.form, "rtol": RTOL},
            "cpu_baseline": {"value": value, "unit": "s/DoF", "cores": smp["threads"], "kind": "oracle",
                             "sample": sample, "apply_gdof_s_all_threads": round(smp["gdof_all"], 4),
                             "apply_gdof_s_one_thread": round(smp["gdof_one"], 5),
                             "oracle_solve_measured": oracle_solve_measured()},
            "e2e": {"value": value, "unit": "s/DoF", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "extrapolated": True}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------
def run_ours(args, cfg, world, rank, local):
    import torch
    import paper_1604_07994_b200 as stk

    log = (lambda s: print(s, file=sys.stderr, flush=True)) if rank == 0 else (lambda s: None)
    nid = None
    if world > 1:
        import torch.distributed as dist
        obj = [stk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    stream = torch.cuda.current_stream()
    kry = args.krylov if args.krylov is not None else DEFAULT_KRYLOV[cfg.name]
    ctx = stk.StokesContext(cfg.n, args.form, cfg.faces, krylov=kry,
                            ncolors_u=4 if args.form == "sym" else 2, rank=rank, nranks=world,
                            stream=stream, nccl_id=nid)
    t0 = time.time()
    cls, fcls, f, xin = slab_inputs(cfg, ctx)
    log(f"inputs {time.time() - t0:.1f}s")
    lay = ctx.layout(0)
    V_own = lay.n_vertices
    dofs = cfg.dofs
    # device-resident inputs
    cls_pin = torch.from_numpy(cls).pin_memory()
    f4 = np.zeros((4, V_own))
    if f is not None:
        f4[:3] = f
    f_pin = torch.from_numpy(f4).pin_memory()
    fcls_pin = torch.from_numpy(fcls).pin_memory()
    ctx.set_viscosity(cls, cfg.class_mu)
    ctx.assemble()
    fvec = ctx.import_(f_pin.cuda(), mask=False)
    x_apply = ctx.import_(torch.from_numpy(xin).cuda())
    fcls_dev = fcls_pin.cuda()
    y = ctx.new_vector()
    b = ctx.new_vector()
    x = ctx.new_vector()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tab = np.ascontiguousarray(cfg.force_table, dtype=np.float64).reshape(-1)

    def load_rhs():
        if cfg.forcing == "nodal":
            st = stk.stk_load_vector(ctx.h, 0, fvec.data_ptr(), None, 0, b.data_ptr())
        else:
            st = stk.stk_load_vector(ctx.h, 1, fcls_dev.data_ptr(), tab.ctypes.data, len(tab) // 3,
                                     b.data_ptr())
        assert st == 0, stk.stk_last_error(ctx.h)

    def step():
        ctx.assemble()
        load_rhs()
        ctx.apply(x_apply, y)
        x.zero_()
        _, rep = ctx.solve(b, x, rtol=RTOL, max_cycles=args.max_cycles)
        return rep

    # warm-up (the clock sampler starts here, its samples count from the timed region on)
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        flush.zero_()
        rep = step()
    torch.cuda.synchronize()
    log(f"warm-up done: cycles {rep.cycles} rho {rep.rho:.3f} rel {rep.rel_res:.2e}")

    # timed steps (device time, CUDA events on the solver stream), library profiling off
    l0 = ctx.launch_count()
    ev = []
    reps = []
    clocks.mark()
    for _ in range(args.steps):
        flush.zero_()                       # L2 flushed between steps (outside the events)
        barrier(world)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps.append(step())
        e1.record(stream)
        torch.cuda.synchronize()
        ev.append((e0, e1))
    clk = clocks.stop()
    launches = ctx.launch_count() - l0
    step_ms = [a.elapsed_time(b_) for a, b_ in ev]
    ms = max_over_ranks(float(np.mean(step_ms)), world)
    # one more step, untimed, with profile mode 1: every level-0 launch bracketed by CUDA
    # events on the solver stream (the coarse levels run as one CUDA graph, timed as a
    # whole) -- the per-op split and the dominant kernel's launch time.  (Kept out of the
    # timed steps: creating and recording the events costs host time that the solver's
    # per-iteration synchronisation puts on the critical path.)
    ctx.profile(1)
    ctx.profile_reset()
    flush.zero_()
    torch.cuda.synchronize()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof_step_ms = p0.elapsed_time(p1)
    prof = {op: ctx.profile_read(op, -1) for op in ctx.PROFILE_OPS}
    dom = max((o for o in prof if o in OP_BYTES), key=lambda o: prof[o][1])  # a single kernel
    ctx.profile(False)
    peak, peak_kind = measured_peaks()
    roof = None
    if dom in OP_BYTES:
        n0, ms0 = ctx.profile_read(dom, 0)
        if n0 > 0:
            bytes_launch = OP_BYTES[dom] * V_own
            achieved = bytes_launch / (ms0 / n0 * 1e-3) / 1e9
            kname = (f"k_fsweep<{FORM_IDX[args.form]}>" if dom == "fwd_sweep"
                     else f"k_stream<{FORM_IDX[args.form]}, {OP_IDX[dom]}>")
            roof = {"bound": "hbm", "kernel": f"{kname} ({dom}, level 0)", "achieved": round(achieved, 1),
                    "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                    "traffic": ncu_traffic(kname), "traffic_source": "profiles/ncu_traffic.json (ncu --set full, "
                    "dram__bytes_read.sum + dram__bytes_write.sum per launch, bytes)",
                    "bytes_per_launch": bytes_launch, "launches_level0": n0,
                    "avg_launch_ms": ms0 / n0,
                    "share_of_step": round(prof[dom][1] / prof_step_ms, 4),
                    "profiled_step_ms": round(prof_step_ms, 3)}
    ops_ms = {k: round(v[1], 3) for k, v in prof.items() if v[0]}

    # operator apply alone (the BASELINE apply metric): L2 flushed before each
    ams = []
    for r in range(args.steps + 3):
        flush.zero_()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        ctx.apply(x_apply, y)
        a1.record(stream)
        torch.cuda.synchronize()
        if r >= 3:
            ams.append(a0.elapsed_time(a1))
    a_ms = max_over_ranks(float(np.median(ams)), world)
    apply_obj = {"gdof_s": round(dofs / (a_ms * 1e-3) / 1e9, 2),
                 "hbm_gbs": round(65 * cfg.vertices / (a_ms * 1e-3) / 1e9, 1),
                 "frac_of_peak": round(65 * cfg.vertices / (a_ms * 1e-3) / 1e9 / peak, 4),
                 "ms": round(a_ms, 4), "bytes_per_vertex": 65}

    # end-to-end through the public API from pinned host buffers: inputs in, the
    # solution (4 fields, canonical layout) out, every step
    e2e_ms = []
    h2d = cls.nbytes + (f4.nbytes if f is not None else fcls.nbytes)
    xcan = torch.empty((4, V_own), dtype=torch.float64, device="cuda")
    xhost = torch.empty((4, V_own), dtype=torch.float64).pin_memory()
    d2h = 0
    for r in range(args.steps + 1):
        flush.zero_()
        barrier(world)
        torch.cuda.synchronize()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        ctx.set_viscosity(cls_pin.numpy(), cfg.class_mu)      # H2D: element classes
        ctx.assemble()
        if cfg.forcing == "nodal":
            fv = ctx.import_(f_pin.numpy(), out=fvec, mask=False)  # H2D: forcing
            st = stk.stk_load_vector(ctx.h, 0, fv.data_ptr(), None, 0, b.data_ptr())
        else:
            fcls_dev.copy_(fcls_pin, non_blocking=True)         # H2D: forcing classes
            st = stk.stk_load_vector(ctx.h, 1, fcls_dev.data_ptr(), tab.ctypes.data, len(tab) // 3,
                                     b.data_ptr())
        assert st == 0
        ctx.apply(x_apply, y)
        x.zero_()
        _, rep = ctx.solve(b, x, rtol=RTOL, max_cycles=args.max_cycles)   # D2H: norms per cycle
        ctx.export_device(x, out=xcan)
        xhost.copy_(xcan, non_blocking=True)                    # D2H: the solution
        c1.record(stream)
        torch.cuda.synchronize()
        if r >= 1:
            e2e_ms.append(c0.elapsed_time(c1))
            d2h = xhost.numel() * 8 + 48 * (rep.cycles + 2)
    e2e_ms_v = max_over_ranks(float(np.mean(e2e_ms)), world)

    rep = reps[-1]
    converged = all(r_.rel_res <= RTOL for r_ in reps)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            smp = oracle_apply_sample(cfg, args.form, reps=1)
            value_cpu, applies = oracle_solve_extrapolated(cfg, smp["t_all"], rep.cycles, kry)
            cpu = {"value": value_cpu, "unit": "s/DoF", "cores": smp["threads"], "kind": "oracle",
                   "sample": (f"one oracle apply (plain C element loop, {smp['threads']} threads) on the full "
                              f"{cfg.name} n={cfg.n} grid: {smp['t_all']:.2f} s; the solve extrapolated as "
                              f"{applies:.0f} such products (the oracle multigrid's cost of the GPU's "
                              f"{rep.cycles} preconditioner cycles); one-thread apply on a "
                              f"{smp['slab_planes']}-plane slab: {smp['t_one_slab']:.2f} s"),
                   "apply_gdof_s_all_threads": round(smp["gdof_all"], 4),
                   "apply_gdof_s_one_thread": round(smp["gdof_one"], 5),
                   "oracle_solve_measured": oracle_solve_measured(),
                   "extrapolated": True}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "s/DoF", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": ms * 1e-3 / dofs, "unit": "s/DoF", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "step_ms": [round(t, 3) for t in step_ms],
                "higher_is_better": False, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": workload_name(cfg.name), "n": cfg.n,
                           "dofs": dofs, "form": args.form, "rtol": RTOL,
                           "solver": f"GMRES({kry}) + V_var(3,3)" if kry else "V_var(3,3) iteration",
                           "step": "assemble + load vector + apply + solve", "l2": "flushed between steps",
                           "parallelism": f"z-slab x{world}"},
                "solve": {"iterations": rep.cycles, "rho": round(rep.rho, 4), "rel_res": rep.rel_res,
                          "solve_s": rep.t_total_s, "converged_every_step": converged,
                          "t_level_s": {"finest": round(rep.t_level_s[0], 5),
                                        "levels_ge_1": round(rep.t_level_s[1], 5)}},
                "apply": apply_obj,
                "roofline": roof,
                "ops_ms_per_step": ops_ms,
                "clocks": clk,
                "e2e": {"value": e2e_ms_v * 1e-3 / dofs, "unit": "s/DoF", "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h)},
                "gpu_launches": int(launches),
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=list(CFG_INDEX))
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--form", default="mod", choices=["mod", "sym", "grad"])
    ap.add_argument("--krylov", type=int, default=None)
    ap.add_argument("--max-cycles", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the workload's n on every N; weak (SURVEY NEXT-3, the JUQUEEN "
                         "ladder P:1341-1346): n = n_1 * N^(1/3) with n_1 = --n (default 512), N a cube")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    n = args.n
    if args.scaling == "weak":
        c = round(world ** (1.0 / 3.0))
        if c ** 3 != world:
            raise SystemExit(f"--scaling weak needs a cube number of GPUs (1, 8, 64), got {world}")
        n = (args.n or 512) * c
    cfg = synth.get_config(args.workload, n=n)
    if args.impl == "reference":
        rc = run_reference(args, cfg, world, rank)
    else:
        rc = run_ours(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
