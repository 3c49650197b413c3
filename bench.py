"""bench.py — B200 benchmark of the matrix-free Stokes hot path (arXiv:1604.07994).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2] [--n N] [--form mod] [--krylov 0]

One JSON line (rank 0).  A *step* is one pass of the whole hot path
over the workload: assemble (coarse classes, classification, constant stencils,
coarse inverse) -> load vector -> one operator apply -> multigrid solve of
K x = b to relative residual 1e-8 from x = 0.

* metric / unit: BASELINE.json's metric; `value` = device-timed seconds per step
  per DoF (DoF = 4 (n+1)^3, the paper's convention), inputs resident in
  HBM; lower is better.  `apply` reports the operator-apply GDoF/s and HBM GB/s
  (separate timed loop, L2 flushed before every apply).
* e2e: the same step through the public API from pinned host buffers (element
  classes and forcing copied in every step; the residual history read back).
* roofline: the dominant kernel of the step (by summed device time, CUDA events
  around every launch on the solver stream during the timed steps) against the
  measured HBM copy bandwidth in MEASURED_PEAKS.json.
* cpu_baseline: the oracle (oracle/, test infrastructure) timed on the host on a
  bounded sample: one V-cycle of the oracle multigrid (plain C element-loop
  products, all host threads) on the same workload, extrapolated by the GPU's
  cycle count.  `--impl reference` times the same oracle as the reference arm.
* Default workload: BASELINE.json configs[1] (n = 128, plane interface with
  mu1/mu2 = 1e3, traction-free top), form "mod".  --gpus N > 1 (torchrun) shards
  the grid in z-slabs over N ranks (weak scaling is not used: total work fixed).
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
CFG_INDEX = {"cfg1": 0, "cfg2": 1, "cfg3": 2, "cfg4": 3, "cfg5": 4}
# algorithmic bytes per owned vertex of each profiled op
OP_BYTES = {"apply": 65, "residual": 97, "vel_pass": 81, "p_pass1": 49, "p_pass2": 25}


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

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

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
# reference arm: the oracle multigrid on the host (bounded sample per step)
# ------------------------------------------------------------------------------
def oracle_cycle_sample(cfg, form, cycles, gpu_cycles=None, log=None):
    """Time `cycles` V-cycles of the oracle (matrix-free C products, all host
    threads) on the workload; returns (seconds per cycle list, residual history,
    threads, setup seconds)."""
    from oracle import capi, mg_mf
    t0 = time.time()
    cls, fcls = synth.element_classes(cfg)
    h = mg_mf.MFHierarchy(cfg.n, cls, cfg.class_mu, cfg.faces, form=form,
                          ncolors_u=4 if form == "sym" else 2)
    pr = h.levels[0].prob
    if cfg.forcing == "nodal":
        f = synth.nodal_forcing(cfg)
        # b_u = M f by the element loop: M f = sum_T |T|/20 (sum_q f_q + f_i)
        b = _oracle_load_nodal(cfg, f)
    else:
        b = _oracle_load_element(cfg, np.asarray(cfg.force_table)[fcls])
    b = np.where(pr.free, b, 0.0)
    setup = time.time() - t0
    x = np.zeros_like(b)
    nb = np.linalg.norm(b)
    hist = [1.0]
    times = []
    for c in range(cycles):
        t1 = time.time()
        x = h.vcycle(b, x)
        times.append(time.time() - t1)
        hist.append(np.linalg.norm(b - pr.apply(x)) / nb)
        if log:
            log(f"oracle cycle {c}: {times[-1]:.2f}s rel {hist[-1]:.2e}")
    return times, hist, capi.num_threads(), setup


def _oracle_load_nodal(cfg, f):
    from oracle import fem
    n = cfg.n
    V = cfg.vertices
    h = 1.0 / n
    b = np.zeros((3, V))
    for t in range(6):
        vid = fem._element_vertex_ids(n, t)
        M = fem.element_matrices(t, h, "grad")["M"]
        for a in range(3):
            loc = f[a][vid] @ M.T
            np.add.at(b[a], vid.reshape(-1), loc.reshape(-1))
    return np.concatenate([b.reshape(-1), np.zeros(V)])


def _oracle_load_element(cfg, fe):
    from oracle import fem
    n, V = cfg.n, cfg.vertices
    fe = fe.reshape(n, n, n, 6, 3)
    b = np.zeros((3, V))
    vol = (1.0 / n) ** 3 / 6
    for t in range(6):
        vid = fem._element_vertex_ids(n, t)
        ft = fe[..., t, :].reshape(-1, 3)
        for a in range(3):
            np.add.at(b[a], vid.reshape(-1), np.repeat(ft[:, a] * vol / 4.0, 4))
    return np.concatenate([b.reshape(-1), np.zeros(V)])


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return 0
    dofs = cfg.dofs
    times, hist, threads, setup = oracle_cycle_sample(cfg, args.form, args.warmup + args.steps,
                                                      log=lambda s: print(s, file=sys.stderr))
    tt = times[args.warmup:]
    rho = (hist[-1] / hist[0]) ** (1.0 / max(1, len(hist) - 1))
    need = math.ceil(math.log(RTOL) / math.log(rho)) if 0 < rho < 1 else None
    t_cycle = float(np.median(tt))
    value = t_cycle * need / dofs if need else None
    sample = (f"one oracle V_var(3,3) cycle per step (matrix-free C element loop, {threads} host threads) "
              f"on the full {cfg.name} n={cfg.n} grid; solve time extrapolated as median cycle time x "
              f"cycles to rtol 1e-8 at the oracle's observed rate rho={rho:.3f} ({need} cycles)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/DoF", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_cycle * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name} (BASELINE configs[{CFG_INDEX[cfg.name]}])", "n": cfg.n,
                       "dofs": dofs, "form": args.form, "rtol": RTOL},
            "cpu_baseline": {"value": value, "unit": "s/DoF", "cores": threads, "kind": "oracle",
                             "sample": sample},
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
    ctx = stk.StokesContext(cfg.n, args.form, cfg.faces, krylov=args.krylov,
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
    fvec = ctx.import_(f_pin.cuda())
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

    # warm-up
    for _ in range(args.warmup):
        flush.zero_()
        rep = step()
    torch.cuda.synchronize()
    log(f"warm-up done: cycles {rep.cycles} rho {rep.rho:.3f} rel {rep.rel_res:.2e}")

    # timed steps (device time, CUDA events on the solver stream).  Profile mode 1
    # brackets every level-0 launch with CUDA events on the same stream (the
    # coarse levels run as one CUDA graph, timed as a whole)
    clocks = Clocks(local)
    ctx.profile(1)
    ctx.profile_reset()
    l0 = ctx.launch_count()
    ev = []
    reps = []
    clocks.start()
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
    # dominant kernel of the step
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
            kname = f"k_stream<{FORM_IDX[args.form]}, {OP_IDX[dom]}>"
            roof = {"bound": "hbm", "kernel": f"{kname} ({dom}, level 0)", "achieved": round(achieved, 1),
                    "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                    "traffic": ncu_traffic(kname), "traffic_source": "profiles/ncu_traffic.json (ncu --set full, "
                    "dram__bytes_read.sum + dram__bytes_write.sum per launch, bytes)",
                    "bytes_per_launch": bytes_launch, "launches_level0": n0,
                    "avg_launch_ms": ms0 / n0,
                    "share_of_step": round(prof[dom][1] / sum(step_ms), 4)}
    ops_ms = {k: round(v[1] / args.steps, 3) for k, v in prof.items() if v[0]}

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

    # end-to-end through the public API from pinned host buffers
    e2e_ms = []
    h2d = cls.nbytes + (f4.nbytes if f is not None else fcls.nbytes)
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
            fv = ctx.import_(f_pin.numpy(), out=fvec)           # H2D: forcing
            st = stk.stk_load_vector(ctx.h, 0, fv.data_ptr(), None, 0, b.data_ptr())
        else:
            fcls_dev.copy_(fcls_pin, non_blocking=True)         # H2D: forcing classes
            st = stk.stk_load_vector(ctx.h, 1, fcls_dev.data_ptr(), tab.ctypes.data, len(tab) // 3,
                                     b.data_ptr())
        assert st == 0
        ctx.apply(x_apply, y)
        x.zero_()
        _, rep = ctx.solve(b, x, rtol=RTOL, max_cycles=args.max_cycles)   # D2H: norms per cycle
        c1.record(stream)
        torch.cuda.synchronize()
        if r >= 1:
            e2e_ms.append(c0.elapsed_time(c1))
            d2h = 48 * (rep.cycles + 2)
    e2e_ms_v = max_over_ranks(float(np.mean(e2e_ms)), world)

    rep = reps[-1]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            times, hist, threads, setup = oracle_cycle_sample(cfg, args.form, 1)
            t_solve = times[0] * max(rep.cycles, 1) + setup
            cpu = {"value": t_solve / dofs, "unit": "s/DoF", "cores": threads, "kind": "oracle",
                   "sample": (f"1 V_var(3,3) cycle of the oracle multigrid (matrix-free C element loop, "
                              f"{threads} threads) on the full {cfg.name} n={cfg.n} grid ({times[0]:.1f} s) "
                              f"+ oracle setup ({setup:.1f} s), extrapolated to the GPU's {rep.cycles} cycles"),
                   "extrapolated": True}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "s/DoF", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": ms * 1e-3 / dofs, "unit": "s/DoF", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"{cfg.name} (BASELINE configs[{CFG_INDEX[cfg.name]}])", "n": cfg.n,
                           "dofs": dofs, "form": args.form, "rtol": RTOL,
                           "solver": f"GMRES({args.krylov}) + V_var(3,3)" if args.krylov else "V_var(3,3) iteration",
                           "step": "assemble + load vector + apply + solve", "l2": "flushed between steps",
                           "parallelism": f"z-slab x{world}"},
                "solve": {"cycles": rep.cycles, "rho": round(rep.rho, 4), "rel_res": rep.rel_res,
                          "solve_s": rep.t_total_s},
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
    ap.add_argument("--workload", default="cfg2", choices=list(CFG_INDEX))
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--form", default="mod", choices=["mod", "sym", "grad"])
    ap.add_argument("--krylov", type=int, default=0)
    ap.add_argument("--max-cycles", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.get_config(args.workload, n=args.n)
    world, rank, local = dist_setup(args)
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
