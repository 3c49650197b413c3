"""One bench step (bench.py's workload and step: assemble + load + apply + solve) with
cudaProfilerStart/Stop around it, for `ncu --profile-from-start off` launch lists:

    ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
        --csv --log-file gpurun_out/launches.csv python tools/step_profiled.py [cfg3] [n] [krylov]
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import synth
import paper_1604_07994_b200 as stk

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = synth.get_config(name, n=n)
kry = int(sys.argv[3]) if len(sys.argv) > 3 else bench.DEFAULT_KRYLOV[name]
ctx = stk.StokesContext(cfg.n, "mod", cfg.faces, krylov=kry)
cls, fcls = synth.element_classes(cfg)
xin = synth.apply_input(cfg)
ctx.set_viscosity(cls, cfg.class_mu)
ctx.assemble()
f = synth.nodal_forcing(cfg) if cfg.forcing == "nodal" else None
fvec = ctx.import_(np.concatenate([f, np.zeros((1, cfg.vertices))]), mask=False) if f is not None else None
fcls_dev = torch.from_numpy(fcls).cuda()
tab = np.ascontiguousarray(cfg.force_table, dtype=np.float64).reshape(-1)
x_apply = ctx.import_(xin)
y, b, x = ctx.new_vector(), ctx.new_vector(), ctx.new_vector()


def step():
    ctx.assemble()
    if f is not None:
        stk.stk_load_vector(ctx.h, 0, fvec.data_ptr(), None, 0, b.data_ptr())
    else:
        stk.stk_load_vector(ctx.h, 1, fcls_dev.data_ptr(), tab.ctypes.data, len(tab) // 3, b.data_ptr())
    ctx.apply(x_apply, y)
    x.zero_()
    return ctx.solve(b, x, rtol=bench.RTOL, max_cycles=300)[1]


step()
torch.cuda.synchronize()
l0 = ctx.launch_count()
torch.cuda.profiler.start()
rep = step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{name} n={cfg.n}: {rep.cycles} iterations, rel {rep.rel_res:.2e}, {ctx.launch_count() - l0} library launches "
      f"(+ the coarse-graph kernels counted per graph launch)", file=sys.stderr)
