"""The N > 1 path on CPU: the z-slab partition the library uses (stk_partition,
host-only C ABI), its halo exchange pattern and reductions, run by world_size-2
gloo process groups against the oracle (no GPU).

Each rank keeps ONLY its slab: owned vertex planes, the one-plane halos received
from its neighbours over gloo (the exchange Comm::halo performs with NCCL), and
the stored cube layers of element classes; everything else is NaN.  The oracle
element loop then evaluates the owned rows of K x from that slab; the union over
ranks must equal the single-process oracle apply bit for bit, which proves that
the partition and the halo width cover every row's 24-tet star.
"""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import capi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partition(n, P, r):
    import paper_1604_07994_b200 as stk
    return stk.partition(n, P, r)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [16, 64, 128])
def test_partition_owns_every_plane_once(n, P):
    parts = [_partition(n, P, r) for r in range(P)]
    nlev = len(parts[0])
    assert [lv["n"] for lv in parts[0]] == [n >> l for l in range(nlev)]
    for l in range(nlev):
        m = n >> l
        levs = [parts[r][l] for r in range(P)]
        if levs[0]["replicated"]:
            assert all(lv["replicated"] and lv["z0"] == 0 and lv["nzl"] == m + 1 for lv in levs)
            continue
        owned = np.zeros(m + 1, int)
        for lv in levs:
            owned[lv["z0"]:lv["z0"] + lv["nzl"]] += 1
            # stored cube layers cover the stars of the owned planes
            assert lv["cz0"] == max(0, lv["z0"] - 1) and lv["cz1"] == min(m, lv["z0"] + lv["nzl"])
            assert lv["nzl"] >= 2          # one-plane halos suffice for the 15-point stencil
        assert np.all(owned == 1)
        if l > 0:
            assert not parts[0][l - 1]["replicated"]  # replicated levels form a coarse tail
    # restriction onto the first replicated level: the K ranges partition it
    for l in range(nlev - 1):
        if not parts[0][l]["replicated"] and parts[0][l + 1]["replicated"]:
            mc = n >> (l + 1)
            cover = np.zeros(mc + 1, int)
            for r in range(P):
                lv = parts[r][l]
                assert lv["K0"] >= 0
                cover[lv["K0"]:lv["K1"]] += 1
                # every restricted coarse plane K reads fine planes 2K-1..2K+1: owned or halo
                for K in range(lv["K0"], lv["K1"]):
                    assert lv["z0"] - 1 <= 2 * K - 1 and 2 * K + 1 <= lv["z0"] + lv["nzl"]
            assert np.all(cover == 1)


def _worker(rank, world, port, n, q, cfgname="cfg4"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.get_config(cfgname, n=n)
        cls, _ = synth.element_classes(cfg)
        x = synth.apply_input(cfg)                       # (4, V) global, same seed on every rank
        N1 = n + 1
        lv = _partition(n, world, rank)[0]
        z0, nzl = lv["z0"], lv["nzl"]
        # this rank's slab: owned planes, halos from the neighbours, NaN elsewhere
        xs = np.full((4, N1, N1 * N1), np.nan)            # [field][k][j*N1+i]
        xg = x.reshape(4, N1, N1 * N1)
        xs[:, z0:z0 + nzl] = xg[:, z0:z0 + nzl]
        reqs, halo_lo, halo_hi = [], None, None
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(xs[:, z0])), rank - 1))
            halo_lo = torch.empty(4, N1 * N1, dtype=torch.float64)
            reqs.append(dist.irecv(halo_lo, rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(xs[:, z0 + nzl - 1])), rank + 1))
            halo_hi = torch.empty(4, N1 * N1, dtype=torch.float64)
            reqs.append(dist.irecv(halo_hi, rank + 1))
        for r_ in reqs:
            r_.wait()
        if halo_lo is not None:
            xs[:, z0 - 1] = halo_lo.numpy()
        if halo_hi is not None:
            xs[:, z0 + nzl] = halo_hi.numpy()
        # element classes: only the stored cube layers; others point at a NaN viscosity
        nan_cls = len(cfg.class_mu)
        mu = np.append(np.asarray(cfg.class_mu, float), np.nan)
        c4 = cls.reshape(n, n, n, 6).copy()
        c4[:lv["cz0"]] = nan_cls
        c4[lv["cz1"]:] = nan_cls
        y = capi.apply_slab(n, "mod", 1 / 12, cfg.faces, c4.reshape(-1), mu, xs.reshape(4, -1),
                            kv0=z0, kv1=z0 + nzl).reshape(4, N1, N1 * N1)
        mine = np.ascontiguousarray(y[:, z0:z0 + nzl])
        # owned-row squared norms, summed over ranks (the NCCL allreduce of the solver)
        nrm = torch.tensor([float(np.sum(mine ** 2))], dtype=torch.float64)
        dist.all_reduce(nrm)
        gathered = [torch.empty(0)] * world
        dist.all_gather_object(gathered, (z0, nzl, mine))
        if rank == 0:
            q.put((gathered, float(nrm.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfgname", [(2, "cfg4"), (2, "cols")])
def test_slab_apply_with_gloo_halo_exchange_equals_global_oracle(world, cfgname):
    import torch.multiprocessing as mp
    n = 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, cfgname)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, nrm = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.get_config(cfgname, n=n)
    cls, _ = synth.element_classes(cfg)
    x = synth.apply_input(cfg)
    N1 = n + 1
    y = capi.apply_slab(n, "mod", 1 / 12, cfg.faces, cls, cfg.class_mu, x).reshape(4, N1, N1 * N1)
    covered = np.zeros(N1, int)
    for z0, nzl, part in gathered:
        assert np.all(np.isfinite(part)), "a row read outside its slab (halo or cube layers too thin)"
        assert np.array_equal(part, y[:, z0:z0 + nzl])   # bit for bit: same rows, same data
        covered[z0:z0 + nzl] += 1
    assert np.all(covered == 1)
    assert nrm == pytest.approx(float(np.sum(y ** 2)), rel=1e-14)
