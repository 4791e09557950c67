"""Multi-process (gloo, world size 2 and 3, CPU) tests of the C5 sharded
path's host logic: slab decomposition, neighbour halo exchange and particle
migration.  Density on each rank is computed by the oracle over own+ghost
particles and must equal the single-process oracle density of the same
particles (same pair formula, f64).  The GPU runs the same functions with
NCCL and the sm_100a density kernel."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def population(n, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3))
    from paper_2512_05516_b200.sharded import grid_for
    h, nc, cell = grid_for(n)
    return x, np.full(n, 1.0 / n), np.full(n, h), nc, cell


def velocities_pressures(n, seed=4):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (n, 3)), rng.uniform(0.2, 1.2, n)


def _worker(rank, world, port, outdir, n):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2512_05516_b200.sharded import (Slab, density_with_ghosts, exchange_ghost_fields, exchange_halo,
                                               force_with_ghosts, migrate_rows)

    x, m, h, nc, cell = population(n)
    slab = Slab(nc, cell, rank, world)
    xt = torch.tensor(x)
    ix = slab.layer(xt[:, 0])
    own = ((ix >= slab.x0) & (ix < slab.x1)).numpy()
    ids = np.nonzero(own)[0]
    xo, mo, ho = torch.tensor(x[own]), torch.tensor(m[own]), torch.tensor(h[own])

    def oracle_backend(xc, mc, hc, slab, n_own):
        rho = O.density_cells(xc.numpy().reshape(-1), mc.numpy(), hc.numpy(), 0.0, 1.0, slab.cell)
        return torch.tensor(rho[:n_own])

    gx, gm, gh = exchange_halo(xo, mo, ho, slab)
    rho = density_with_ghosts(xo, mo, ho, gx, gm, gh, slab, oracle_backend).numpy()

    # force: second halo of (x, v, m, h, rho, P) after every rank has its rho
    v, P = velocities_pressures(n)
    own_f = [xo, torch.tensor(v[own]), mo, ho, torch.tensor(rho), torch.tensor(P[own])]
    ghosts = exchange_ghost_fields(own_f, xo[:, 0], slab)

    def oracle_force(xc, vc, mc, hc, rc, pc, slab, n_own):
        a, du, _, _ = O.force_cells(xc.numpy().reshape(-1), vc.numpy().reshape(-1), mc.numpy(), hc.numpy(),
                                    rc.numpy(), pc.numpy(), 0.0, 1.0, slab.cell)
        return torch.tensor(a[:n_own]), torch.tensor(du[:n_own])

    fa, fdu = force_with_ghosts(own_f, ghosts, slab, oracle_force)

    # migration: push every particle by +-0.6 cell in x, wrap into the box
    rng = np.random.default_rng(100 + rank)
    xm = x[own].copy()
    xm[:, 0] = np.clip(xm[:, 0] + rng.choice([-0.6, 0.6], size=len(xm)) * cell, 0.0, 1.0 - 1e-12)
    rows = torch.tensor(np.concatenate([ids[:, None].astype(np.float64), xm], axis=1))
    moved = migrate_rows(rows, rows[:, 1], slab)
    lay = slab.layer(moved[:, 1])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=ids, rho=rho, nghost=len(gm), fa=fa.numpy(),
             fdu=fdu.numpy(), nghost_f=len(ghosts[0]),
             mig_ids=moved[:, 0].numpy().astype(np.int64),
             mig_ok=bool(((lay >= slab.x0) & (lay < slab.x1)).all()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_and_migration_gloo(tmp_path, world):
    n = 6000
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), n), nprocs=world, join=True)
    import oracle as O
    x, m, h, nc, cell = population(n)
    want = O.density_cells(x.reshape(-1), m, h, 0.0, 1.0, cell)
    v, P = velocities_pressures(n)
    rho_all = np.zeros(n)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        rho_all[d["ids"]] = d["rho"]
    wa, wdu, sa, sd = O.force_cells(x.reshape(-1), v.reshape(-1), m, h, rho_all, P, 0.0, 1.0, cell)
    seen, mig = [], []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        np.testing.assert_allclose(d["rho"], want[d["ids"]], rtol=1e-12, atol=0)
        # per-rank force over own + ghost rows == the single-process force (summation order differs)
        ids = d["ids"]
        assert np.all(np.linalg.norm(d["fa"] - wa[ids], axis=1) <= 1e-12 * sa[ids])
        assert np.all(np.abs(d["fdu"] - wdu[ids]) <= 1e-12 * sd[ids] + 1e-300)
        assert d["nghost_f"] == d["nghost"]
        assert d["nghost"] > 0
        assert bool(d["mig_ok"])
        seen.append(d["ids"])
        mig.append(d["mig_ids"])
    assert sorted(np.concatenate(seen).tolist()) == list(range(n))   # a partition
    assert sorted(np.concatenate(mig).tolist()) == list(range(n))    # nothing lost/duplicated


def test_slab_geometry():
    from paper_2512_05516_b200.sharded import Slab, grid_for
    h, nc, cell = grid_for(1 << 27)
    assert nc == 200 and cell >= 2 * h            # 200 cells per side
    for world in (1, 2, 4, 8):
        slabs = [Slab(nc, cell, r, world) for r in range(world)]
        assert slabs[0].x0 == 0 and slabs[-1].x1 == nc
        assert all(a.x1 == b.x0 for a, b in zip(slabs, slabs[1:]))
