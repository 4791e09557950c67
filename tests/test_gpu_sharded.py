"""C5 sharded path on one B200: a full N=1 step against the oracle, and the
per-rank density with ghost layers (simulated 2- and 4-rank splits of one
population) against the global oracle density."""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2512_05516_b200 import api
from paper_2512_05516_b200.sharded import ShardedState, Slab, density_with_ghosts, gpu_density_backend, grid_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_single_rank_step_matches_oracle(halo):
    n = 1 << 15
    h, nc, cell = grid_for(n)
    st = ShardedState(n, Slab(nc, cell, 0, 1), prec=32, h=h, halo=halo)
    st.sort_by_cell()
    before = {k: st.stream(k).double().cpu().numpy().copy() for k in ["x", "v", "u", "a", "du", "m", "h"]}
    st.step(1e-3)
    torch.cuda.synchronize()
    # kick then drift, binary64 arithmetic on the binary32 stored lanes, stored back as binary32
    v2, u2 = O.kick(before["v"], before["u"], before["a"], before["du"], 1e-3)
    v2 = v2.astype(np.float32).astype(np.float64)
    u2 = u2.astype(np.float32).astype(np.float64)
    x2 = O.drift(before["x"], v2, 1e-3).astype(np.float32).astype(np.float64)
    np.testing.assert_array_equal(st.stream("v").double().cpu().numpy(), v2)
    np.testing.assert_array_equal(st.stream("u").double().cpu().numpy(), u2)
    np.testing.assert_array_equal(st.stream("x").double().cpu().numpy(), x2)
    want = O.density_cells(x2.reshape(-1), before["m"], before["h"], 0.0, 1.0, cell)
    got = st.stream("rho").double().cpu().numpy()
    np.testing.assert_allclose(got, want.astype(np.float32), rtol=2e-5)


@pytest.mark.parametrize("world", [2, 4])
def test_rank_density_with_ghost_layers(world):
    n = 1 << 15
    rng = np.random.default_rng(9)
    x = rng.random((n, 3))
    h, nc, cell = grid_for(n)
    hh = np.full(n, h)
    m = np.full(n, 1.0 / n)
    want = O.density_cells(x.reshape(-1), m, hh, 0.0, 1.0, cell)
    layer = np.minimum(np.floor(x[:, 0] / cell).astype(int), nc - 1)
    seen = np.zeros(n, bool)
    for r in range(world):
        slab = Slab(nc, cell, r, world)
        own = (layer >= slab.x0) & (layer < slab.x1)
        ghost = ((layer == slab.x0 - 1) | (layer == slab.x1)) & ~own
        t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
        rho = density_with_ghosts(t(x[own]), t(m[own]), t(hh[own]), t(x[ghost]), t(m[ghost]), t(hh[ghost]), slab,
                                  gpu_density_backend(api.SF_PREC_NATIVE))
        np.testing.assert_allclose(rho.double().cpu().numpy(), want[own], rtol=1e-5)
        seen |= own
    assert seen.all()


@pytest.mark.parametrize("world", [2, 4])
def test_rank_force_with_ghost_layers(world):
    """Per-rank cell-linked force over own + ghost (x, v, m, h, rho, P) rows
    (simulated splits of one population) against the global oracle force."""
    from paper_2512_05516_b200.sharded import force_with_ghosts, gpu_force_backend
    n = 1 << 15
    rng = np.random.default_rng(10)
    x = rng.random((n, 3))
    v = rng.uniform(-1, 1, (n, 3))
    h, nc, cell = grid_for(n)
    hh, m = np.full(n, h), np.full(n, 1.0 / n)
    rho, P = rng.uniform(0.5, 1.5, n), rng.uniform(0.2, 1.2, n)
    t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
    dec = lambda a: t(a).double().cpu().numpy()  # noqa: E731  (the stored binary32 values)
    wa, wdu, sa, sd = O.force_cells(dec(x).reshape(-1), dec(v).reshape(-1), dec(m), dec(hh), dec(rho), dec(P),
                                    0.0, 1.0, cell)
    layer = np.minimum(np.floor(x[:, 0] / cell).astype(int), nc - 1)
    seen = np.zeros(n, bool)
    for r in range(world):
        slab = Slab(nc, cell, r, world)
        own = (layer >= slab.x0) & (layer < slab.x1)
        ghost = ((layer == slab.x0 - 1) | (layer == slab.x1)) & ~own
        a, du = force_with_ghosts([t(f[own]) for f in (x, v, m, hh, rho, P)],
                                  [t(f[ghost]) for f in (x, v, m, hh, rho, P)], slab,
                                  gpu_force_backend(api.SF_PREC_NATIVE))
        assert np.all(np.linalg.norm(a.double().cpu().numpy() - wa[own], axis=1) <= 2e-5 * sa[own])
        assert np.all(np.abs(du.double().cpu().numpy() - wdu[own]) <= 2e-5 * sd[own] + 1e-30)
        seen |= own
    assert seen.all()


@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_single_rank_full_step_runs_reference_order(halo):
    """density -> force -> kick -> drift on one rank: a/du come from the force
    on the fresh rho, then kick/drift use them (checked against the oracle)."""
    n = 1 << 15
    h, nc, cell = grid_for(n)
    st = ShardedState(n, Slab(nc, cell, 0, 1), prec=32, h=h, halo=halo)
    st.sort_by_cell()
    st.stream("P").copy_(torch.rand(st.n, device="cuda") + 0.2)
    before = {k: st.stream(k).double().cpu().numpy().copy() for k in ["x", "v", "u", "m", "h", "P"]}
    st.full_step(1e-3)
    torch.cuda.synchronize()
    rho = st.stream("rho").double().cpu().numpy()
    want_rho = O.density_cells(before["x"].reshape(-1), before["m"], before["h"], 0.0, 1.0, cell)
    np.testing.assert_allclose(rho, want_rho.astype(np.float32), rtol=2e-5)
    wa, wdu, sa, sd = O.force_cells(before["x"].reshape(-1), before["v"].reshape(-1), before["m"], before["h"], rho,
                                    before["P"], 0.0, 1.0, cell)
    a = st.stream("a").double().cpu().numpy()
    assert np.all(np.linalg.norm(a - wa, axis=1) <= 2e-5 * sa + 1e-6 * np.abs(wa).max())
    # kick used the stored a/du
    du = st.stream("du").double().cpu().numpy()
    v2, u2 = O.kick(before["v"], before["u"], a, du, 1e-3)
    np.testing.assert_array_equal(st.stream("v").double().cpu().numpy(), v2.astype(np.float32).astype(np.float64))


def _slab_blocks(x, m, h, nc, cell, world, refine):
    """Per slab: own particles binned on the slab's own layers and packed
    (the persistent block a rank exposes to its neighbours)."""
    fine = cell / refine
    layer = np.minimum(np.floor(x[:, 0] / cell).astype(int), nc - 1)
    out = []
    for r in range(world):
        slab = Slab(nc, cell, r, world)
        own = (layer >= slab.x0) & (layer < slab.x1)
        x0, nx = slab.x0 * refine, (slab.x1 - slab.x0) * refine
        t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
        xt, mt, ht = t(x[own]), t(m[own]), t(h[own])
        n = int(own.sum())
        cs, perm = api.bin_particles(xt, (x0 * fine, 0.0, 0.0), fine, (nx, nc * refine, nc * refine))
        pos = torch.empty(n, 4, device="cuda")
        hs = torch.empty(n, device="cuda")
        hmax = torch.zeros(4, dtype=torch.int32, device="cuda")
        api.cells_pack(xt, mt, ht, perm, pos, hs, hmax)
        out.append(dict(own=own, n=n, perm=perm, keep=(xt, mt, ht, cs, pos, hs, hmax),
                        block=api.cell_block(pos, hs, cs, hmax, x0, nx, x0 * fine)))
    return out


@pytest.mark.parametrize("world,refine", [(2, 2), (4, 2), (3, 1)])
def test_density_blocks_read_neighbours_in_place(world, refine):
    """The fused-halo density: each slab's homes read the neighbouring slabs'
    packed blocks in place (here through same-device pointers; across GPUs the
    same addresses come from CUDA IPC over NVLink) — no ghost rows at all."""
    n = 1 << 15
    rng = np.random.default_rng(21)
    x = rng.random((n, 3))
    h, nc, cell = grid_for(n)
    hh = np.full(n, h) * rng.uniform(0.9, 1.0, n)
    m = rng.uniform(0.5, 1.5, n) / n
    dec = lambda a: torch.tensor(a, dtype=torch.float32).double().numpy()  # noqa: E731
    want = O.density_cells(dec(x).reshape(-1), dec(m), dec(hh), 0.0, 1.0, cell)
    S = _slab_blocks(x, m, hh, nc, cell, world, refine)
    seen = np.zeros(n, bool)
    for r in range(world):
        blocks = [S[r]["block"]] + [S[q]["block"] for q in (r - 1, r + 1) if 0 <= q < world]
        rho = api.density_cells_blocks(blocks, S[r]["n"], S[r]["perm"], (0.0, 0.0), cell / refine, nc * refine,
                                       nc * refine, nc * refine, reach=refine)
        np.testing.assert_allclose(rho[: S[r]["n"]].double().cpu().numpy(), want[S[r]["own"]], rtol=1e-5)
        seen |= S[r]["own"]
    assert seen.all()

    # the force over the same blocks: every slab packs (v, P/rho^2) in its cell order
    v = rng.uniform(-1, 1, (n, 3))
    rho = rng.uniform(0.5, 1.5, n)
    P = rng.uniform(0.2, 1.2, n)
    wa, wdu, sa, sd = O.force_cells(dec(x).reshape(-1), dec(v).reshape(-1), dec(m), dec(hh), dec(rho), dec(P),
                                    0.0, 1.0, cell)
    t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
    fb = []
    for r in range(world):
        own, k = S[r]["own"], S[r]["n"]
        vel = torch.empty(k, 4, device="cuda")
        api.force_pack(t(v[own]), t(rho[own]), t(P[own]), S[r]["perm"], vel)
        xt, mt, ht, cs, pos, hs, hmax = S[r]["keep"]
        S[r]["fkeep"] = vel
        fb.append(api.force_block(pos, vel, hs, cs, hmax, S[r]["block"].x0, S[r]["block"].nx, S[r]["block"].x_origin))
    for r in range(world):
        blocks = [fb[r]] + [fb[q] for q in (r - 1, r + 1) if 0 <= q < world]
        a, du = api.force_cells_blocks(blocks, S[r]["n"], S[r]["perm"], (0.0, 0.0), cell / refine, nc * refine,
                                       nc * refine, nc * refine, reach=refine)
        own = S[r]["own"]
        err = np.linalg.norm(a[: S[r]["n"]].double().cpu().numpy() - wa[own], axis=1)
        assert np.all(err <= 2e-5 * sa[own])
        assert np.all(np.abs(du[: S[r]["n"]].double().cpu().numpy() - wdu[own]) <= 2e-5 * sd[own] + 1e-30)


def _population(n):
    rng = np.random.default_rng(31)
    x = rng.random((n, 3))
    h, nc, cell = grid_for(n)
    m = rng.uniform(0.5, 1.5, n) / n
    v = np.random.default_rng(32).uniform(-1, 1, (n, 3))
    P = np.random.default_rng(33).uniform(0.2, 1.2, n)
    return x, m, h, nc, cell, v, P


def _shard_worker(rank, world, port, outdir, n):
    """One rank of api.Shard (the C++ sharded step behind the C ABI): its
    slab's particles of a shared population, density then force."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # every rank on the one device: CUDA IPC between processes of one GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_05516_b200.sharded import _handle_exchange
    x, m, h, nc, cell, v, P = _population(n)
    layer = np.minimum(np.floor(x[:, 0] / cell).astype(int), nc - 1)
    slab = Slab(nc, cell, rank, world)
    own = (layer >= slab.x0) & (layer < slab.x1)
    k = int(own.sum())
    S = api.Schema.default()
    buf = api.PackedBuffer.empty(api.View(S, k, "soa", None, 32))
    vals = {"x": x[own], "id": np.nonzero(own)[0], "v": v[own], "u": np.ones(k), "m": m[own], "h": np.full(k, h),
            "rho": np.ones(k), "P": P[own], "cs": np.zeros(k), "a": np.zeros((k, 3)), "du": np.zeros(k),
            "dt": np.full(k, 1e-3)}
    for name, arr in vals.items():
        base, _, w, ar = buf.view.lane(name)
        t = torch.tensor(arr, dtype=torch.int64 if name == "id" else torch.float32, device="cuda")
        buf.data[base // 8: base // 8 + t.numel() * t.element_size()].copy_(t.reshape(-1).view(torch.uint8))
    sh = api.Shard(rank, world, nc, cell, 2, 3 * n // world, _handle_exchange(None))
    sh.load(buf)
    sh.step("density")
    rho = sh.field("rho").clone()
    ids = sh.field("id").clone()
    sh.step("density")  # again: epochs advance, the blocks are rebuilt in place
    assert torch.equal(sh.field("rho"), rho)
    m1 = sh.step("force", timed=True)
    np.savez(os.path.join(outdir, f"p{rank}.npz"), id=ids.cpu().numpy(), rho=rho.cpu().numpy(),
             a=sh.field("a").cpu().numpy(), du=sh.field("du").cpu().numpy(), n=sh.count,
             force_ms=m1["force_ms"])
    torch.cuda.synchronize()
    dist.barrier()
    sh.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_across_processes_reads_neighbours_in_place(tmp_path, world):
    """api.Shard in `world` processes sharing one GPU: each maps its
    neighbours' blocks by CUDA IPC handle (the multi-GPU mechanism), the
    ranks order each other with device-side epochs, and the per-rank density
    and force equal the global oracle's."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n = 1 << 15
    mp.spawn(_shard_worker, args=(world, port, str(tmp_path), n), nprocs=world, join=True)
    x, m, h, nc, cell, v, P = _population(n)
    dec = lambda a: torch.tensor(a, dtype=torch.float32).double().numpy()  # noqa: E731
    want = O.density_cells(dec(x).reshape(-1), dec(m), dec(np.full(n, h)), 0.0, 1.0, cell)
    rho_all, seen = np.zeros(n), np.zeros(n, bool)
    outs = [np.load(tmp_path / f"p{r}.npz") for r in range(world)]
    for d in outs:
        ids = d["id"]
        np.testing.assert_allclose(d["rho"], want[ids], rtol=1e-5)
        assert not seen[ids].any()
        seen[ids] = True
        rho_all[ids] = d["rho"]
    assert seen.all()
    wa, wdu, sa, sd = O.force_cells(dec(x).reshape(-1), dec(v).reshape(-1), dec(m), dec(np.full(n, h)), rho_all,
                                    dec(P), 0.0, 1.0, cell)
    for d in outs:
        ids = d["id"]
        assert np.all(np.linalg.norm(d["a"] - wa[ids], axis=1) <= 2e-5 * sa[ids])
        assert np.all(np.abs(d["du"] - wdu[ids]) <= 2e-5 * sd[ids] + 1e-30)


def _state_worker(rank, world, port, outdir, n, full):
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, nc, cell = grid_for(n)
    st = ShardedState(n, Slab(nc, cell, rank, world), prec=32, h=h, group=None)
    for _ in range(3):  # large dt: particles cross slab planes every step
        if full:
            st.stream("P").copy_(st.stream("rho") * 0.7)
            st.full_step(0.02)
        else:
            st.step(0.02)
    if full:  # full_step ends with kick/drift + migration: refresh rho for the final positions
        st.density()
    torch.cuda.synchronize()
    lay = st.slab.layer(st.stream("x")[:, 0])
    np.savez(os.path.join(outdir, f"s{rank}.npz"), id=st.stream_bytes("id").cpu().numpy().view(np.int64).ravel(),
             x=st.stream("x").double().cpu().numpy(), rho=st.stream("rho").double().cpu().numpy(),
             m=st.stream("m").double().cpu().numpy(), h=st.stream("h").double().cpu().numpy(),
             inside=bool(((lay >= st.slab.x0) & (lay < st.slab.x1)).all()), n=st.n,
             sent=(st.last_metrics or {}).get("sent", -1))
    dist.barrier()
    st.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("full", [False, True])
def test_sharded_state_steps_across_processes(tmp_path, full):
    """ShardedState on 2 ranks sharing one GPU (gloo control, CUDA IPC peer
    blocks): after steps with migration every particle is owned by exactly one
    rank, lies in its slab, and the densities equal the global oracle's."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n, world = 1 << 16, 2
    mp.spawn(_state_worker, args=(world, port, str(tmp_path), n, full), nprocs=world, join=True)
    d = [np.load(tmp_path / f"s{r}.npz") for r in range(world)]
    ids = np.concatenate([q["id"] for q in d])
    assert sorted(ids.tolist()) == list(range(n))          # conserved, no duplicates
    assert all(bool(q["inside"]) for q in d)
    assert sum(int(q["n"]) for q in d) == n and all(0 < int(q["n"]) < n for q in d)
    x = np.concatenate([q["x"] for q in d])
    m = np.concatenate([q["m"] for q in d])
    hh = np.concatenate([q["h"] for q in d])
    rho = np.concatenate([q["rho"] for q in d])
    h, nc, cell = grid_for(n)
    want = O.density_cells(x.reshape(-1), m, hh, 0.0, 1.0, cell)
    np.testing.assert_allclose(rho, want.astype(np.float32), rtol=2e-5)


@pytest.mark.parametrize("refine", [1, 2])
def test_uniform_h_and_general_paths_agree(refine):
    """With one smoothing length everywhere the pair loops take the uniform-h
    path (1/h_ij hoisted per home, one float4 load per candidate, m_j w
    accumulated by FFMA); zeroing the block's h-range word [1] ("range
    unknown") forces the general path.  Both match the oracle and each other
    to fp32 summation rounding."""
    n = 1 << 14
    rng = np.random.default_rng(5)
    x = rng.random((n, 3))
    h, nc, cell = grid_for(n)
    hh = np.full(n, h)
    m = rng.uniform(0.5, 1.5, n) / n
    S = _slab_blocks(x, m, hh, nc, cell, 1, refine)[0]
    xt, mt, ht, cs, pos, hs, hmax = S["keep"]
    assert hmax[0].item() == int(np.float32(h).view(np.int32))
    assert (~hmax[1].item()) & 0xffffffff == int(np.float32(h).view(np.uint32))
    args = (n, S["perm"], (0.0, 0.0), cell / refine, nc * refine, nc * refine, nc * refine)
    fast = api.density_cells_blocks([S["block"]], *args, reach=refine).clone()
    v = torch.tensor(rng.uniform(-1, 1, (n, 3)), dtype=torch.float32, device="cuda")
    P = torch.tensor(rng.uniform(0.2, 1.2, n), dtype=torch.float32, device="cuda")
    vel = torch.empty(n, 4, device="cuda")
    api.force_pack(v, fast[:n].contiguous(), P, S["perm"], vel)
    fb = api.force_block(pos, vel, hs, cs, hmax, 0, nc * refine, 0.0)
    fa, fdu = (t.clone() for t in api.force_cells_blocks([fb], *args, reach=refine))
    hmax[1] = 0  # range unknown: the general path
    slow = api.density_cells_blocks([S["block"]], *args, reach=refine)
    sa, sdu = api.force_cells_blocks([fb], *args, reach=refine)
    torch.testing.assert_close(fast, slow, rtol=2e-6, atol=0)
    torch.testing.assert_close(fa, sa, rtol=1e-5, atol=1e-5 * float(sa.abs().max()))
    torch.testing.assert_close(fdu, sdu, rtol=1e-5, atol=1e-5 * float(sdu.abs().max()))
    dec = lambda a: torch.tensor(a, dtype=torch.float32).double().numpy()  # noqa: E731
    want = O.density_cells(dec(x).reshape(-1), dec(m), dec(hh), 0.0, 1.0, cell)
    np.testing.assert_allclose(fast[:n].double().cpu().numpy(), want, rtol=1e-5)
    np.testing.assert_allclose(slow[:n].double().cpu().numpy(), want, rtol=1e-5)


@pytest.mark.parametrize("workload", ["c2", "c5"])
def test_bench_under_torchrun_two_ranks_one_device(workload, tmp_path):
    """bench.py under torchrun with 2 ranks (both on cuda:0 over gloo,
    SFB_BENCH_ONE_DEVICE=1): one JSON line from rank 0, n_gpus = 2, the
    whole-job value over both ranks (C2 at its full 16M per rank, C5 small)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # c2 with extras: at 2 ranks the only extra is the sharded C5 timestep (small here), in the same line
    extra = ["--no-e2e", "--no-cpu", "--c5-n", str(1 << 20)] if workload == "c2" else \
        ["--workload", "c5", "--c5-n", str(1 << 20), "--no-cpu"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(29600 + (workload == "c5")), os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, SFB_BENCH_ONE_DEVICE="1"), cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    if workload == "c2":
        c5 = d["sharded_c5"]
        assert "unavailable" not in c5, c5
        assert c5["n_gpus"] == 2 and c5["value"] > 0 and c5["particles_total"] == 1 << 20
        assert c5["phases_ms_max_over_ranks"]["force"] > 0


@pytest.mark.parametrize("world,refine,spread,clustered", [(1, 2, False, False), (3, 2, True, False),
                                                          (2, 1, False, False), (2, 2, False, True)])
def test_masked_force_after_density_matches_oracle(world, refine, spread, clustered):
    """One step's density writes window masks (sf_b200_density_cells_blocks_masked)
    and the force sweeps exactly the marked pairs (..._force_cells_blocks_masked):
    same rho, and a / du within the force tolerance of the oracle, across
    slabs (peer blocks), with spread h (general pair term) and with clustered
    particles whose dense windows exceed 32 candidates (those homes fall back
    to the window sweep)."""
    n = 1 << 14
    rng = np.random.default_rng(31 + world + refine)
    x = rng.random((n, 3))
    if clustered:  # a tight clump: windows far beyond 32 candidates
        k = n // 8
        x[:k] = np.clip(0.5 + rng.normal(0, 0.004, (k, 3)), 0, 1 - 1e-9)
    h, nc, cell = grid_for(n)
    hh = np.full(n, h) * (rng.uniform(0.85, 1.0, n) if spread else 1.0)
    m = rng.uniform(0.5, 1.5, n) / n
    v = rng.uniform(-1, 1, (n, 3))
    P = rng.uniform(0.2, 1.2, n)
    dec = lambda a: torch.tensor(a, dtype=torch.float32).double().numpy()  # noqa: E731
    S = _slab_blocks(x, m, hh, nc, cell, world, refine)
    rho_all = np.zeros(n)
    masks, vels = [], []
    grid = lambda r: (S[r]["n"], S[r]["perm"], (0.0, 0.0), cell / refine, nc * refine, nc * refine,  # noqa: E731
                      nc * refine)
    for r in range(world):
        blocks = [S[r]["block"]] + [S[q]["block"] for q in (r - 1, r + 1) if 0 <= q < world]
        mk = api.window_masks(S[r]["n"], refine)
        plain = api.density_cells_blocks(blocks, *grid(r), reach=refine).clone()
        rho = api.density_cells_blocks(blocks, *grid(r), reach=refine, masks=mk)
        torch.testing.assert_close(rho, plain, rtol=0, atol=0)  # the masks do not change rho
        rho_all[S[r]["own"]] = rho[:S[r]["n"]].double().cpu().numpy()
        masks.append(mk)
    t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
    for r in range(world):
        own = S[r]["own"]
        vel = torch.empty(S[r]["n"], 4, device="cuda")
        api.force_pack(t(v[own]), t(rho_all[own]), t(P[own]), S[r]["perm"], vel)
        vels.append(vel)
    wa, wdu, sa, sd = O.force_cells(dec(x).reshape(-1), dec(v).reshape(-1), dec(m), dec(hh),
                                    dec(rho_all), dec(P), 0.0, 1.0, cell)
    FORCE_TOL = 2e-5
    for r in range(world):
        fb = lambda q: api.force_block(S[q]["keep"][4], vels[q], S[q]["keep"][5], S[q]["keep"][3],  # noqa: E731
                                       S[q]["keep"][6], S[q]["block"].x0, S[q]["block"].nx,
                                       S[q]["block"].x_origin)
        blocks = [fb(r)] + [fb(q) for q in (r - 1, r + 1) if 0 <= q < world]
        a, du = api.force_cells_blocks(blocks, *grid(r), reach=refine, masks=masks[r])
        pa, pdu = api.force_cells_blocks(blocks, *grid(r), reach=refine)
        own = S[r]["own"]
        a_np, du_np = a[:S[r]["n"]].double().cpu().numpy(), du[:S[r]["n"]].double().cpu().numpy()
        assert np.all(np.linalg.norm(a_np - wa[own], axis=1) <= FORCE_TOL * sa[own])
        assert np.all(np.abs(du_np - wdu[own]) <= FORCE_TOL * sd[own] + 1e-30)
        # the masked and the window sweep agree to summation rounding
        torch.testing.assert_close(a, pa, rtol=1e-4, atol=2e-5 * float(pa.abs().max()))


@pytest.mark.parametrize("seed", range(int(os.environ.get("SFB_RANDOM_MASKED", "4"))))
def test_random_masked_density_force_vs_oracle(seed):
    """Random cases for the window-mask hand-off: particle count, slabs 1-3,
    reach 1 / 2, uniform or spread h, a clustered fraction (windows beyond
    32 candidates); rho with and without masks bit-identical, the masked force
    within the force tolerance of the binary64 oracle."""
    rng = np.random.default_rng(9100 + seed)
    n = int(rng.integers(3000, 24000))
    world, refine = int(rng.integers(1, 4)), int(rng.integers(1, 3))
    x = rng.random((n, 3))
    k = int(n * rng.uniform(0, 0.25))
    if k:
        c = rng.random((3, 3)) * 0.8 + 0.1
        x[:k] = np.clip(c[rng.integers(0, 3, k)] + rng.normal(0, rng.choice([0.003, 0.02]), (k, 3)), 0, 1 - 1e-9)
    h, nc, cell = grid_for(n)
    if nc < 2 * world:
        world = 1
    hh = np.full(n, h) * (rng.uniform(0.8, 1.0, n) if rng.random() < 0.5 else 1.0)
    m = rng.uniform(0.5, 1.5, n) / n
    v, P = rng.uniform(-1, 1, (n, 3)), rng.uniform(0.2, 1.2, n)
    dec = lambda a: torch.tensor(a, dtype=torch.float32).double().numpy()  # noqa: E731
    t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
    S = _slab_blocks(x, m, hh, nc, cell, world, refine)
    grid = lambda r: (S[r]["n"], S[r]["perm"], (0.0, 0.0), cell / refine, nc * refine, nc * refine,  # noqa: E731
                      nc * refine)
    rho_all, masks = np.zeros(n), []
    for r in range(world):
        blocks = [S[r]["block"]] + [S[q]["block"] for q in (r - 1, r + 1) if 0 <= q < world]
        mk = api.window_masks(S[r]["n"], refine)
        plain = api.density_cells_blocks(blocks, *grid(r), reach=refine).clone()
        rho = api.density_cells_blocks(blocks, *grid(r), reach=refine, masks=mk)
        assert torch.equal(rho, plain)
        rho_all[S[r]["own"]] = rho[:S[r]["n"]].double().cpu().numpy()
        masks.append(mk)
    np.testing.assert_allclose(rho_all, O.density_cells(dec(x).reshape(-1), dec(m), dec(hh), 0.0, 1.0, cell),
                               rtol=1e-5)
    vels = []
    for r in range(world):
        own = S[r]["own"]
        vel = torch.empty(S[r]["n"], 4, device="cuda")
        api.force_pack(t(v[own]), t(rho_all[own]), t(P[own]), S[r]["perm"], vel)
        vels.append(vel)
    wa, wdu, sa, sd = O.force_cells(dec(x).reshape(-1), dec(v).reshape(-1), dec(m), dec(hh), dec(rho_all), dec(P),
                                    0.0, 1.0, cell)
    for r in range(world):
        fb = lambda q: api.force_block(S[q]["keep"][4], vels[q], S[q]["keep"][5], S[q]["keep"][3],  # noqa: E731
                                       S[q]["keep"][6], S[q]["block"].x0, S[q]["block"].nx, S[q]["block"].x_origin)
        blocks = [fb(r)] + [fb(q) for q in (r - 1, r + 1) if 0 <= q < world]
        a, du = api.force_cells_blocks(blocks, *grid(r), reach=refine, masks=masks[r])
        own = S[r]["own"]
        a_np, du_np = a[:S[r]["n"]].double().cpu().numpy(), du[:S[r]["n"]].double().cpu().numpy()
        assert np.all(np.linalg.norm(a_np - wa[own], axis=1) <= 2e-5 * sa[own])
        assert np.all(np.abs(du_np - wdu[own]) <= 2e-5 * sd[own] + 1e-30)


def test_masked_density_force_with_ghost_particles():
    """n_home < n: the masks cover the homes only (ghosts feed their
    neighbours) and the masked force writes no ghost."""
    n = 1 << 13
    rng = np.random.default_rng(77)
    x = rng.random((n, 3))
    h, nc, cell = grid_for(n)
    hh, m = np.full(n, h), rng.uniform(0.5, 1.5, n) / n
    v, P = rng.uniform(-1, 1, (n, 3)), rng.uniform(0.2, 1.2, n)
    dec = lambda a: torch.tensor(a, dtype=torch.float32).double().numpy()  # noqa: E731
    S = _slab_blocks(x, m, hh, nc, cell, 1, 2)[0]
    n_home = n - 700  # particle indices >= n_home are ghosts
    geo = (n, S["perm"], (0.0, 0.0), cell / 2, 2 * nc, 2 * nc, 2 * nc)
    mk = api.window_masks(n, 2)
    rho = api.density_cells_blocks([S["block"]], *geo, n_home=n_home, reach=2, masks=mk)
    want = O.density_cells(dec(x).reshape(-1), dec(m), dec(hh), 0.0, 1.0, cell)
    np.testing.assert_allclose(rho[:n_home].double().cpu().numpy(), want[:n_home], rtol=1e-5)
    rho_all = want.astype(np.float32)  # ghosts carry the oracle's rho (as a neighbour rank would)
    t = lambda a: torch.tensor(a, device="cuda", dtype=torch.float32)  # noqa: E731
    vel = torch.empty(n, 4, device="cuda")
    api.force_pack(t(v), t(rho_all), t(P), S["perm"], vel)
    xt, mt, ht, cs, pos, hs, hmax = S["keep"]
    fb = api.force_block(pos, vel, hs, cs, hmax, 0, 2 * nc, 0.0)
    a, du = api.force_cells_blocks([fb], *geo, n_home=n_home, reach=2, masks=mk)
    wa, wdu, sa, sd = O.force_cells(dec(x).reshape(-1), dec(v).reshape(-1), dec(m), dec(hh), dec(rho_all), dec(P),
                                    0.0, 1.0, cell)
    a_np, du_np = a.double().cpu().numpy(), du.double().cpu().numpy()
    assert np.all(np.linalg.norm(a_np[:n_home] - wa[:n_home], axis=1) <= 2e-5 * sa[:n_home])
    assert np.all(np.abs(du_np[:n_home] - wdu[:n_home]) <= 2e-5 * sd[:n_home] + 1e-30)
    assert np.all(a_np[n_home:] == 0) and np.all(du_np[n_home:] == 0)
