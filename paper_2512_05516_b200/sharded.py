"""Cell-sharded SPH step across GPUs (BASELINE C5).

Particles are decomposed into x-slabs of whole cell layers (cells of side
>= 2h, so every neighbour of a particle lies in the 27 surrounding cells).
Rank r owns layers [x0, x1).  One step:

    kick, drift           in place on the rank's SoA buffer (sm_100a kernels)
    migrate               particles whose layer left [x0, x1) move to the
                          neighbouring rank (one neighbour exchange)
    halo                  boundary layers x0 and x1-1 of (x, m, h) go to the
                          left/right neighbours: ncclSend/ncclRecv pairs in
                          one group (torch.distributed batch_isend_irecv)
    density               counting-sort own+ghost particles into the local
                          grid (own layers + one ghost layer each side), then
                          the cell-linked density over the own layers only

`full_step` runs the reference's timestep order instead: density, the
cell-linked force (its halo: the neighbours' (x, h, v, m, P/rho^2)), kick,
drift, migrate.

halo="peer" (default) is a thin caller of the C++ shard behind the C ABI
(sf_b200_shard_*, csrc/shard.cu): the whole step — binning, packing, the
density and force reading the neighbours' packed cell blocks in place
through CUDA IPC peer pointers, kick, drift, and migration through
peer-memory outboxes, ordered between ranks by device-side epoch words —
is one library call; this module only exchanges the 64-byte handles once.
halo="nccl" keeps a Python orchestration that sends ghost rows with NCCL
point-to-point (torch.distributed), for fp16 state and for comparison.

NVSwitch makes every peer equidistant, so slab r simply maps to rank r.  The
exchange uses only neighbour point-to-point traffic; there is no collective
on the data path.  The same code runs with gloo on CPU tensors (tests) with
a pluggable density backend.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import torch

FIELD_DTYPES = {64: torch.float64, 32: torch.float32, 16: torch.float16}


@dataclass
class Slab:
    """x-slab of cell layers owned by one rank."""
    nc: int      # cells per side of the global grid
    cell: float  # cell side (>= 2h)
    rank: int
    world: int

    @property
    def x0(self) -> int:
        return self.rank * self.nc // self.world

    @property
    def x1(self) -> int:
        return (self.rank + 1) * self.nc // self.world

    def layer(self, xcol: torch.Tensor) -> torch.Tensor:
        return torch.clamp(torch.floor(xcol.float() / self.cell), 0, self.nc - 1).to(torch.int32)

    @property
    def local_lo(self) -> int:  # first layer of the local grid (one ghost layer)
        return max(self.x0 - 1, 0)

    @property
    def local_hi(self) -> int:
        return min(self.x1 + 1, self.nc)


def grid_for(n_global: int, neighbours: float = 64.0, multiple: int = 8) -> Tuple[float, int, float]:
    """h with ~`neighbours` particles inside 2h for a uniform unit box, and
    the cell grid: side 1/nc >= 2h, nc rounded down to a multiple of 8 so
    1/2/4/8 ranks get equal slabs (200 cells at 2^27)."""
    h = 0.5 * (3.0 * neighbours / (4.0 * math.pi * n_global)) ** (1.0 / 3.0)
    nc = int(math.floor(1.0 / (2.0 * h)))
    if nc >= 2 * multiple:
        nc -= nc % multiple
    return h, max(nc, 1), 1.0 / max(nc, 1)


def neighbour_exchange(send_left: torch.Tensor, send_right: torch.Tensor, rank: int, world: int,
                       group=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Rows to rank-1 / rank+1; returns rows received from rank-1 / rank+1.
    Counts first, then the payloads, each as one grouped send/recv batch
    (ncclGroupStart; ncclSend/ncclRecv x 4; ncclGroupEnd under NCCL)."""
    import torch.distributed as dist
    dev = send_left.device
    if dev.type == "cuda" and dist.get_backend(group) == "gloo":
        # gloo has no point-to-point for CUDA tensors: stage through the host (tests / CPU fallback
        # of the plumbing only; the NCCL path sends device buffers directly)
        rl, rr = neighbour_exchange(send_left.cpu(), send_right.cpu(), rank, world, group)
        return rl.to(dev), rr.to(dev)
    row = tuple(send_left.shape[1:])
    cnt_out = {d: torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
               for d, t in ((-1, send_left), (1, send_right))}
    cnt_in = {d: torch.zeros(1, dtype=torch.int64, device=dev) for d in (-1, 1)}
    peers = [d for d in (-1, 1) if 0 <= rank + d < world]
    ops = []
    for d in peers:
        ops.append(dist.P2POp(dist.isend, cnt_out[d], rank + d, group))
        ops.append(dist.P2POp(dist.irecv, cnt_in[d], rank + d, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    recv = {d: torch.empty((int(cnt_in[d].item()),) + row, dtype=send_left.dtype, device=dev) for d in (-1, 1)}
    ops = []
    for d in peers:
        out = send_left if d == -1 else send_right
        if out.shape[0]:
            ops.append(dist.P2POp(dist.isend, out.contiguous(), rank + d, group))
        if recv[d].shape[0]:
            ops.append(dist.P2POp(dist.irecv, recv[d], rank + d, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return recv[-1], recv[1]


def halo_rows(x: torch.Tensor, m: torch.Tensor, h: torch.Tensor, slab: Slab):
    """Boundary-layer rows (x0, y, z, m, h) for the left and right neighbours."""
    ix = slab.layer(x[:, 0])
    rows = torch.cat([x, m[:, None], h[:, None]], dim=1)
    left = rows[ix == slab.x0] if slab.rank > 0 else rows[:0]
    right = rows[ix == slab.x1 - 1] if slab.rank < slab.world - 1 else rows[:0]
    return left, right


def exchange_halo(x, m, h, slab: Slab, group=None):
    """Ghost particles (x, m, h) received from the neighbouring slabs."""
    if slab.world == 1:
        return x[:0], m[:0], h[:0]
    left, right = halo_rows(x, m, h, slab)
    gl, gr = neighbour_exchange(left, right, slab.rank, slab.world, group)
    g = torch.cat([gl, gr], dim=0)
    return g[:, 0:3].contiguous(), g[:, 3].contiguous(), g[:, 4].contiguous()


def migrate_rows(rows: torch.Tensor, xcol: torch.Tensor, slab: Slab, group=None) -> torch.Tensor:
    """Particles (one row each, any dtype) whose layer left the slab move to
    the neighbour; returns the rank's new row set (kept + received)."""
    ix = slab.layer(xcol)
    go_l = ix < slab.x0
    go_r = ix >= slab.x1
    keep = ~(go_l | go_r)
    if slab.world == 1:
        return rows
    rl, rr = neighbour_exchange(rows[go_l], rows[go_r], slab.rank, slab.world, group)
    return torch.cat([rows[keep], rl, rr], dim=0)


def exchange_ghost_fields(fields: List[torch.Tensor], xcol: torch.Tensor, slab: Slab, group=None) -> List[torch.Tensor]:
    """Ghost copies of per-particle fields ((n,) or (n,k), one dtype) of the
    neighbours' boundary layers — the force step's halo (x, v, m, h, rho, P
    after the density step has produced rho on every rank)."""
    cols = [f.reshape(f.shape[0], -1) for f in fields]
    if slab.world == 1:
        return [f[:0] for f in fields]
    rows = torch.cat(cols, dim=1)
    ix = slab.layer(xcol)
    left = rows[ix == slab.x0] if slab.rank > 0 else rows[:0]
    right = rows[ix == slab.x1 - 1] if slab.rank < slab.world - 1 else rows[:0]
    gl, gr = neighbour_exchange(left, right, slab.rank, slab.world, group)
    g = torch.cat([gl, gr], dim=0)
    out, c = [], 0
    for f, col in zip(fields, cols):
        k = col.shape[1]
        out.append(g[:, c:c + k].reshape((g.shape[0],) + tuple(f.shape[1:])).contiguous())
        c += k
    return out


DensityFn = Callable[[torch.Tensor, torch.Tensor, torch.Tensor, Slab, int], torch.Tensor]
ForceFn = Callable[..., Tuple[torch.Tensor, torch.Tensor]]


def density_with_ghosts(x, m, h, gx, gm, gh, slab: Slab, backend: DensityFn) -> torch.Tensor:
    """rho of the own particles given the ghosts: own rows come first in the
    combined set, ghosts after; backend(xc, mc, hc, slab, n_own) -> rho[n_own]."""
    if gm.shape[0] == 0:  # single slab: no ghost rows, no copy
        return backend(x, m, h, slab, x.shape[0])
    xc = torch.cat([x, gx.to(x.dtype)], dim=0)
    mc = torch.cat([m, gm.to(m.dtype)], dim=0)
    hc = torch.cat([h, gh.to(h.dtype)], dim=0)
    return backend(xc, mc, hc, slab, x.shape[0])


PHASES: dict = {}  # optional CUDA-event phase log (bench instrumentation)


def _mark(name):
    if PHASES.get("_on"):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        PHASES.setdefault("_events", []).append((name, e))


def local_grid(slab: Slab, refine: int):
    """Binning grid of a rank: own layers plus one ghost layer per side, the
    slab cells split `refine` times per axis."""
    lo_layer, hi_layer = slab.local_lo, slab.local_hi
    cell = slab.cell / refine
    dims = ((hi_layer - lo_layer) * refine, slab.nc * refine, slab.nc * refine)
    return (lo_layer * slab.cell, 0.0, 0.0), cell, dims


def gpu_density_backend(prec: int, refine: int = 2, keep: Optional[dict] = None):
    """bin_particles + density_cells on the rank's local grid (own layers plus
    one ghost layer per side).  Binning cells are the slab cells split
    `refine` times per axis (side >= 2h/refine), searched with reach=refine:
    ~42% fewer candidate pairs at refine 2 than 27 cells of side 2h.  With
    `keep`, the binning is left there for a following force on the same
    own+ghost rows."""
    from . import api

    def run(xc, mc, hc, slab: Slab, n_own: int) -> torch.Tensor:
        lo, cell, dims = local_grid(slab, refine)
        _mark("bin")
        cs, perm = api.bin_particles(xc.float().contiguous(), lo, cell, dims)
        if keep is not None:
            keep.update(cs=cs, perm=perm, n=xc.shape[0])
        _mark("pairs")
        rho = api.density_cells(xc.contiguous(), mc.contiguous(), hc.contiguous(), cs, perm, lo, cell, dims,
                                n_home=n_own, reach=refine, prec=prec)
        _mark("store")
        return rho[:n_own]

    return run


def force_with_ghosts(own: List[torch.Tensor], ghosts: List[torch.Tensor], slab: Slab,
                      backend: ForceFn) -> Tuple[torch.Tensor, torch.Tensor]:
    """(a, du) of the own particles: own rows first, ghosts after;
    backend(x, v, m, h, rho, P, slab, n_own) -> (a[n_own,3], du[n_own])."""
    n_own = own[0].shape[0]
    if ghosts[2].shape[0] == 0:
        return backend(*own, slab, n_own)
    comb = [torch.cat([o, g.to(o.dtype)], dim=0) for o, g in zip(own, ghosts)]
    return backend(*comb, slab, n_own)


def gpu_force_backend(prec: int, refine: int = 2, binning: Optional[dict] = None):
    """bin_particles + force_cells on the rank's local grid (as the density).
    `binning` from the density of the same rows (same positions, same ghost
    rows in the same order) skips the second counting sort."""
    from . import api

    def run(x, v, m, h, rho, P, slab: Slab, n_own: int):
        lo, cell, dims = local_grid(slab, refine)
        if binning and binning.get("n") == x.shape[0]:
            cs, perm = binning["cs"], binning["perm"]
        else:
            cs, perm = api.bin_particles(x.float().contiguous(), lo, cell, dims)
        a, du = api.force_cells(x.contiguous(), v.contiguous(), m.contiguous(), h.contiguous(), rho.contiguous(),
                                P.contiguous(), cs, perm, lo, cell, dims, n_home=n_own, reach=refine, prec=prec)
        return a[:n_own], du[:n_own]

    return run


def _align(v: int, a: int = 256) -> int:
    return (v + a - 1) // a * a


def _handle_exchange(group):
    """All ranks' 64-byte shard handles in rank order, over the process group."""
    import torch.distributed as dist

    def run(mine: bytes):
        every = [None] * dist.get_world_size(group)
        dist.all_gather_object(every, mine, group=group)
        return every
    return run


class ShardedState:
    """One rank's particles: SoA of the reference's default schema at uniform
    storage precision `prec` (32 or 16; positions included).  halo="peer"
    (default, prec 32): the state lives in the C++ shard (api.Shard) and every
    step is one library call; halo="nccl": the Python ghost-row path."""

    NAMES = ["x", "id", "v", "u", "m", "h", "rho", "P", "cs", "a", "du", "dt"]

    def __init__(self, n_global: int, slab: Slab, prec: int = 32, seed: int = 7, device="cuda",
                 h: Optional[float] = None, halo: str = "peer", group=None, refine: int = 2,
                 capacity: Optional[int] = None):
        from . import api
        self.api, self.slab, self.prec, self.device, self.group = api, slab, prec, device, group
        if halo not in ("peer", "nccl"):
            raise ValueError("halo must be 'peer' (neighbour blocks read in place) or 'nccl' (ghost rows sent)")
        if halo == "peer" and prec != 32:
            raise ValueError("the C++ shard holds binary32 state (C5 storage); use halo='nccl' for prec 16")
        self.halo, self.refine = halo, refine
        self.schema = api.Schema.default()
        self.h = h if h is not None else grid_for(n_global)[0]
        # one capacity for every rank (the shards check it when they connect)
        self.capacity = capacity or (3 * n_global) // (2 * slab.world) + (1 << 16)
        self._shard = None
        self.last_metrics = None
        n = n_global // slab.world
        g = torch.Generator(device=device).manual_seed(seed + slab.rank)
        x = torch.rand(n, 3, generator=g, device=device, dtype=torch.float64)
        x[:, 0] = (slab.x0 + x[:, 0] * (slab.x1 - slab.x0)) * slab.cell
        fields = {
            "x": x, "id": torch.arange(n, device=device, dtype=torch.int64) + slab.rank * n,
            "v": torch.rand(n, 3, generator=g, device=device, dtype=torch.float64) * 2 - 1,
            "u": torch.rand(n, generator=g, device=device, dtype=torch.float64) + 0.5,
            "m": torch.full((n,), 1.0 / n_global, device=device, dtype=torch.float64),
            "h": torch.full((n,), self.h, device=device, dtype=torch.float64),
            "rho": torch.ones(n, device=device, dtype=torch.float64),
            "P": torch.zeros(n, device=device, dtype=torch.float64),
            "cs": torch.zeros(n, device=device, dtype=torch.float64),
            "a": torch.rand(n, 3, generator=g, device=device, dtype=torch.float64) * 2 - 1,
            "du": torch.rand(n, generator=g, device=device, dtype=torch.float64) * 2 - 1,
            "dt": torch.full((n,), 1e-3, device=device, dtype=torch.float64),
        }
        self.set_fields(fields)

    # -- buffer plumbing ------------------------------------------------------
    def view(self, n):
        return self.api.View(self.schema, n, "soa", None, self.prec)

    @property
    def n(self) -> int:
        return self._shard.count if self._shard is not None else self._n

    def set_fields(self, fields):
        if self._shard is not None:
            raise RuntimeError("the state already lives in the C++ shard")
        self._binning = None
        n = fields["id"].shape[0]
        self._n = n
        self.buf = self.api.PackedBuffer.empty(self.view(n), self.device)
        for name, t in fields.items():
            _, _, w, _ = self.buf.view.lane(name)
            dt = torch.int64 if name == "id" else FIELD_DTYPES[w]
            self.stream_bytes(name).copy_(t.to(dt).contiguous().view(torch.uint8).reshape(n, -1))

    def shard(self):
        """The C++ shard (created and loaded on first use; halo='peer')."""
        if self._shard is None:
            s = self.slab
            exchange = _handle_exchange(self.group) if s.world > 1 else None
            self._shard = self.api.Shard(s.rank, s.world, s.nc, s.cell, self.refine, self.capacity, exchange)
            self._shard.load(self.buf)
            self.buf = None
        return self._shard

    def stream_bytes(self, name) -> torch.Tensor:
        """The field's stream as (n, bytes per particle) uint8 — valid at any
        offset (the reference SoA packs streams back to back, so e.g. the
        int64 id stream of an odd particle count is not 8-byte aligned)."""
        if self._shard is not None:
            t = self._shard.field(name)
            return t.contiguous().view(torch.uint8).reshape(t.shape[0], -1)
        base, stride, w, ar = self.buf.view.lane(name)
        nbytes = self._n * ar * w // 8
        return self.buf.data[base // 8: base // 8 + nbytes].view(self._n, ar * w // 8)

    def stream(self, name) -> torch.Tensor:
        """Typed view of a field's stream ((n, 3) for x / v / a)."""
        if self._shard is not None:
            return self._shard.field(name)
        base, stride, w, ar = self.buf.view.lane(name)
        dt = torch.int64 if name == "id" else FIELD_DTYPES[w]
        nbytes = self._n * ar * w // 8
        t = self.buf.data[base // 8: base // 8 + nbytes].view(dt)
        return t.view(self._n, ar) if ar == 3 else t

    def rows(self) -> torch.Tensor:
        """All fields of every particle as one byte row (for migration)."""
        return torch.cat([self.stream_bytes(k) for k in self.NAMES], dim=1)

    def from_rows(self, rows: torch.Tensor):
        n = rows.shape[0]
        fields, c = {}, 0
        for k in self.NAMES:
            _, _, w, ar = self.buf.view.lane(k)
            wb = (w // 8) * ar
            b = rows[:, c: c + wb].contiguous()
            c += wb
            dt = torch.int64 if k == "id" else FIELD_DTYPES[w]
            fields[k] = b.view(dt).reshape(n, ar) if ar == 3 else b.view(dt).reshape(n)
        self.set_fields(fields)

    # -- the step ---------------------------------------------------------------
    def _run(self, kernels: str, dt: float = 1e-3, timed: bool = False):
        self.last_metrics = self.shard().step(kernels, dt, timed=timed)
        return self.last_metrics

    def kick_drift(self, dt=1e-3):
        if self.halo == "peer":  # the shard migrates right after the drift
            self._run("kick,drift", dt)
            return
        self._binning = None  # positions change
        self.api.run_kernel(self.buf, "kick", dt, buffer_size=1)
        self.api.run_kernel(self.buf, "drift", dt, buffer_size=1)

    def migrate(self, group=None):
        """Particles whose layer left the slab move to the neighbour (the
        peer-halo shard migrates inside every step; this is the nccl path's).
        Only the leaving particles are packed into rows and sent; the new SoA
        buffer is written in one pass per field (kept particles gathered in
        order, then the received rows)."""
        if self.slab.world == 1 or self.halo == "peer":
            return
        ix = self.slab.layer(self.stream("x")[:, 0])
        go_l, go_r = ix < self.slab.x0, ix >= self.slab.x1
        keep = (~(go_l | go_r)).nonzero().squeeze(1)
        old = {k: self.stream_bytes(k) for k in self.NAMES}
        pack = lambda idx: torch.cat([old[k][idx] for k in self.NAMES], dim=1)  # noqa: E731
        rl, rr = neighbour_exchange(pack(go_l.nonzero().squeeze(1)), pack(go_r.nonzero().squeeze(1)),
                                    self.slab.rank, self.slab.world, group)
        recv = torch.cat([rl, rr], dim=0)
        keep_buf = self.buf  # alive until every field is copied out
        nk = keep.numel()
        self._n = nk + recv.shape[0]
        self.buf = self.api.PackedBuffer.empty(self.view(self._n), self.device)
        self._binning = None
        c = 0
        for k in self.NAMES:
            dst = self.stream_bytes(k)
            wb = dst.shape[1]
            torch.index_select(old[k], 0, keep, out=dst[:nk])
            dst[nk:] = recv[:, c:c + wb]
            c += wb
        del keep_buf

    def density(self, group=None):
        if self.halo == "peer":
            self._run("density")
            return
        x, m, h = self.stream("x"), self.stream("m"), self.stream("h")
        _mark("halo")
        gx, gm, gh = exchange_halo(x, m, h, self.slab, group)
        prec = {32: self.api.SF_PREC_NATIVE, 16: 16}[self.prec]
        self._binning = {}
        rho = density_with_ghosts(x, m, h, gx, gm, gh, self.slab, gpu_density_backend(prec, self.refine,
                                                                                          keep=self._binning))
        self.stream("rho").copy_(rho.to(self.stream("rho").dtype))
        _mark("end")

    def force(self, group=None):
        """Cell-linked force with the neighbours' (x, v, m, h, rho, P) as
        ghosts (second halo, after every rank has its rho)."""
        if self.halo == "peer":
            self._run("force")
            return
        names = ["x", "v", "m", "h", "rho", "P"]
        own = [self.stream(k) for k in names]
        _mark("halo2")
        ghosts = exchange_ghost_fields(own, own[0][:, 0], self.slab, group)
        prec = {32: self.api.SF_PREC_NATIVE, 16: 16}[self.prec]
        a, du = force_with_ghosts(own, ghosts, self.slab, gpu_force_backend(prec, self.refine, binning=self._binning))
        self.stream("a").copy_(a.to(self.stream("a").dtype))
        self.stream("du").copy_(du.to(self.stream("du").dtype))
        _mark("end2")

    def full_step(self, dt=1e-3, group=None, timed: bool = False):
        """The reference timestep order (density -> force -> kick -> drift,
        pipelines.cpp / bench.cpp kernel lists), then migration."""
        if self.halo == "peer":
            return self._run("density,force,kick,drift", dt, timed)
        self.density(group)
        self.force(group)
        self.kick_drift(dt)
        self.migrate(group)
        return None

    def sort_by_cell(self, refine: int = 2):
        """Reorder every field into cell order (the density binning's order),
        before the first step: each step's permutation is then near-identity
        and its gathers stay coherent (the peer-halo shard keeps the order
        itself: its migration rewrites the stayers in cell order)."""
        if self._shard is not None:
            raise RuntimeError("sort_by_cell runs before the first step")
        from . import api
        cell = self.slab.cell / refine
        lo_layer = self.slab.local_lo
        dims = ((self.slab.local_hi - lo_layer) * refine, self.slab.nc * refine, self.slab.nc * refine)
        x = self.stream("x")
        _, perm = api.bin_particles(x.float().contiguous(), (lo_layer * self.slab.cell, 0.0, 0.0), cell, dims)
        p = perm[: self.n].long()
        self.from_rows(self.rows()[p])

    def step(self, dt=1e-3, group=None):
        """kick, drift, migrate, then density of the new positions."""
        self.kick_drift(dt)
        self.migrate(group)
        self.density(group)

    def close(self):
        if self._shard is not None:
            self._shard.close()
            self._shard = None
