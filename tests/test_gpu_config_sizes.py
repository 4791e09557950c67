"""Parity at the BASELINE.json config sizes (C1 1M, C2 16M, C3 4M, C4 64M,
C5 128M), through the C ABI, against the pinned oracle or the live
reference:

  C2  the full 16M-record gather (binary16 and bf16), every output byte vs
      the oracle's per-lane rule, with NaN payloads / +-inf / subnormals /
      fp16 overflow salted in; the fused drift vs the oracle with non-NaN
      salting (NaN arithmetic is pinned against the live reference at small
      size in test_gpu_parity.py).
  C1  kick then drift in place on the 1M-record default AoS, bit-exact vs
      the unmodified reference on the same bytes.
  C3  4M uniform particles at grid_for(4M), refine 2, fp32 / fp16 / bf16:
      rho and (a, du) of every home inside sampled sub-boxes (interior and a
      domain corner) vs the oracle over every particle of the sub-box.
  C4  64M host-resident records, every run_host mode: sampled records vs
      the oracle composition (T16 SoA, kick, drift, merge back).
  C5  one 128M-particle N=1 sharded step (density, force, kick, drift):
      sampled homes vs the oracle, kick/drift bit-exact on a sample.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
from helpers import apply_kernel

from paper_2512_05516_b200 import api

pytestmark = pytest.mark.gpu

FORCE_TOL = 2e-5  # |a - a_oracle| <= FORCE_TOL * sum_j |term_j| (test_gpu_parity.py)


def _host(t: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy()


def salted_default_aos(n: int, seed: int, nan: bool):
    """Default 88-B records (f64 x, i64 id, f32 rest), uniform values, with
    ~1% of the x / v lanes replaced by edge values: +-inf, -0, subnormals of
    the destination formats, values overflowing binary16 and (nan=True) NaN
    with random payloads.  x-infinity and v-overflow go to disjoint records,
    so the drift never forms inf - inf."""
    P = api.Schema.default()
    v = api.View(P, n, "aos")
    src = api.PackedBuffer.empty(v)
    rec = src.data[: v.nbytes].view(n, 88)
    g = torch.Generator(device="cuda").manual_seed(seed)
    step = 1 << 22
    for b in range(0, n, step):
        e = min(n, b + step)
        m = e - b
        f = torch.rand(m, 17, device="cuda", generator=g)
        xd = (f[:, 0:3].double() * 4 - 2)
        vf = f[:, 3:6] * 2 - 1
        sel = torch.rand(m, 3, device="cuda", generator=g)
        half = torch.arange(b, e, device="cuda") % 2 == 0  # x edge values on even records, v on odd ones
        xe = torch.tensor([float("inf"), -float("inf"), -0.0, 3e-8, 6.1e-5, 70000.0, 1e-40, 5e-324],
                          device="cuda", dtype=torch.float64)
        ve = torch.tensor([float("inf"), -0.0, 2e-7, 1e5, -65520.0, 1e-39, 3.4e38, 1e-45],
                          device="cuda", dtype=torch.float32)
        kx = torch.randint(0, len(xe), (m, 3), device="cuda", generator=g)
        kv = torch.randint(0, len(ve), (m, 3), device="cuda", generator=g)
        xd = torch.where((sel < 0.01) & half[:, None], xe[kx], xd)
        vf = torch.where((sel < 0.01) & ~half[:, None], ve[kv], vf)
        rec[b:e, 0:24] = xd.contiguous().view(torch.uint8).view(m, 24)
        rec[b:e, 24:32] = torch.arange(b, e, device="cuda", dtype=torch.int64).view(torch.uint8).view(m, 8)
        rest = f[:, 3:17].clone()
        rest[:, 0:3] = vf
        rec[b:e, 32:88] = rest.contiguous().view(torch.uint8).view(m, 56)
        if nan:  # NaN payloads (quiet and signalling) in ~0.2% of the x and v lanes
            w = rec[b:e]
            r = torch.rand(m, 6, device="cuda", generator=g) < 0.002
            pay64 = torch.randint(1, 1 << 51, (m, 3), device="cuda", generator=g, dtype=torch.int64)
            nan64 = (pay64 | 0x7FF0000000000000) | (torch.randint(0, 2, (m, 3), device="cuda", generator=g) << 63)
            xs = w[:, 0:24].contiguous().view(torch.int64).view(m, 3)
            xs = torch.where(r[:, 0:3], nan64, xs)
            w[:, 0:24] = xs.contiguous().view(torch.uint8).view(m, 24)
            pay32 = torch.randint(1, 1 << 22, (m, 3), device="cuda", generator=g, dtype=torch.int32)
            nan32 = pay32 | 0x7F800000 | (torch.randint(0, 2, (m, 3), device="cuda", generator=g,
                                                          dtype=torch.int32) << 31)
            vs = w[:, 32:44].contiguous().view(torch.int32).view(m, 3)
            vs = torch.where(r[:, 3:6], nan32, vs)
            w[:, 32:44] = vs.contiguous().view(torch.uint8).view(m, 12)
    return P, v, src


def _oracle_aos(host_bytes: np.ndarray, n: int) -> O.Buffer:
    S = O.default_schema()
    ob = O._alloc(S, 0, "aos", range(len(S.fields)), [f.fmt(False) for f in S.fields])
    ob.count = n
    ob.data = host_bytes
    return ob


@pytest.mark.parametrize("prec,fmt", [(16, O.NATIVE(16)), (api.SF_PREC_BF16, O.OR_BF16)])
def test_c2_16m_gather_every_byte_vs_oracle(prec, fmt):
    n = 1 << 24
    P, v, src = salted_default_aos(n, 11 if prec == 16 else 12, nan=True)
    dv = api.View(P, n, "soa", "drift", prec)
    got = _host(api.gather(src, dv).data[: dv.nbytes])
    ob = _oracle_aos(_host(src.data[: v.nbytes]), n)
    sub = ob.schema.subset("drift")
    want = O.transform(ob, "soa", subset=sub, fmts=[fmt] * len(sub))
    assert want.data.size == dv.nbytes
    bad = np.nonzero(got != want.data)[0]
    assert bad.size == 0, "first mismatching bytes at %s" % bad[:8]


@pytest.mark.parametrize("prec,fmt", [(16, O.NATIVE(16)), (api.SF_PREC_BF16, O.OR_BF16)])
def test_c2_16m_fused_drift_every_byte_vs_oracle(prec, fmt):
    n = 1 << 24
    P, v, src = salted_default_aos(n, 21 if prec == 16 else 22, nan=False)
    dv = api.View(P, n, "soa", "drift", prec)
    got = _host(api.gather_kernel(src, dv, "drift", 1e-3).data[: dv.nbytes])
    ob = _oracle_aos(_host(src.data[: v.nbytes]), n)
    sub = ob.schema.subset("drift")
    soa = O.transform(ob, "soa", subset=sub, fmts=[fmt] * len(sub))
    want = apply_kernel(soa, "drift", 1e-3)
    bad = np.nonzero(got != want.data)[0]
    assert bad.size == 0, "first mismatching bytes at %s" % bad[:8]


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
def test_c1_1m_kick_drift_vs_live_reference():
    """C1: the reference's own 1M-particle default AoS (seed 42, a/du seeded
    43 so kick is not a no-op), kick then drift in one pass on the GPU vs
    run_kernel_chunked(kick), run_kernel_chunked(drift) in the reference."""
    n = 1 << 20
    R = O.RefLib()
    h = R.from_ics(n, 42, 0, "", None, 43, 1e-3)
    start = R.bytes(h)
    threads = os.cpu_count() or 1
    R.run_kernel(h, "kick", 64, 1e-3, threads=threads)
    R.run_kernel(h, "drift", 64, 1e-3, threads=threads)
    want = R.bytes(h)
    R.free(h)
    P = api.Schema.default()
    buf = api.PackedBuffer.from_host(api.View(P, n, "aos"), start)
    api.run_kernel(buf, "kick,drift", 1e-3, buffer_size=64)
    got = _host(buf.data[: buf.view.nbytes])
    assert not np.array_equal(start, want)
    np.testing.assert_array_equal(got, want)


def _subbox_homes(x: torch.Tensor, lo, side: float, margin: float):
    """Particles inside the cube [lo, lo+side)^3 and, among them, the homes
    whose support lies inside the cube (margin = 2 h_max from every face
    that is not a face of the unit domain)."""
    lo_t = torch.tensor(lo, device=x.device, dtype=x.dtype)
    # a box touching the domain's upper face keeps everything beyond it (fp16 / bf16 positions round up to 1.0)
    hi_t = torch.where(lo_t + side >= 1, torch.full_like(lo_t, float("inf")), lo_t + side)
    inside = ((x >= lo_t) & (x < hi_t)).all(dim=1)
    idx = inside.nonzero().squeeze(1)
    xs = x[idx]
    lo_in = torch.where(lo_t <= 0, torch.full_like(lo_t, -1.0), lo_t + margin)
    hi_in = torch.where(lo_t + side >= 1, torch.full_like(lo_t, 2.0), lo_t + side - margin)
    home = ((xs >= lo_in) & (xs < hi_in)).all(dim=1)
    return idx, home.nonzero().squeeze(1)


def _check_cells_sample(x, m, h, rho, idx, homes, lo, side, v=None, rho_in=None, P=None, a=None, du=None):
    """rho (and a, du) of the homes (indices into the sub-box list idx) vs
    the oracle over every particle of the sub-box."""
    xd = x[idx].double().cpu().numpy()
    md, hd = m[idx].double().cpu().numpy(), h[idx].double().cpu().numpy()
    hn = homes.cpu().numpy().astype(np.uint64)
    cell = float(2.0 * hd.max()) * 1.0001
    glo, ghi = float(min(lo)), float(max(lo)) + side  # one cube around the sub-box (the oracle grid is cubic)
    want = O.density_cells_at(xd.reshape(-1), md, hd, glo, ghi, cell, hn)
    got = rho[idx[homes]].double().cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
    if a is None:
        return len(hn)
    vd, rd, Pd = (t[idx].double().cpu().numpy() for t in (v, rho_in, P))
    wa, wdu, sa, sd = O.force_cells_at(xd.reshape(-1), vd.reshape(-1), md, hd, rd, Pd, glo, ghi, cell, hn)
    ga = a[idx[homes]].double().cpu().numpy()
    gdu = du[idx[homes]].double().cpu().numpy()
    assert np.all(np.linalg.norm(ga - wa, axis=1) <= FORCE_TOL * sa)
    assert np.all(np.abs(gdu - wdu) <= FORCE_TOL * sd + 1e-30)
    return len(hn)


@pytest.mark.parametrize("name,prec,dt", [("fp32", api.SF_PREC_NATIVE, torch.float32),
                                          ("fp16", 16, torch.float16), ("bf16", api.SF_PREC_BF16, torch.bfloat16)])
def test_c3_4m_density_and_force_sampled_vs_oracle(name, prec, dt):
    from paper_2512_05516_b200.sharded import grid_for
    n = 1 << 22
    hh, nc, cell = grid_for(n)
    refine = 2
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(n, 3, generator=g, device="cuda").to(dt)
    m = torch.full((n,), 1.0 / n, device="cuda").to(dt)
    h = torch.full((n,), hh, device="cuda").to(dt)
    vel = (torch.rand(n, 3, generator=g, device="cuda") * 2 - 1).to(dt)
    xf = x.float().contiguous()
    dims = (nc * refine,) * 3
    cs, perm = api.bin_particles(xf, (0, 0, 0), cell / refine, dims)
    rho = api.density_cells(x, m, h, cs, perm, (0, 0, 0), cell / refine, dims, reach=refine, prec=prec)
    rho_s = rho.to(dt)
    pres = (rho * (2.0 / 3.0)).to(dt)
    a, du = api.force_cells(x, vel, m, h, rho_s, pres, cs, perm, (0, 0, 0), cell / refine, dims, reach=refine,
                            prec=prec)
    hmax = float(h.float().max())
    checked = 0
    for lo in ((0.41, 0.37, 0.52), (0.0, 0.0, 0.0), (0.85, 0.0, 0.6)):
        side = 0.15
        idx, homes = _subbox_homes(xf, lo, side, 2 * hmax * 1.001)
        checked += _check_cells_sample(x, m, h, rho, idx, homes, lo, side, vel, rho_s, pres, a, du)
    assert checked > 15000


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_c4_64m_run_host_sampled_vs_oracle(mode):
    n = 1 << 26
    P, v, src = salted_default_aos(n, 40 + mode, nan=False)
    hb = api.HostBuffer(v.nbytes, 1 if mode in (1, 3) else 0)
    host_t = torch.from_numpy(hb.numpy())
    for b in range(0, v.nbytes, 1 << 30):  # device -> pinned / managed host memory, no pageable staging
        e = min(v.nbytes, b + (1 << 30))
        host_t[b:e].copy_(src.data[b:e])
    torch.cuda.synchronize()
    rng = np.random.default_rng(mode)
    k = 200000
    sample = np.sort(rng.choice(n, k, replace=False))
    sample[:3] = [0, n // 2, n - 1]
    rows = hb.numpy()[: v.nbytes].reshape(n, 88)[sample].copy()
    dst = api.View(P, n, "soa", None, 16)
    m = api.run_host(v, hb, dst, "kick,drift", 1e-3, chunk=1 << 21, mode=mode)
    assert m["h2d_bytes"] == v.nbytes
    assert m["d2h_bytes"] == (n * 40 if mode == 0 else v.nbytes)  # streamed: x, v, u written back in place
    # oracle on the sampled records (the step is record-local)
    ob = _oracle_aos(rows.reshape(-1).copy(), k)
    S = ob.schema
    soa = O.transform(ob, "soa", fmts=[O.NATIVE(16) if f.is_float else O.OR_I64 for f in S.fields])
    soa = apply_kernel(apply_kernel(soa, "kick"), "drift")
    O.merge_into(soa, ob, ["v", "u", "x"])
    got = hb.numpy()[: v.nbytes].reshape(n, 88)[sample]
    np.testing.assert_array_equal(got.reshape(-1), ob.data)
    hb.free()


def test_c5_128m_step_sampled_vs_oracle():
    """One N=1 C5 step on 2^27 particles (the reference timestep order):
    density and force of the homes in sampled sub-boxes vs the oracle, then
    kick + drift bit-exact on 10^5 sampled particles."""
    from paper_2512_05516_b200.sharded import ShardedState, Slab, grid_for
    n = 1 << 27
    hh, nc, cell = grid_for(n)
    st = ShardedState(n, Slab(nc, cell, 0, 1), prec=32, h=hh)
    st.sort_by_cell()
    st.density()
    x, m, h = st.stream("x"), st.stream("m"), st.stream("h")
    rho = st.stream("rho")
    checked = 0
    for lo in ((0.31, 0.62, 0.17), (0.0, 0.0, 0.0)):
        side = 0.06
        idx, homes = _subbox_homes(x, lo, side, 2 * hh * 1.001)
        checked += _check_cells_sample(x, m, h, rho, idx, homes, lo, side)
    assert checked > 20000
    # force with an EOS pressure (P = (gamma - 1) rho u), a / du written in place
    st.stream("P").copy_(st.stream("rho") * (2.0 / 3.0) * st.stream("u"))
    st.force()
    a, du = st.stream("a"), st.stream("du")
    lo, side = (0.52, 0.12, 0.77), 0.06
    idx, homes = _subbox_homes(x, lo, side, 2 * hh * 1.001)
    _check_cells_sample(x, m, h, rho, idx, homes, lo, side, st.stream("v"), rho, st.stream("P"), a, du)
    # kick + drift on a sample of particles: binary64 arithmetic, binary32 storage, bit-exact
    g = torch.Generator(device="cuda").manual_seed(9)
    smp = torch.randint(0, st.n, (100000,), device="cuda", generator=g)
    before = {k: st.stream(k)[smp].double().cpu().numpy() for k in ("x", "v", "u", "a", "du")}
    st.kick_drift(1e-3)
    v2, u2 = O.kick(before["v"], before["u"], before["a"], before["du"], 1e-3)
    v2 = O.decode(O.encode(v2, O.NATIVE(32)), O.NATIVE(32)).reshape(-1, 3)
    u2 = O.decode(O.encode(u2, O.NATIVE(32)), O.NATIVE(32))
    x2 = O.decode(O.encode(O.drift(before["x"], v2, 1e-3), O.NATIVE(32)), O.NATIVE(32)).reshape(-1, 3)
    np.testing.assert_array_equal(st.stream("v")[smp].double().cpu().numpy(), v2)
    np.testing.assert_array_equal(st.stream("u")[smp].double().cpu().numpy(), u2)
    np.testing.assert_array_equal(st.stream("x")[smp].double().cpu().numpy(), x2)
