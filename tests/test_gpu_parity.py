"""GPU parity: libsoaforge_b200.so (called through its C ABI) against the
oracle and the reference's golden checksums.  Bit-exact for every layout /
precision conversion and for fp64-exact kick/drift/density; stated
tolerances for the fp32 math mode and the cell-linked density."""
import copy
import os

import numpy as np
import pytest
import torch

import oracle as O
from helpers import apply_kernel, compressed_fmts, golden, native_fmts, schema_for

from paper_2512_05516_b200 import api

pytestmark = pytest.mark.gpu

G = golden("pipeline.json") if True else None


def dev(ob: O.Buffer, view: api.View) -> api.PackedBuffer:
    return api.PackedBuffer.from_host(view, ob.data)


def host(pb: api.PackedBuffer) -> np.ndarray:
    torch.cuda.synchronize()
    return pb.to_host()


def csum(pb: api.PackedBuffer) -> int:
    return O.checksum(host(pb), pb.view.nbytes * 8 if pb.view.nbytes else 0)


def csum_bits(pb: api.PackedBuffer, bits: int) -> int:
    return O.checksum(host(pb), bits)


def default_aos(n=None, seed=None, accel=43):
    n = n or G["n"]
    seed = seed or G["seed"]
    S0 = O.default_schema()
    ob = O.store_state(O.random_ics(n, seed, accel, G["dt"]), S0)
    P = api.Schema.default()
    return ob, P, dev(ob, api.View(P, n, "aos"))


# ----------------------------------------------------------- golden pipelines
@pytest.mark.parametrize("name", ["t16_xincl", "t16_xexcl", "t32_xincl"])
def test_northstar_composition_goldens(name):
    T, ex = {"t16_xincl": (16, ""), "t16_xexcl": (16, "x"), "t32_xincl": (32, "")}[name]
    want = {k: int(v, 16) for k, v in G["northstar"][name].items()}
    _, P, src = default_aos()
    n = G["n"]
    # store_state(T) on the device: default AoS -> T-bit AoS
    aos_t = api.convert(src, api.View(P, n, "aos", None, api.SF_PREC_PACKED + T, ex))
    assert csum(aos_t) == want["aos_t"]
    full = api.gather(src, api.View(P, n, "soa", None, T, ex))
    assert csum(full) == want["soa_full"]
    for k in ["drift", "kick", "density"]:
        v = api.View(P, n, "soa", k, T, ex)
        soa = api.gather(src, v)
        assert csum(soa) == want[f"{k}_soa"], k
        api.run_kernel(soa, k, G["dt"])
        assert csum(soa) == want[f"{k}_soa_after"], k
        merged = api.convert(src, aos_t.view)
        api.widen_merge(soa, merged, k)
        assert csum(merged) == want[f"{k}_merged_t"], k
        if k != "density":
            fused = api.gather_kernel(src, v, k, G["dt"])
            assert csum(fused) == want[f"{k}_soa_after"], k


def test_survey_golden_c2_path():
    """drift-set SoA 0635880f517e24e8, after drift 6fab44d025d6f18c,
    default AoS after exact x scatter-back b95ebdfd606469ca."""
    _, P, src = default_aos(accel=0)
    v = api.View(P, 4096, "soa", "drift", 16)
    assert csum(api.gather(src, v)) == 0x0635880f517e24e8
    fused = api.gather_kernel(src, v, "drift", 1e-3)
    assert csum(fused) == 0x6fab44d025d6f18c
    api.widen_merge(fused, src, "drift")
    assert csum(src) == 0xb95ebdfd606469ca


SWEEPS = {"default": (0, "", 43), "t16_xexcl": (16, "x", 43), "t16_xincl": (16, "", 43),
          "t64_xexcl": (64, "x", 43), "t32_xexcl": (32, "x", 43), "default_ics": (0, "", 0)}


@pytest.mark.parametrize("name", list(SWEEPS))
def test_kernel_sweep_goldens(name):
    """bench kernels composition (bench.cpp:269-316) on AoS and SoA, in place."""
    T, ex, acc = SWEEPS[name]
    want = {k: int(v, 16) for k, v in G["sweeps"][name].items()}
    S = schema_for(T, ex)
    P = api.Schema(S.text())
    n = G["n"]
    ob = O.store_state(O.random_ics(n, G["seed"], acc, G["dt"]), S)
    aos = dev(ob, api.View(P, n, "aos"))
    assert csum(aos) == want["aos"]
    nat = api.convert(aos, api.View(P, n, "aos", None, api.SF_PREC_NATIVE))
    soa = api.gather(aos, api.View(P, n, "soa", None, api.SF_PREC_NATIVE))
    assert csum(soa) == want["soa_full"]
    packed_view = api.View(P, n, "aos")
    for k in ["drift", "kick", "density", "force", "density,force"]:
        for layout, buf in [("aos", nat), ("soa", soa)]:
            work = api.PackedBuffer(buf.view, buf.data.clone())
            for kk in k.split(","):
                api.run_kernel(work, kk, G["dt"])
            assert csum(api.convert(work, packed_view)) == want[f"{k}_{layout}"], (k, layout)
    for k in ["density", "force"]:
        work = api.PackedBuffer(nat.view, nat.data.clone())
        api.run_kernel(work, k, G["dt"], per_access=True)
        assert csum(api.convert(work, packed_view)) == want[f"{k}_aos_peraccess"], k


# ----------------------------------------------------------- codec coverage
def random_bits_schema():
    return O.Schema("bits", [O.Field("p", "f64", 3), O.Field("q", "f32", 3), O.Field("k", "i64"),
                             O.Field("r", "f32")], {"all": (["p", "q", "k", "r"], [])})


@pytest.mark.parametrize("prec", [16, api.SF_PREC_BF16, 12, 20, 24, 33, 40, 64])
def test_random_bit_patterns_bit_exact(prec):
    """10^6 random lanes incl. NaN payloads, +-inf, subnormals, huge values."""
    S = random_bits_schema()
    n = 1 << 17  # 8 float lanes per record -> ~1.05 M lanes
    rng = np.random.default_rng(prec)
    ob = O._alloc(S, n, "aos", range(4), [f.fmt() for f in S.fields])
    ob.data[:] = rng.integers(0, 256, size=ob.data.size, dtype=np.uint8)
    # salt with special values
    specials64 = np.array([0x7ff8000000000000, 0xfff0000000000001, 0x7ff0000000000000, 1, 0x8000000000000001,
                           0x000fffffffffffff, 0x3f10000000000000, 0x40f0000000000000, 0x47f0000000000000],
                          dtype=np.uint64)
    p_bits = ob.field_bits("p")
    p_bits[: specials64.size * 100] = np.tile(specials64, 100)
    from helpers import set_field  # noqa: F401
    O._write_field_bits(ob, 0, p_bits)
    P = api.Schema(S.text())
    src = dev(ob, api.View(P, n, "aos"))
    fmt_of = (lambda f: O.OR_BF16) if prec == api.SF_PREC_BF16 else (lambda f: O.NATIVE(prec))
    fmts = [fmt_of(f) if f.is_float else O.OR_I64 for f in S.fields]
    want = O.transform(ob, "soa", fmts=fmts)
    got = api.gather(src, api.View(P, n, "soa", None, prec))
    np.testing.assert_array_equal(host(got), want.data)
    # generic (non-tiled) kernel, AoS -> AoS
    want_aos = O.transform(ob, "aos", fmts=fmts)
    got_aos = api.convert(src, api.View(P, n, "aos", None, prec))
    np.testing.assert_array_equal(host(got_aos), want_aos.data)


def test_bit_packed_truncated_schema():
    """Non-byte-aligned @truncate widths: tiled gather from a bit-packed AoS
    and scatter-merge back into it (bit-level atomics path)."""
    S = O.Schema("tp", [O.Field("x", "f64", 3, 40), O.Field("id", "i64"), O.Field("v", "f32", 3, 20),
                        O.Field("u", "f32", 1, 12), O.Field("m", "f32", 1, 17)],
                 {"drift": (["x", "v"], ["x"]), "kick2": (["u", "m"], ["u"])})
    n = 3001
    ics = O.random_ics(n, 5, 7)
    ob = O.store_state(ics, S)
    P = api.Schema(S.text())
    assert P.record_bits == S.record_bits == 3 * 40 + 64 + 60 + 12 + 17
    src = dev(ob, api.View(P, n, "aos"))
    for access in [None, "drift"]:
        want = O.transform(ob, "soa", subset=S.subset(access), fmts=[S.fields[i].fmt(True) for i in S.subset(access)])
        got = api.gather(src, api.View(P, n, "soa", access, api.SF_PREC_NATIVE))
        np.testing.assert_array_equal(host(got), want.data)
    soa = api.gather(src, api.View(P, n, "soa", "drift", api.SF_PREC_NATIVE))
    api.run_kernel(soa, "drift", 1e-3, buffer_size=1)
    ref_soa = apply_kernel(O.transform(ob, "soa", subset=S.subset("drift"),
                                       fmts=[S.fields[i].fmt(True) for i in S.subset("drift")]), "drift")
    np.testing.assert_array_equal(host(soa), ref_soa.data)
    api.widen_merge(soa, src, "drift")
    merged = copy.deepcopy(ob)
    O.merge_into(ref_soa, merged, ["x"])
    np.testing.assert_array_equal(host(src), merged.data)


@pytest.mark.parametrize("n", [1, 7, 127, 128, 129, 1000, 4101, 20000])
def test_ragged_counts(n):
    """Partial tiles, sub-16-byte tails, single records."""
    ob, P, src = default_aos(n=n)
    S16 = schema_for(16)
    st = O.transform(ob, "aos", fmts=compressed_fmts(S16), schema=S16)
    want = O.transform(st, "soa", subset=S16.subset("drift"))
    v = api.View(P, n, "soa", "drift", 16)
    np.testing.assert_array_equal(host(api.gather(src, v)), want.data)
    after = apply_kernel(want, "drift")
    fused = api.gather_kernel(src, v, "drift", 1e-3)
    np.testing.assert_array_equal(host(fused), after.data)
    api.widen_merge(fused, src, "drift")
    O.merge_into(after, ob, ["x"])
    np.testing.assert_array_equal(host(src), ob.data)


def test_zero_records():
    P = api.Schema.default()
    src = api.PackedBuffer.empty(api.View(P, 0, "aos"))
    out = api.gather(src, api.View(P, 0, "soa", "drift", 16))
    api.run_kernel(out, "drift", 1e-3, buffer_size=1)
    torch.cuda.synchronize()


def test_kick_fused_and_bf16():
    ob, P, src = default_aos(n=8192)
    for prec, fmt in [(api.SF_PREC_BF16, O.OR_BF16), (16, O.NATIVE(16)), (32, O.NATIVE(32))]:
        S = O.default_schema()
        sub = S.subset("kick")
        ref = apply_kernel(O.transform(ob, "soa", subset=sub, fmts=[fmt] * len(sub)), "kick")
        got = api.gather_kernel(src, api.View(P, 8192, "soa", "kick", prec), "kick", 1e-3)
        np.testing.assert_array_equal(host(got), ref.data)


def test_fp32_math_within_one_storage_ulp():
    ob, P, src = default_aos(n=1 << 16)
    v = api.View(P, 1 << 16, "soa", "drift", 16)
    exact = api.gather_kernel(src, v, "drift", 1e-3, api.SF_MATH_FP64_EXACT)
    fast = api.gather_kernel(src, v, "drift", 1e-3, api.SF_MATH_FP32)
    a = host(exact)[: v.nbytes].view(np.float16).astype(np.float64)
    b = host(fast)[: v.nbytes].view(np.float16).astype(np.float64)
    assert np.all(np.abs(a - b) <= np.abs(a) * 2.0 ** -10 + 2.0 ** -24)


# ----------------------------------------------------------- full-size properties
def test_c2_full_size_roundtrip_properties():
    """16M particles (BASELINE configs[1]): size-independent properties."""
    n = 1 << 24
    P = api.Schema.default()
    aos_v = api.View(P, n, "aos")
    g = torch.Generator(device="cuda").manual_seed(1)
    src = api.PackedBuffer.empty(aos_v)
    # synthetic f64/f32 records: random finite values in [-4, 4)
    f = torch.rand(n, 22, device="cuda", generator=g, dtype=torch.float32) * 8 - 4
    rec = src.data[: aos_v.nbytes].view(n, 88)
    rec[:, 0:24] = f[:, 0:3].double().contiguous().view(torch.uint8).view(n, 24)
    rec[:, 24:32] = torch.arange(n, device="cuda", dtype=torch.int64).view(torch.uint8).view(n, 8)
    rec[:, 32:88] = f[:, 3:17].contiguous().view(torch.uint8).view(n, 56)
    orig = src.data.clone()
    # lossless U∘N∘C then C^T: identity on the full record
    soa = api.gather(src, api.View(P, n, "soa", None, api.SF_PREC_NATIVE))
    back = api.convert(soa, aos_v)
    assert torch.equal(back.data[: aos_v.nbytes], orig[: aos_v.nbytes])
    # narrowing is idempotent: gather(T16) == gather(T16 of the T16 AoS)
    v16 = api.View(P, n, "soa", "drift", 16)
    s1 = api.gather(src, v16)
    aos16 = api.convert(src, api.View(P, n, "aos", None, 1016))
    s2 = api.gather(aos16, v16)
    assert torch.equal(s1.data, s2.data)
    # fused drift == gather then drift
    fused = api.gather_kernel(src, v16, "drift", 1e-3)
    api.run_kernel(s1, "drift", 1e-3, buffer_size=1)
    assert torch.equal(fused.data, s1.data)
    # scatter-back of x only: every other byte of the record is untouched
    api.widen_merge(fused, src, "drift")
    recs = src.data[: aos_v.nbytes].view(n, 88)
    o = orig[: aos_v.nbytes].view(n, 88)
    assert torch.equal(recs[:, 24:], o[:, 24:])
    x16 = fused.data[: n * 6].view(torch.float16).view(n, 3)
    assert torch.equal(recs[:, :24].contiguous().view(torch.float64).view(n, 3), x16.double())


# ----------------------------------------------------------- cell density
@pytest.mark.parametrize("prec", [api.SF_PREC_NATIVE, 16, api.SF_PREC_BF16])
@pytest.mark.parametrize("refine", [1, 2])
def test_density_cells_vs_oracle(prec, refine):
    n = 1 << 15
    rng = np.random.default_rng(3)
    x = rng.random((n, 3))
    h = np.full(n, 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3)) * rng.uniform(0.8, 1.2, n)
    m = rng.uniform(0.5, 1.5, n) / n
    dt = {api.SF_PREC_NATIVE: torch.float32, 16: torch.float16, api.SF_PREC_BF16: torch.bfloat16}[prec]
    xt = torch.tensor(x, device="cuda").to(dt)
    mt = torch.tensor(m, device="cuda").to(dt)
    ht = torch.tensor(h, device="cuda").to(dt)
    nc = int(np.floor(1.0 / float(2 * ht.float().max())))
    cell = 1.0 / nc / refine
    dims = (nc * refine,) * 3
    cs, perm = api.bin_particles(xt.float().contiguous(), (0, 0, 0), cell, dims)
    rho = api.density_cells(xt, mt, ht, cs, perm, (0, 0, 0), cell, dims, reach=refine, prec=prec)
    # oracle on exactly the stored (decoded) inputs, binary64
    xd, md, hd = (t.double().cpu().numpy() for t in (xt, mt, ht))
    want = O.density_cells(xd.reshape(-1), md, hd, 0.0, 1.0, 1.0 / nc)
    np.testing.assert_allclose(rho.double().cpu().numpy(), want, rtol=1e-5, atol=0)
    # binning is a stable counting sort
    cs_h, perm_h = cs.cpu().numpy(), perm.cpu().numpy()
    assert cs_h[-1] == n and np.all(np.diff(cs_h) >= 0)
    assert sorted(perm_h.tolist()) == list(range(n))
    for c in range(0, len(cs_h) - 1, 97):  # ascending particle index inside each cell
        assert np.all(np.diff(perm_h[cs_h[c]:cs_h[c + 1]]) > 0)


@pytest.mark.parametrize("refine", [3, 4])
def test_cells_reach_3_and_4_vs_oracle(refine):
    """Reach 3 / 4 (49 / 81 neighbour columns: more than one 32-column batch
    per warp group), spread h (the general pair term), density and force."""
    n = 1 << 14
    ts, (xd, vd, md, hd, rd, Pd) = _force_case(n, 40 + refine, api.SF_PREC_NATIVE)
    nc = int(np.floor(1.0 / float(2 * ts[3].max())))
    cell = 1.0 / nc / refine
    dims = (nc * refine,) * 3
    cs, perm = api.bin_particles(ts[0].contiguous(), (0, 0, 0), cell, dims)
    rho = api.density_cells(ts[0], ts[2], ts[3], cs, perm, (0, 0, 0), cell, dims, reach=refine)
    want = O.density_cells(xd.reshape(-1), md, hd, 0.0, 1.0, 1.0 / nc)
    np.testing.assert_allclose(rho.double().cpu().numpy(), want, rtol=1e-5, atol=0)
    a, du = api.force_cells(*ts, cs, perm, (0, 0, 0), cell, dims, reach=refine)
    want_a, want_du, sa, sd = O.force_cells(xd.reshape(-1), vd.reshape(-1), md, hd, rd, Pd, 0.0, 1.0, 1.0 / nc)
    assert np.all(np.linalg.norm(a.double().cpu().numpy() - want_a, axis=1) <= FORCE_TOL * sa)
    assert np.all(np.abs(du.double().cpu().numpy() - want_du) <= FORCE_TOL * sd + 1e-30)


def test_density_cells_homes_and_ghosts():
    """Only the first n_home particles are computed; the rest (ghosts) feed
    their neighbours only and keep rho untouched."""
    n = 1 << 14
    rng = np.random.default_rng(4)
    x = rng.random((n, 3))
    h = np.full(n, 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3))
    m = np.full(n, 1.0 / n)
    nc = int(np.floor(1.0 / (2 * h[0])))
    n_home = n - 3000
    xt, mt, ht = (torch.tensor(a, device="cuda", dtype=torch.float32) for a in (x, m, h))
    cs, perm = api.bin_particles(xt, (0, 0, 0), 1.0 / nc, (nc, nc, nc))
    rho = torch.full((n,), -1.0, device="cuda")
    api.density_cells(xt, mt, ht, cs, perm, (0, 0, 0), 1.0 / nc, (nc, nc, nc), n_home=n_home, rho=rho)
    rho = rho.cpu().numpy()
    want = O.density_cells(x.reshape(-1), m, h, 0.0, 1.0, 1.0 / nc)
    np.testing.assert_allclose(rho[:n_home], want[:n_home], rtol=1e-5)
    assert np.all(rho[n_home:] == -1.0)


# ----------------------------------------------------------- cell force
def _force_case(n, seed, prec):
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3))
    h = np.full(n, 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3)) * rng.uniform(0.8, 1.2, n)
    m = rng.uniform(0.5, 1.5, n) / n
    v = rng.uniform(-1, 1, (n, 3))
    rho = rng.uniform(0.5, 1.5, n)
    P = rng.uniform(0.2, 1.2, n)
    dt = {api.SF_PREC_NATIVE: torch.float32, 16: torch.float16, api.SF_PREC_BF16: torch.bfloat16}[prec]
    ts = [torch.tensor(a, device="cuda").to(dt) for a in (x, v, m, h, rho, P)]
    return ts, [t.double().cpu().numpy() for t in ts]


# Tolerance: binary32 sums of binary32 terms (approximate rcp/rsqrt) vs the
# binary64 oracle on the identical stored inputs.  Forces cancel (a_i is a sum
# of terms of both signs), so the error is bounded relative to the sum of the
# term magnitudes the oracle reports: |a - a_ref| <= 2e-5 * sum_j |a_ij|.
FORCE_TOL = 2e-5


@pytest.mark.parametrize("prec", [api.SF_PREC_NATIVE, 16, api.SF_PREC_BF16])
@pytest.mark.parametrize("refine", [1, 2])
def test_force_cells_vs_oracle(prec, refine):
    n = 1 << 15
    ts, (xd, vd, md, hd, rd, Pd) = _force_case(n, 5, prec)
    nc = int(np.floor(1.0 / float(2 * ts[3].float().max())))
    cell = 1.0 / nc / refine
    dims = (nc * refine,) * 3
    cs, perm = api.bin_particles(ts[0].float().contiguous(), (0, 0, 0), cell, dims)
    a, du = api.force_cells(*ts, cs, perm, (0, 0, 0), cell, dims, reach=refine, prec=prec)
    want_a, want_du, sa, sd = O.force_cells(xd.reshape(-1), vd.reshape(-1), md, hd, rd, Pd, 0.0, 1.0, 1.0 / nc)
    err_a = np.linalg.norm(a.double().cpu().numpy() - want_a, axis=1)
    err_du = np.abs(du.double().cpu().numpy() - want_du)
    assert np.all(err_a <= FORCE_TOL * sa), (err_a / sa).max()
    assert np.all(err_du <= FORCE_TOL * sd + 1e-30), (err_du / np.maximum(sd, 1e-300)).max()
    # not trivially zero: the accelerations are of the order of their scale
    assert np.median(np.linalg.norm(want_a, axis=1) / sa) > 1e-3


def test_force_cells_homes_and_degenerate():
    n = 1 << 14
    ts, (xd, vd, md, hd, rd, Pd) = _force_case(n, 6, api.SF_PREC_NATIVE)
    nc = int(np.floor(1.0 / float(2 * ts[3].max())))
    cs, perm = api.bin_particles(ts[0].contiguous(), (0, 0, 0), 1.0 / nc, (nc, nc, nc))
    n_home = n // 2
    a, du = api.force_cells(*ts, cs, perm, (0, 0, 0), 1.0 / nc, (nc, nc, nc), n_home=n_home)
    want_a, want_du, sa, sd = O.force_cells(xd.reshape(-1), vd.reshape(-1), md, hd, rd, Pd, 0.0, 1.0, 1.0 / nc)
    err = np.linalg.norm(a.double().cpu().numpy() - want_a, axis=1)
    assert np.all(err[:n_home] <= FORCE_TOL * sa[:n_home])
    assert np.all(a.cpu().numpy()[n_home:] == 0) and np.all(du.cpu().numpy()[n_home:] == 0)
    ts[4][17] = 0.0  # rho == 0 anywhere: the reference's domain_error
    with pytest.raises(api.L.SfError, match="rho == 0"):
        api.force_cells(*ts, cs, perm, (0, 0, 0), 1.0 / nc, (nc, nc, nc))


def test_cells_outside_grid_offset_origin_and_empty():
    """Particles beyond the grid clamp into the face cells (binning), whose
    extent the culled windows treat as unbounded; a non-zero origin; n = 0."""
    n = 1 << 14
    rng = np.random.default_rng(9)
    lo, hi = -0.5, 0.5
    x = rng.random((n, 3)) - 0.5
    out = rng.random(n) < 0.05           # 5% pushed up to 0.02 beyond a face
    ax = rng.integers(0, 3, n)
    x[out, ax[out]] = np.where(x[out, ax[out]] > 0, hi, lo) + np.sign(x[out, ax[out]]) * rng.random(out.sum()) * 0.02
    h = np.full(n, 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3)) * rng.uniform(0.9, 1.1, n)
    m = rng.uniform(0.5, 1.5, n) / n
    nc = int(np.floor((hi - lo) / (2 * h.max())))
    cell = (hi - lo) / nc
    xt, mt, ht = (torch.tensor(a, device="cuda", dtype=torch.float32) for a in (x, m, h))
    xd, md, hd = (t.double().cpu().numpy() for t in (xt, mt, ht))
    for refine in (1, 2):
        dims = (nc * refine,) * 3
        cs, perm = api.bin_particles(xt, (lo, lo, lo), cell / refine, dims)
        rho = api.density_cells(xt, mt, ht, cs, perm, (lo, lo, lo), cell / refine, dims, reach=refine)
        want = O.density_cells(xd.reshape(-1), md, hd, lo, hi, (hi - lo) / nc)
        np.testing.assert_allclose(rho.double().cpu().numpy(), want, rtol=1e-5, atol=0)
        v = torch.rand(n, 3, device="cuda") - 0.5
        r32, P = rho.clone(), rho * 0.7
        a, du = api.force_cells(xt, v, mt, ht, r32, P, cs, perm, (lo, lo, lo), cell / refine, dims, reach=refine)
        wa, wdu, sa, sd = O.force_cells(xd.reshape(-1), v.double().cpu().numpy().reshape(-1), md, hd,
                                        r32.double().cpu().numpy(), P.double().cpu().numpy(), lo, hi, (hi - lo) / nc)
        assert np.all(np.linalg.norm(a.double().cpu().numpy() - wa, axis=1) <= FORCE_TOL * sa)
        assert np.all(np.abs(du.double().cpu().numpy() - wdu) <= FORCE_TOL * sd + 1e-30)
    # n = 0: nothing launched, nothing written
    e = torch.zeros(0, 3, device="cuda")
    z = torch.zeros(0, device="cuda")
    cs, perm = api.bin_particles(e, (0, 0, 0), 0.25, (4, 4, 4))
    assert int(cs.cpu()[-1]) == 0
    api.density_cells(e, z, z, cs, perm, (0, 0, 0), 0.25, (4, 4, 4))
    api.force_cells(e, e, z, z, z, z, cs, perm, (0, 0, 0), 0.25, (4, 4, 4))


def test_force_degenerate_state_is_an_error():
    """force with rho == 0 raises like the reference's std::domain_error."""
    n = 128
    ics = O.random_ics(n, 9)
    ics["rho"][:] = 0.0
    S = schema_for(64)
    ob = O.store_state(ics, S)
    P = api.Schema(S.text())
    buf = dev(ob, api.View(P, n, "aos"))
    with pytest.raises(api.L.SfError, match="rho == 0"):
        api.run_kernel(buf, "force", 1e-3, 64)


def test_density_buffer_fp64_matches_oracle_random():
    """Reference-semantics density on random h and masses (exact)."""
    n = 64 * 50
    rng = np.random.default_rng(11)
    ics = O.random_ics(n, 9)
    ics["h"] = rng.uniform(0.05, 0.6, n)
    ics["m"] = rng.uniform(0.1, 2.0, n)
    S = schema_for(64)
    ob = O.store_state(ics, S)
    P = api.Schema(S.text())
    buf = dev(ob, api.View(P, n, "aos"))
    api.run_kernel(buf, "density", 1e-3, 64)
    ref = apply_kernel(ob, "density")
    np.testing.assert_array_equal(host(buf), ref.data)


# ----------------------------------------------------------- host orchestration
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("subset", ["all", "kick"])
def test_run_host_streamed_managed_inplace(mode, subset):
    n = 100000
    ob, P, _ = default_aos(n=n)
    aos_v = api.View(P, n, "aos")
    hb = api.HostBuffer(aos_v.nbytes, 1 if mode in (1, 3) else 0)
    hb.numpy()[:] = ob.data
    kernels = "kick,drift" if subset == "all" else "kick"
    dst = api.View(P, n, "soa", None if subset == "all" else "kick", 16)
    m = api.run_host(aos_v, hb, dst, kernels, 1e-3, chunk=16384, mode=mode)
    if mode == 0:  # zero copy: the lanes the SoA view reads, the write set's lanes back
        assert m["h2d_bytes"] == n * (32 if subset == "kick" else 88)   # kick: v, u, a, du
        assert m["d2h_bytes"] == n * (16 if subset == "kick" else 40)   # v, u (+ x)
    else:
        assert m["h2d_bytes"] == aos_v.nbytes and m["d2h_bytes"] == aos_v.nbytes
    # oracle: T16 SoA of everything, kick then drift, merge v,u,x back (exact widen)
    S = O.default_schema()
    soa = O.transform(ob, "soa", fmts=[O.NATIVE(16) if f.is_float else O.OR_I64 for f in S.fields])
    soa = apply_kernel(soa, "kick")
    if subset == "all":
        soa = apply_kernel(soa, "drift")
    O.merge_into(soa, ob, ["v", "u", "x"] if subset == "all" else ["v", "u"])
    np.testing.assert_array_equal(hb.numpy(), ob.data)
    hb.free()


def test_run_host_streamed_soa_out_drift_span():
    """C2 end to end, zero copy: only x and v (36 of the 88 B) of each record are read over PCIe."""
    n = 50000
    ob, P, src = default_aos(n=n)
    aos_v = api.View(P, n, "aos")
    hb = api.HostBuffer(aos_v.nbytes, 0)
    hb.numpy()[:] = ob.data
    v = api.View(P, n, "soa", "drift", 16)
    hs = api.HostBuffer(v.nbytes, 0)
    m = api.run_host(aos_v, hb, v, "drift", 1e-3, chunk=8192, soa_out=hs)
    assert m["h2d_bytes"] == n * 36 and m["d2h_bytes"] == n * 12
    want = api.gather_kernel(src, v, "drift", 1e-3)
    np.testing.assert_array_equal(hs.numpy()[: v.nbytes], host(want))
    hb.free()
    hs.free()


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("prec", [16, 32])
def test_nan_inf_drift_matches_live_reference(prec):
    """NaN / inf / overflow lanes through store_state(T) -> drift: the GPU
    reproduces the reference's x86 NaN propagation bit for bit."""
    n = 4096
    ob, P, src = default_aos(n=n)
    rec = ob.data.reshape(n, 88)
    rng = np.random.default_rng(5)
    specials64 = np.array([np.nan, -np.nan, np.inf, -np.inf, 1e300, -1e300, 5e-324, 0.0, -0.0])
    nanpay = np.array([0x7ff0000000000001, 0xfff4000000000000, 0x7ff8000000000123], dtype=np.uint64)
    for k in range(0, n, 7):
        lane = int(rng.integers(0, 3))
        v = specials64[k % specials64.size]
        rec[k, 8 * lane: 8 * lane + 8] = np.array([v]).view(np.uint8)
        if k % 3 == 0:
            rec[k, 0:8] = nanpay[k % 3:k % 3 + 1].view(np.uint8)
        vl = np.float32([np.nan, np.inf, -np.inf, 3e38][k % 4])
        rec[k, 32 + 4 * lane: 36 + 4 * lane] = np.array([vl]).view(np.uint8)
    src = dev(ob, api.View(P, n, "aos"))
    R = O.RefLib()
    h = R.L.ref_buf_from_bytes(None, 0, b"", n, O._p(ob.data), ob.data.size)
    assert h
    st = R.restore(h, prec)
    u = R.op(st, "unpack")
    nw = R.op(u, "narrow", "drift")
    so = R.op(nw, "aos_to_soa")
    R.run_kernel(so, "drift", 64, 1e-3)
    want = R.bytes(so)
    got = api.gather_kernel(src, api.View(P, n, "soa", "drift", prec), "drift", 1e-3)
    np.testing.assert_array_equal(host(got), want)
    # generic (non-tiled) path: run_kernel in place on the gathered SoA
    soa = api.gather(src, api.View(P, n, "soa", "drift", prec))
    api.run_kernel(soa, "drift", 1e-3, 64)
    np.testing.assert_array_equal(host(soa), want)
    R.free(h, st, u, nw, so)


def test_cells_non_cubic_grid():
    """A box of 1 x 0.5 x 0.25 on a non-cubic cell grid (nx != ny != nz);
    the oracle's cubic cell list only enumerates candidates, so any grid with
    cells >= 2 h_max must give the same sums."""
    n = 1 << 14
    rng = np.random.default_rng(13)
    x = rng.random((n, 3)) * np.array([1.0, 0.5, 0.25])
    h = np.full(n, 0.5 * (3 * 64 * 0.125 / (4 * np.pi * n)) ** (1 / 3))
    m = np.full(n, 1.0 / n)
    nc = int(np.floor(1.0 / (2 * h[0])))
    cell = 1.0 / nc
    dims = (nc, int(np.ceil(0.5 / cell)), int(np.ceil(0.25 / cell)))
    xt, mt, ht = (torch.tensor(a, device="cuda", dtype=torch.float32) for a in (x, m, h))
    xd, md, hd = (t.double().cpu().numpy() for t in (xt, mt, ht))
    want = O.density_cells(xd.reshape(-1), md, hd, 0.0, 1.0, cell)
    for refine in (1, 2):
        d = tuple(k * refine for k in dims)
        cs, perm = api.bin_particles(xt, (0, 0, 0), cell / refine, d)
        rho = api.density_cells(xt, mt, ht, cs, perm, (0, 0, 0), cell / refine, d, reach=refine)
        np.testing.assert_allclose(rho.double().cpu().numpy(), want, rtol=1e-5)


def test_cells_coincident_particles():
    """Distinct particles at identical positions (r = 0): density counts
    m_j W(0) for each, the force's grad W(0) = 0 (sph.cpp:35-40) — no NaN."""
    n = 1 << 13
    rng = np.random.default_rng(17)
    x = rng.random((n, 3))
    x[1::7] = x[0::7][: len(x[1::7])]   # every 7th pair coincides exactly
    h = np.full(n, 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3))
    m = rng.uniform(0.5, 1.5, n) / n
    v = rng.uniform(-1, 1, (n, 3))
    nc = int(np.floor(1.0 / (2 * h[0])))
    ts = [torch.tensor(a, device="cuda", dtype=torch.float32) for a in (x, v, m, h)]
    xd, vd, md, hd = (t.double().cpu().numpy() for t in ts)
    cs, perm = api.bin_particles(ts[0], (0, 0, 0), 1.0 / nc, (nc, nc, nc))
    rho = api.density_cells(ts[0], ts[2], ts[3], cs, perm, (0, 0, 0), 1.0 / nc, (nc, nc, nc))
    want = O.density_cells(xd.reshape(-1), md, hd, 0.0, 1.0, 1.0 / nc)
    np.testing.assert_allclose(rho.double().cpu().numpy(), want, rtol=1e-5)
    P = rho * 0.6
    a, du = api.force_cells(ts[0], ts[1], ts[2], ts[3], rho, P, cs, perm, (0, 0, 0), 1.0 / nc, (nc, nc, nc))
    assert torch.isfinite(a).all() and torch.isfinite(du).all()
    wa, wdu, sa, sd = O.force_cells(xd.reshape(-1), vd.reshape(-1), md, hd, rho.double().cpu().numpy(),
                                    P.double().cpu().numpy(), 0.0, 1.0, 1.0 / nc)
    assert np.all(np.linalg.norm(a.double().cpu().numpy() - wa, axis=1) <= FORCE_TOL * sa)


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("prec", [16, 32])
def test_nan_inf_kick_matches_live_reference(prec):
    """NaN / inf / overflow in v, u, a, du through store_state(T) -> kick (the
    fused gather's x + y*dt and max(0, .) lanes): bit for bit vs the reference."""
    n = 4096
    ob, P, src = default_aos(n=n)
    rec = ob.data.reshape(n, 88)
    f32 = np.float32([np.nan, -np.nan, np.inf, -np.inf, 3e38, -3e38, 1e-45, 0.0, -0.0])
    for k in range(0, n, 5):
        lane = k % 3
        rec[k, 32 + 4 * lane: 36 + 4 * lane] = f32[k % f32.size: k % f32.size + 1].view(np.uint8)      # v
        rec[k, 68 + 4 * lane: 72 + 4 * lane] = f32[(k + 3) % f32.size:(k + 3) % f32.size + 1].view(np.uint8)  # a
        if k % 2 == 0:
            rec[k, 44:48] = f32[(k + 1) % f32.size:(k + 1) % f32.size + 1].view(np.uint8)   # u
            rec[k, 80:84] = f32[(k + 5) % f32.size:(k + 5) % f32.size + 1].view(np.uint8)   # du
    src = dev(ob, api.View(P, n, "aos"))
    R = O.RefLib()
    h = R.L.ref_buf_from_bytes(None, 0, b"", n, O._p(ob.data), ob.data.size)
    assert h
    st = R.restore(h, prec)
    u = R.op(st, "unpack")
    nw = R.op(u, "narrow", "kick")
    so = R.op(nw, "aos_to_soa")
    R.run_kernel(so, "kick", 64, 1e-3)
    want = R.bytes(so)
    got = api.gather_kernel(src, api.View(P, n, "soa", "kick", prec), "kick", 1e-3)
    np.testing.assert_array_equal(host(got), want)
    R.free(h, st, u, nw, so)


def _random_schema(rng):
    """A random record (test_layout_ops.cpp:31-52 / acceptance.cpp:77-100 in
    spirit): 1-12 fields of f32/f64/i64, arity 1 or 3, some @truncate(7..w)."""
    fields = []
    for i in range(int(rng.integers(1, 13))):
        base = str(rng.choice(["f32", "f64", "i64"]))
        ar = 3 if rng.random() < 0.3 else 1
        trunc = 0
        if base != "i64" and rng.random() < 0.4:
            trunc = int(rng.integers(7, 33 if base == "f32" else 65))
        fields.append(O.Field(f"f{i}", base, ar, trunc))
    names = [f.name for f in fields]
    k = max(1, len(names) // 2)
    reads = sorted(rng.choice(names, size=k, replace=False).tolist())
    writes = [w for w in reads if rng.random() < 0.5 and fields[names.index(w)].base != "i64"] or []
    return O.Schema("rnd", fields, {"k": (reads, writes)})


@pytest.mark.parametrize("seed", range(int(os.environ.get("SFB_RANDOM_SCHEMAS", "24"))))
def test_random_schemas_match_oracle(seed):
    """Random schemas x random bit patterns x every precision code, through
    whichever kernel each plan selects (TMA tiles, many-stream direct loads,
    typed / sector / generic conversions): bit-exact vs the oracle moves."""
    rng = np.random.default_rng(9000 + seed)
    S = _random_schema(rng)
    n = int(rng.integers(1, 3000))
    ob = O._alloc(S, n, "aos", list(range(len(S.fields))), [f.fmt(False) for f in S.fields])
    ob.data[:] = rng.integers(0, 256, ob.data.size, dtype=np.uint8)
    tail = ob.length_bits % 8
    if tail:
        ob.data[-1] &= (1 << tail) - 1
    P = api.Schema(S.text())
    assert P.record_bits == S.record_bits
    src = dev(ob, api.View(P, n, "aos"))
    codes = [(api.SF_PREC_STORED, lambda f: f.fmt(False)), (api.SF_PREC_NATIVE, lambda f: f.fmt(True)),
             (16, lambda f: O.NATIVE(16) if f.is_float else O.OR_I64),
             (api.SF_PREC_BF16, lambda f: O.OR_BF16 if f.is_float else O.OR_I64),
             (api.SF_PREC_PACKED + 12, lambda f: 12 if f.is_float else O.OR_I64)]
    for access in (None, "k"):
        sub = S.subset(access)
        for code, fmt in codes:
            fm = [fmt(S.fields[i]) for i in sub]
            want = O.transform(ob, "soa", subset=sub, fmts=fm)
            got = api.gather(src, api.View(P, n, "soa", access, code))
            np.testing.assert_array_equal(host(got), want.data, err_msg=f"{S.text()} access={access} code={code}")
            if code == api.SF_PREC_STORED and access is None:  # lossless: back to the AoS bit for bit
                back = api.convert(got, api.View(P, n, "aos"))
                np.testing.assert_array_equal(host(back), ob.data)
    # N^T: the access set's write set from a binary16 SoA merged into the stored AoS
    w = S.kernels["k"][1]
    if w:
        sub = S.subset("k")
        narrowed = O.transform(ob, "soa", subset=sub, fmts=[O.NATIVE(16) if S.fields[i].is_float else O.OR_I64
                                                              for i in sub])
        soa = api.gather(src, api.View(P, n, "soa", "k", 16))
        api.widen_merge(soa, src, "k")
        merged = copy.deepcopy(ob)
        O.merge_into(narrowed, merged, w)
        np.testing.assert_array_equal(host(src), merged.data)


def _salted_default(n, seed):
    """The default 88-B AoS with NaN / inf / overflow salted into v, u, a, du
    (and x), so the sequence kernel's exact-rule lanes are exercised."""
    ob, P, _ = default_aos(n=n, seed=seed)
    rec = ob.data.reshape(n, 88)
    f32 = np.float32([np.nan, -np.nan, np.inf, -np.inf, 3e38, -3e38, 1e-45, 0.0, -0.0])
    f64 = np.float64([np.nan, np.inf, -np.inf, 1.7e308, -0.0])
    for k in range(0, n, 7):
        lane = k % 3
        rec[k, 32 + 4 * lane: 36 + 4 * lane] = f32[k % 9: k % 9 + 1].view(np.uint8)              # v
        rec[k, 68 + 4 * lane: 72 + 4 * lane] = f32[(k + 3) % 9:(k + 3) % 9 + 1].view(np.uint8)  # a
        rec[k, 44:48] = f32[(k + 1) % 9:(k + 1) % 9 + 1].view(np.uint8)                          # u
        rec[k, 80:84] = f32[(k + 5) % 9:(k + 5) % 9 + 1].view(np.uint8)                          # du
        if k % 3 == 0:
            rec[k, 8 * lane: 8 * lane + 8] = f64[k % 5: k % 5 + 1].view(np.uint8)                # x
    return ob, P


@pytest.mark.parametrize("prec", [api.SF_PREC_NATIVE, 16, api.SF_PREC_BF16, 32, 12])
@pytest.mark.parametrize("math", [api.SF_MATH_FP64_EXACT, api.SF_MATH_FP32])
@pytest.mark.parametrize("seq", ["kick", "drift", "kick,drift", "drift,kick", "kick,kick", "drift,drift,kick",
                                 "kick,drift,kick"])
def test_kernel_sequence_on_aos_equals_soa_kernels(prec, math, seq):
    """run_kernel(seq) in place on an AoS (one shared-memory pass,
    k_update_rec_tile, for IEEE lanes; the per-kernel loop for bit-packed
    T=12 or more than kMaxSeq ops) = the same kernels one launch each on the
    SoA (k_update_soa / k_convert), bit for bit, NaN / inf salted; n is not a
    multiple of the 256-record tile."""
    n = 50001
    ob, P = _salted_default(n, 11)
    src = dev(ob, api.View(P, n, "aos"))
    aos = api.convert(src, api.View(P, n, "aos", None, prec))
    soa = api.gather(src, api.View(P, n, "soa", None, prec))
    for k in seq.split(","):
        api.run_kernel(soa, k, 1e-3, buffer_size=1, math=math)
    api.run_kernel(aos, seq, 1e-3, buffer_size=1, math=math)
    np.testing.assert_array_equal(host(aos), host(api.convert(soa, aos.view)))


@pytest.mark.parametrize("n", [1, 31, 255, 256, 257, 4097])
def test_kernel_sequence_ragged_tails_and_odd_strides(n):
    """Tile tails (n % 256), a 52-B record (32-B chunks straddle records, the
    stride is not a multiple of 8) and a 16-B-aligned buffer (not 32: the
    per-lane kernels)."""
    S = O.Schema("s36", [O.Field("x", "f32", 3), O.Field("v", "f32", 3), O.Field("id", "i64"),
                          O.Field("u", "f32"), O.Field("a", "f32", 3), O.Field("du", "f32")],
                 {"kick": (["v", "a", "u", "du"], ["v", "u"]), "drift": (["x", "v"], ["x"])})
    assert S.record_bits == 8 * 52
    rng = np.random.default_rng(n)
    ob = O._alloc(S, n, "aos", list(range(len(S.fields))), [f.fmt(False) for f in S.fields])
    ob.data[:] = rng.integers(0, 256, ob.data.size, dtype=np.uint8)
    P = api.Schema(S.text())
    aos = dev(ob, api.View(P, n, "aos"))
    soa = api.gather(aos, api.View(P, n, "soa"))
    for k in ("kick", "drift"):
        api.run_kernel(soa, k, 1e-3, buffer_size=1)
    want = host(api.convert(soa, aos.view))
    api.run_kernel(aos, "kick,drift", 1e-3, buffer_size=1)
    np.testing.assert_array_equal(host(aos), want)
    # the same records 16 B into a larger allocation: not 32-B aligned
    raw = torch.zeros(ob.data.size + 64, dtype=torch.uint8, device="cuda")
    raw[16:16 + ob.data.size] = torch.from_numpy(ob.data).cuda()
    off = api.PackedBuffer(aos.view, raw[16:16 + ob.data.size])
    api.run_kernel(off, "kick,drift", 1e-3, buffer_size=1)
    np.testing.assert_array_equal(host(off), want)


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("prec", [16, 32])
def test_kernel_sequence_matches_live_reference(prec):
    """store_state(T) -> unpack -> run_kernel(kick) -> run_kernel(drift) in the
    reference vs one run_kernel("kick,drift") here, NaN / inf salted."""
    n = 4096
    ob, P = _salted_default(n, 5)
    src = dev(ob, api.View(P, n, "aos"))
    R = O.RefLib()
    h = R.L.ref_buf_from_bytes(None, 0, b"", n, O._p(ob.data), ob.data.size)
    assert h
    st = R.restore(h, prec)
    u = R.op(st, "unpack")
    R.run_kernel(u, "kick", 64, 1e-3)
    R.run_kernel(u, "drift", 64, 1e-3)
    want = R.bytes(u)
    got = api.convert(src, api.View(P, n, "aos", None, prec))
    api.run_kernel(got, "kick,drift", 1e-3)
    np.testing.assert_array_equal(host(got), want)
    R.free(h, st, u)
    with pytest.raises(Exception):
        api.run_kernel(got, "kick,drift", 1e-3, buffer_size=3)  # 3 does not divide 4096: rejected like one call


@pytest.mark.parametrize("n,dims", [(0, (3, 4, 5)), (1, (2, 2, 2)), (5000, (7, 9, 11)), (1 << 20, (100, 100, 100)),
                                    (1 << 20, (260, 260, 260))])
def test_bin_particles_is_a_stable_counting_sort(n, dims):
    """cell_start / perm equal numpy's stable argsort of the x-major cell ids
    (same binary32 formula, clamped at the faces), incl. particles outside the
    grid; the 260^3 grid takes the scan's two-level recursion (> 4096 tiles)."""
    rng = np.random.default_rng(n + dims[0])
    lo = np.float32([-0.1, 0.05, 0.0])
    cell = 1.1 / max(dims)
    x = (rng.random((n, 3)) * 1.3 - 0.15).astype(np.float32)
    if n > 100:
        x[:n // 2] = np.sort(x[:n // 2], axis=0)  # half nearly cell-ordered, half random
    inv = np.float32(1.0) / np.float32(cell)
    c = [np.clip(np.floor((x[:, a] - lo[a]) * inv).astype(np.int64), 0, dims[a] - 1) for a in range(3)]
    cid = (c[0] * dims[1] + c[1]) * dims[2] + c[2]
    want_perm = np.argsort(cid, kind="stable")
    want_start = np.searchsorted(cid[want_perm], np.arange(np.prod(dims) + 1), side="left")
    xt = torch.tensor(x, device="cuda").reshape(max(n, 0), 3)
    cs, perm = api.bin_particles(xt, tuple(float(v) for v in lo), cell, dims)
    np.testing.assert_array_equal(cs.cpu().numpy(), want_start)
    np.testing.assert_array_equal(perm[:n].cpu().numpy(), want_perm)


def test_wide_records_take_the_unstaged_kernels():
    """Records wider than the staged kernels' 384-B limit (424 B: the default
    fields plus fourteen f64x3 padding fields) go through the direct /
    per-lane kernels: gather, the scatter-back, and kick,drift in place stay
    bit-exact vs the oracle and vs the same kernels on the SoA."""
    base = O.default_schema()
    fields = list(base.fields) + [O.Field("pad%d" % i, "f64", 3) for i in range(14)]
    kernels = dict(base.kernels)
    kernels["kd"] = (["x", "v", "a", "u", "du"], ["x", "v", "u"])
    S = O.Schema("wide", fields, kernels)
    assert S.record_bits // 8 > 384
    n = 3001
    rng = np.random.default_rng(77)
    ob = O._alloc(S, n, "aos", list(range(len(S.fields))), [f.fmt(False) for f in S.fields])
    ob.data[:] = rng.integers(0, 256, ob.data.size, dtype=np.uint8)
    P = api.Schema(S.text())
    src = dev(ob, api.View(P, n, "aos"))
    sub = S.subset("drift")
    want = O.transform(ob, "soa", subset=sub, fmts=[O.NATIVE(16) for _ in sub])
    got = api.gather(src, api.View(P, n, "soa", "drift", 16))
    np.testing.assert_array_equal(host(got), want.data)
    merged = copy.deepcopy(ob)
    O.merge_into(want, merged, S.kernels["drift"][1])
    api.widen_merge(got, src, "drift")
    np.testing.assert_array_equal(host(src), merged.data)
    soa = api.gather(src, api.View(P, n, "soa", "kd"))
    for k in ("kick", "drift"):
        api.run_kernel(soa, k, 1e-3, buffer_size=1)
    ref = api.PackedBuffer(src.view, src.data.clone())
    api.widen_merge(soa, ref, "kd")
    api.run_kernel(src, "kick,drift", 1e-3, buffer_size=1)
    np.testing.assert_array_equal(host(src), host(ref))


@pytest.mark.parametrize("shift", [8, 16, 48])
def test_gather_and_scatter_from_shifted_buffers(shift):
    """AoS buffers that start 16 / 48 bytes into an allocation (16-B but not
    32-B aligned): the scatter and in-place kernels hand off to their per-lane
    forms, the same bytes either way.  8 bytes breaks the ABI's 16-B buffer
    alignment and is rejected (SF_INVALID_ARG), never silently misread."""
    n = 20001
    ob, P, src = default_aos(n=n)
    raw = torch.zeros(ob.data.size + 128, dtype=torch.uint8, device="cuda")
    raw[shift:shift + ob.data.size] = torch.from_numpy(ob.data).cuda()
    sh = api.PackedBuffer(src.view, raw[shift:shift + ob.data.size])
    if shift % 16:
        with pytest.raises(ValueError):
            api.gather(sh, api.View(P, n, "soa", "drift", 16))
        return
    for access, prec in ((None, 16), ("drift", api.SF_PREC_BF16), ("kick", 32)):
        dst = api.View(P, n, "soa", access, prec)
        np.testing.assert_array_equal(host(api.gather(sh, dst)), host(api.gather(src, dst)))
    fused = api.gather_kernel(sh, api.View(P, n, "soa", "drift", 16), "drift", 1e-3)
    np.testing.assert_array_equal(host(fused), host(api.gather_kernel(src, api.View(P, n, "soa", "drift", 16),
                                                                      "drift", 1e-3)))
    ref = api.PackedBuffer(src.view, src.data.clone())
    api.widen_merge(fused, ref, "drift")
    api.widen_merge(fused, sh, "drift")
    np.testing.assert_array_equal(host(sh), host(ref))
    api.run_kernel(ref, "kick,drift", 1e-3, buffer_size=1)
    api.run_kernel(sh, "kick,drift", 1e-3, buffer_size=1)
    np.testing.assert_array_equal(host(sh), host(ref))


def _random_kd_schema(rng):
    """kick / drift fields in random order and formats among random extra
    fields (f32/f64, optional @truncate), so the in-place sequence runs on
    every format pair, aligned or bit-packed."""
    def fld(name, ar):
        base = str(rng.choice(["f32", "f64"]))
        trunc = int(rng.integers(10, 33 if base == "f32" else 65)) if rng.random() < 0.25 else 0
        return O.Field(name, base, ar, trunc)
    fields = [fld("x", 3), fld("v", 3), fld("a", 3), fld("u", 1), fld("du", 1)]
    for i in range(int(rng.integers(0, 5))):
        fields.append(O.Field("e%d" % i, str(rng.choice(["f32", "f64", "i64"])), int(rng.choice([1, 3]))))
    order = rng.permutation(len(fields))
    fields = [fields[k] for k in order]
    return O.Schema("kd", fields, {"kick": (["v", "a", "u", "du"], ["v", "u"]), "drift": (["x", "v"], ["x"])})


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(int(os.environ.get("SFB_RANDOM_KD", "16"))))
def test_random_kick_drift_layouts_match_live_reference(seed):
    """run_kernel("kick,drift") in place on a random stored AoS (byte-aligned
    IEEE lanes: the one-pass tile kernel; truncated lanes: the generic path)
    vs the unmodified reference running kick then drift on the same bytes."""
    rng = np.random.default_rng(4000 + seed)
    S = _random_kd_schema(rng)
    n = int(rng.integers(1, 4000))
    ob = O._alloc(S, n, "aos", list(range(len(S.fields))), [f.fmt(False) for f in S.fields])
    vals = rng.standard_normal(ob.data.size // 4 + 1).astype(np.float32)  # finite lanes in every format
    ob.data[:] = vals.view(np.uint8)[: ob.data.size]
    for i, f in enumerate(S.fields):  # finite, representable values in every float lane
        if f.is_float:
            O._write_field_bits(ob, i, O.encode(rng.uniform(-2, 2, n * f.arity), f.fmt(False)))
    tail = ob.length_bits % 8
    if tail:
        ob.data[-1] &= (1 << tail) - 1
    R = O.RefLib()
    h = R._chk(R.L.ref_buf_from_bytes(S.text().encode(), 0, b"", n, O._p(ob.data), ob.data.size))
    R.run_kernel(h, "kick", 1, 1e-3)
    R.run_kernel(h, "drift", 1, 1e-3)
    want = R.bytes(h)
    R.free(h)
    P = api.Schema(S.text())
    src = dev(ob, api.View(P, n, "aos"))
    api.run_kernel(src, "kick,drift", 1e-3, buffer_size=1)
    np.testing.assert_array_equal(host(src), want, err_msg=S.text())


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(int(os.environ.get("SFB_RANDOM_DF", "8"))))
def test_random_density_force_layouts_match_live_reference(seed):
    """Buffer-mode density then force (64-particle buffers, binary64, the
    reference's association order) in place on random stored AoS layouts vs
    the unmodified reference on the same bytes: bit for bit."""
    rng = np.random.default_rng(5000 + seed)

    def fld(name, ar):
        base = str(rng.choice(["f32", "f64"]))
        trunc = int(rng.integers(12, 33 if base == "f32" else 65)) if rng.random() < 0.2 else 0
        return O.Field(name, base, ar, trunc)
    fields = [fld("x", 3), fld("v", 3), fld("m", 1), fld("h", 1), fld("rho", 1), fld("P", 1), fld("a", 3),
              fld("du", 1)]
    for i in range(int(rng.integers(0, 3))):
        fields.append(O.Field("e%d" % i, "i64", 1))
    fields = [fields[k] for k in rng.permutation(len(fields))]
    S = O.Schema("df", fields, {"density": (["x", "m", "h"], ["rho"]),
                                 "force": (["x", "v", "m", "h", "rho", "P"], ["a", "du"])})
    n = 64 * int(rng.integers(1, 40))
    ob = O._alloc(S, n, "aos", list(range(len(S.fields))), [f.fmt(False) for f in S.fields])
    ranges = {"x": (0, 1), "v": (-1, 1), "m": (0.5 / 64, 1.5 / 64), "h": (0.2, 0.6), "rho": (0.5, 1.5),
              "P": (0.1, 1.0), "a": (-1, 1), "du": (-1, 1)}
    for i, f in enumerate(S.fields):
        if f.is_float:
            lo, hi = ranges[f.name]
            O._write_field_bits(ob, i, O.encode(rng.uniform(lo, hi, n * f.arity), f.fmt(False)))
        else:
            O._write_field_bits(ob, i, rng.integers(0, 1 << 62, n, dtype=np.int64).view(np.uint64))
    R = O.RefLib()
    h = R._chk(R.L.ref_buf_from_bytes(S.text().encode(), 0, b"", n, O._p(ob.data), ob.data.size))
    R.run_kernel(h, "density", 64, 1e-3)
    R.run_kernel(h, "force", 64, 1e-3)
    want = R.bytes(h)
    R.free(h)
    P = api.Schema(S.text())
    src = dev(ob, api.View(P, n, "aos"))
    api.run_kernel(src, "density", 1e-3, buffer_size=64)
    api.run_kernel(src, "force", 1e-3, buffer_size=64)
    np.testing.assert_array_equal(host(src), want, err_msg=S.text())


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(int(os.environ.get("SFB_RANDOM_FUSED", "12"))))
def test_random_fused_gather_kernel_matches_live_reference(seed):
    """The north-star composition on random layouts: store_state(T) -> unpack
    -> narrow(k) -> aos_to_soa -> run_kernel(k) in the reference vs one fused
    gather_kernel (T in {16, 24, 32}, k in {kick, drift}), bit for bit."""
    rng = np.random.default_rng(6000 + seed)
    S = _random_kd_schema(rng)
    n = int(rng.integers(1, 3000))
    ob = O._alloc(S, n, "aos", list(range(len(S.fields))), [f.fmt(False) for f in S.fields])
    for i, f in enumerate(S.fields):
        if f.is_float:
            O._write_field_bits(ob, i, O.encode(rng.uniform(-2, 2, n * f.arity), f.fmt(False)))
    T = int(rng.choice([16, 24, 32]))
    k = str(rng.choice(["kick", "drift"]))
    R = O.RefLib()
    h = R._chk(R.L.ref_buf_from_bytes(S.text().encode(), 0, b"", n, O._p(ob.data), ob.data.size))
    st = R.restore(h, T, "", S.text())
    u = R.op(st, "unpack")
    nw = R.op(u, "narrow", k)
    so = R.op(nw, "aos_to_soa")
    R.run_kernel(so, k, 1, 1e-3)
    want = R.bytes(so)
    R.free(h, st, u, nw, so)
    P = api.Schema(S.text())
    src = dev(ob, api.View(P, n, "aos"))
    got = api.gather_kernel(src, api.View(P, n, "soa", k, T), k, 1e-3)
    np.testing.assert_array_equal(host(got), want, err_msg="%s T=%d %s" % (S.text(), T, k))


@pytest.mark.parametrize("layout,prec", [("aos", None), ("soa", None), ("soa", 16), ("aos", api.SF_PREC_NATIVE)])
def test_permute_records(layout, prec):
    """sf_b200_permute: record k of the result = record perm[k], every lane."""
    n = 12345
    ob, P, src = default_aos(n=n)
    v = api.View(P, n, layout, None, api.SF_PREC_STORED if prec is None else prec)
    buf = api.convert(src, v)
    perm = torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)).int()
    out = api.permute(buf, perm)
    back = api.convert(out, api.View(P, n, "aos", None, api.SF_PREC_STORED if prec is None else prec))
    orig = api.convert(buf, back.view)
    rb = back.view.nbytes // n
    np.testing.assert_array_equal(host(back)[: n * rb].reshape(n, rb), host(orig)[: n * rb].reshape(n, rb)[
        perm.cpu().numpy()])


@pytest.mark.parametrize("seed", range(int(os.environ.get("SFB_RANDOM_CELLS", "6"))))
def test_random_cell_density_and_force_vs_oracle(seed):
    """Random cell-linked cases: particle count, h spread (uniform h takes the
    hoisted loop, spread h the general one), a clustered fraction (dense cells,
    long runs), reach 1 / 2 and storage precision; rho within rel 1e-5 and
    a / du within 2e-5 of sum_j |term| of the binary64 oracle."""
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(2000, 20000))
    x = rng.random((n, 3))
    k = int(n * rng.uniform(0, 0.3))  # clustered particles around a few centres
    if k:
        centres = rng.random((4, 3)) * 0.8 + 0.1
        x[:k] = np.clip(centres[rng.integers(0, 4, k)] + rng.normal(0, 0.02, (k, 3)), 0, 1 - 1e-9)
    h0 = 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3)
    spread = float(rng.choice([0.0, 0.1, 0.3]))
    h = np.full(n, h0) * rng.uniform(1 - spread, 1 + spread * 0.2, n) if spread else np.full(n, h0)
    m = rng.uniform(0.5, 1.5, n) / n
    prec = [api.SF_PREC_NATIVE, 16, api.SF_PREC_BF16][int(rng.integers(0, 3))]
    refine = int(rng.integers(1, 3))
    dt = {api.SF_PREC_NATIVE: torch.float32, 16: torch.float16, api.SF_PREC_BF16: torch.bfloat16}[prec]
    v, rho0, P = rng.uniform(-1, 1, (n, 3)), rng.uniform(0.5, 1.5, n), rng.uniform(0.2, 1.2, n)
    ts = [torch.tensor(a, device="cuda").to(dt) for a in (x, v, m, h, rho0, P)]
    xd, vd, md, hd, rd, Pd = (t.double().cpu().numpy() for t in ts)
    nc = int(np.floor(1.0 / float(2 * ts[3].float().max())))
    cell = 1.0 / nc / refine
    dims = (nc * refine,) * 3
    cs, perm = api.bin_particles(ts[0].float().contiguous(), (0, 0, 0), cell, dims)
    rho = api.density_cells(ts[0], ts[2], ts[3], cs, perm, (0, 0, 0), cell, dims, reach=refine, prec=prec)
    want = O.density_cells(xd.reshape(-1), md, hd, 0.0, 1.0, 1.0 / nc)
    np.testing.assert_allclose(rho.double().cpu().numpy(), want, rtol=1e-5, atol=0)
    a, du = api.force_cells(*ts, cs, perm, (0, 0, 0), cell, dims, reach=refine, prec=prec)
    want_a, want_du, sa, sd = O.force_cells(xd.reshape(-1), vd.reshape(-1), md, hd, rd, Pd, 0.0, 1.0, 1.0 / nc)
    assert np.all(np.linalg.norm(a.double().cpu().numpy() - want_a, axis=1) <= FORCE_TOL * sa)
    assert np.all(np.abs(du.double().cpu().numpy() - want_du) <= FORCE_TOL * sd + 1e-30)


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("bs", [616, 1024])
def test_force_large_buffers_match_live_reference(bs):
    """Buffer-mode density + force with buffers above the 48 KB default of
    dynamic shared memory (force stages 80 B per particle): bit for bit."""
    n = bs * 4
    R = O.RefLib()
    h = R.from_ics(n, 42, 0, "", None, 43, 1e-3)
    start = R.bytes(h)
    R.run_kernel(h, "density", bs, 1e-3)
    R.run_kernel(h, "force", bs, 1e-3)
    want = R.bytes(h)
    R.free(h)
    P = api.Schema.default()
    buf = api.PackedBuffer.from_host(api.View(P, n, "aos"), start)
    api.run_kernel(buf, "density", 1e-3, buffer_size=bs)
    api.run_kernel(buf, "force", 1e-3, buffer_size=bs)
    np.testing.assert_array_equal(host(buf), want)
