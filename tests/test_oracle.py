"""The oracle (oracle/soa_oracle.c + oracle.py) against the reference's golden
vectors (tests/golden/, generated from the unmodified reference by
tests/golden/make_golden.py) and, when oracle/_ref is built, against the
reference library itself on random inputs."""
import ctypes as C
import struct

import numpy as np
import pytest

import oracle as O
from helpers import apply_kernel, compressed_fmts, golden, native_fmts, schema_for


@pytest.fixture(scope="module")
def codec():
    return golden("codec.json")


def test_layout_for_table():
    # acceptance.cpp:32-48
    assert O.layout_for(64) == (1, 11, 52)
    assert O.layout_for(32) == (1, 8, 23)
    assert O.layout_for(16) == (1, 5, 10)
    for t in range(7, 65):
        e = 11 if t >= 33 else 8 if t >= 17 else 5
        assert O.layout_for(t) == (1, e, t - 1 - e)
    with pytest.raises(ValueError):
        O.layout_for(6)


def test_known_answers():
    # test_fpcodec.cpp:33-40, bench.cpp:431-432
    assert O.lib().or_quantize(np.pi, 17) == 3.140625
    assert O.lib().or_quantize(np.pi, 32) == 3.1415927410125732
    assert O.lib().or_quantize(1e300, 20) == float("inf")
    assert np.signbit(O.lib().or_quantize(-0.0, 16))
    assert np.isnan(O.lib().or_quantize(float("nan"), 7))
    # test_sph.cpp:52-63
    assert O.w(0.0, 1.0) == pytest.approx(1 / np.pi, rel=1e-15)
    assert O.w(0.5, 1.0) == pytest.approx(0.71875 / np.pi, rel=1e-15)
    assert O.w(2.0, 1.0) == 0.0


def test_bitpack_known_answer():
    # test_bitpack.cpp:11-18
    buf = np.zeros(2, np.uint8)
    O.lib().or_write_bits(O._p(buf), 7, 3, 0b101)
    assert buf.tolist() == [0x80, 0x02]
    assert O.lib().or_read_bits(O._p(buf), 7, 3) == 0b101


@pytest.mark.parametrize("T", [7, 10, 12, 16, 17, 20, 24, 32, 33, 40, 48, 56, 63, 64])
def test_encode_matches_reference(codec, T):
    x = np.array([int(b, 16) for b in codec["inputs"]], dtype=np.uint64).view(np.float64)
    want = np.array([int(b, 16) for b in codec["encode"][str(T)]], dtype=np.uint64)
    np.testing.assert_array_equal(O.encode(x, T), want)


@pytest.mark.parametrize("em", ["8,7", "5,10", "8,23"])
def test_narrow_matches_reference(codec, em):
    e, m = map(int, em.split(","))
    x = np.array([int(b, 16) for b in codec["inputs"]], dtype=np.uint64).view(np.float64)
    want = np.array([int(b, 16) for b in codec["narrow"][em]], dtype=np.uint64)
    got = np.array([O.lib().or_narrow_to_ieee(float(v), e, m) for v in x], dtype=np.uint64)
    np.testing.assert_array_equal(got, want)


def test_decode_matches_reference(codec):
    pats = np.arange(0, 65536, 7, dtype=np.uint64)
    want16 = np.array([int(b, 16) for b in codec["decode16"]], dtype=np.uint64)
    np.testing.assert_array_equal(O.decode(pats, 16).view(np.uint64), want16)
    wantbf = np.array([int(b, 16) for b in codec["widen_bf16"]], dtype=np.uint64)
    np.testing.assert_array_equal(O.decode(pats, O.OR_BF16).view(np.uint64), wantbf)


def test_layouts_match_reference():
    g = golden("layouts.json")
    for name, (T, ex) in {"default": (0, ""), "t16_xexcl": (16, "x"), "t16_xincl": (16, ""),
                          "t64_xexcl": (64, "x"), "t20": (20, "")}.items():
        S = schema_for(T, ex)
        assert S.record_bits == g[name]["record_bits"], name
        offs = S.offsets()
        for f, off, row in zip(S.fields, offs, g[name]["fields"]):
            assert [off, f.stored_width, f.arity] == row[:3]
    assert schema_for(0).record_bits == 704           # test_schema.cpp:13
    assert schema_for(16, "x").record_bits == 480     # test_schema.cpp:32


SWEEPS = {"default": (0, "", 43), "t16_xexcl": (16, "x", 43), "t16_xincl": (16, "", 43),
          "t64_xexcl": (64, "x", 43), "t32_xexcl": (32, "x", 43),
          "default_ics": (0, "", 0), "t16_xincl_ics": (16, "", 0)}


@pytest.mark.parametrize("name", list(SWEEPS))
def test_kernel_sweeps_match_reference(name):
    g = golden("pipeline.json")
    T, ex, acc = SWEEPS[name]
    want = {k: int(v, 16) for k, v in g["sweeps"][name].items()}
    S = schema_for(T, ex)
    ics = O.random_ics(g["n"], g["seed"], acc, g["dt"])
    aos = O.store_state(ics, S)
    assert aos.checksum() == want["aos"]
    nat = O.transform(aos, "aos", fmts=native_fmts(S))
    soa = O.transform(nat, "soa")
    assert soa.checksum() == want["soa_full"]
    for k in ["drift", "kick", "density"]:
        for layout, buf in [("aos", nat), ("soa", soa)]:
            after = apply_kernel(buf, k, g["dt"])
            packed = O.transform(after, "aos", fmts=compressed_fmts(S))
            assert packed.checksum() == want[f"{k}_{layout}"], (k, layout)
    after = apply_kernel(nat, "density", g["dt"], per_access=True)
    packed = O.transform(after, "aos", fmts=compressed_fmts(S))
    assert packed.checksum() == want["density_aos_peraccess"]


@pytest.mark.parametrize("name", ["t16_xincl", "t16_xexcl", "t32_xincl"])
def test_northstar_composition_matches_reference(name):
    """default AoS -> store_state(T) -> U -> N(k) -> C -> k -> C^T U^T N^T."""
    g = golden("pipeline.json")
    T, ex = {"t16_xincl": (16, ""), "t16_xexcl": (16, "x"), "t32_xincl": (32, "")}[name]
    want = {k: int(v, 16) for k, v in g["northstar"][name].items()}
    S0 = O.default_schema()
    ST = schema_for(T, ex)
    src = O.store_state(O.random_ics(g["n"], g["seed"], 43, g["dt"]), S0)
    st = O.transform(src, "aos", fmts=compressed_fmts(ST), schema=ST)
    assert st.checksum() == want["aos_t"]
    nat = O.transform(st, "aos", fmts=native_fmts(ST))
    assert O.transform(nat, "soa").checksum() == want["soa_full"]
    for k in ["drift", "kick", "density"]:
        soa = O.transform(nat, "soa", subset=ST.subset(k))
        assert soa.checksum() == want[f"{k}_soa"], k
        after = apply_kernel(soa, k, g["dt"])
        assert after.checksum() == want[f"{k}_soa_after"], k
        merged = O.transform(st, "aos")
        O.merge_into(after, merged, ST.kernels[k][1])
        assert merged.checksum() == want[f"{k}_merged_t"], k


def test_survey_goldens():
    """SURVEY §8c tables (recorded from the reference during the survey)."""
    S0 = O.default_schema()
    src = O.store_state(O.random_ics(4096, 42), S0)
    assert src.checksum() == 0xb5bdc583f81920d5
    S16 = schema_for(16)
    st = O.transform(src, "aos", fmts=compressed_fmts(S16), schema=S16)
    soa = O.transform(st, "soa", subset=S16.subset("drift"))
    assert soa.checksum() == 0x0635880f517e24e8
    after = apply_kernel(soa, "drift")
    assert after.checksum() == 0x6fab44d025d6f18c
    O.merge_into(after, src, ["x"])
    assert src.checksum() == 0xb95ebdfd606469ca


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
def test_random_values_against_live_reference():
    R = O.RefLib()
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 2 ** 64, size=20000, dtype=np.uint64)
    x = bits.view(np.float64).copy()
    for T in [9, 16, 21, 32, 45, 64]:
        want = np.zeros(x.size, np.uint64)
        R.L.ref_encode_array(O._p(x), x.size, T, O._p(want))
        np.testing.assert_array_equal(O.encode(x, T), want)
    want = np.zeros(x.size, np.uint64)
    R.L.ref_narrow_array(O._p(x), x.size, 8, 7, O._p(want))
    np.testing.assert_array_equal(O.encode(x, O.OR_BF16), want)


def _t64_records(x, v, m, h, rho, P):
    """The default schema at T=64, x included (every field binary64, id i64):
    144-B records in declaration order x3 id v3 u m h rho P cs a3 du dt."""
    n = len(m)
    rec = np.zeros((n, 18), np.float64)
    rec[:, 0:3] = x
    rec[:, 3] = np.arange(n, dtype=np.int64).view(np.float64)
    rec[:, 4:7] = v
    rec[:, 7] = 1.0
    rec[:, 8], rec[:, 9], rec[:, 10], rec[:, 11] = m, h, rho, P
    rec[:, 12] = 1.0
    return rec


def _cells_case(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3))
    h0 = 0.5 * (3 * 64 / (4 * np.pi * n)) ** (1 / 3)
    h = h0 * rng.uniform(0.8, 1.2, n)
    m = rng.uniform(0.5, 1.5, n) / n
    v = rng.uniform(-1, 1, (n, 3))
    nc = int(np.floor(1.0 / (2 * h.max())))
    return x, v, m, h, 1.0 / nc


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
def test_cell_oracles_pinned_to_reference_all_pairs():
    """The cell-linked restatements (27 cells of side >= 2 h_max, ascending j)
    equal the reference's own density_kernel / force_kernel run over ONE buffer
    holding every particle (all pairs, sph.cpp:176-245): the terms beyond the
    support are exact zeros, so the sums agree bit for bit."""
    R = O.RefLib()
    n = 2048
    x, v, m, h, cell = _cells_case(n, 11)
    rng = np.random.default_rng(12)
    P = rng.uniform(0.5, 1.5, n)
    rec = _t64_records(x, v, m, h, np.ones(n), P)
    hb = R._chk(R.L.ref_buf_from_bytes(None, 64, b"", n, rec.ctypes.data_as(C.c_void_p), rec.nbytes))
    R.run_kernel(hb, "density", bs=n)
    out = R.bytes(hb).view(np.float64).reshape(n, 18)
    rho = O.density_cells(x.reshape(-1), m, h, 0.0, 1.0, cell)
    assert np.array_equal(out[:, 10], rho)
    # force on the reference's own densities
    R.run_kernel(hb, "force", bs=n)
    out = R.bytes(hb).view(np.float64).reshape(n, 18)
    a, du, sa, sd = O.force_cells(x.reshape(-1), v.reshape(-1), m, h, rho, P, 0.0, 1.0, cell)
    assert np.array_equal(out[:, 13:16], a) and np.array_equal(out[:, 16], du)
    assert np.all(sa > 0) and np.all(sd >= 0)
    R.free(hb)


def test_cell_oracle_subsets_equal_full_population():
    """or_density_cells_at / or_force_cells_at (the large-size parity
    checkers) equal the full-population oracle at the listed homes."""
    rng = np.random.default_rng(4)
    n = 4000
    x = rng.random((n, 3)).reshape(-1)
    m, h = rng.uniform(0.5, 1.5, n) / n, rng.uniform(0.04, 0.06, n)
    v, rho, P = rng.uniform(-1, 1, 3 * n), rng.uniform(0.5, 1.5, n), rng.uniform(0.2, 1.0, n)
    homes = rng.choice(n, 300, replace=False)
    full = O.density_cells(x, m, h, 0.0, 1.0, 0.125)
    np.testing.assert_array_equal(O.density_cells_at(x, m, h, 0.0, 1.0, 0.125, homes), full[homes])
    fa = O.force_cells(x, v, m, h, rho, P, 0.0, 1.0, 0.125)
    sa = O.force_cells_at(x, v, m, h, rho, P, 0.0, 1.0, 0.125, homes)
    for a, b in zip(fa, sa):
        np.testing.assert_array_equal(a[homes], b)
