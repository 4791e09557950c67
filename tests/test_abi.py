"""CPU tests of the drop-in boundary (no GPU compute): the C-ABI library
loads, exports every symbol include/soaforge_b200.h declares, and its host
logic (schema DSL, layout math, codec scalars, config keys, views) matches the
reference — the same checks as the reference's test_capi.cpp /
test_schema.cpp, run through libsoaforge_b200.so."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from helpers import golden, schema_for

from paper_2512_05516_b200 import _lib as L
from paper_2512_05516_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "soaforge_b200.h")).read()
    declared = set(re.findall(r"SF_API\s+[\w\s\*]+?\b(sf_\w+)\s*\(", hdr))
    assert len(declared) >= 19 + 15
    lib = C.CDLL(L.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == {s[0] for s in L.SYMBOLS}
    # the 19 reference symbols (soaforge.h:33-82) are all present
    ref19 = {"sf_version", "sf_last_error", "sf_layout_for", "sf_quantize", "sf_schema_parse",
             "sf_schema_destroy", "sf_schema_record_bits", "sf_schema_field_count", "sf_schema_print",
             "sf_config_create", "sf_config_destroy", "sf_config_set_string", "sf_config_set_int",
             "sf_config_set_double", "sf_run_bench_transform", "sf_run_bench_kernels",
             "sf_run_bench_pipeline", "sf_run_study_truncation", "sf_run_validate"}
    assert ref19 <= declared


def test_version_and_errors():  # test_capi.cpp:9-29
    assert api.version()
    assert api.layout_for(32) == (1, 8, 23)
    assert api.quantize(3.14159265358979312, 17) == 3.140625
    with pytest.raises(L.SfInvalidArg):
        api.layout_for(6)
    assert L.lib().sf_last_error()
    with pytest.raises(L.SfInvalidArg):
        api.quantize(1.0, 99)
    e, m = C.c_int(), C.c_int()
    assert L.lib().sf_layout_for(16, None, C.byref(e), C.byref(m)) == L.SF_INVALID_ARG


def test_quantize_matches_reference_codec():
    g = golden("codec.json")
    xs = np.array([int(b, 16) for b in g["inputs"]], dtype=np.uint64).view(np.float64)[:1500]
    for T in [7, 12, 16, 17, 20, 32, 40, 64]:
        want = O.decode(np.array([int(b, 16) for b in g["encode"][str(T)]][:1500], dtype=np.uint64), T)
        got = np.array([api.quantize(float(x), T) for x in xs])
        np.testing.assert_array_equal(got.view(np.uint64), want.view(np.uint64))


def test_schema_handles():  # test_capi.cpp:31-54
    s = api.Schema("schema s { field a : f64 x3; field b : f32 @truncate(20); }")
    assert s.record_bits == 192 + 20
    assert s.field_count == 2
    again = api.Schema(s.print())
    assert again.record_bits == s.record_bits
    with pytest.raises(L.SfParseError):
        api.Schema("schema { oops")


@pytest.mark.parametrize("text,err", [
    ("schema s { field a : f16; }", "unknown base kind"),
    ("schema s { field a : f32; field a : f64; }", "duplicate field"),
    ("schema s { field a : i64 @truncate(16); }", "not allowed on i64"),
    ("schema s { field a : f32 @truncate(6); }", "outside 7..64"),
    ("schema s { field a : f32 @bogus(6); }", "unknown attribute"),
    ("kernel k reads a;", "no schema block"),
    ("schema s { field a : f32; } schema t { field b : f32; }", "only one schema block"),
    ("schema s { field a : f32; } kernel k;", "neither reads nor writes"),
])
def test_schema_diagnostics(text, err):  # test_schema.cpp:55-68
    with pytest.raises(L.SfParseError) as ei:
        api.Schema(text)
    assert err in str(ei.value)
    assert re.match(r"\d+:\d+: ", str(ei.value))


def test_unknown_kernel_field_is_invalid_argument():  # schema.cpp:311-317
    with pytest.raises(L.SfInvalidArg):
        api.Schema("schema s { field a : f32; } kernel k reads b;")


def test_default_schema_layout_and_fixpoint():  # test_schema.cpp:10-26, :87-93
    s = api.Schema.default()
    assert s.record_bits == 704
    txt = s.print()
    assert api.Schema(txt).print() == txt
    assert "kernel drift reads x, v writes x;" in txt
    lay = golden("layouts.json")
    for name, (T, ex) in {"default": (0, ""), "t16_xexcl": (16, "x"), "t16_xincl": (16, ""),
                          "t64_xexcl": (64, "x"), "t20": (20, "")}.items():
        S = api.Schema(schema_for(T, ex).text())
        assert S.record_bits == lay[name]["record_bits"]
        v = api.View(S, 5, "aos")
        for f, row in zip(schema_for(T, ex).fields, lay[name]["fields"]):
            base, stride, w, ar = v.lane(f.name)
            assert (base, w, ar, stride) == (row[0], row[1], row[2], lay[name]["record_bits"])


def test_views_match_oracle_geometry():
    S = schema_for(16)
    P = api.Schema(S.text())
    n = 1000
    for access in [None, "drift", "kick", "density", "force"]:
        for layout in ["aos", "soa"]:
            v = api.View(P, n, layout, access, api.SF_PREC_NATIVE)
            sub = S.subset(access)
            ob = O.Buffer(S, n, layout, sub, [S.fields[i].fmt(True) for i in sub], np.zeros(0, np.uint8))
            assert v.nbytes == (ob.length_bits + 7) // 8
            for pos, i in enumerate(sub):
                base, stride, w, ar = v.lane(S.fields[i].name)
                assert (base, stride) == ob.lane_geometry(pos)
                assert w == ob.widths[pos] and ar == S.fields[i].arity
    with pytest.raises(L.SfInvalidArg):
        api.View(P, n, "soa", "nonexistent")


def test_config_keys_validate():  # test_capi.cpp:56-70
    lib = L.lib()
    cfg = C.c_void_p()
    L.check(lib.sf_config_create(C.byref(cfg)))
    ok, bad = L.SF_OK, L.SF_INVALID_ARG
    assert lib.sf_config_set_int(cfg, b"particles", 128) == ok
    assert lib.sf_config_set_int(cfg, b"buffer-size", 64) == ok
    assert lib.sf_config_set_int(cfg, b"particles", -1) == bad
    assert lib.sf_config_set_int(cfg, b"warp-speed", 9) == bad
    assert lib.sf_config_set_string(cfg, b"variants", b"cpu-baseline,dev-soa") == ok
    assert lib.sf_config_set_string(cfg, b"variants", b"warp") == bad
    assert lib.sf_config_set_string(cfg, b"writeback", b"per-access") == ok
    assert lib.sf_config_set_string(cfg, b"writeback", b"sometimes") == bad
    assert lib.sf_config_set_double(cfg, b"bandwidth", 0.0) == bad
    assert lib.sf_config_set_double(cfg, b"latency", 1e-6) == ok
    lib.sf_config_destroy(cfg)


def test_gpu_entry_points_fail_loudly_without_device():
    """No CPU fallback: without a CUDA device every compute entry is SF_ERROR."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    S = api.Schema.default()
    src = api.View(S, 128, "aos")
    dst = api.View(S, 128, "soa", "drift", 16)
    buf = (C.c_uint8 * (src.nbytes + 16))()
    out = (C.c_uint8 * (dst.nbytes + 16))()
    st = L.lib().sf_b200_gather(src.handle, C.cast(buf, C.c_void_p), dst.handle, C.cast(out, C.c_void_p), None)
    assert st == L.SF_ERROR
    assert "no CUDA device" in L.lib().sf_last_error().decode()
    perm = (C.c_int32 * 128)(*range(128))
    st = L.lib().sf_b200_permute(src.handle, C.cast(buf, C.c_void_p), C.cast(out, C.c_void_p),
                                 C.cast(perm, C.c_void_p), None)
    assert st == L.SF_ERROR and "no CUDA device" in L.lib().sf_last_error().decode()
    st = L.lib().sf_b200_run_kernel(src.handle, C.cast(buf, C.c_void_p), b"kick,drift", 1e-3, 64, 0, 0, None)
    assert st == L.SF_ERROR and "no CUDA device" in L.lib().sf_last_error().decode()
    with pytest.raises(L.SfError, match="no CUDA device"):
        api.Shard(0, 1, 8, 0.125)


def test_shard_argument_checks():
    """sf_b200_shard_*: null arguments are SF_INVALID_ARG before any device work."""
    lib = L.lib()
    assert lib.sf_b200_shard_create(0, 1, 8, 0.125, 2, 1000, None) == L.SF_INVALID_ARG
    assert lib.sf_b200_shard_step(None, b"density", 1e-3, None, None) == L.SF_INVALID_ARG
    assert lib.sf_b200_shard_connect(None, None) == L.SF_INVALID_ARG
    lib.sf_b200_shard_destroy(None)  # no-op, like the reference's *_destroy(NULL)


def test_plain_c_consumer_links_and_runs(tmp_path):
    """tests/c/capi_check.c: a C program built against include/soaforge_b200.h."""
    import subprocess
    exe = tmp_path / "capi_check"
    libdir = os.path.dirname(L.LIB_PATH)
    subprocess.run(["/usr/bin/gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "capi_check.c"), "-L", libdir, "-lsoaforge_b200",
                    "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and "capi ok" in out.stdout, out.stdout


@pytest.mark.parametrize("prec,exclude,want", [
    (api.SF_PREC_STORED, "", {"x": 64, "id": 64, "v": 32, "rho": 32}),
    (api.SF_PREC_NATIVE, "", {"x": 64, "id": 64, "v": 32, "rho": 32}),
    (16, "", {"x": 16, "id": 64, "v": 16, "rho": 16}),
    (16, "x", {"x": 64, "id": 64, "v": 16, "rho": 16}),
    (20, "", {"x": 32, "id": 64, "v": 32, "rho": 32}),           # truncated T held in its base width
    (api.SF_PREC_PACKED + 20, "", {"x": 20, "id": 64, "v": 20, "rho": 20}),
    (api.SF_PREC_PACKED + 40, "v", {"x": 40, "id": 64, "v": 32, "rho": 40}),
    (api.SF_PREC_BF16, "x,rho", {"x": 64, "id": 64, "v": 16, "rho": 32}),
])
def test_view_precision_codes(prec, exclude, want):
    """Lane widths chosen by each precision code (include/soaforge_b200.h)."""
    v = api.View(api.Schema.default(), 10, "aos", None, prec, exclude)
    for f, w in want.items():
        assert v.lane(f)[2] == w, f


def test_view_rejects_bad_arguments():
    S = api.Schema.default()
    for bad in [2, 6, 65, 999, 1006, 1065]:
        with pytest.raises(L.SfInvalidArg):
            api.View(S, 10, "aos", None, bad)
    with pytest.raises(L.SfInvalidArg):
        api.View(S, 10, "soa", "no_such_kernel")
    h = C.c_void_p()
    assert L.lib().sf_b200_view_create(S.handle, None, 7, 0, None, 10, C.byref(h)) == L.SF_INVALID_ARG
    v = api.View(S, 10, "soa", "drift", 16)
    with pytest.raises(L.SfInvalidArg):
        v.lane("rho")  # not in the drift access set


def test_cell_entry_points_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    n = 64
    f = (C.c_float * (3 * n))()
    i32 = (C.c_int32 * (n + 8))()
    lo = (C.c_float * 3)(0, 0, 0)
    p = lambda a: C.cast(a, C.c_void_p)  # noqa: E731
    st = L.lib().sf_b200_density_cells(p(f), p(f), p(f), 1, n, p(i32), p(i32), p(lo), 0.5, 2, 2, 2, 1, n, p(f), None)
    assert st == L.SF_ERROR and "no CUDA device" in L.lib().sf_last_error().decode()
    st = L.lib().sf_b200_force_cells(p(f), p(f), p(f), p(f), p(f), p(f), 1, n, p(i32), p(i32), p(lo), 0.5, 2, 2, 2,
                                     1, n, p(f), p(f), None)
    assert st == L.SF_ERROR and "no CUDA device" in L.lib().sf_last_error().decode()
    st = L.lib().sf_b200_force_cells(None, p(f), p(f), p(f), p(f), p(f), 1, n, p(i32), p(i32), p(lo), 0.5, 2, 2, 2,
                                     1, n, p(f), p(f), None)
    assert st == L.SF_INVALID_ARG


def test_block_and_ipc_entry_points_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    n = 64
    f = (C.c_float * (4 * n))()
    i32 = (C.c_int32 * (n + 8))()
    p = lambda a: C.cast(a, C.c_void_p)  # noqa: E731
    lib = L.lib()
    assert lib.sf_b200_cells_pack(p(f), p(f), p(f), 1, n, p(i32), p(f), p(f), p(i32), None) == L.SF_ERROR
    assert "no CUDA device" in lib.sf_last_error().decode()
    blk = L.SfCellBlock(C.cast(f, C.c_void_p).value, C.cast(f, C.c_void_p).value, C.cast(i32, C.c_void_p).value,
                        C.cast(i32, C.c_void_p).value, 0, 2, 0.0, 0)
    lo = (C.c_float * 2)(0, 0)
    arr = (L.SfCellBlock * 1)(blk)
    assert lib.sf_b200_density_cells_blocks(p(arr), 1, n, p(i32), n, p(lo), 0.5, 2, 2, 2, 1, p(f), None) == L.SF_ERROR
    assert lib.sf_b200_force_pack(p(f), p(f), p(f), 1, n, p(i32), p(f), None) == L.SF_ERROR
    # window masks (one step's density -> force): size, reach and alignment checked before any device work
    assert lib.sf_b200_window_mask_bytes(n, 2) == 4 * (2 * 25 + 1) * n
    assert lib.sf_b200_window_mask_bytes(n, 1) == 4 * (2 * 9 + 1) * n
    assert lib.sf_b200_window_mask_bytes(n, 3) == 0
    masks = (C.c_int64 * ((lib.sf_b200_window_mask_bytes(n, 2) + 15) // 8))()
    assert lib.sf_b200_density_cells_blocks_masked(p(arr), 1, n, p(i32), n, p(lo), 0.5, 2, 2, 2, 3, p(f), p(masks),
                                                   None) == L.SF_INVALID_ARG
    assert lib.sf_b200_density_cells_blocks_masked(p(arr), 1, n, p(i32), n, p(lo), 0.5, 2, 2, 2, 2, p(f),
                                                   C.c_void_p(C.cast(masks, C.c_void_p).value + 4), None) \
        == L.SF_INVALID_ARG
    assert lib.sf_b200_density_cells_blocks_masked(p(arr), 1, n, p(i32), n, p(lo), 0.5, 2, 2, 2, 2, p(f), None,
                                                   None) == L.SF_INVALID_ARG
    assert lib.sf_b200_density_cells_blocks_masked(p(arr), 1, n, p(i32), n, p(lo), 0.5, 2, 2, 2, 2, p(f), p(masks),
                                                   None) == L.SF_ERROR  # no device
    out = C.c_void_p()
    assert lib.sf_b200_dev_alloc(1024, C.byref(out)) == L.SF_ERROR
    assert "no CUDA device" in lib.sf_last_error().decode()
    h = (C.c_uint8 * L.SF_IPC_HANDLE_BYTES)()
    assert lib.sf_b200_ipc_open(p(h), C.byref(out)) == L.SF_ERROR
    assert lib.sf_b200_ipc_handle(None, p(h)) == L.SF_INVALID_ARG
