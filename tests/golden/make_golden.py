"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref, built by `make -C oracle`
from /root/reference sources):

    python tests/golden/make_golden.py

Outputs (committed, small):
  codec.json     reference encode/narrow/decode over special + random values
  pipeline.json  FNV-1a checksums of reference operator compositions
  layouts.json   record layouts of the sweep schemas
"""
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

R = O.RefLib()
L = R.L


def special_values():
    vals = [0.0, -0.0, 1.0, -1.0, np.pi, -np.pi, 0.1, 1e-3, 65504.0, 65520.0, 65536.0, 1e5,
            -1e5, 1e300, -1e300, 1e-300, 5e-324, 2.0 ** -14, 2.0 ** -24, 2.0 ** -25,
            2.0 ** -25 * 1.0000001, 2.0 ** -126, 2.0 ** -149, 2.0 ** -150, 3.4e38, 3.5e38,
            float("inf"), float("-inf"), 1.0009765625, 1.00048828125, 1.000732421875,
            6.097555160522461e-05, 0.333333333333, 2.0 ** -133]
    nan_bits = [0x7ff8000000000000, 0xfff8000000000000, 0x7ff0000000000001, 0x7ff4000000000000,
                0x7ff0000020000000, 0x7ffc000000000123]
    return [struct.unpack("<Q", struct.pack("<d", v))[0] for v in vals] + nan_bits


def codec():
    rng = np.random.default_rng(2025)
    bits = np.array(special_values(), dtype=np.uint64)
    rand = rng.integers(0, 2 ** 64, size=1000, dtype=np.uint64)
    # f32-representable values (what a binary32 AoS lane decodes to)
    f32 = rng.integers(0, 2 ** 32, size=1000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    with np.errstate(invalid="ignore"):
        f32 = f32.astype(np.float64).view(np.uint64)
    # log-uniform magnitudes across the binary16 range
    mags = np.exp(rng.uniform(np.log(1e-9), np.log(1e6), size=1000)) * rng.choice([-1, 1], 1000)
    allbits = np.concatenate([bits, rand, f32, mags.view(np.uint64)])
    x = allbits.view(np.float64).copy()
    out = {"inputs": [f"{b:016x}" for b in allbits.tolist()], "encode": {}, "narrow": {}}
    for T in [7, 10, 12, 16, 17, 20, 24, 32, 33, 40, 48, 56, 63, 64]:
        enc = np.zeros(x.size, np.uint64)
        L.ref_encode_array(O._p(x), x.size, T, O._p(enc))
        out["encode"][str(T)] = [f"{b:x}" for b in enc.tolist()]
    for (e, m) in [(8, 7), (5, 10), (8, 23)]:
        nar = np.zeros(x.size, np.uint64)
        L.ref_narrow_array(O._p(x), x.size, e, m, O._p(nar))
        out["narrow"][f"{e},{m}"] = [f"{b:x}" for b in nar.tolist()]
    # decode of every 16-bit pattern through T=16 and bf16 (8,7)
    out["decode16"] = [f"{struct.unpack('<Q', struct.pack('<d', L.ref_decode_bits(b, 16)))[0]:x}"
                       for b in range(0, 65536, 7)]
    out["widen_bf16"] = [f"{struct.unpack('<Q', struct.pack('<d', L.ref_widen_from_ieee(b, 8, 7)))[0]:x}"
                         for b in range(0, 65536, 7)]
    out["quantize"] = {"pi17": L.ref_quantize(np.pi, 17), "pi32": L.ref_quantize(np.pi, 32)}
    return out


def pipeline():
    n, seed, dt = 4096, 42, 1e-3
    out = {"n": n, "seed": seed, "dt": dt, "accel_seed": 43, "sweeps": {}, "northstar": {}}
    sweeps = {"default": (0, "", 43), "t16_xexcl": (16, "x", 43), "t16_xincl": (16, "", 43),
              "t64_xexcl": (64, "x", 43), "t32_xexcl": (32, "x", 43),
              "default_ics": (0, "", 0), "t16_xincl_ics": (16, "", 0)}
    for name, (T, ex, acc) in sweeps.items():
        rec = {}
        aos = R.from_ics(n, seed, T, ex, accel_seed=acc, dt=dt)
        rec["aos"] = R.checksum(aos)
        nat = R.op(aos, "unpack")
        soa = R.op(nat, "aos_to_soa")
        rec["soa_full"] = R.checksum(soa)
        for k in ["drift", "kick", "density", "force", "density,force"]:
            for layout, buf in [("aos", nat), ("soa", soa)]:
                h = R.L.ref_buf_clone(buf)
                for kk in k.split(","):
                    R.run_kernel(h, kk, 64, dt)
                back = R.op(h, "soa_to_aos") if layout == "soa" else R.L.ref_buf_clone(h)
                packed = R.op(back, "pack")
                rec[f"{k}_{layout}"] = R.checksum(packed)
                R.free(h, back, packed)
        # per-access density writeback
        h = R.L.ref_buf_clone(nat)
        R.run_kernel(h, "density", 64, dt, per_access=True)
        packed = R.op(h, "pack")
        rec["density_aos_peraccess"] = R.checksum(packed)
        R.free(h, packed)
        h = R.L.ref_buf_clone(nat)
        R.run_kernel(h, "force", 64, dt, per_access=True)
        packed = R.op(h, "pack")
        rec["force_aos_peraccess"] = R.checksum(packed)
        R.free(h, packed, aos, nat, soa)
        out["sweeps"][name] = {k: f"{v:016x}" for k, v in rec.items()}
    # north-star composition: default AoS -> T-bit store -> narrow drift -> SoA -> drift -> merge
    for name, (T, ex) in {"t16_xincl": (16, ""), "t16_xexcl": (16, "x"),
                          "t32_xincl": (32, "")}.items():
        rec = {}
        src = R.from_ics(n, seed, 0, "", accel_seed=43, dt=dt)
        st = R.restore(src, T, ex)
        rec["aos_t"] = R.checksum(st)
        u = R.op(st, "unpack")
        full = R.op(u, "aos_to_soa")
        rec["soa_full"] = R.checksum(full)
        for k in ["drift", "kick", "density"]:
            nw = R.op(u, "narrow", k)
            so = R.op(nw, "aos_to_soa")
            rec[f"{k}_soa"] = R.checksum(so)
            R.run_kernel(so, k, 64, dt)
            rec[f"{k}_soa_after"] = R.checksum(so)
            back = R.op(so, "soa_to_aos")
            pk = R.op(back, "pack")
            merged = R.L.ref_buf_clone(st)
            R.widen_merge(pk, merged, k)
            rec[f"{k}_merged_t"] = R.checksum(merged)
            R.free(nw, so, back, pk, merged)
        R.free(src, st, u, full)
        out["northstar"][name] = {k: f"{v:016x}" for k, v in rec.items()}
    return out


def layouts():
    out = {}
    for name, (T, ex) in {"default": (0, ""), "t16_xexcl": (16, "x"), "t16_xincl": (16, ""),
                          "t64_xexcl": (64, "x"), "t20": (20, "")}.items():
        rb = np.zeros(1, np.uint64)
        rows = np.zeros(4 * 32, np.int64)
        nf = np.zeros(1, np.int32)
        assert L.ref_schema_layout(None, T, ex.encode(), O._p(rb), O._p(rows), 32, O._p(nf)) == 0
        out[name] = {"record_bits": int(rb[0]),
                     "fields": rows[: 4 * int(nf[0])].reshape(-1, 4).tolist()}
    return out


def streamed():
    out = {}
    for k in ["kick", "drift", "density", "force"]:
        for v in ["dev-soa", "host-soa-stream", "cpu-soa"]:
            out[f"{k}:{v}"] = int(L.ref_streamed_bytes_one_way(None, 0, b"", k.encode(), 4096, v.encode()))
    return out


if __name__ == "__main__":
    for fname, fn in [("codec.json", codec), ("pipeline.json", pipeline),
                      ("layouts.json", layouts), ("streamed.json", streamed)]:
        with open(os.path.join(HERE, fname), "w") as f:
            json.dump(fn(), f, indent=None if fname == "codec.json" else 1, sort_keys=True,
                      separators=(",", ":") if fname == "codec.json" else None)
        print("wrote", fname)
