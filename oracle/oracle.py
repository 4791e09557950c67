"""TEST INFRASTRUCTURE — Python face of the CPU oracle.

Restates the reference's record layout math (schema.hpp:35-67,
schema.cpp:216-224 compute_layout, schema.cpp:296-309
with_uniform_precision, layout_ops.cpp:13-39 lane_offset) and drives the C
restatement in ``liboracle.so`` (soa_oracle.c) for the per-lane codec, the
bit streams and the SPH kernels.  ``RefLib`` wraps the unmodified reference
library built by ``oracle/Makefile`` into ``oracle/_ref`` (available in the
build container and on the GPU box when shipped; never read from
/root/reference at run time).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.  The product (paper_2512_05516_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field as dfield
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OR_BF16 = -2
OR_I64 = -1


def NATIVE(t: int) -> int:
    return 1000 + t


# ---------------------------------------------------------------- library
class _Move(C.Structure):
    _fields_ = [("arity", C.c_int), ("src_fmt", C.c_int), ("dst_fmt", C.c_int),
                ("src_base", C.c_uint64), ("src_stride", C.c_uint64),
                ("dst_base", C.c_uint64), ("dst_stride", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        L = C.CDLL(path)
        u64, d, i = C.c_uint64, C.c_double, C.c_int
        P = C.c_void_p
        for name, res, args in [
            ("or_narrow_to_ieee", u64, [d, i, i]),
            ("or_widen_from_ieee", d, [u64, i, i]),
            ("or_encode_bits", u64, [d, i]),
            ("or_decode_bits", d, [u64, i]),
            ("or_quantize", d, [d, i]),
            ("or_encode_fmt", u64, [d, i]),
            ("or_decode_fmt", d, [u64, i]),
            ("or_encode_array", None, [P, u64, i, P]),
            ("or_decode_array", None, [P, u64, i, P]),
            ("or_write_bits", None, [P, u64, i, u64]),
            ("or_read_bits", u64, [P, u64, i]),
            ("or_apply_moves", None, [P, P, u64, P, i]),
            ("or_checksum", u64, [P, u64, u64]),
            ("or_w", d, [d, d]),
            ("or_density_buffer", None, [P, P, P, u64, u64, i, P]),
            ("or_density_cells", None, [P, P, P, u64, d, d, d, P]),
            ("or_force_cells", i, [P] * 6 + [u64, d, d, d] + [P] * 4),
            ("or_density_cells_at", None, [P, P, P, u64, d, d, d, P, u64, P]),
            ("or_force_cells_at", i, [P] * 6 + [u64, d, d, d, P, u64] + [P] * 4),
            ("or_dw_dr", d, [d, d]),
            ("or_random_ics", None, [u64, u64, u64, d] + [P] * 12),
            ("or_fmt_width", i, [i]),
        ]:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- codec
def layout_for(t: int):
    """fpcodec.cpp:28-37"""
    if t < 7 or t > 64:
        raise ValueError(f"total_bits {t} outside 7..64")
    e = 11 if t >= 33 else 8 if t >= 17 else 5
    return 1, e, t - 1 - e


def base_bits(t: int) -> int:
    return {11: 64, 8: 32, 5: 16}[layout_for(t)[1]]


def fmt_width(fmt: int) -> int:
    return lib().or_fmt_width(fmt)


def encode(x: np.ndarray, fmt: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    out = np.empty(x.size, dtype=np.uint64)
    lib().or_encode_array(_p(x), x.size, fmt, _p(out))
    return out


def decode(b: np.ndarray, fmt: int) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint64).ravel()
    out = np.empty(b.size, dtype=np.float64)
    lib().or_decode_array(_p(b), b.size, fmt, _p(out))
    return out


def checksum(data: bytes | np.ndarray, length_bits: Optional[int] = None) -> int:
    """pipelines.cpp:51-60"""
    a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) \
        else np.ascontiguousarray(data).view(np.uint8).ravel()
    a = np.ascontiguousarray(a)
    if length_bits is None:
        length_bits = a.size * 8
    return int(lib().or_checksum(_p(a), a.size, length_bits))


# ---------------------------------------------------------------- schema
@dataclass
class Field:
    """schema.hpp:35-51 FieldDecl"""
    name: str
    base: str            # "f32" | "f64" | "i64"
    arity: int = 1
    trunc: Optional[int] = None

    @property
    def is_float(self) -> bool:
        return self.base != "i64"

    @property
    def base_width(self) -> int:
        return 32 if self.base == "f32" else 64

    @property
    def stored_width(self) -> int:
        return self.trunc if self.trunc else self.base_width

    @property
    def native_width(self) -> int:
        return base_bits(self.stored_width) if self.is_float else self.base_width

    def fmt(self, native: bool = False) -> int:
        if not self.is_float:
            return OR_I64
        return NATIVE(self.stored_width) if native else self.stored_width


@dataclass
class Schema:
    name: str
    fields: List[Field]
    kernels: Dict[str, tuple] = dfield(default_factory=dict)   # name -> (reads, writes)

    def index(self, name: str) -> int:
        for i, f in enumerate(self.fields):
            if f.name == name:
                return i
        return -1

    @property
    def record_bits(self) -> int:
        """schema.cpp:216-224"""
        return sum(f.arity * f.stored_width for f in self.fields)

    def offsets(self) -> List[int]:
        out, off = [], 0
        for f in self.fields:
            out.append(off)
            off += f.arity * f.stored_width
        return out

    def with_uniform_precision(self, t: int, exclude: Sequence[str] = ()) -> "Schema":
        """schema.cpp:296-309"""
        if t < 7 or t > 64:
            raise ValueError("truncation width outside 7..64")
        fs = [Field(f.name, f.base, f.arity,
                    (t if (f.is_float and f.name not in exclude) else f.trunc)) for f in self.fields]
        return Schema(self.name, fs, dict(self.kernels))

    def subset(self, kernel: Optional[str]) -> List[int]:
        """layout_ops.cpp:86-101 — reads ∪ writes in declaration order"""
        if kernel is None:
            return list(range(len(self.fields)))
        r, w = self.kernels[kernel]
        return [i for i, f in enumerate(self.fields) if f.name in r or f.name in w]

    def text(self) -> str:
        lines = [f"schema {self.name} {{"]
        for f in self.fields:
            s = f"  field {f.name} : {f.base}"
            if f.arity == 3:
                s += " x3"
            if f.trunc:
                s += f" @truncate({f.trunc})"
            lines.append(s + ";")
        lines.append("}")
        for k, (r, w) in self.kernels.items():
            s = f"kernel {k}"
            if r:
                s += " reads " + ", ".join(r)
            if w:
                s += " writes " + ", ".join(w)
            lines.append(s + ";")
        return "\n".join(lines) + "\n"


def default_schema() -> Schema:
    """sph.cpp:445-467 (default_schema_text)"""
    f = Field
    return Schema("particle", [
        f("x", "f64", 3), f("id", "i64"), f("v", "f32", 3), f("u", "f32"), f("m", "f32"),
        f("h", "f32"), f("rho", "f32"), f("P", "f32"), f("cs", "f32"), f("a", "f32", 3),
        f("du", "f32"), f("dt", "f32")], {
        "density": (["x", "m", "h"], ["rho"]),
        "force": (["x", "v", "m", "h", "rho", "P", "cs"], ["a", "du"]),
        "kick": (["v", "u", "a", "du"], ["v", "u"]),
        "drift": (["x", "v"], ["x"]),
        "identity": (["x"], ["x"]),
    })


# ---------------------------------------------------------------- buffers
@dataclass
class Buffer:
    """layout_ops.hpp:76-98 PackedBuffer, restated: bytes + per-field formats."""
    schema: Schema
    count: int
    layout: str                 # "aos" | "soa"
    subset: List[int]
    fmts: List[int]             # per subset position
    data: np.ndarray            # uint8

    @property
    def widths(self) -> List[int]:
        return [fmt_width(f) for f in self.fmts]

    @property
    def record_bits(self) -> int:
        return sum(self.schema.fields[i].arity * w for i, w in zip(self.subset, self.widths))

    @property
    def length_bits(self) -> int:
        return self.record_bits * self.count

    def lane_geometry(self, pos: int):
        """(base, stride) in bits of subset position `pos` (layout_ops.cpp:25-39)."""
        ws = self.widths
        ar = [self.schema.fields[i].arity for i in self.subset]
        if self.layout == "aos":
            return sum(ar[p] * ws[p] for p in range(pos)), self.record_bits
        return sum(self.count * ar[p] * ws[p] for p in range(pos)), ar[pos] * ws[pos]

    def checksum(self) -> int:
        return checksum(self.data, self.length_bits)

    def field_values(self, name: str) -> np.ndarray:
        """Decoded binary64 values of one field, shape (count, arity)."""
        i = self.schema.index(name)
        pos = self.subset.index(i)
        ar = self.schema.fields[i].arity
        bits = self.field_bits(name)
        if self.schema.fields[i].is_float:
            return decode(bits, self.fmts[pos]).reshape(self.count, ar)
        return bits.view(np.int64).astype(np.float64).reshape(self.count, ar)

    def field_bits(self, name: str) -> np.ndarray:
        """Raw lane bits of one field as uint64, record-major."""
        i = self.schema.index(name)
        pos = self.subset.index(i)
        ar = self.schema.fields[i].arity
        w = self.widths[pos]
        base, stride = self.lane_geometry(pos)
        fmt = self.fmts[pos]
        mv = (_Move * 1)(_Move(ar, fmt, fmt, base, stride, 0, ar * w))
        dense = np.zeros((self.count * ar * w + 7) // 8 + 8, dtype=np.uint8)
        lib().or_apply_moves(_p(self.data), _p(dense), self.count, mv, 1)
        return unpack_lanes(dense, self.count * ar, w)


def unpack_lanes(dense: np.ndarray, n: int, w: int) -> np.ndarray:
    if w in (16, 32, 64):
        dt = {16: np.uint16, 32: np.uint32, 64: np.uint64}[w]
        return dense[: n * w // 8].view(dt).astype(np.uint64)
    L = lib()
    return np.array([L.or_read_bits(_p(dense), k * w, w) for k in range(n)], dtype=np.uint64)


def _alloc(schema, count, layout, subset, fmts) -> Buffer:
    b = Buffer(schema, count, layout, list(subset), list(fmts), np.zeros(0, np.uint8))
    b.data = np.zeros((b.length_bits + 7) // 8, dtype=np.uint8)
    return b


def transform(src: Buffer, layout: str, subset: Optional[List[int]] = None,
              fmts: Optional[List[int]] = None, schema: Optional[Schema] = None) -> Buffer:
    """General lane move: dst lane = encode(decode(src lane)); the restated
    composition of N (narrow_into, layout_ops.cpp:86-112), U/U^T
    (convert_precision, :164-191), C/C^T (convert_layout, :150-162) and the
    load_state/store_state narrowing (sph.cpp:385-443)."""
    subset = list(src.subset if subset is None else subset)
    if fmts is None:
        fmts = [src.fmts[src.subset.index(i)] for i in subset]
    dst = _alloc(schema or src.schema, src.count, layout, subset, fmts)
    moves = []
    for pos, idx in enumerate(subset):
        spos = src.subset.index(idx)
        sb, ss = src.lane_geometry(spos)
        db, ds = dst.lane_geometry(pos)
        moves.append(_Move(src.schema.fields[idx].arity, src.fmts[spos], fmts[pos], sb, ss, db, ds))
    arr = (_Move * len(moves))(*moves)
    lib().or_apply_moves(_p(src.data), _p(dst.data), src.count, arr, len(moves))
    return dst


def merge_into(narrowed: Buffer, original: Buffer, names: Sequence[str]) -> None:
    """N^T (widen_merge, layout_ops.cpp:120-146): overwrite only `names`
    (the write set) of `original`, converting through its formats."""
    moves = []
    for name in names:
        idx = original.schema.index(name)
        spos, dpos = narrowed.subset.index(idx), original.subset.index(idx)
        sb, ss = narrowed.lane_geometry(spos)
        db, ds = original.lane_geometry(dpos)
        moves.append(_Move(original.schema.fields[idx].arity, narrowed.fmts[spos],
                           original.fmts[dpos], sb, ss, db, ds))
    arr = (_Move * len(moves))(*moves)
    lib().or_apply_moves(_p(narrowed.data), _p(original.data), original.count, arr, len(moves))


# ---------------------------------------------------------------- ICs/state
STATE_FIELDS = ["x", "v", "a", "u", "m", "h", "rho", "P", "cs", "du", "dt", "id"]


def random_ics(n: int, seed: int = 42, accel_seed: int = 0, dt: float = 1e-3) -> Dict[str, np.ndarray]:
    """sph.cpp:325-349 via the C restatement (mt19937_64)."""
    s = {k: np.zeros((n, 3) if k in ("x", "v", "a") else n, dtype=np.float64) for k in STATE_FIELDS}
    s["id"] = np.zeros(n, dtype=np.int64)
    lib().or_random_ics(n, seed, accel_seed, dt, *[_p(s[k]) for k in
                        ["x", "v", "a", "u", "m", "h", "rho", "P", "cs", "du", "dt", "id"]])
    return s


def store_state(state: Dict[str, np.ndarray], schema: Schema, layout: str = "aos",
                native: bool = False) -> Buffer:
    """sph.cpp:385-412 — binary64 state written through the schema formats."""
    n = len(state["id"])
    fmts = [f.fmt(native) for f in schema.fields]
    buf = _alloc(schema, n, layout, range(len(schema.fields)), fmts)
    for pos, f in enumerate(schema.fields):
        if f.name not in state:
            continue
        vals = np.ascontiguousarray(state[f.name])
        if f.is_float:
            bits = encode(vals.astype(np.float64), fmts[pos])
        else:
            bits = vals.astype(np.int64).view(np.uint64).ravel()
        _write_field_bits(buf, pos, bits)
    return buf


def _write_field_bits(buf: Buffer, pos: int, bits: np.ndarray) -> None:
    idx = buf.subset[pos]
    ar = buf.schema.fields[idx].arity
    w = buf.widths[pos]
    dense = np.ascontiguousarray(bits.astype(np.uint64))
    db, ds = buf.lane_geometry(pos)
    # source: a 64-bit-per-lane stream; raw move keeps the low w bits
    mv = (_Move * 1)(_Move(ar, OR_I64, OR_I64, 0, ar * 64, db, ds))
    if w != 64:
        # pack to w-bit lanes first
        packed = np.zeros((dense.size * w + 7) // 8 + 8, dtype=np.uint8)
        if w in (16, 32):
            packed[: dense.size * w // 8] = dense.astype(np.uint16 if w == 16 else np.uint32).view(np.uint8)
        else:
            for k in range(dense.size):
                lib().or_write_bits(_p(packed), k * w, w, int(dense[k]))
        fmt = buf.fmts[pos]
        mv = (_Move * 1)(_Move(ar, fmt, fmt, 0, ar * w, db, ds))
        lib().or_apply_moves(_p(packed), _p(buf.data), buf.count, mv, 1)
        return
    lib().or_apply_moves(_p(dense.view(np.uint8)), _p(buf.data), buf.count, mv, 1)


def load_state(buf: Buffer) -> Dict[str, np.ndarray]:
    """sph.cpp:414-443"""
    out = {}
    for idx in buf.subset:
        f = buf.schema.fields[idx]
        v = buf.field_values(f.name)
        out[f.name] = v if f.arity == 3 else v[:, 0]
    return out


# ---------------------------------------------------------------- kernels
def kick(v: np.ndarray, u: np.ndarray, a: np.ndarray, du: np.ndarray, dt: float):
    """sph.cpp:247-256 in binary64: v += a*dt; u = max(0, u + du*dt)."""
    v2 = v + a * dt
    u2 = u + du * dt
    u2 = np.where(u2 < 0.0, 0.0, u2)
    return v2, u2


def drift(x: np.ndarray, v: np.ndarray, dt: float) -> np.ndarray:
    """sph.cpp:258-264 in binary64: x += v*dt."""
    return x + v * dt


def density_buffer(x, m, h, bs: int = 64, rho_fmt: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64); m = np.ascontiguousarray(m, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    rho = np.zeros(len(m), np.float64)
    lib().or_density_buffer(_p(x), _p(m), _p(h), len(m), bs, rho_fmt, _p(rho))
    return rho


def density_cells(x, m, h, lo: float, hi: float, cell: float) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64); m = np.ascontiguousarray(m, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    rho = np.zeros(len(m), np.float64)
    lib().or_density_cells(_p(x), _p(m), _p(h), len(m), lo, hi, cell, _p(rho))
    return rho


def force_cells(x, v, m, h, rho, P, lo: float, hi: float, cell: float):
    """Cell-linked restatement of force_kernel (sph.cpp:201-245): returns
    (a[n,3], du[n], a_scale[n], du_scale[n]); raises on rho == 0 like the
    reference's domain_error."""
    x, v, m, h, rho, P = (np.ascontiguousarray(t, np.float64) for t in (x, v, m, h, rho, P))
    n = len(m)
    a = np.zeros(3 * n); du = np.zeros(n); sa = np.zeros(n); sd = np.zeros(n)
    if lib().or_force_cells(_p(x), _p(v), _p(m), _p(h), _p(rho), _p(P), n, lo, hi, cell,
                            _p(a), _p(du), _p(sa), _p(sd)) != 0:
        raise ArithmeticError("force: degenerate state, rho == 0")
    return a.reshape(n, 3), du, sa, sd


def density_cells_at(x, m, h, lo: float, hi: float, cell: float, homes) -> np.ndarray:
    """or_density_cells for the listed homes (indices into x/m/h) only."""
    x = np.ascontiguousarray(x, np.float64); m = np.ascontiguousarray(m, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    homes = np.ascontiguousarray(homes, np.uint64)
    rho = np.zeros(len(homes), np.float64)
    lib().or_density_cells_at(_p(x), _p(m), _p(h), len(m), lo, hi, cell, _p(homes), len(homes), _p(rho))
    return rho


def force_cells_at(x, v, m, h, rho, P, lo: float, hi: float, cell: float, homes):
    """or_force_cells for the listed homes only: (a[k,3], du[k], a_scale[k], du_scale[k])."""
    x, v, m, h, rho, P = (np.ascontiguousarray(t, np.float64) for t in (x, v, m, h, rho, P))
    homes = np.ascontiguousarray(homes, np.uint64)
    k = len(homes)
    a = np.zeros(3 * k); du = np.zeros(k); sa = np.zeros(k); sd = np.zeros(k)
    if lib().or_force_cells_at(_p(x), _p(v), _p(m), _p(h), _p(rho), _p(P), len(m), lo, hi, cell, _p(homes), k,
                               _p(a), _p(du), _p(sa), _p(sd)) != 0:
        raise ArithmeticError("force: degenerate state, rho == 0")
    return a.reshape(k, 3), du, sa, sd


def w(r: float, h: float) -> float:
    return lib().or_w(r, h)


# ---------------------------------------------------------------- reference
class RefLib:
    """The unmodified reference (oracle/_ref/libref_driver.so)."""

    PATH = os.path.join(HERE, "_ref", "libref_driver.so")

    def __init__(self):
        L = C.CDLL(self.PATH)
        P, u64, d, i, s = C.c_void_p, C.c_uint64, C.c_double, C.c_int, C.c_char_p
        for name, res, args in [
            ("ref_last_error", s, []),
            ("ref_narrow_to_ieee", u64, [d, i, i]),
            ("ref_widen_from_ieee", d, [u64, i, i]),
            ("ref_encode_bits", u64, [d, i]),
            ("ref_decode_bits", d, [u64, i]),
            ("ref_quantize", d, [d, i]),
            ("ref_narrow_array", None, [P, u64, i, i, P]),
            ("ref_encode_array", None, [P, u64, i, P]),
            ("ref_schema_layout", i, [s, i, s, P, P, i, P]),
            ("ref_buf_from_ics", P, [s, i, s, u64, u64, u64, d]),
            ("ref_buf_from_bytes", P, [s, i, s, u64, P, u64]),
            ("ref_buf_restore", P, [P, s, i, s]),
            ("ref_buf_clone", P, [P]),
            ("ref_buf_op", P, [P, s, s]),
            ("ref_buf_widen_merge", i, [P, P, s]),
            ("ref_buf_run_kernel", i, [P, s, u64, d, i, i]),
            ("ref_buf_nbytes", u64, [P]),
            ("ref_buf_bits", u64, [P]),
            ("ref_buf_copy_bytes", None, [P, P]),
            ("ref_buf_checksum", u64, [P]),
            ("ref_buf_free", None, [P]),
            ("ref_streamed_bytes_one_way", u64, [s, i, s, s, u64, s]),
            ("ref_time_c2", d, [u64, i, i, u64, d]),
        ]:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def _chk(self, h):
        if not h:
            raise RuntimeError(self.L.ref_last_error().decode())
        return h

    @staticmethod
    def _s(x):
        return None if x is None else x.encode()

    def from_ics(self, n, seed=42, T=0, exclude="", text=None, accel_seed=0, dt=1e-3):
        return self._chk(self.L.ref_buf_from_ics(self._s(text), T, self._s(exclude), n, seed,
                                                  accel_seed, dt))

    def restore(self, h, T, exclude="", text=None):
        return self._chk(self.L.ref_buf_restore(h, self._s(text), T, self._s(exclude)))

    def op(self, h, op, kernel=None):
        return self._chk(self.L.ref_buf_op(h, op.encode(), self._s(kernel)))

    def run_kernel(self, h, kernel, bs=64, dt=1e-3, per_access=False, threads=1):
        if self.L.ref_buf_run_kernel(h, kernel.encode(), bs, dt, int(per_access), threads) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def widen_merge(self, narrowed, original, kernel):
        if self.L.ref_buf_widen_merge(narrowed, original, kernel.encode()) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def bytes(self, h) -> np.ndarray:
        out = np.zeros(self.L.ref_buf_nbytes(h), dtype=np.uint8)
        self.L.ref_buf_copy_bytes(h, _p(out))
        return out

    def checksum(self, h) -> int:
        return int(self.L.ref_buf_checksum(h))

    def free(self, *hs):
        for h in hs:
            self.L.ref_buf_free(h)

    def time_c2(self, n_per_thread, threads, T=16, seed=42, dt=1e-3) -> float:
        return self.L.ref_time_c2(n_per_thread, threads, T, seed, dt)
