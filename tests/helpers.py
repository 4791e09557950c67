"""Shared test helpers: oracle-side compositions of the reference operators."""
import copy
import json
import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def set_field(buf: O.Buffer, name: str, values: np.ndarray) -> None:
    """BufferView::set over every lane of `name` (sph.cpp:114-126)."""
    pos = buf.subset.index(buf.schema.index(name))
    O._write_field_bits(buf, pos, O.encode(np.ascontiguousarray(values).ravel(), buf.fmts[pos]))


def apply_kernel(buf: O.Buffer, kernel: str, dt: float = 1e-3, per_access: bool = False,
                 bs: int = 64) -> O.Buffer:
    """run_kernel_chunked (sph.cpp:286-308) restated over an oracle buffer:
    decode -> binary64 arithmetic -> encode through the field's format."""
    out = copy.deepcopy(buf)
    st = O.load_state(out)
    if kernel == "drift":
        set_field(out, "x", O.drift(st["x"], st["v"], dt))
    elif kernel == "kick":
        v2, u2 = O.kick(st["v"], st["u"], st["a"], st["du"], dt)
        set_field(out, "v", v2)
        set_field(out, "u", u2)
    elif kernel == "density":
        rpos = out.subset.index(out.schema.index("rho"))
        rho = O.density_buffer(st["x"], st["m"], st["h"], bs,
                               out.fmts[rpos] if per_access else 0)
        set_field(out, "rho", rho)
    else:
        raise ValueError(kernel)
    return out


def schema_for(T: int, exclude: str = "") -> O.Schema:
    S = O.default_schema()
    return S.with_uniform_precision(T, [e for e in exclude.split(",") if e]) if T else S


def compressed_fmts(S: O.Schema):
    return [f.fmt(False) for f in S.fields]


def native_fmts(S: O.Schema):
    return [f.fmt(True) for f in S.fields]
