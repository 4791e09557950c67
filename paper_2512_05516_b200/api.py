"""Python mirror of the reference operator interface, executed on the B200.

Names follow the reference (proj/include/soaforge/*.hpp): a ``Schema`` is
parsed from the same DSL (schema.hpp:12-21); a ``PackedBuffer`` is a view
(layout, field subset, lane formats) over caller-owned device bytes
(layout_ops.hpp:76-98); the operators are the reference's N/U/C and their
transposes (layout_ops.hpp:100-128) and run_kernel (sph.hpp:97-104), but each
call is one fused sm_100a kernel launched through libsoaforge_b200.so on
torch's current CUDA stream.  Errors map the reference's exception classes:
ValueError subclasses for invalid arguments and parse errors.

torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

from . import _lib as L
from ._lib import (SF_LAYOUT_AOS, SF_LAYOUT_SOA, SF_MATH_FP32, SF_MATH_FP64_EXACT, SF_PREC_BF16,  # noqa: F401
                   SF_PREC_NATIVE, SF_PREC_PACKED, SF_PREC_STORED, check, enc, lib)

# sph.cpp:445-467 — the built-in particle schema, same text
DEFAULT_SCHEMA_TEXT = """# SWIFT-style particle record; positions stay binary64, the rest binary32.
schema particle {
  field x : f64 x3;
  field id : i64;
  field v : f32 x3;
  field u : f32;
  field m : f32;
  field h : f32;
  field rho : f32;
  field P : f32;
  field cs : f32;
  field a : f32 x3;
  field du : f32;
  field dt : f32;
}
kernel density reads x, m, h writes rho;
kernel force reads x, v, m, h, rho, P, cs writes a, du;
kernel kick reads v, u, a, du writes v, u;
kernel drift reads x, v writes x;
kernel identity reads x writes x;
"""


def version() -> str:
    return lib().sf_version().decode()


def layout_for(total_bits: int) -> Tuple[int, int, int]:
    """fpcodec::layout_for (fpcodec.cpp:28-37)."""
    s, e, m = C.c_int(), C.c_int(), C.c_int()
    check(lib().sf_layout_for(total_bits, C.byref(s), C.byref(e), C.byref(m)))
    return s.value, e.value, m.value


def quantize(x: float, total_bits: int) -> float:
    """fpcodec::quantize (fpcodec.cpp:151-155)."""
    out = C.c_double()
    check(lib().sf_quantize(float(x), total_bits, C.byref(out)))
    return out.value


class Schema:
    """schema::parse_file over the DSL; owns an sf_schema handle."""

    def __init__(self, text: str = DEFAULT_SCHEMA_TEXT):
        h = C.c_void_p()
        check(lib().sf_schema_parse(text.encode(), C.byref(h)))
        self._h = h

    @classmethod
    def default(cls) -> "Schema":
        return cls(DEFAULT_SCHEMA_TEXT)

    @property
    def handle(self):
        return self._h

    @property
    def record_bits(self) -> int:
        v = C.c_uint64()
        check(lib().sf_schema_record_bits(self._h, C.byref(v)))
        return v.value

    @property
    def field_count(self) -> int:
        v = C.c_int()
        check(lib().sf_schema_field_count(self._h, C.byref(v)))
        return v.value

    def print(self) -> str:
        out = C.c_char_p()
        check(lib().sf_schema_print(self._h, C.byref(out)))
        return out.value.decode()

    def __del__(self):
        try:
            if getattr(self, "_h", None) and L._lib is not None:
                L._lib.sf_schema_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: module globals already gone
            pass


class View:
    """A packed-buffer descriptor (PackedBuffer without the bytes)."""

    def __init__(self, schema: Schema, count: int, layout: str = "aos", access_set: Optional[str] = None,
                 precision: int = SF_PREC_STORED, exclude: str = ""):
        self.schema, self.count, self.layout = schema, int(count), layout
        self.access_set, self.precision, self.exclude = access_set, precision, exclude
        h = C.c_void_p()
        check(lib().sf_b200_view_create(schema.handle, enc(access_set), SF_LAYOUT_AOS if layout == "aos" else SF_LAYOUT_SOA,
                                        precision, enc(exclude), self.count, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def nbytes(self) -> int:
        v = C.c_uint64()
        check(lib().sf_b200_view_bytes(self._h, C.byref(v)))
        return v.value

    def lane(self, field: str) -> Tuple[int, int, int, int]:
        """(base_bits, stride_bits, width_bits, arity) of a field (layout_ops.cpp:25-39)."""
        b, s, w, a = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_int()
        check(lib().sf_b200_view_lane(self._h, field.encode(), C.byref(b), C.byref(s), C.byref(w), C.byref(a)))
        return b.value, s.value, w.value, a.value

    def with_count(self, count: int) -> "View":
        return View(self.schema, count, self.layout, self.access_set, self.precision, self.exclude)

    def like(self, layout=None, access_set=-1, precision=None, exclude=None) -> "View":
        return View(self.schema, self.count, layout or self.layout,
                    self.access_set if access_set == -1 else access_set,
                    self.precision if precision is None else precision,
                    self.exclude if exclude is None else exclude)

    def __del__(self):
        try:
            if getattr(self, "_h", None) and L._lib is not None:
                L._lib.sf_b200_view_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown: module globals already gone
            pass


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


@dataclass
class PackedBuffer:
    """View + device bytes (torch uint8 tensor, caller-owned storage)."""
    view: View
    data: "object"

    @staticmethod
    def empty(view: View, device="cuda") -> "PackedBuffer":
        import torch
        # +16: every buffer is a whole number of 16-B words (vector stores)
        return PackedBuffer(view, torch.zeros(view.nbytes + 16, dtype=torch.uint8, device=device))

    @staticmethod
    def from_host(view: View, host_bytes, device="cuda") -> "PackedBuffer":
        import numpy as np
        import torch
        b = PackedBuffer.empty(view, device)
        arr = np.frombuffer(bytes(host_bytes), dtype=np.uint8) if not isinstance(host_bytes, np.ndarray) \
            else host_bytes.view(np.uint8).ravel()
        if arr.size != view.nbytes:
            raise ValueError(f"expected {view.nbytes} bytes, got {arr.size}")
        b.data[: view.nbytes].copy_(torch.from_numpy(arr.copy()))
        return b

    def to_host(self):
        return self.data[: self.view.nbytes].cpu().numpy()


# ---------------------------------------------------------------- operators
def gather(src: PackedBuffer, dst_view: View, out: Optional[PackedBuffer] = None) -> PackedBuffer:
    """U∘N∘C (+ narrowing) in one kernel: narrow_into + unpack_into +
    aos_to_soa_into (layout_ops.cpp:86-191) and store_state(T)."""
    out = out or PackedBuffer.empty(dst_view, src.data.device)
    check(lib().sf_b200_gather(src.view.handle, _ptr(src.data), dst_view.handle, _ptr(out.data), _stream()))
    return out


def gather_kernel(src: PackedBuffer, dst_view: View, kernel: str, dt: float = 1e-3,
                  math: int = SF_MATH_FP64_EXACT, out: Optional[PackedBuffer] = None) -> PackedBuffer:
    """Gather fused with kick/drift (the conversion is the kernel's load)."""
    out = out or PackedBuffer.empty(dst_view, src.data.device)
    check(lib().sf_b200_gather_kernel(src.view.handle, _ptr(src.data), dst_view.handle, _ptr(out.data),
                                      kernel.encode(), dt, math, _stream()))
    return out


def convert(src: PackedBuffer, dst_view: View, out: Optional[PackedBuffer] = None) -> PackedBuffer:
    """Any view -> any view, lane by lane (C, C^T, U, U^T, narrowing)."""
    out = out or PackedBuffer.empty(dst_view, src.data.device)
    check(lib().sf_b200_convert(src.view.handle, _ptr(src.data), dst_view.handle, _ptr(out.data), _stream()))
    return out


def widen_merge(narrowed: PackedBuffer, original: PackedBuffer, kernel: str) -> None:
    """N^T: overwrite `kernel`'s write set of `original` (layout_ops.cpp:120-146)."""
    check(lib().sf_b200_scatter_merge(narrowed.view.handle, _ptr(narrowed.data), original.view.handle,
                                      _ptr(original.data), kernel.encode(), _stream()))


scatter_merge = widen_merge


def permute(src: PackedBuffer, perm, out: Optional[PackedBuffer] = None) -> PackedBuffer:
    """Record k of the result = record perm[k] of src (every lane; perm: int32
    cuda tensor of src.view.count entries, e.g. bin_particles' perm)."""
    out = out if out is not None else PackedBuffer.empty(src.view)
    check(lib().sf_b200_permute(src.view.handle, _ptr(src.data), _ptr(out.data), _ptr(perm), _stream()))
    return out


def run_kernel(buf: PackedBuffer, kernel: str, dt: float = 1e-3, buffer_size: int = 64,
               per_access: bool = False, math: int = SF_MATH_FP64_EXACT) -> None:
    """run_kernel_chunked (sph.cpp:286-308) in place on the device.  `kernel`:
    kick | drift | density | force, or a comma-separated list ("kick,drift")
    run in order with the same result as one call each (one pass over the
    records on an AoS of plain IEEE lanes)."""
    check(lib().sf_b200_run_kernel(buf.view.handle, _ptr(buf.data), kernel.encode(), dt, buffer_size,
                                   int(per_access), math, _stream()))


def _prec_dtype(prec: int):
    import torch
    if prec in (SF_PREC_NATIVE, 32):
        return torch.float32
    if prec == 16:
        return torch.float16
    if prec == SF_PREC_BF16:
        return torch.bfloat16
    raise L.SfInvalidArg(L.SF_INVALID_ARG, "precision must be SF_PREC_NATIVE (fp32), 16 or SF_PREC_BF16")


def _streams(prec: int, **tensors):
    """The kernels reinterpret each stream's bytes in `prec`: every tensor
    must be a contiguous CUDA tensor of that dtype."""
    want = _prec_dtype(prec)
    for name, t in tensors.items():
        if not t.is_cuda:
            raise L.SfInvalidArg(L.SF_INVALID_ARG, f"{name} must be a CUDA tensor")
        if not t.is_contiguous():
            raise L.SfInvalidArg(L.SF_INVALID_ARG, f"{name} must be contiguous")
        if t.dtype != want:
            raise L.SfInvalidArg(L.SF_INVALID_ARG, f"{name} is {t.dtype}, precision code {prec} needs {want}")


def _int32s(**tensors):
    import torch
    for name, t in tensors.items():
        if t is not None and (not t.is_cuda or not t.is_contiguous() or t.dtype != torch.int32):
            raise L.SfInvalidArg(L.SF_INVALID_ARG, f"{name} must be a contiguous int32 CUDA tensor")


def _f32s(**tensors):
    import torch
    for name, t in tensors.items():
        if t is not None and (not t.is_cuda or not t.is_contiguous() or t.dtype != torch.float32):
            raise L.SfInvalidArg(L.SF_INVALID_ARG, f"{name} must be a contiguous float32 CUDA tensor")


def bin_particles(x, lo, cell: float, dims, cell_start=None, perm=None):
    """Counting sort into cells (x-major ids), stable by particle index.
    x: (n,3) float32 cuda tensor.  Returns (cell_start[ncell+1], perm[n])."""
    import torch
    n = x.shape[0]
    nx, ny, nz = dims
    ncell = nx * ny * nz
    cell_start = cell_start if cell_start is not None else torch.empty(ncell + 1, dtype=torch.int32, device=x.device)
    perm = perm if perm is not None else torch.empty(max(n, 1), dtype=torch.int32, device=x.device)
    nbytes = lib().sf_b200_bin_scratch_bytes(n, nx, ny, nz)
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    lo_arr = (C.c_float * 3)(*[float(v) for v in lo])
    check(lib().sf_b200_bin_particles(_ptr(x), n, C.cast(lo_arr, C.c_void_p), float(cell), nx, ny, nz,
                                      _ptr(cell_start), _ptr(perm), _ptr(scratch), nbytes, _stream()))
    return cell_start, perm


def density_cells(x, m, h, cell_start, perm, lo, cell: float, dims, n_home=None, reach: int = 1,
                  prec: int = SF_PREC_NATIVE, rho=None):
    """Cell-linked density.  x: (n,3), m, h: (n,) in particle order stored
    as fp32 (SF_PREC_NATIVE), fp16 (16) or bf16 (SF_PREC_BF16); cell_start /
    perm from bin_particles on the same grid.  Returns rho (fp32, particle
    order); only the first n_home particles (default all) are computed, the
    rest are neighbours only (ghosts)."""
    import torch
    nx, ny, nz = dims
    n = m.shape[0]
    n_home = n if n_home is None else n_home
    rho = rho if rho is not None else torch.zeros(max(n, 1), dtype=torch.float32, device=m.device)
    _streams(prec, x=x, m=m, h=h)
    _int32s(cell_start=cell_start, perm=perm)
    _f32s(rho=rho)
    lo_arr = (C.c_float * 3)(*[float(v) for v in lo])
    check(lib().sf_b200_density_cells(_ptr(x), _ptr(m), _ptr(h), prec, n, _ptr(perm) if perm is not None else None,
                                      _ptr(cell_start), C.cast(lo_arr, C.c_void_p), float(cell), nx, ny, nz, reach,
                                      n_home, _ptr(rho), _stream()))
    return rho


def force_cells(x, v, m, h, rho, P, cell_start, perm, lo, cell: float, dims, n_home=None, reach: int = 1,
                prec: int = SF_PREC_NATIVE, a=None, du=None):
    """Cell-linked force (force_kernel, sph.cpp:201-245, over cell
    neighbours).  x, v: (n,3); m, h, rho, P: (n,), particle order, stored as
    fp32 / fp16 / bf16 per `prec`; grid as for density_cells.  Returns
    (a (n,3) fp32, du (n,) fp32) for the first n_home particles (default
    all; the rest are ghosts).  rho == 0 raises SfError (the reference's
    domain_error)."""
    import torch
    nx, ny, nz = dims
    n = m.shape[0]
    n_home = n if n_home is None else n_home
    a = a if a is not None else torch.zeros((max(n, 1), 3), dtype=torch.float32, device=m.device)
    du = du if du is not None else torch.zeros(max(n, 1), dtype=torch.float32, device=m.device)
    _streams(prec, x=x, v=v, m=m, h=h, rho=rho, P=P)
    _int32s(cell_start=cell_start, perm=perm)
    _f32s(a=a, du=du)
    lo_arr = (C.c_float * 3)(*[float(t) for t in lo])
    check(lib().sf_b200_force_cells(_ptr(x), _ptr(v), _ptr(m), _ptr(h), _ptr(rho), _ptr(P), prec, n,
                                    _ptr(perm) if perm is not None else None, _ptr(cell_start),
                                    C.cast(lo_arr, C.c_void_p), float(cell), nx, ny, nz, reach, n_home,
                                    _ptr(a), _ptr(du), _stream()))
    return a, du


def cells_pack(x, m, h, perm, pos, hs, hmax, prec: int = SF_PREC_NATIVE):
    """Pack x (n,3), m, h (n,) through perm (sorted position -> particle) into
    caller-owned float4 pos (n,4) = (x, y, z, m), hs (n,) = h and hmax (>= 2
    int32 words: the h range, [0] bits of the largest h, [1] ~bits of the
    smallest)."""
    n = m.shape[0]
    _streams(prec, x=x, m=m, h=h)
    _int32s(perm=perm)
    _f32s(pos=pos, hs=hs)
    check(lib().sf_b200_cells_pack(_ptr(x), _ptr(m), _ptr(h), prec, n, _ptr(perm) if perm is not None else None,
                                   _ptr(pos), _ptr(hs), _ptr(hmax), _stream()))


def cell_block(pos, hs, cell_start, hmax, x0: int, nx: int, x_origin: float) -> "L.SfCellBlock":
    """One sf_cell_block from device tensors or raw device addresses (ints);
    x_origin = the lo[0] the block's bin_particles used."""
    addr = lambda t: t if isinstance(t, int) else t.data_ptr()  # noqa: E731
    return L.SfCellBlock(addr(pos), addr(hs), addr(cell_start), addr(hmax), x0, nx, float(x_origin), 0)


def window_masks(n: int, reach: int):
    """Device buffer for the window masks one density hands to the force of
    the same step (reach 1 or 2)."""
    import torch
    nbytes = int(lib().sf_b200_window_mask_bytes(n, reach))
    if nbytes == 0:
        raise L.SfInvalidArg("window masks need reach 1 or 2")
    return torch.empty((nbytes + 7) // 8, dtype=torch.int64, device="cuda")  # 8-B aligned (int2 windows)


def density_cells_blocks(blocks, n: int, perm, lo_yz, cell: float, nx_global: int, ny: int, nz: int, n_home=None,
                         reach: int = 1, rho=None, masks=None):
    """Cell-linked density of blocks[0]'s first n_home particles with
    candidates from every block (own slab + neighbouring slabs in place).
    masks (window_masks(n, reach)): also record every home's in-support
    pairs for force_cells_blocks(..., masks=) of the same step."""
    import torch
    n_home = n if n_home is None else n_home
    alloc = torch.empty if n_home == n else torch.zeros  # entries past n_home are not written
    rho = rho if rho is not None else alloc(max(n, 1), dtype=torch.float32, device="cuda")
    arr = (L.SfCellBlock * len(blocks))(*blocks)
    lo_arr = (C.c_float * 2)(*[float(t) for t in lo_yz])
    args = (C.cast(arr, C.c_void_p), len(blocks), n, _ptr(perm) if perm is not None else None, n_home,
            C.cast(lo_arr, C.c_void_p), float(cell), nx_global, ny, nz, reach, _ptr(rho))
    if masks is None:
        check(lib().sf_b200_density_cells_blocks(*args, _stream()))
    else:
        check(lib().sf_b200_density_cells_blocks_masked(*args, _ptr(masks), _stream()))
    return rho


def force_pack(v, rho, P, perm, vel, prec: int = SF_PREC_NATIVE):
    """(v, P/rho^2) -> float4 vel (n,4) in perm's order; rho == 0 raises
    SfError (domain error)."""
    n = rho.shape[0]
    _streams(prec, v=v, rho=rho, P=P)
    _int32s(perm=perm)
    _f32s(vel=vel)
    check(lib().sf_b200_force_pack(_ptr(v), _ptr(rho), _ptr(P), prec, n,
                                   _ptr(perm) if perm is not None else None, _ptr(vel), _stream()))


def force_block(pos, vel, hs, cell_start, hmax, x0: int, nx: int, x_origin: float) -> "L.SfForceBlock":
    addr = lambda t: t if isinstance(t, int) else t.data_ptr()  # noqa: E731
    return L.SfForceBlock(addr(pos), addr(vel), addr(hs), addr(cell_start), addr(hmax), x0, nx, float(x_origin), 0)


def force_cells_blocks(blocks, n: int, perm, lo_yz, cell: float, nx_global: int, ny: int, nz: int, n_home=None,
                       reach: int = 1, a=None, du=None, masks=None):
    """Cell-linked force of blocks[0]'s first n_home particles with
    candidates from every block; returns (a (n,3), du (n,)).  masks: the
    window masks density_cells_blocks(..., masks=) wrote for these blocks
    (the force then evaluates exactly the in-support pairs)."""
    import torch
    n_home = n if n_home is None else n_home
    alloc = torch.empty if n_home == n else torch.zeros  # entries past n_home are not written
    a = a if a is not None else alloc((max(n, 1), 3), dtype=torch.float32, device="cuda")
    du = du if du is not None else alloc(max(n, 1), dtype=torch.float32, device="cuda")
    arr = (L.SfForceBlock * len(blocks))(*blocks)
    lo_arr = (C.c_float * 2)(*[float(t) for t in lo_yz])
    args = (C.cast(arr, C.c_void_p), len(blocks), n, _ptr(perm) if perm is not None else None, n_home,
            C.cast(lo_arr, C.c_void_p), float(cell), nx_global, ny, nz, reach, _ptr(a), _ptr(du))
    if masks is None:
        check(lib().sf_b200_force_cells_blocks(*args, _stream()))
    else:
        check(lib().sf_b200_force_cells_blocks_masked(*args, _ptr(masks), _stream()))
    return a, du


class DeviceBuffer:
    """cudaMalloc'd device memory (an IPC-shareable allocation base), or a
    mapping of another process's buffer opened from its IPC handle."""

    def __init__(self, nbytes: int = 0, handle: Optional[bytes] = None):
        p = C.c_void_p()
        if handle is not None:
            h = (C.c_uint8 * L.SF_IPC_HANDLE_BYTES).from_buffer_copy(handle)
            check(lib().sf_b200_ipc_open(C.cast(h, C.c_void_p), C.byref(p)))
            self.opened = True
        else:
            check(lib().sf_b200_dev_alloc(nbytes, C.byref(p)))
            self.opened = False
        self.ptr, self.nbytes = p.value, nbytes

    def ipc_handle(self) -> bytes:
        h = (C.c_uint8 * L.SF_IPC_HANDLE_BYTES)()
        check(lib().sf_b200_ipc_handle(C.c_void_p(self.ptr), C.cast(h, C.c_void_p)))
        return bytes(h)

    def tensor(self, offset: int, shape, dtype):
        """A torch view of [offset, offset + size) of this buffer (no copy)."""
        import torch
        itemsize = torch.empty((), dtype=dtype).element_size()
        typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.float64: "<f8", torch.uint8: "|u1"}[dtype]
        shape = tuple(shape)

        class _Iface:
            __cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (self.ptr + offset, False),
                                        "version": 3, "strides": None}
        t = torch.as_tensor(_Iface(), device="cuda")
        assert t.data_ptr() == self.ptr + offset and t.element_size() == itemsize
        return t

    def free(self):
        if self.ptr:
            if self.opened:
                check(lib().sf_b200_ipc_close(C.c_void_p(self.ptr)))
            else:
                check(lib().sf_b200_dev_free(C.c_void_p(self.ptr)))
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Shard:
    """One rank of the cell-sharded timestep (sf_b200_shard_*): an x-slab of
    an nc^3 cell grid over the unit box, its particles an SoA of the default
    schema at T=32 held by the library at a fixed capacity.  `exchange`
    gathers every rank's 64-byte handle (rank order) — e.g. torch.distributed
    all_gather_object; None for a single rank."""

    FIELDS = ("x", "id", "v", "u", "m", "h", "rho", "P", "cs", "a", "du", "dt")

    def __init__(self, rank: int, world: int, cells_per_side: int, cell: float, refine: int = 2,
                 capacity: int = 0, exchange=None):
        h = C.c_void_p()
        check(lib().sf_b200_shard_create(rank, world, cells_per_side, float(cell), refine, int(capacity),
                                         C.byref(h)))
        self._h, self.rank, self.world = h, rank, world
        mine = (C.c_uint8 * L.SF_IPC_HANDLE_BYTES)()
        check(lib().sf_b200_shard_handle(self._h, C.cast(mine, C.c_void_p)))
        every = exchange(bytes(mine)) if (exchange is not None and world > 1) else [bytes(mine)] * world
        allh = (C.c_uint8 * (L.SF_IPC_HANDLE_BYTES * world)).from_buffer_copy(b"".join(every))
        check(lib().sf_b200_shard_connect(self._h, C.cast(allh, C.c_void_p)))

    def load(self, soa: "PackedBuffer") -> None:
        """The rank's particles: an SoA PackedBuffer of the default schema at
        T=32 (x included, every field)."""
        check(lib().sf_b200_shard_load(self._h, _ptr(soa.data), soa.view.count, _stream()))

    @property
    def count(self) -> int:
        p, n, b = C.c_void_p(), C.c_uint64(), C.c_int()
        check(lib().sf_b200_shard_field(self._h, b"x", C.byref(p), C.byref(n), C.byref(b)))
        return n.value

    def field(self, name: str):
        """The field's stream of the current state as a torch tensor (a view
        of library memory, valid until the next step): (n, 3) float32 for
        x / v / a, (n,) float32 for scalars, (n,) int64 for id."""
        import torch
        p, n, b = C.c_void_p(), C.c_uint64(), C.c_int()
        check(lib().sf_b200_shard_field(self._h, name.encode(), C.byref(p), C.byref(n), C.byref(b)))
        count, per = n.value, b.value
        typestr = "<i8" if name == "id" else "<f4"
        shape = (count, 3) if per == 12 else (count,)

        class _Iface:
            __cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (p.value or 0, False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_Iface(), device="cuda") if count else torch.empty(
            shape, dtype=torch.int64 if name == "id" else torch.float32, device="cuda")

    def step(self, kernels: str = "density,force,kick,drift", dt: float = 1e-3, timed: bool = False):
        """One timestep (then migration).  timed: returns the metrics dict."""
        m = (C.c_double * 9)() if timed else None
        check(lib().sf_b200_shard_step(self._h, kernels.encode(), dt, _stream(), m))
        if not timed:
            return None
        names = kernels.split(",")
        out = {"particles": int(m[0]), "step_ms": m[1], "migrate_ms": m[6], "sent": int(m[7]), "step": int(m[8])}
        for i, k in enumerate(names):
            out[k + "_ms"] = m[2 + i]
        return out

    def close(self):
        if getattr(self, "_h", None) and L._lib is not None:
            L._lib.sf_b200_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostBuffer:
    """Pinned (mode 0) or managed (mode 1) host memory for run_host."""

    def __init__(self, nbytes: int, mode: int = 0):
        p = C.c_void_p()
        check(lib().sf_b200_host_alloc(nbytes, mode, C.byref(p)))
        self.ptr, self.nbytes, self.mode = p, nbytes, mode

    def numpy(self):
        import numpy as np
        return np.ctypeslib.as_array(C.cast(self.ptr, C.POINTER(C.c_uint8)), shape=(self.nbytes,))

    def free(self):
        if self.ptr:
            check(lib().sf_b200_host_free(self.ptr, self.mode))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def run_host(src_view: View, host: HostBuffer, dst_view: View, kernels: str = "drift", dt: float = 1e-3,
             math: int = SF_MATH_FP64_EXACT, chunk: int = 1 << 21, soa_out: Optional[HostBuffer] = None,
             mode: Optional[int] = None) -> dict:
    """One whole-population step on host-resident AoS: mode 0 streamed
    (narrowed 2-D DMA, pinned), 1 managed (host buffer must be managed),
    2 in-place (whole records, pinned); default: the host buffer's kind.
    With `soa_out` the SoA result lands in host memory instead of being
    scattered back into the AoS."""
    m = (C.c_double * 5)()
    check(lib().sf_b200_run_host(src_view.handle, host.ptr, dst_view.handle, kernels.encode(), dt, math,
                                 host.mode if mode is None else mode, chunk,
                                 soa_out.ptr if soa_out is not None else None, m))
    return {"seconds": m[0], "h2d_bytes": int(m[1]), "d2h_bytes": int(m[2]), "chunks": int(m[3]),
            "launches": int(m[4])}


def launch_count() -> int:
    return int(lib().sf_b200_launch_count())
