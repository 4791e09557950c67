"""ctypes binding of libsoaforge_b200.so (include/soaforge_b200.h).

The shared library is the product; this module only declares signatures and
maps sf_status codes to Python exceptions.  Importing it fails loudly when
the library has not been built — there is no Python or CPU fallback.
"""
import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libsoaforge_b200.so")

SF_OK, SF_ERROR, SF_INVALID_ARG, SF_PARSE_ERROR, SF_CHECK_FAILED = range(5)
SF_LAYOUT_AOS, SF_LAYOUT_SOA = 0, 1
SF_PREC_STORED, SF_PREC_NATIVE, SF_PREC_BF16, SF_PREC_PACKED = 0, 1, 100, 1000
SF_MATH_FP64_EXACT, SF_MATH_FP32 = 0, 1
SF_MODE_STREAMED, SF_MODE_MANAGED, SF_MODE_INPLACE, SF_MODE_MANAGED_MAPPED = 0, 1, 2, 3


class SfCellBlock(C.Structure):
    """sf_cell_block (include/soaforge_b200.h)."""
    _fields_ = [("pos", C.c_void_p), ("h", C.c_void_p), ("cell_start", C.c_void_p), ("hmax", C.c_void_p),
                ("x0", C.c_int32), ("nx", C.c_int32), ("x_origin", C.c_float), ("reserved", C.c_int32)]


class SfForceBlock(C.Structure):
    """sf_force_block (include/soaforge_b200.h)."""
    _fields_ = [("pos", C.c_void_p), ("vel", C.c_void_p), ("h", C.c_void_p), ("cell_start", C.c_void_p),
                ("hmax", C.c_void_p), ("x0", C.c_int32), ("nx", C.c_int32), ("x_origin", C.c_float),
                ("reserved", C.c_int32)]


SF_IPC_HANDLE_BYTES = 64


class SfError(RuntimeError):
    """SF_ERROR (generic failure, including CUDA errors / missing device)."""

    def __init__(self, status, message):
        super().__init__(message)
        self.status = status


class SfInvalidArg(SfError, ValueError):
    """SF_INVALID_ARG (the reference's std::invalid_argument)."""


class SfParseError(SfError, ValueError):
    """SF_PARSE_ERROR (schema::ParseError, message carries line:column)."""


class SfCheckFailed(SfError):
    """SF_CHECK_FAILED (validate ran and at least one check failed)."""


_EXC = {SF_ERROR: SfError, SF_INVALID_ARG: SfInvalidArg, SF_PARSE_ERROR: SfParseError,
        SF_CHECK_FAILED: SfCheckFailed}

# (name, restype, argtypes) for every symbol in include/soaforge_b200.h
P, u64, i32, f64, s = C.c_void_p, C.c_uint64, C.c_int, C.c_double, C.c_char_p
PP = C.POINTER(C.c_void_p)
SYMBOLS = [
    ("sf_version", s, []),
    ("sf_last_error", s, []),
    ("sf_layout_for", i32, [i32, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("sf_quantize", i32, [f64, i32, C.POINTER(C.c_double)]),
    ("sf_schema_parse", i32, [s, PP]),
    ("sf_schema_destroy", None, [P]),
    ("sf_schema_record_bits", i32, [P, C.POINTER(C.c_uint64)]),
    ("sf_schema_field_count", i32, [P, C.POINTER(C.c_int)]),
    ("sf_schema_print", i32, [P, C.POINTER(C.c_char_p)]),
    ("sf_config_create", i32, [PP]),
    ("sf_config_destroy", None, [P]),
    ("sf_config_set_string", i32, [P, s, s]),
    ("sf_config_set_int", i32, [P, s, C.c_int64]),
    ("sf_config_set_double", i32, [P, s, f64]),
    ("sf_run_bench_transform", i32, [P, C.POINTER(C.c_char_p)]),
    ("sf_run_bench_kernels", i32, [P, C.POINTER(C.c_char_p)]),
    ("sf_run_bench_pipeline", i32, [P, C.POINTER(C.c_char_p)]),
    ("sf_run_study_truncation", i32, [P, C.POINTER(C.c_char_p)]),
    ("sf_run_validate", i32, [P, C.POINTER(C.c_char_p)]),
    ("sf_b200_view_create", i32, [P, s, i32, i32, s, u64, PP]),
    ("sf_b200_view_destroy", None, [P]),
    ("sf_b200_view_bytes", i32, [P, C.POINTER(C.c_uint64)]),
    ("sf_b200_view_lane", i32, [P, s, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]),
    ("sf_b200_gather", i32, [P, P, P, P, P]),
    ("sf_b200_gather_kernel", i32, [P, P, P, P, s, f64, i32, P]),
    ("sf_b200_convert", i32, [P, P, P, P, P]),
    ("sf_b200_scatter_merge", i32, [P, P, P, P, s, P]),
    ("sf_b200_permute", i32, [P, P, P, P, P]),
    ("sf_b200_run_kernel", i32, [P, P, s, f64, u64, i32, i32, P]),
    ("sf_b200_density_cells", i32, [P, P, P, i32, u64, P, P, P, C.c_float, i32, i32, i32, i32, u64, P, P]),
    ("sf_b200_force_cells", i32, [P] * 6 + [i32, u64, P, P, P, C.c_float] + [i32] * 4 + [u64, P, P, P]),
    ("sf_b200_cells_pack", i32, [P, P, P, i32, u64, P, P, P, P, P]),
    ("sf_b200_density_cells_blocks", i32, [P, i32, u64, P, u64, P, C.c_float, i32, i32, i32, i32, P, P]),
    ("sf_b200_force_pack", i32, [P, P, P, i32, u64, P, P, P]),
    ("sf_b200_force_cells_blocks", i32, [P, i32, u64, P, u64, P, C.c_float, i32, i32, i32, i32, P, P, P]),
    ("sf_b200_window_mask_bytes", u64, [u64, i32]),
    ("sf_b200_density_cells_blocks_masked", i32, [P, i32, u64, P, u64, P, C.c_float, i32, i32, i32, i32, P, P, P]),
    ("sf_b200_force_cells_blocks_masked", i32, [P, i32, u64, P, u64, P, C.c_float, i32, i32, i32, i32, P, P, P,
                                                P]),
    ("sf_b200_dev_alloc", i32, [u64, PP]),
    ("sf_b200_dev_free", i32, [P]),
    ("sf_b200_ipc_handle", i32, [P, P]),
    ("sf_b200_ipc_open", i32, [P, PP]),
    ("sf_b200_ipc_close", i32, [P]),
    ("sf_b200_shard_create", i32, [i32, i32, i32, f64, i32, u64, PP]),
    ("sf_b200_shard_destroy", None, [P]),
    ("sf_b200_shard_handle", i32, [P, P]),
    ("sf_b200_shard_connect", i32, [P, P]),
    ("sf_b200_shard_load", i32, [P, P, u64, P]),
    ("sf_b200_shard_field", i32, [P, s, PP, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
    ("sf_b200_shard_step", i32, [P, s, f64, P, C.POINTER(C.c_double)]),
    ("sf_b200_bin_particles", i32, [P, u64, P, C.c_float, i32, i32, i32, P, P, P, u64, P]),
    ("sf_b200_bin_scratch_bytes", u64, [u64, i32, i32, i32]),
    ("sf_b200_run_host", i32, [P, P, P, s, f64, i32, i32, u64, P, C.POINTER(C.c_double)]),
    ("sf_b200_host_alloc", i32, [u64, i32, PP]),
    ("sf_b200_host_free", i32, [P, i32]),
    ("sf_b200_launch_count", u64, []),
]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2512_05516_b200.build` "
                              "(there is no fallback implementation)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status):
    if status != SF_OK:
        msg = lib().sf_last_error().decode(errors="replace")
        raise _EXC.get(status, SfError)(status, msg)


def enc(x):
    return None if x is None else x.encode()
