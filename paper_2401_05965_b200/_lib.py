"""ctypes binding of the C ABI in include/hap_b200.h (libhap_b200.so).

This is the only door to the GPU kernels.  There is no fallback: if the
library is missing or does not export a declared symbol, loading raises
:class:`LibraryError` and the executor refuses to run.
"""
from __future__ import annotations

import ctypes
import os
import re

from ctypes import c_float, c_int, c_int64, c_uint32, c_void_p, POINTER

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HAP_LIB_PATH", os.path.join(PKG, "libhap_b200.so"))   # override: A/B builds
HEADER = os.path.join(os.path.dirname(PKG), "include", "hap_b200.h")

F32, BF16 = 0, 1
UNARY_TAGS = {"exp": 0, "neg": 1, "relu": 2, "sigmoid": 3, "tanh": 4}
BINARY_TAGS = {"add": 0, "mul": 1}
GEMM_TCGEN05, GEMM_SIMT = 0, 1

_P = c_void_p
_I64P = POINTER(c_int64)

class GemmDesc(ctypes.Structure):
    """hap_gemm_desc (include/hap_b200.h)."""
    _fields_ = [("A", c_void_p), ("lda", c_int64), ("transA", c_int), ("B", c_void_p), ("ldb", c_int64),
                ("transB", c_int), ("C", c_void_p), ("ldc", c_int64), ("M", c_int64), ("N", c_int64),
                ("K", c_int64), ("accumulate", c_int), ("epi", c_int), ("epi_tag", c_int), ("R", c_void_p),
                ("ldr", c_int64), ("R2", c_void_p), ("ldr2", c_int64), ("Y", c_void_p), ("ldy", c_int64),
                ("Z", c_void_p), ("ldz", c_int64)]


EPI_NONE, EPI_ADD, EPI_ADD2, EPI_SWISH, EPI_SWISH_BWD = range(5)


# name -> (restype, argtypes); must cover every function include/hap_b200.h declares.
SIGNATURES = {
    "hap_last_error": (ctypes.c_char_p, []),
    "hap_abi_version": (c_int, []),
    "hap_sm_count": (c_int, []),
    "hap_matmul": (c_int, [_P, c_int64, c_int, _P, c_int64, c_int, _P, c_int64, c_int64, c_int64,
                           c_int64, c_int, c_int, c_int, c_int, _P]),
    "hap_matmul_batch": (c_int, [POINTER(GemmDesc), c_int, c_int, c_int, c_int, c_int, _P]),
    "hap_matmul_tune": (c_int, [POINTER(GemmDesc), c_int, c_int, c_int, c_int, c_int, _P]),
    "hap_matmul_tune_export": (c_int64, [ctypes.c_char_p, c_int64]),
    "hap_matmul_tune_import": (c_int, [ctypes.c_char_p]),
    "hap_matmul_tune_clear": (None, []),
    "hap_matmul_engine": (c_int, [_P, c_int64, c_int, _P, c_int64, c_int, c_int64, c_int64, c_int64,
                                  c_int]),
    "hap_unary": (c_int, [c_int, _P, c_int, _P, c_int, c_int64, c_int, _P]),
    "hap_unary_grad": (c_int, [c_int, _P, _P, c_int, _P, c_int, _P, c_int, c_int64, c_int, c_int, _P]),
    "hap_binary": (c_int, [c_int, _P, _P, c_int, _P, c_int, c_int64, c_int, _P]),
    "hap_mul_grad": (c_int, [_P, _P, c_int, _P, c_int, _P, _P, c_int, c_int64, c_int, c_int, _P]),
    "hap_swish_fwd": (c_int, [c_int, _P, _P, _P, c_int, c_int64, c_int, _P]),
    "hap_swish_bwd": (c_int, [c_int, _P, _P, _P, _P, c_int, c_int64, c_int, c_int, _P]),
    "hap_gate_fwd": (c_int, [c_int, _P, _P, _P, _P, _P, _P, c_int, c_int64, c_int, _P]),
    "hap_gate_bwd": (c_int, [c_int, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int, c_int64, c_int, c_int, c_int,
                             c_int, _P]),
    "hap_reduce": (c_int, [_P, c_int, _I64P, c_int, c_uint32, _P, c_int, c_int, c_int, _P]),
    "hap_unreduce": (c_int, [_P, c_int, _I64P, c_int, c_uint32, _P, c_int, c_int, c_int, _P]),
    "hap_copy_block": (c_int, [_P, c_int, c_int64, c_int64, _P, c_int, c_int64, c_int64, c_int64,
                               c_int64, c_int64, c_int, c_int, _P]),
    "hap_axpy": (c_int, [c_float, _P, c_int, _P, c_int, c_int64, c_int, c_int, _P]),
    "hap_fill": (c_int, [_P, c_int, c_float, c_int64, _P]),
    "hap_sgd": (c_int, [_P, _P, _P, c_int, c_float, c_int64, c_int, _P]),
    "hap_sgd_multi": (c_int, [_P, c_int, c_int64, c_int, c_float, c_int, _P]),
    "hap_nccl_version": (c_int, []),
    "hap_comm_unique_id": (c_int, [ctypes.c_char_p]),
    "hap_comm_init": (c_int, [POINTER(c_void_p), ctypes.c_char_p, c_int, c_int]),
    "hap_comm_destroy": (c_int, [_P]),
    "hap_all_reduce": (c_int, [_P, _P, _P, c_int64, c_int, _P]),
    "hap_all_gather_v": (c_int, [_P, _P, _P, _I64P, c_int, c_int, _P, _P]),
    "hap_grouped_broadcast": (c_int, [_P, _P, _P, _I64P, c_int, _P]),
    "hap_reduce_scatter_v": (c_int, [_P, _P, _P, _I64P, c_int, _P, _P]),
    "hap_all_to_all_v": (c_int, [_P, _P, _I64P, _P, _I64P, c_int, _P]),
    "hap_symm_create": (c_int, [POINTER(c_void_p), c_int64, c_int, c_int]),
    "hap_symm_handle": (c_int, [_P, ctypes.c_char_p]),
    "hap_symm_open": (c_int, [_P, ctypes.c_char_p]),
    "hap_symm_destroy": (c_int, [_P]),
    "hap_symm_capacity": (c_int64, [_P]),
    "hap_symm_open_local": (c_int, [_P, _I64P]),
    "hap_symm_local_base": (c_void_p, [_P]),
    "hap_symm_peek": (c_int, [_P, _P]),
    "hap_p2p_all_reduce": (c_int, [_P, _P, _P, c_int, c_int64, c_int, _P]),
    "hap_p2p_all_to_all": (c_int, [_P, _P, _P, c_int, _P, _P, _P, c_int64, c_int, _P]),
    "hap_p2p_probe": (c_int, [_P, c_int, c_int64, c_int, _P]),
    "hap_p2p_buffer_handle": (c_int, [_P, _P, _P, POINTER(c_int64), POINTER(c_int64)]),
    "hap_p2p_buffer_open": (c_int, [_P, _P, _P, _P, _P, _P]),
    "hap_p2p_reduce_scatter_direct": (c_int, [_P, _P, _P, c_int, c_int64, c_int64, c_int64, _P, _P, c_int64,
                                              c_int, _P]),
    "hap_p2p_all_gather_push": (c_int, [_P, _P, _P, c_int, c_int64, c_int64, c_int64, _P, _P, c_int64, c_int,
                                        _P]),
    "hap_p2p_all_gather_v": (c_int, [_P, _P, _P, c_int, c_int64, c_int64, c_int64, _P, _P, c_int64, c_int,
                                     _P]),
    "hap_p2p_reduce_scatter_v": (c_int, [_P, _P, _P, c_int, c_int64, c_int64, c_int64, _P, _P, c_int, _P]),
}


class LibraryError(RuntimeError):
    pass


class HapError(RuntimeError):
    pass


def declared_symbols(header: str = HEADER) -> list[str]:
    """Function names declared in include/hap_b200.h."""
    with open(header, encoding="utf-8") as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hap_[a-z0-9_]+)\s*\(", text)))


_LIB = None


def lib():
    """Load (once) and return the bound library; raises LibraryError."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise LibraryError(f"{LIB_PATH} is missing: run `python -m paper_2401_05965_b200.build` "
                           "(the executor has no CPU fallback)")
    handle = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        try:
            fn = getattr(handle, name)
        except AttributeError:
            raise LibraryError(f"{LIB_PATH} does not export {name}") from None
        fn.restype = res
        fn.argtypes = args
    _LIB = handle
    return handle


TUNE_TABLE = os.environ.get("HAP_TUNE_TABLE", os.path.join(PKG, "tune_b200.txt"))
_TUNE_LOADED = False


def load_tune_table(path: str = TUNE_TABLE) -> int:
    """Import the committed GEMM tuning table (tile shape and split-K factor
    per launch signature, measured on a B200 by tools/tune_table.py) once per
    process.  With it every process picks the same shapes — and so rounds
    every GEMM the same way.  Returns the number of signatures imported."""
    global _TUNE_LOADED
    if _TUNE_LOADED or not os.path.exists(path):
        return 0
    with open(path, "rb") as fh:
        text = fh.read()
    check(lib().hap_matmul_tune_import(text), "hap_matmul_tune_import")
    _TUNE_LOADED = True
    return text.count(b"\n")


def export_tune_table() -> str:
    n = lib().hap_matmul_tune_export(None, 0)
    buf = ctypes.create_string_buffer(int(n))
    lib().hap_matmul_tune_export(buf, n)
    return buf.value.decode()


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().hap_last_error().decode(errors="replace")
        raise HapError(f"{what or 'hap call'} failed (status {status}): {msg}")


def i64_array(values) -> ctypes.Array:
    return (c_int64 * len(values))(*[int(v) for v in values])
