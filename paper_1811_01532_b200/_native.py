"""ctypes binding of the C ABI declared in include/wap_b200.h.

This is the only door from Python into the sm_100a kernels. There is no CPU
fallback: if the library is missing or CUDA is unavailable, every call raises
(`NativeUnavailable`), so a GPU run can never silently degrade to host code.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import EvalError, WorkloadError

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libwapb200.so"
# diagnostics only (tools/): load an alternative in-tree build, e.g. a traced GEMM
if os.environ.get("WAP_LIB_VARIANT"):
    _LIB_PATH = _LIB_PATH.with_name(f"libwapb200_{os.environ['WAP_LIB_VARIANT']}.so")
MAX_TAPS = 32
POOL_RELU_FUSED = 1  # include/wap_b200.h WAP_POOL_RELU_FUSED
AR_MAX_RANKS = 8     # WAP_AR_MAX_RANKS
AR_SLOTS = 64        # WAP_AR_SLOTS
AR_FLAG_WORDS = 2 * AR_SLOTS * AR_MAX_RANKS


class NativeUnavailable(RuntimeError):
    """The CUDA extension could not be loaded (no GPU path available)."""


class wap_operand_t(C.Structure):
    _fields_ = [
        ("ptr", C.c_void_p),
        ("inner", C.c_int64),
        ("outer", C.c_int64),
        ("ld", C.c_int64),
        ("mn_major", C.c_int32),
        ("tap_period", C.c_int32),
        ("ntaps", C.c_int32),
        ("off", C.c_int32 * MAX_TAPS),
    ]


class wap_gemm_desc_t(C.Structure):
    _fields_ = [
        ("M", C.c_int64),
        ("N", C.c_int64),
        ("K", C.c_int64),
        ("a", wap_operand_t),
        ("b", wap_operand_t),
        ("c", C.c_void_p),
        ("ldc", C.c_int64),
        ("bias", C.c_void_p),
        ("relu", C.c_int32),
        ("mask", C.c_void_p),
        ("ldm", C.c_int64),
        ("halo_pad", C.c_int32),
        ("halo_h", C.c_int32),
        ("halo_w", C.c_int32),
        ("precision", C.c_int32),
        ("splits", C.c_int32),
        ("block_n", C.c_int32),
        ("cluster", C.c_int32),
        ("window", C.c_int32),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_int64),
        ("mbits_out", C.c_void_p),
        ("mbits_out_ld", C.c_int64),
        ("mbits_in", C.c_void_p),
        ("mbits_in_ld", C.c_int64),
    ]


class wap_layout_t(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("W", C.c_int32), ("C", C.c_int32),
                ("pad", C.c_int32), ("ld", C.c_int32)]


class wap_wau_layer_t(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_grad", C.c_int32), ("batch", C.c_int64),
                ("out_h", C.c_int64), ("out_w", C.c_int64), ("cin", C.c_int64),
                ("cout", C.c_int64), ("k", C.c_int64), ("weight_elems", C.c_int64)]


class wap_wau_profile_t(C.Structure):
    _fields_ = [("peak_flops", C.c_double), ("efficiency_knee_flops", C.c_double),
                ("link_bandwidth", C.c_double), ("link_latency", C.c_double),
                ("allreduce_chunk_latency", C.c_double)]


class wap_ar_group_t(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("mode", C.c_int32), ("reserved", C.c_int32),
                ("grad", C.c_void_p * AR_MAX_RANKS), ("var", C.c_void_p * AR_MAX_RANKS),
                ("grad_mc", C.c_void_p), ("var_mc", C.c_void_p), ("flags", C.c_void_p * AR_MAX_RANKS),
                ("epochs", C.c_void_p), ("done", C.c_void_p), ("status", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the native library."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise NativeUnavailable(
                f"{_LIB_PATH} not built; run `python -m paper_1811_01532_b200.build`"
            )
        _lib = C.CDLL(str(_LIB_PATH))
        _declare(_lib)
    return _lib


def lib_path() -> Path:
    return _LIB_PATH


def _declare(L: C.CDLL) -> None:
    for name, res, args in _SIGNATURES:
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_F = C.c_float
_D = C.c_double

# (name, restype, argtypes) for every symbol include/wap_b200.h declares.
_SIGNATURES: list[tuple[str, object, list]] = [
    ("wap_version", C.c_char_p, []),
    ("wap_last_error", C.c_char_p, []),
    ("wap_launch_count", C.c_longlong, []),
    ("wap_gemm_workspace_bytes", _I64, [C.POINTER(wap_gemm_desc_t)]),
    ("wap_gemm", _I, [C.POINTER(wap_gemm_desc_t), _P]),
    ("wap_gemm_plan_create", _I, [C.POINTER(wap_gemm_desc_t), C.POINTER(_P)]),
    ("wap_gemm_plan_run", _I, [_P, _P]),
    ("wap_gemm_plan_destroy", None, [_P]),
    ("wap_gemm_plan_info", _I, [_P, C.POINTER(C.c_int64)]),
    ("wap_im2col", _I, [_P, wap_layout_t, _I, _I, _I, _I, _I, _I, _P, _I64, _P]),
    ("wap_s2d_input", _I, [_P, wap_layout_t, _I, _I, _I, _I, _P, _I, _P]),
    ("wap_conv_direct", _I, [_P, wap_layout_t, _P, _I, _I, _I, _P, _I, _P, wap_layout_t, _P, _I64, _P]),
    ("wap_conv_wgrad_direct_work_floats", _I64, [wap_layout_t]),
    ("wap_conv_wgrad_direct", _I, [_P, wap_layout_t, _P, wap_layout_t, _I, _I, _P, _I, _P, _P]),
    ("wap_s2d_weight", _I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P]),
    ("wap_col2im", _I, [_P, _I64, _I, _I, _I, _I, _I, _I, _P, wap_layout_t, _P, wap_layout_t, _P]),
    ("wap_elementwise", _I, [_I, _P, wap_layout_t, _P, wap_layout_t, _P, _P, wap_layout_t, _P]),
    ("wap_add_n", _I, [C.POINTER(_P), _I, wap_layout_t, _P, _P]),
    ("wap_bias_grad_work_floats", _I64, [wap_layout_t]),
    ("wap_bias_grad", _I, [_P, wap_layout_t, _P, _P, _P]),
    ("wap_maxpool_fwd", _I, [_P, wap_layout_t, _I, _I, _P, wap_layout_t, _P, _P]),
    ("wap_maxpool_fwd_ex", _I, [_P, wap_layout_t, _I, _I, _P, wap_layout_t, _P, _I, _P]),
    ("wap_maxpool_bwd", _I, [_P, _P, wap_layout_t, _I, _I, _P, wap_layout_t, _P, wap_layout_t, _P]),
    ("wap_lrn_maxpool_fwd", _I, [_P, wap_layout_t, _I, _F, _F, _F, _I, _I, _P, wap_layout_t, _P, _P]),
    ("wap_maxpool_lrn_bwd", _I, [_P, _P, wap_layout_t, _I, _I, _P, wap_layout_t, _I, _F, _F, _F, _P,
                                 wap_layout_t, _P, wap_layout_t, _P]),
    ("wap_lrn_fwd", _I, [_P, wap_layout_t, _I, _F, _F, _F, _P, wap_layout_t, _P]),
    ("wap_lrn_bwd", _I, [_P, wap_layout_t, _P, wap_layout_t, _I, _F, _F, _F, _P, wap_layout_t, _P,
                         wap_layout_t, _P]),
    ("wap_xent_fwd_bwd", _I, [_P, _I64, _P, _I64, _I, _I, _F, _P, _P, _I64, _P, _P]),
    ("wap_pack", _I, [_P, wap_layout_t, _P, _I, _P]),
    ("wap_sgd", _I, [_P, _P, _F, _P, _I64, _P]),
    ("wap_allreduce_sgd", _I, [C.POINTER(wap_ar_group_t), _I64, _I64, _F, _F, _I, _P]),
    ("wap_tf32_probe_flops", _D, [_I]),
    ("wap_tf32_probe", _I, [_I, _P]),
    ("wap_wau_select", _I, [C.POINTER(wap_wau_layer_t), _I, _I64, _I, wap_wau_profile_t, _I, _P, _P,
                            _P, _P, _P, _P]),
]


def exported_symbols() -> list[str]:
    return [s[0] for s in _SIGNATURES]


def check(rc: int, what: str = "native call", exc: type = EvalError) -> None:
    """Map a C status onto the reference exception hierarchy (errors.py)."""
    if rc != 0:
        msg = lib().wap_last_error().decode(errors="replace")
        if rc == -1 and exc is EvalError:
            exc = WorkloadError if "degree" in msg else EvalError
        raise exc(f"{what} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(lib().wap_launch_count())


def version() -> str:
    return lib().wap_version().decode()


def stream_ptr(stream=None) -> int:
    """cudaStream_t of a torch stream (current stream when None)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def operand(t, inner: int, outer: int, ld: int, mn_major: bool, tap_period: int = 0,
            offsets: tuple[int, ...] = (0,)) -> wap_operand_t:
    if len(offsets) > MAX_TAPS:
        raise ValueError(f"at most {MAX_TAPS} taps, got {len(offsets)}")
    op = wap_operand_t()
    op.ptr = t if isinstance(t, int) else t.data_ptr()
    op.inner, op.outer, op.ld = inner, outer, ld
    op.mn_major = 1 if mn_major else 0
    op.tap_period = tap_period
    op.ntaps = len(offsets)
    for i, o in enumerate(offsets):
        op.off[i] = int(o)
    return op


def ptr(t) -> int | None:
    if t is None:
        return None
    return t if isinstance(t, int) else t.data_ptr()


os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")
