"""The C-ABI library loads on a machine without a GPU, exports every symbol the
header declares, and rejects bad arguments before touching the device."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1811_01532_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "wap_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wap_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.exported_symbols())


def test_version_and_error_strings():
    assert "sm_100a" in N.version()
    assert isinstance(N.lib().wap_last_error(), bytes)


def test_invalid_gemm_rejected_without_gpu():
    d = N.wap_gemm_desc_t()
    d.M, d.N, d.K = 0, 8, 8
    rc = N.lib().wap_gemm(C.byref(d), None)
    assert rc == -1
    assert b"bad GEMM shape" in N.lib().wap_last_error()


def test_invalid_wau_rejected_without_gpu():
    prof = N.wap_wau_profile_t(1e12, 0.0, 1e9, 0.0, 0.0)
    rc = N.lib().wap_wau_select(None, 0, 16, 0, prof, 0, None, None, None, None, None, None)
    assert rc == -1
    assert b"device set" in N.lib().wap_last_error()


def test_errors_map_to_reference_exceptions():
    from paper_1811_01532_b200.errors import EvalError

    d = N.wap_gemm_desc_t()
    with pytest.raises(EvalError):
        N.check(N.lib().wap_gemm(C.byref(d), None), "gemm")


def test_product_path_has_no_cpu_fallback():
    """Program refuses to run without CUDA instead of falling back to host math."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1811_01532_b200 import models
    from paper_1811_01532_b200.runtime import Program

    with pytest.raises(N.NativeUnavailable):
        Program(models.mlp(8))


def test_allreduce_sgd_rejects_bad_groups_without_gpu():
    """wap_allreduce_sgd validates the group before any launch (no device needed)."""
    L = N.lib()
    assert L.wap_allreduce_sgd(None, 0, 4, C.c_float(0.1), C.c_float(1.0), 0, None) == -1
    g = N.wap_ar_group_t()
    g.world, g.rank = 0, 0
    assert L.wap_allreduce_sgd(C.byref(g), 0, 4, C.c_float(0.1), C.c_float(1.0), 0, None) == -1
    assert b"world" in L.wap_last_error()
    g.world, g.rank = 2, 2
    assert L.wap_allreduce_sgd(C.byref(g), 0, 4, C.c_float(0.1), C.c_float(1.0), 0, None) == -1
    g.rank = 0
    assert L.wap_allreduce_sgd(C.byref(g), 0, 4, C.c_float(0.1), C.c_float(1.0), N.AR_SLOTS, None) == -1
    assert b"slot" in L.wap_last_error()
    # counters present but rank 1's buffers not mapped
    g.epochs = g.done = g.status = 16
    assert L.wap_allreduce_sgd(C.byref(g), 0, 4, C.c_float(0.1), C.c_float(1.0), 0, None) == -1
    assert b"not mapped" in L.wap_last_error()
    assert C.sizeof(N.wap_ar_group_t) == 16 + 8 * (3 * N.AR_MAX_RANKS + 5)
