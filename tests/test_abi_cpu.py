"""The C-ABI library loads and exports every symbol include/flashkmeans.h declares.

CPU only: no kernel is launched.  Argument validation happens before any
device access, so invalid calls return FK_EINVAL even without a GPU.
"""

import ctypes
import os
import re

import pytest

from paper_2603_09229_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashkmeans.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FK_API\s+[\w\s\*]+?\b(fk_\w+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("fk_assign", "fk_update", "fk_normalize", "fk_assign_workspace",
              "fk_update_workspace", "fk_row_norms", "fk_objective", "fk_status_string"):
        assert s in syms
    assert set(syms) == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    # raw dlsym as well, independent of the ctypes declarations
    raw = ctypes.CDLL(_native.LIB_PATH)
    for s in declared_symbols():
        getattr(raw, s)


def test_version_and_status_strings():
    L = _native.lib()
    assert b"sm_100a" in L.fk_version()
    assert L.fk_status_string(0) == b"ok"
    assert L.fk_status_string(1) == b"invalid argument"


def test_validation_before_any_launch():
    L = _native.lib()
    # B = 0
    st = L.fk_assign(_native.FK_BF16, 16, 16, None, 0, 10, 4, 8, 16, 16, None, None, None, 0, None)
    assert st == _native.FK_EINVAL
    # null output pointers
    st = L.fk_assign(_native.FK_F32, 16, 16, None, 1, 10, 4, 8, None, None, None, None, None, 0, None)
    assert st == _native.FK_EINVAL
    # idx_prev without a changed flag
    st = L.fk_assign(_native.FK_F32, 16, 16, None, 1, 10, 4, 8, 16, 16, 16, None, None, 0, None)
    assert st == _native.FK_EINVAL
    # bad dtype
    st = L.fk_update(9, 16, 16, 1, 10, 4, 8, 5, 0, 16, 16, None, 16, 1 << 20, None)
    assert st == _native.FK_EINVAL
    # update_chunk < 1
    st = L.fk_update(_native.FK_F32, 16, 16, 1, 10, 4, 8, 0, 0, 16, 16, None, 16, 1 << 20, None)
    assert st == _native.FK_EINVAL
    # workspace too small
    st = L.fk_update(_native.FK_F32, 16, 16, 1, 10, 4, 8, 5, 0, 16, 16, None, 16, 1, None)
    assert st == _native.FK_EWORKSPACE
    # normalize master must be f32/f64
    st = L.fk_normalize(_native.FK_BF16, 16, 16, 16, 16, 0, None, None, None, 1, 4, 8, None, None)
    assert st == _native.FK_EINVAL
    # a bias operand needs a bf16/fp16 operand
    st = L.fk_normalize(_native.FK_F32, 16, 16, 16, 16, 0, None, None, None, 1, 4, 8, 16, None)
    assert st == _native.FK_EINVAL
    # bias of f32 centroids
    assert L.fk_assign_bias(_native.FK_F32, 16, 1, 4, 8, 16, None) == _native.FK_EINVAL
    assert L.fk_assign_bias_rows(300) == 512 and L.fk_assign_bias_rows(256) == 256


def test_workspace_queries():
    L = _native.lib()
    assert L.fk_assign_workspace(_native.FK_BF16, 1, 1 << 23, 4096, 128) >= 4096 * 4
    assert L.fk_assign_workspace(_native.FK_F32, 2, 100, 7, 5) >= (200 + 14) * 4
    assert L.fk_update_workspace(_native.FK_BF16, 1, 1 << 23, 4096, 128) >= (1 << 23) * 4
    assert L.fk_objective_workspace(3, 100000) >= 3 * 13 * 8


def test_no_cpu_fallback():
    """Operators refuse host tensors instead of computing on the CPU."""
    import torch

    from paper_2603_09229_b200 import ops

    x = torch.zeros((1, 8, 8), dtype=torch.bfloat16)
    with pytest.raises((ValueError, NotImplementedError, RuntimeError)):
        ops.assign(x, x[:, :2].contiguous())
