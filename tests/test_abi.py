"""The C-ABI library builds, loads without a GPU, and exports every symbol include/cce_b200.h declares."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "cce_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cce_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("cce_fwd", "cce_bwd", "cce_merge_shards", "cce_vocab_order", "cce_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2411_09009_b200 import _build, _lib

    _build.build()
    lib = ctypes.CDLL(str(_lib.lib_path()))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table mirrors the header one to one
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_error_channel_without_gpu():
    from paper_2411_09009_b200 import _lib

    lib = _lib.load()
    assert lib.cce_abi_version() == 1
    assert isinstance(lib.cce_last_error(), bytes)
    # argument validation happens before any device work
    assert lib.cce_fwd(None, None, None, 4, 12, 5, -100, 0, 0.0, None, 0, None, None, None) != 0
    assert b"multiple of 8" in lib.cce_last_error()


def test_product_rejects_cpu_tensors():
    import torch
    from paper_2411_09009_b200 import linear_cross_entropy

    e = torch.randn(4, 8).bfloat16()
    c = torch.randn(5, 8).bfloat16()
    t = torch.zeros(4, dtype=torch.int64)
    with pytest.raises(ValueError, match="CUDA"):
        linear_cross_entropy(e, c, t)
