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


_C2CTYPES = {
    "int64_t": "c_int64", "size_t": "c_size_t", "float": "c_float", "int": "c_int",
}


def _header_signatures():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    sigs = {}
    for m in re.finditer(r"\b(?:int|size_t|const char\*)\s+(cce_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text):
        args = [a.strip() for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        kinds = []
        for a in args:
            a = re.sub(r"\s+\w+$", "", a)  # drop the parameter name
            kinds.append("c_void_p" if "*" in a else _C2CTYPES[a.replace("const ", "").strip()])
        sigs[m.group(1)] = kinds
    return sigs


def test_ctypes_table_matches_header_argument_types():
    """Every ctypes argtypes entry agrees with the C prototype (count and kind)."""
    import ctypes as ct

    from paper_2411_09009_b200 import _lib

    for name, kinds in _header_signatures().items():
        _, argtypes = _lib.SIGNATURES[name]
        got = [t.__name__ for t in argtypes]
        # c_size_t is an alias of c_ulong on LP64
        want = [ct.c_size_t.__name__ if k == "c_size_t" else getattr(ct, k).__name__ for k in kinds]
        assert got == want, (name, got, want)
