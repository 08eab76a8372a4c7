"""ctypes binding of libcce_b200.so (include/cce_b200.h).

This is the product path's only route to compute: if the shared library is missing or fails to
load, every op raises.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libcce_b200.so"
# CCE_LIB selects another in-tree build of the same ABI (A/B experiments: `_build.py --variant`)
if os.environ.get("CCE_LIB"):
    _LIB_PATH = Path(__file__).resolve().parent / os.environ["CCE_LIB"]
_lib = None

c_void_p = ctypes.c_void_p
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_int = ctypes.c_int
c_size = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/cce_b200.h one to one
SIGNATURES = {
    "cce_last_error": (ctypes.c_char_p, []),
    "cce_abi_version": (c_int, []),
    "cce_launch_count": (ctypes.c_ulonglong, []),
    "cce_fwd_workspace_bytes": (c_size, [c_i64, c_i64, c_i64]),
    "cce_fwd": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_f32,
                        c_void_p, c_size, c_void_p, c_void_p, c_void_p]),
    "cce_merge_shards": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_void_p,
                                 c_void_p, c_void_p]),
    "cce_merge_shards_checked": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64,
                                         c_void_p, c_void_p, c_void_p, c_void_p]),
    "cce_ebar_workspace_bytes": (c_size, [c_i64, c_i64]),
    "cce_ebar": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_i64, c_void_p, c_void_p, c_size, c_void_p]),
    "cce_sort_workspace_bytes": (c_size, [c_i64]),
    "cce_vocab_order": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_void_p,
                                c_void_p, c_size, c_void_p]),
    "cce_compact_rows": (c_int, [c_void_p, c_i64, c_i64, c_void_p, c_void_p, c_void_p]),
    "cce_bwd_prep": (c_int, [c_void_p, c_i64, c_void_p, c_i64, c_i64, c_i64, c_void_p, c_void_p,
                             c_void_p, c_void_p]),
    "cce_bwd_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_i64, c_i64]),
    "cce_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                        c_void_p, c_void_p, c_i64, c_i64, c_i64, c_f32, c_f32, c_i64, c_i64,
                        c_void_p, c_int, c_void_p, c_size, c_void_p, c_int, c_void_p, c_void_p,
                        c_void_p, c_void_p]),
    "cce_tile_max_bytes": (c_size, [c_i64, c_i64]),
    "cce_fwd_tiles": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64, c_i64,
                              c_f32, c_void_p, c_size, c_void_p, c_void_p, c_void_p, c_void_p, c_i64,
                              c_void_p, c_void_p, c_void_p, c_void_p]),
    "cce_fwd_gather": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64,
                               c_i64, c_f32, c_void_p, c_size, c_void_p, c_void_p, c_void_p, c_void_p]),
    "cce_fwd_group": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64,
                              c_i64, c_i64, c_f32, c_void_p, c_size, c_void_p, c_void_p, c_void_p, c_void_p]),
    "cce_fwd_group_ex": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64,
                                 c_i64, c_i64, c_f32, c_void_p, c_size, c_void_p, c_void_p, c_void_p, c_int,
                                 c_void_p]),
    "cce_fwd_group_sync": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64,
                                   c_i64, c_i64, c_f32, c_void_p, c_size, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_int, c_void_p, c_void_p, c_i64, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
    "cce_fwd_splits": (c_int, [c_i64, c_i64, c_i64]),
    "cce_combine_parts": (c_int, [c_void_p, c_int, c_i64, c_void_p, c_void_p]),
    "cce_bwd_stream_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_i64]),
    "cce_bwd_stream_debug_layout": (c_int, [c_i64, c_i64, c_i64, c_i64, c_void_p]),
    "cce_bwd_stream": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64, c_f32, c_f32, c_int,
                               c_void_p, c_i64, c_void_p, c_size, c_void_p, c_int, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "cce_bwd_stream_ex": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64, c_f32, c_f32, c_int,
                                  c_void_p, c_i64, c_void_p, c_size, c_void_p, c_int, c_void_p, c_void_p,
                                  c_void_p, c_int, c_void_p]),
    "cce_unpermute_rows": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_size, c_void_p]),
    "cce_bwd_kept_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_i64, c_i64]),
    "cce_bwd_kept": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64,
                             c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64, c_f32, c_f32, c_int, c_void_p,
                             c_i64, c_void_p, c_void_p, c_void_p, c_i64, c_void_p, c_size, c_void_p,
                             c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "cce_bwd_lowmem_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_i64]),
    "cce_bwd_lowmem": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_i64, c_i64, c_i64, c_f32, c_f32, c_int, c_i64, c_void_p,
                               c_size, c_void_p, c_void_p, c_void_p, c_void_p]),
    "cce_label_terms_workspace_bytes": (c_size, [c_i64]),
    "cce_label_terms": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_i64, c_i64, c_i64, c_f32, c_void_p, c_size, c_void_p, c_int,
                                c_void_p, c_void_p]),
    "cce_reduce_loss": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_int, c_void_p, c_void_p]),
    "cce_upstream": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_int, c_void_p, c_void_p]),
    "cce_gather_rows": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_void_p]),
    "cce_f32_to_bf16": (c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "cce_indexed_dot": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64, c_i64, c_i64,
                                c_f32, c_void_p, c_void_p]),
}


class CceError(RuntimeError):
    pass


def lib_path() -> Path:
    return _LIB_PATH


def load():
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise CceError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2411_09009_b200._build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(_LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().cce_last_error().decode(errors="replace")
        raise CceError(f"{what} failed: {msg}")
