"""Torch-facing wrappers of the C ABI (include/cce_b200.h).

Each function validates, allocates outputs/workspaces with torch (so every byte shows up in
torch.cuda.max_memory_allocated, mirroring instrument.py's scratch/output accounting) and calls
exactly one or two C entry points on the current CUDA stream.  No function here computes
anything on the host; if libcce_b200.so is missing, the first call raises.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import _lib

BLOCK_TOKENS = 128      # GPU tile rows  (reference BlockSpec.n_b)
BLOCK_VOCAB = 256       # GPU tile cols  (reference BlockSpec.m_b)
EPSILON_DEFAULT = 2.0 ** -12   # core.py:27


# Optional CUDA-event timing of the two tcgen05 kernels (bench.py's roofline leg).  When
# enabled, an event pair is recorded on the launching stream around each cce_fwd / cce_bwd call.
KERNEL_EVENTS: dict[str, list] | None = None
LAST_COUNTERS: dict = {}
LAST_OVERFLOW = {"count": 0}  # backward reruns caused by S-hat slot overflow
LAUNCHES = {"count": 0}   # kernels launched from libcce_b200.so (bench.py's gpu_launches)


def _ev_begin(name: str):
    if KERNEL_EVENTS is None:
        return None
    a = torch.cuda.Event(enable_timing=True)
    a.record()
    return a


def _ev_end(name: str, a) -> None:
    if a is None:
        return
    b = torch.cuda.Event(enable_timing=True)
    b.record()
    KERNEL_EVENTS.setdefault(name, []).append((a, b))


def _p(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def check_operands(e: torch.Tensor, c: torch.Tensor, targets: torch.Tensor | None = None) -> None:
    """Shape/dtype/device validation (core.py:39-114, kernels.py:168-170) -> ValueError."""
    if e.dim() != 2 or c.dim() != 2:
        raise ValueError(f"e and c must be 2-D, got {tuple(e.shape)} and {tuple(c.shape)}")
    if e.shape[1] != c.shape[1]:
        raise ValueError(f"feature dims differ: embeddings {e.shape[1]} vs classifier {c.shape[1]}")
    if c.shape[0] < 1:
        raise ValueError("classifier needs at least 1 rows, got 0")
    if e.shape[1] % 8 != 0:
        raise ValueError(f"hidden size {e.shape[1]} must be a multiple of 8 (16-byte TMA rows)")
    for name, t in (("e", e), ("c", c)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
        if t.dtype != torch.bfloat16:
            raise ValueError(f"{name} must be bfloat16, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    if targets is not None:
        if targets.dim() != 1 or targets.shape[0] != e.shape[0]:
            raise ValueError(f"label count {targets.shape[0] if targets.dim() else 0} != token count {e.shape[0]}")
        if targets.dtype != torch.int64:
            raise ValueError(f"targets must be int64, got {targets.dtype}")


def forward_local(e, c, targets, ignore_index: int, vocab_start: int = 0, softcap: float = 0.0):
    """Per-row log-sum-exp over this shard's vocabulary and the owned target logit.

    Replaces indexed_matmul (kernels.py:204-251) + lse_forward (kernels.py:254-319) with one
    fused tcgen05 kernel; the only transient is splits x N float2 partials.
    """
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    lse_local = torch.empty(n, dtype=torch.float32, device=dev)
    correct = torch.empty(n, dtype=torch.float32, device=dev)
    if n == 0:
        return lse_local, correct
    ws_bytes = lib.cce_fwd_workspace_bytes(n, d, v)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    ev = _ev_begin("fwd")
    _lib.check(lib.cce_fwd(_p(e), _p(c), _p(targets), n, d, v, int(ignore_index), int(vocab_start),
                           float(softcap or 0.0), _p(ws), ws_bytes, _p(lse_local), _p(correct),
                           _stream(dev)), "cce_fwd")
    _ev_end("fwd", ev)
    LAUNCHES["count"] += 3
    return lse_local, correct


def merge_shards(lse_parts, correct_parts, targets, ignore_index: int):
    """log_add_exp merge over shards (kernels.py:121-137) + the cce_loss scatter (:539-547)."""
    lib = _lib.load()
    p, n = lse_parts.shape
    lse = torch.empty(n, dtype=torch.float32, device=lse_parts.device)
    loss = torch.empty(n, dtype=torch.float32, device=lse_parts.device)
    if n:
        _lib.check(lib.cce_merge_shards(p, _p(lse_parts.contiguous()), _p(correct_parts.contiguous()),
                                        _p(targets), int(ignore_index), n, _p(lse), _p(loss),
                                        _stream(lse_parts.device)), "cce_merge_shards")
        LAUNCHES["count"] += 1
    return lse, loss


def indexed_dot(e, c, targets, ignore_index: int, vocab_start: int = 0, softcap: float = 0.0):
    """out[i] = C[x_i] . E[i], 0 at ignored rows (indexed_matmul, kernels.py:204-251)."""
    lib = _lib.load()
    n, d = e.shape
    out = torch.empty(n, dtype=torch.float32, device=e.device)
    if n:
        _lib.check(lib.cce_indexed_dot(_p(e), _p(c), _p(targets), n, d, c.shape[0], int(ignore_index),
                                       int(vocab_start), float(softcap or 0.0), _p(out),
                                       _stream(e.device)), "cce_indexed_dot")
    return out


def vocab_order(e, c, targets, ignore_index: int, n_valid: int):
    """(perm, mean_logits): stable descending sort of C . mean(E[valid]) (kernels.py:145-160)."""
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    ebar = torch.empty(d, dtype=torch.float32, device=dev)
    _lib.check(lib.cce_ebar(_p(e), _p(targets), int(ignore_index), n, d, _p(ebar), _stream(dev)), "cce_ebar")
    perm = torch.empty(v, dtype=torch.int32, device=dev)
    key = torch.empty(v, dtype=torch.float32, device=dev)
    ws_bytes = lib.cce_sort_workspace_bytes(v)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _lib.check(lib.cce_vocab_order(_p(c), _p(ebar), int(n_valid), v, d, _p(perm), _p(key), _p(ws),
                                   ws_bytes, _stream(dev)), "cce_vocab_order")
    LAUNCHES["count"] += 3 + 5  # ebar, sort key, iota + CUB onesweep radix sort passes
    return perm, key


@dataclass
class BackwardStats:
    """Tile accounting of one backward pass (BackwardStats, kernels.py:66-76)."""

    total_tiles: int = 0
    skipped_epsilon: int = 0
    skipped_zero_upstream: int = 0

    @property
    def skipped_tiles(self) -> int:
        return self.skipped_epsilon + self.skipped_zero_upstream

    @property
    def kept_tiles(self) -> int:
        return self.total_tiles - self.skipped_tiles


def _pad_to(x: torch.Tensor, mult: int, value: int = 0) -> torch.Tensor:
    n = x.shape[0]
    m = -(-n // mult) * mult
    if m == n:
        return x.contiguous()
    out = torch.full((m,), value, dtype=x.dtype, device=x.device)
    out[:n] = x
    return out


def backward(e, c, targets, lse, upstream, *, ignore_index: int, vocab_start: int = 0,
             softcap: float = 0.0, eps: float | None = EPSILON_DEFAULT, vocab_sorting: bool = True,
             perm: torch.Tensor | None = None, fp32_de: bool = False):
    """Filtered, vocab-sorted CCE backward (lse_backward, kernels.py:327-486).

    Ignored rows are compacted first (filter_ignored, kernels.py:494-510) so token tiles hold
    valid rows only, exactly as cce_loss does before calling lse_backward.  `upstream` must be
    0 at ignored rows.  Returns (dE, dC, counters[3] tensor, perm).  With fp32_de the fp32 dE
    accumulator is returned instead of its bf16 cast (vocab-parallel all-reduces it first).
    """
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    stream = _stream(dev)
    valid = targets != ignore_index
    idx = torch.nonzero(valid).squeeze(1)
    n_valid = int(idx.numel())
    if n_valid == n:
        row_map = None
        lse_c, up_c, tg_c = lse, upstream, targets
    else:
        row_map = _pad_to(idx.to(torch.int32), BLOCK_TOKENS)
        lse_c, up_c, tg_c = lse[idx].contiguous(), upstream[idx].contiguous(), targets[idx].contiguous()
    lse_c = lse_c.to(torch.float32).contiguous()
    up_c = up_c.to(torch.float32).contiguous()

    if vocab_sorting and perm is None and n_valid > 0:
        perm, _ = vocab_order(e, c, targets, ignore_index, n_valid)
    vpad = -(-v // BLOCK_VOCAB) * BLOCK_VOCAB
    nt = max(1, -(-n_valid // BLOCK_TOKENS))
    perm_padded = torch.empty(vpad, dtype=torch.int32, device=dev) if perm is not None else None
    inv_perm = torch.empty(v, dtype=torch.int32, device=dev) if perm is not None else None
    pos = torch.empty(max(n_valid, 1), dtype=torch.int32, device=dev)
    block_zero = torch.empty(nt, dtype=torch.uint8, device=dev)
    _lib.check(lib.cce_bwd_prep(_p(perm), v, _p(tg_c), int(ignore_index), int(vocab_start), _p(up_c),
                                n_valid, _p(perm_padded), _p(inv_perm), _p(pos), _p(block_zero),
                                stream), "cce_bwd_prep")
    LAUNCHES["count"] += 3 if perm is not None else 2
    compacted = row_map is not None
    de_dtype = torch.float32 if fp32_de else torch.bfloat16
    de = (torch.zeros if compacted or n_valid == 0 else torch.empty)(n, d, dtype=de_dtype, device=dev)
    dc = (torch.zeros if n_valid == 0 else torch.empty)(v, d, dtype=torch.bfloat16, device=dev)
    counters = torch.zeros(3, dtype=torch.int64, device=dev)
    if n_valid == 0:
        return de, dc, counters, perm
    filt_eps = 0.0 if (eps is None or eps == 0) else float(eps)
    mt = -(-v // BLOCK_VOCAB)
    budget = shat_budget_tiles()
    # first try: every token tile in one group, compact S-hat slots up to the budget
    plans = [(nt, min(budget, nt * mt))]
    if plans[0][1] < nt * mt:
        g = max(1, budget // mt)          # fallback: groups whose worst case fits the budget
        plans.append((g, g * mt))
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    # Vocabulary order: materialise C[perm] once (1 HBM read + write of C) so every tile load in
    # the backward is a plain TMA box; CCE_SORT_GATHER=1 instead gathers rows with TMA gather4
    # inside the kernels (no copy, but gather-bound).
    c_src, c_sorted = c, 0
    if perm is not None and os.environ.get("CCE_SORT_GATHER", "0") != "1":
        c_src = torch.empty_like(c)
        _lib.check(lib.cce_gather_rows(_p(c), _p(perm), v, d, _p(c_src), stream), "cce_gather_rows")
        LAUNCHES["count"] += 1
        c_sorted = 1
    for i, (g, cap) in enumerate(plans):
        ws_bytes = lib.cce_bwd_workspace_bytes(n_valid, d, v, g, cap)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        if i:
            counters.zero_()
        ev = _ev_begin("bwd")
        _lib.check(lib.cce_bwd(_p(e), n, _p(c_src), _p(perm_padded), _p(row_map), _p(pos), _p(lse_c),
                               _p(up_c), _p(block_zero), n_valid, d, v, float(softcap or 0.0), filt_eps,
                               g, cap, c_sorted, _p(ws), ws_bytes, _p(de), int(fp32_de), _p(dc),
                               _p(counters), _p(overflow), stream), "cce_bwd")
        _ev_end("bwd", ev)
        LAUNCHES["count"] += 3 * (-(-nt // g))
        del ws
        # the single-group plan can only overflow when the budget is below the worst case;
        # checking needs one host read, paid only in that situation
        if i + 1 == len(plans) or int(overflow.item()) == 0:
            break
        overflow.zero_()
        LAST_OVERFLOW["count"] += 1
    LAST_COUNTERS["counters"] = counters
    return de, dc, counters, perm


def shat_budget_tiles() -> int:
    """S-hat slots (64 KiB each) the backward may hold: CCE_SHAT_BUDGET_MB (default 2048)."""
    budget = int(os.environ.get("CCE_SHAT_BUDGET_MB", "2048")) << 20
    return max(1, budget // (BLOCK_TOKENS * BLOCK_VOCAB * 2))


def f32_to_bf16(x: torch.Tensor) -> torch.Tensor:
    lib = _lib.load()
    y = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    _lib.check(lib.cce_f32_to_bf16(_p(x.contiguous()), _p(y), x.numel(), _stream(x.device)), "cce_f32_to_bf16")
    return y


def stats_from_counters(counters: torch.Tensor, n_valid: int, v: int) -> BackwardStats:
    k = counters.tolist()
    nt = -(-n_valid // BLOCK_TOKENS)
    mt = -(-v // BLOCK_VOCAB)
    return BackwardStats(total_tiles=nt * mt, skipped_epsilon=int(k[1]), skipped_zero_upstream=int(k[2]))
