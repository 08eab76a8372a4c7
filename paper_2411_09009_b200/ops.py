"""Torch-facing wrappers of the C ABI (include/cce_b200.h).

Each function validates, allocates outputs/workspaces with torch (so every byte shows up in
torch.cuda.max_memory_allocated, mirroring instrument.py's scratch/output accounting) and calls
exactly one or two C entry points on the current CUDA stream.  No function here computes
anything on the host; if libcce_b200.so is missing, the first call raises.
"""

from __future__ import annotations

import ctypes
import functools
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
LAST_OVERFLOW: dict = {}  # device flag of the last backward: 1 if the fallback pass ran
LAST_STATS: dict = {}     # tile-path backward: [label tiles stored by the forward, tiles recomputed]


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


def recorded_event() -> torch.cuda.Event:
    """A CUDA event that already exists (recorded once on the current stream), so its handle can
    go to the C ABI: a torch Event is created lazily and its handle is 0 until first recorded, and
    the library re-records it (cudaEventRecord) only when the handle is nonzero."""
    ev = torch.cuda.Event()
    ev.record()
    return ev


def _event_handle(ev) -> ctypes.c_void_p:
    if ev is None:
        return ctypes.c_void_p(0)
    if ev.cuda_event == 0:
        ev.record()
    return ctypes.c_void_p(ev.cuda_event)


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


def adapt_operands(e: torch.Tensor, c: torch.Tensor):
    """Bring caller operands to the kernels' layout: floating inputs are cast to bf16 (the compute
    type), a strided classifier is made contiguous, and a hidden size that is not a multiple of 8
    (16-byte TMA rows; the reference tests use d=4, test_kernels.py:361) is zero-padded -- zero
    columns add nothing to any logit, and autograd slices the padding off dE / dC.  Anything that
    is not a float, not 2-D or has mismatched feature dims is left for check_operands to reject."""
    def cast(t):
        if t.is_floating_point() and t.dtype != torch.bfloat16:
            t = t.to(torch.bfloat16)
        return t if t.is_contiguous() else t.contiguous()

    e, c = cast(e), cast(c)
    if e.dim() == 2 and c.dim() == 2 and e.shape[1] == c.shape[1] and e.shape[1] % 8:
        pad = 8 - e.shape[1] % 8
        e = torch.nn.functional.pad(e, (0, pad))
        c = torch.nn.functional.pad(c, (0, pad))
    return e, c


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
    return lse_local, correct


def merge_shards(lse_parts, correct_parts, targets, ignore_index: int, v_total: int = 0):
    """log_add_exp merge over shards (kernels.py:121-137) + the cce_loss scatter (:539-547).

    v_total > 0 adds the reference's label-range check (check_vocab, core.py:110-114) on the
    device: a label outside [0, v_total) that is not ignore_index gives a NaN loss and raises
    the sticky device flag that `raise_label_error` reports (no host synchronisation here)."""
    lib = _lib.load()
    p, n = lse_parts.shape
    dev = lse_parts.device
    lse = torch.empty(n, dtype=torch.float32, device=dev)
    loss = torch.empty(n, dtype=torch.float32, device=dev)
    if n:
        flag = _label_state(dev)[0] if v_total > 0 else None
        _lib.check(lib.cce_merge_shards_checked(p, _p(lse_parts.contiguous()), _p(correct_parts.contiguous()),
                                                _p(targets), int(ignore_index), n, int(v_total), _p(flag),
                                                _p(lse), _p(loss), _stream(dev)), "cce_merge_shards_checked")
        if flag is not None:
            _queue_label_flag(dev)
    return lse, loss


# Label-range errors found on the device: per device [flag (device int32, sticky), pinned copy,
# event of the copy in flight].  The flag is copied back asynchronously after each checked merge
# and read (never waited for) by the next call, which raises the reference's ValueError.
_LABEL_STATE: dict = {}


def _label_state(dev: torch.device):
    key = (dev.type, dev.index if dev.index is not None else torch.cuda.current_device())
    st = _LABEL_STATE.get(key)
    if st is None:
        st = _LABEL_STATE[key] = [torch.zeros(1, dtype=torch.int32, device=dev),
                                  torch.zeros(1, dtype=torch.int32).pin_memory(), None]
    return st


def _queue_label_flag(dev: torch.device) -> None:
    if _capturing():
        return
    st = _label_state(dev)
    if st[2] is not None:
        return  # previous copy still in flight; it is read first
    st[1].copy_(st[0], non_blocking=True)
    st[2] = torch.cuda.Event()
    st[2].record()


def raise_label_error(dev: torch.device, v_total: int, wait: bool = False) -> None:
    """Raise ValueError if an earlier call on `dev` saw a label outside [0, v_total) (the device
    flag of merge_shards).  Without `wait`, only a copy that has already landed is read (no host
    synchronisation); the flag is cleared once reported."""
    if _capturing():
        return
    st = _label_state(dev)
    if wait:
        if st[2] is None:
            _queue_label_flag(dev)
        st[2].synchronize()
    if st[2] is None or not st[2].query():
        return
    st[2] = None
    if int(st[1][0]) != 0:
        st[0].zero_()
        st[1].zero_()
        raise ValueError(f"label out of range for vocab size {v_total} (found on the device by an earlier "
                         "call, whose loss is NaN at those rows)")


def shard_targets(targets: torch.Tensor, vocab_rows: torch.Tensor, v_total: int, ignore_index: int) -> torch.Tensor:
    """Labels in the coordinates of a shard holding global rows `vocab_rows` (local row k holds
    global id vocab_rows[k]): an owned label becomes its local row, any other label the first row
    past the shard (owned by another rank, as a label outside [vocab_start, vocab_start + V) is
    for a contiguous shard), ignore_index stays.  On the device, O(N + V), no host read.  Labels
    outside [0, v_total) are caught by merge_shards on the caller's targets."""
    v_loc = vocab_rows.shape[0]
    lut = torch.full((v_total + 1,), v_loc, dtype=torch.int64, device=targets.device)
    lut[vocab_rows.to(torch.int64)] = torch.arange(v_loc, device=targets.device)
    local = lut[targets.clamp(0, v_total)]
    return torch.where(targets == ignore_index, targets, local).contiguous()


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


def vocab_order(e, c, targets, ignore_index: int, n_valid):
    """(perm, mean_logits): stable descending sort of C . mean(E[valid]) (kernels.py:145-160).

    `n_valid` is the device int32 count of valid rows (or a host int)."""
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    if not torch.is_tensor(n_valid):
        n_valid = torch.tensor([int(n_valid)], dtype=torch.int32, device=dev)
    ebar = torch.empty(d, dtype=torch.float32, device=dev)
    ebar_ws_bytes = lib.cce_ebar_workspace_bytes(n, d)
    ebar_ws = torch.empty(max(ebar_ws_bytes, 16), dtype=torch.uint8, device=dev)
    _lib.check(lib.cce_ebar(_p(e), _p(targets), int(ignore_index), n, d, _p(ebar), _p(ebar_ws),
                            ebar_ws_bytes, _stream(dev)), "cce_ebar")
    perm = torch.empty(v, dtype=torch.int32, device=dev)
    key = torch.empty(v, dtype=torch.float32, device=dev)
    ws_bytes = lib.cce_sort_workspace_bytes(v)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _lib.check(lib.cce_vocab_order(_p(c), _p(ebar), _p(n_valid), v, d, _p(perm), _p(key), _p(ws),
                                   ws_bytes, _stream(dev)), "cce_vocab_order")
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


def compact_rows(targets, ignore_index: int):
    """Device-side filter_ignored (kernels.py:494-510): (row_map padded to a multiple of 128,
    n_valid as a device int32[1]).  No host synchronisation."""
    lib = _lib.load()
    n = targets.shape[0]
    dev = targets.device
    row_map = torch.empty(max(1, -(-n // BLOCK_TOKENS) * BLOCK_TOKENS), dtype=torch.int32, device=dev)
    n_valid = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.check(lib.cce_compact_rows(_p(targets), int(ignore_index), n, _p(row_map), _p(n_valid),
                                    _stream(dev)), "cce_compact_rows")
    return row_map, n_valid


NO_COMPACTION = -(2 ** 62)  # an ignore value no label can take: compact_rows keeps every row


def backward(e, c, targets, lse, upstream, *, ignore_index: int, vocab_start: int = 0,
             softcap: float = 0.0, eps: float | None = EPSILON_DEFAULT, vocab_sorting: bool = True,
             perm: torch.Tensor | None = None, fp32_de: bool = False, compact: bool = True):
    """Filtered, vocab-sorted CCE backward (lse_backward, kernels.py:327-486).

    Ignored rows are compacted on the device first (filter_ignored, kernels.py:494-510), so
    token tiles hold valid rows only, exactly as cce_loss does before calling lse_backward.
    `lse` / `upstream` are per original row; `upstream` must be 0 at ignored rows.  Returns
    (dE, dC, counters[3] tensor, perm); with fp32_de, dE stays fp32 (vocab-parallel all-reduces
    it before the cast).  The whole call is asynchronous: no value is read back to the host.
    compact=False keeps every row in place, as the reference's lse_backward does (ignored rows
    then only carry zero upstream), so tile counts follow its uncompacted grid.
    """
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    stream = _stream(dev)
    lse = lse.to(torch.float32).contiguous()
    upstream = upstream.to(torch.float32).contiguous()
    row_map, n_valid = compact_rows(targets, ignore_index if compact else NO_COMPACTION)
    if vocab_sorting and perm is None:
        perm, _ = vocab_order(e, c, targets, ignore_index, n_valid)
    vpad = -(-v // BLOCK_VOCAB) * BLOCK_VOCAB
    nt = max(1, -(-n // BLOCK_TOKENS))
    mt = -(-v // BLOCK_VOCAB)
    perm_padded = torch.empty(vpad, dtype=torch.int32, device=dev) if perm is not None else None
    inv_perm = torch.empty(v, dtype=torch.int32, device=dev) if perm is not None else None
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.cce_bwd_prep(_p(perm), v, _p(targets), int(ignore_index), int(vocab_start), n,
                                _p(perm_padded), _p(inv_perm), _p(pos), stream), "cce_bwd_prep")
    de = torch.zeros(n, d, dtype=torch.float32 if fp32_de else torch.bfloat16, device=dev)
    dc = torch.empty(v, d, dtype=torch.bfloat16, device=dev)
    if n == 0:
        return de, dc.zero_(), torch.zeros(3, dtype=torch.int64, device=dev), perm
    filt_eps = 0.0 if (eps is None or eps == 0) else float(eps)
    gather = os.environ.get("CCE_SORT_GATHER", "0") == "1"
    # Vocabulary order: materialise C[perm] once (one HBM read + write of C) so every tile load of
    # the backward is a plain TMA box; CCE_SORT_GATHER=1 instead gathers rows (C through perm, E
    # through row_map) with TMA gather4 inside the kernels: no copies, but gather-bound.
    c_src, c_sorted = c, 0
    if perm is not None and not gather:
        c_src = torch.empty_like(c)
        _lib.check(lib.cce_gather_rows(_p(c), _p(perm), v, d, _p(c_src), stream), "cce_gather_rows")
        c_sorted = 1
    # S-hat slots: every token tile in one group with compact slots up to the budget; if more
    # tiles are kept than that, a fallback pass over budget-sized groups (worst case fits) runs,
    # gated on the device overflow flag -- no host read either way.
    key = ("filter_pass", d, v, int(vocab_start), filt_eps, float(softcap or 0.0))
    cap0 = shat_capacity(key, nt, mt)
    plans = [(nt, cap0, None)]
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    if cap0 < nt * mt:
        g = max(1, cap0 // mt)
        plans.append((g, g * mt, overflow))
    all_counters = []
    ws_bytes = max(lib.cce_bwd_workspace_bytes(n, d, v, g, cap) for g, cap, _ in plans)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    for g, cap, run_if in plans:
        counters = torch.zeros(3, dtype=torch.int64, device=dev)
        ev = _ev_begin("bwd")
        _lib.check(lib.cce_bwd(_p(e), _p(c_src), _p(perm_padded), c_sorted, _p(row_map), _p(n_valid),
                               _p(pos), _p(lse), _p(upstream), n, d, v, float(softcap or 0.0), filt_eps,
                               g, cap, _p(run_if), int(gather), _p(ws), ws_bytes, _p(de), int(fp32_de),
                               _p(dc), _p(counters), _p(overflow if run_if is None else None), stream),
                   "cce_bwd")
        _ev_end("bwd", ev)
        all_counters.append(counters)
    counters = all_counters[0] if len(plans) == 1 else torch.where(overflow.bool(), all_counters[1], all_counters[0])
    _remember_kept(key, counters, nt)
    LAST_COUNTERS["counters"] = counters
    LAST_OVERFLOW["flag"] = overflow
    return de, dc, counters, perm


def label_terms(e, c, perm_padded, row_map, n_valid, pos, upstream, correct, softcap: float, de, dc):
    """The label term of the paper ordering, applied exactly (cce_label_terms): de[i] and
    dc[x_i] += -upstream_i (1 - tanh^2) C[x_i] / E[i]."""
    lib = _lib.load()
    n, d = e.shape
    if n == 0:
        return
    ws_bytes = lib.cce_label_terms_workspace_bytes(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=e.device)
    _lib.check(lib.cce_label_terms(_p(e), _p(c), _p(perm_padded), _p(row_map), _p(n_valid), _p(pos),
                                   _p(upstream), _p(correct.to(torch.float32).contiguous()), n, d, c.shape[0],
                                   float(softcap or 0.0), _p(ws), ws_bytes, _p(de),
                                   int(de is not None and de.dtype == torch.float32), _p(dc), _stream(e.device)),
               "cce_label_terms")


LOWMEM_SHAT_MB = 256  # S-hat slots of one vocabulary group in the low-memory backward
LOWMEM_CG_MB = 256    # classifier rows of one vocabulary group


GROUPED_SHAT_MB = 128  # low_memory=True (vocabulary groups sized from the learned density)


def lowmem_group_vtiles(n: int, d: int, v: int, default_mb: int = LOWMEM_SHAT_MB) -> int:
    """Vocab tiles per group of the low-memory backward: the worst-case S-hat of a group
    (every token tile x every group vocab tile) within CCE_LOWMEM_SHAT_MB (else default_mb), and
    the group's classifier rows within LOWMEM_CG_MB."""
    budget = int(os.environ.get("CCE_LOWMEM_SHAT_MB", default_mb)) << 20
    nt = max(1, -(-n // BLOCK_TOKENS))
    mt = -(-v // BLOCK_VOCAB)
    by_shat = budget // (nt * BLOCK_TOKENS * BLOCK_VOCAB * 2)
    by_cg = (LOWMEM_CG_MB << 20) // (BLOCK_VOCAB * d * 2)
    return max(1, min(mt, by_shat, by_cg))


GROUP_MARGIN = 1.3  # headroom of the learned kept density when sizing vocabulary groups


def grouped_plan(n: int, d: int, v: int, key) -> tuple[list, int]:
    """(vocab-tile ranges of the groups, S-hat slots per group) for low_memory=True.

    Until kept counts of this shape have been observed: the worst case, equal groups with every
    tile of a group kept (lowmem_group_vtiles).  Afterwards the same memory -- the worst-case
    plan's S-hat slots plus one group's classifier rows -- is split in halves between slots and
    rows, and vocab tiles are packed greedily by the previous call's kept tiles per vocab tile
    (1.3x margin): dense tiles (the head of the sorted vocabulary under Zipf-like logits) form
    small groups, sparse ones large groups.  A group that keeps more than its slots takes the
    on-device overflow path of cce_bwd_kept."""
    nt = max(1, -(-n // BLOCK_TOKENS))
    mt = -(-v // BLOCK_VOCAB)
    # 128 MB measured best for this mode: 13.3 ms / 275 MiB vs 13.0 ms / 443 MiB at 256 MB
    # (Gemma-2-2B, profiles/r1/ab/ab_lowmem_budget.txt)
    gv0 = lowmem_group_vtiles(n, d, v, GROUPED_SHAT_MB)
    worst = ([(m0, min(mt, m0 + gv0)) for m0 in range(0, mt, gv0)], nt * gv0)
    if os.environ.get("CCE_LOWMEM_WORST", "0") == "1":
        return worst
    hint = _KEPT_HINT.get(key + ("per-vtile",))
    if hint is None:
        return worst
    _harvest(hint)
    cnt = hint[2]
    if cnt is None or len(cnt) != mt:
        return worst
    rows_bytes = BLOCK_VOCAB * d * 2
    budget = nt * gv0 * SHAT_TILE_BYTES + gv0 * rows_bytes  # the worst-case plan's memory
    slots = max(1, budget // 2 // SHAT_TILE_BYTES)
    # cce_bwd_kept needs at least one token tile's vocab tiles of slots: groups stay <= slots
    gmax = int(max(1, min(mt, budget // 2 // rows_bytes, slots)))
    bounds, m0, acc = [], 0, 0.0
    for m in range(mt):
        need = GROUP_MARGIN * cnt[m]
        if m > m0 and (m - m0 >= gmax or acc + need + (m + 1 - m0) > slots):
            bounds.append((m0, m))
            m0, acc = m, 0.0
        acc += need
    bounds.append((m0, mt))
    return bounds, int(slots)


def backward_lowmem(e, c, targets, lse, upstream, *, ignore_index: int, vocab_start: int = 0,
                    softcap: float = 0.0, eps: float | None = EPSILON_DEFAULT, vocab_sorting: bool = True,
                    perm: torch.Tensor | None = None, fp32_de: bool = False,
                    label_split: bool = False, correct: torch.Tensor | None = None):
    """lse_backward (kernels.py:327-486) over vocabulary groups with bounded transients.

    Ignored rows are compacted on the device (kernels.py:494-510); the vocabulary order is the
    reference's (kernels.py:145-160).  Per group of vocab tiles: the group's sorted classifier
    rows, the filter pass over every tile of the group (recompute, decision, S-hat), dE
    accumulated in fp32, dC of the group's rows.  Transient memory is the compacted E, an fp32 dE
    accumulator and one group's classifier rows and S-hat slots -- nothing grows with V or with
    the kept-tile count.  Returns (dE, dC, counters[3], perm).
    """
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    stream = _stream(dev)
    lse = lse.to(torch.float32).contiguous()
    upstream = upstream.to(torch.float32).contiguous()
    row_map, n_valid = compact_rows(targets, ignore_index)
    if vocab_sorting and perm is None:
        perm, _ = vocab_order(e, c, targets, ignore_index, n_valid)
    vpad = -(-v // BLOCK_VOCAB) * BLOCK_VOCAB
    perm_padded = torch.empty(vpad, dtype=torch.int32, device=dev) if perm is not None else None
    inv_perm = torch.empty(v, dtype=torch.int32, device=dev) if perm is not None else None
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.cce_bwd_prep(_p(perm), v, _p(targets), int(ignore_index), int(vocab_start), n,
                                _p(perm_padded), _p(inv_perm), _p(pos), stream), "cce_bwd_prep")
    del inv_perm
    de_acc = torch.zeros(n, d, dtype=torch.float32, device=dev)
    dc = torch.empty(v, d, dtype=torch.bfloat16, device=dev)
    counters = torch.zeros(3, dtype=torch.int64, device=dev)
    if n == 0:
        return (de_acc if fp32_de else de_acc.to(torch.bfloat16)), dc.zero_(), counters, perm
    gv = lowmem_group_vtiles(n, d, v)
    ws_bytes = lib.cce_bwd_lowmem_workspace_bytes(n, d, v, gv)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    filt_eps = 0.0 if (eps is None or eps == 0) else float(eps)
    ev = _ev_begin("bwd")
    split = bool(label_split) and filt_eps > 0
    _lib.check(lib.cce_bwd_lowmem(_p(e), _p(c), _p(perm_padded), _p(row_map), _p(n_valid), _p(pos),
                                  _p(lse), _p(upstream), n, d, v, float(softcap or 0.0), filt_eps,
                                  int(split), gv, _p(ws), ws_bytes, _p(de_acc), _p(dc), _p(counters),
                                  stream), "cce_bwd_lowmem")
    del ws
    if split:
        label_terms(e, c, perm_padded, row_map, n_valid, pos, upstream, correct, softcap, de_acc, dc)
    _ev_end("bwd", ev)
    LAST_COUNTERS["counters"] = counters
    de = de_acc if fp32_de else f32_to_bf16(de_acc)
    return de, dc, counters, perm


@dataclass
class TileState:
    """What the filter-from-forward path hands from the forward to the backward.

    e_c      compacted rows of E (filter_ignored, kernels.py:494-510) [n, d] bf16
    c_t      classifier in tile order: C[perm] (vocab sorting) or C itself
    row_map / n_valid   compaction (device), perm / perm_padded (None without sorting)
    pos      label position in tile order per original row (-1 ignored / other shard)
    tile_max [nt, mt, 128] fp32 max raw logit per compact row per tile
    """

    e: torch.Tensor
    c: torch.Tensor
    e_c: torch.Tensor
    c_t: torch.Tensor
    row_map: torch.Tensor
    n_valid: torch.Tensor
    perm: torch.Tensor | None
    perm_padded: torch.Tensor | None
    pos: torch.Tensor
    tile_max: torch.Tensor
    vocab_start: int
    softcap: float
    mean_logits: torch.Tensor | None = None
    # S-hat slots [stored label tiles (lab_cap) | recomputed tiles (rcap)], allocated by the forward
    shat: torch.Tensor | None = None
    lab_cap: int = 0
    rcap: int = 0
    lab_slot: torch.Tensor | None = None
    lab_list: torch.Tensor | None = None
    lab_count: torch.Tensor | None = None
    keys: tuple = ()

    def nbytes(self) -> int:
        own = [self.e_c, self.row_map, self.n_valid, self.pos, self.tile_max]
        own += [t for t in (self.shat, self.lab_slot, self.lab_list, self.lab_count) if t is not None]
        if self.perm is not None:
            own += [self.c_t, self.perm, self.perm_padded]
        return sum(t.numel() * t.element_size() for t in own if t is not None)


def gather_rows(src: torch.Tensor, index: torch.Tensor, rows: int) -> torch.Tensor:
    """dst[i] = src[index[i]] for i < rows (bf16 rows)."""
    lib = _lib.load()
    dst = torch.empty(rows, src.shape[1], dtype=src.dtype, device=src.device)
    if rows:
        _lib.check(lib.cce_gather_rows(_p(src), _p(index), rows, src.shape[1], _p(dst),
                                       _stream(src.device)), "cce_gather_rows")
    return dst


def forward_tiles(e, c, targets, ignore_index: int, vocab_start: int = 0, softcap: float = 0.0,
                  vocab_sorting: bool = True, perm: torch.Tensor | None = None,
                  eps: float = EPSILON_DEFAULT, label_split: bool = False, store_labels: bool = True):
    """Forward of the filter-from-forward path: (lse_local, correct, TileState).

    Same results as forward_local (indexed_matmul + lse_forward, kernels.py:204-319), computed
    the way cce_loss orders the work: ignored rows are compacted first (kernels.py:494-510, 531)
    and, with vocab sorting, the vocabulary order (compute_vocab_order, kernels.py:145-160; the
    mean logit C.ebar is a GEMV of the valid rows' mean) is fixed before the tile sweep so the
    forward visits exactly the backward's tiles and records each row's max logit per tile.
    """
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    stream = _stream(dev)
    row_map, n_valid = compact_rows(targets, ignore_index)
    e_c = gather_rows(e, row_map, n)
    mean_logits = None
    if vocab_sorting and perm is None:
        perm, mean_logits = vocab_order(e, c, targets, ignore_index, n_valid)
    vpad = -(-v // BLOCK_VOCAB) * BLOCK_VOCAB
    perm_padded = torch.empty(vpad, dtype=torch.int32, device=dev) if perm is not None else None
    inv_perm = torch.empty(v, dtype=torch.int32, device=dev) if perm is not None else None
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.cce_bwd_prep(_p(perm), v, _p(targets), int(ignore_index), int(vocab_start), n,
                                _p(perm_padded), _p(inv_perm), _p(pos), stream), "cce_bwd_prep")
    c_t = gather_rows(c, perm, v) if perm is not None else c
    tile_max = torch.empty(lib.cce_tile_max_bytes(n, v) // 4, dtype=torch.float32, device=dev)
    lse_local = torch.empty(n, dtype=torch.float32, device=dev)
    correct = torch.empty(n, dtype=torch.float32, device=dev)
    state = TileState(e, c, e_c, c_t, row_map, n_valid, perm, perm_padded, pos, tile_max,
                      int(vocab_start), float(softcap or 0.0), mean_logits)
    if n == 0:
        return lse_local, correct, state
    # S-hat slots for the backward, allocated here because the forward fills the label region:
    # tiles holding a label are always kept (kernels.py:447-455), so their logits are stored now
    # and turned into S-hat without a recompute
    nt = -(-n // BLOCK_TOKENS)
    mt = -(-v // BLOCK_VOCAB)
    # storing a label tile costs the forward's epilogue a fixed amount per tile, recomputing it
    # costs the backward 2 * 128 * 256 * D: measured break-even between D = 768 (GPT-2: 1.35 vs
    # 1.39 ms per step without) and D = 2304 (Gemma-2-2B: 11.5 vs 12.1 ms with), so small heads
    # recompute (profiles/r1/ab/ab_store_labels_by_d.txt).  CCE_STORE_LABELS=0 / 1 forces it.
    env = os.environ.get("CCE_STORE_LABELS")
    store_labels = store_labels and (env == "1" if env in ("0", "1") else d >= LABEL_STORE_MIN_D)
    # capacity hints are keyed by the head, not the batch: a count observed at another N is
    # rescaled by the token-tile ratio (kept tiles grow linearly with the token tiles)
    rkey = ("recompute", d, v, int(vocab_start), float(eps), float(softcap or 0.0), bool(label_split),
            bool(store_labels))
    lkey = ("labels", d, v, int(vocab_start))
    state.rcap = shat_capacity(rkey, nt, mt)
    state.lab_cap = label_capacity(lkey, nt, mt) if store_labels else 0
    state.keys = (rkey, lkey)
    state.shat = torch.empty((state.lab_cap + state.rcap) * SHAT_TILE_BYTES, dtype=torch.uint8, device=dev)
    if state.lab_cap:
        state.lab_slot = torch.empty(nt * mt, dtype=torch.int32, device=dev)
        state.lab_list = torch.empty(state.lab_cap, 2, dtype=torch.int32, device=dev)
        state.lab_count = torch.empty(1, dtype=torch.int32, device=dev)
    ws_bytes = lib.cce_fwd_workspace_bytes(n, d, v)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    ev = _ev_begin("fwd")
    _lib.check(lib.cce_fwd_tiles(_p(e_c), _p(c_t), _p(row_map), _p(n_valid), _p(pos), 0, n, d, v,
                                 float(softcap or 0.0), _p(ws), ws_bytes, _p(lse_local), _p(correct),
                                 _p(tile_max), _p(state.shat if state.lab_cap else None), state.lab_cap,
                                 _p(state.lab_slot), _p(state.lab_list), _p(state.lab_count), stream),
               "cce_fwd_tiles")
    _ev_end("fwd", ev)
    return lse_local, correct, state


@dataclass
class GatherState:
    """What the copy-free training forward hands to the backward: only O(N + V) maps plus the
    per-row tile maxima -- no compacted E, no sorted classifier (rows are gathered through
    row_map / perm inside the kernels)."""

    e: torch.Tensor
    c: torch.Tensor
    row_map: torch.Tensor
    n_valid: torch.Tensor
    perm: torch.Tensor | None
    perm_padded: torch.Tensor | None
    pos: torch.Tensor
    tile_max: torch.Tensor
    vocab_start: int
    softcap: float
    mean_logits: torch.Tensor | None = None

    def nbytes(self) -> int:
        own = [self.row_map, self.n_valid, self.pos, self.tile_max, self.perm, self.perm_padded]
        return sum(t.numel() * t.element_size() for t in own if t is not None)


def prepare_order(e, c, targets, ignore_index: int, vocab_start: int = 0, vocab_sorting: bool = True,
                  perm: torch.Tensor | None = None, with_inverse: bool = False):
    """Compaction (filter_ignored, kernels.py:494-510), the vocabulary order (compute_vocab_order,
    kernels.py:145-160) and label positions in that order: (row_map, n_valid, perm, perm_padded,
    pos, mean_logits[, inv_perm]).  All on the device, O(N + V)."""
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    row_map, n_valid = compact_rows(targets, ignore_index)
    mean_logits = None
    if vocab_sorting and perm is None:
        perm, mean_logits = vocab_order(e, c, targets, ignore_index, n_valid)
    vpad = -(-v // BLOCK_VOCAB) * BLOCK_VOCAB
    if perm is None:  # natural order: gathers through the identity keep one code path
        perm = torch.arange(v, dtype=torch.int32, device=dev)
    perm_padded = torch.empty(vpad, dtype=torch.int32, device=dev)
    inv_perm = torch.empty(v, dtype=torch.int32, device=dev)
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.cce_bwd_prep(_p(perm), v, _p(targets), int(ignore_index), int(vocab_start), n,
                                _p(perm_padded), _p(inv_perm), _p(pos), _stream(dev)), "cce_bwd_prep")
    if with_inverse:
        return row_map, n_valid, perm, perm_padded, pos, mean_logits, inv_perm
    return row_map, n_valid, perm, perm_padded, pos, mean_logits


def forward_gather(e, c, targets, ignore_index: int, vocab_start: int = 0, softcap: float = 0.0,
                   vocab_sorting: bool = True, perm: torch.Tensor | None = None):
    """Copy-free forward of the training path: (lse_local, correct, GatherState).

    The same sweep as forward_tiles (compacted rows, vocabulary order, per-row tile maxima;
    indexed_matmul + lse_forward, kernels.py:204-319), but the kernels read E through row_map and C
    through the vocabulary order with row gathers, so the transients are O(N + V) plus the tile
    maxima."""
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    row_map, n_valid, perm, perm_padded, pos, mean_logits = prepare_order(e, c, targets, ignore_index,
                                                                          vocab_start, vocab_sorting, perm)
    tile_max = torch.empty(lib.cce_tile_max_bytes(n, v) // 4, dtype=torch.float32, device=dev)
    lse_local = torch.empty(n, dtype=torch.float32, device=dev)
    correct = torch.empty(n, dtype=torch.float32, device=dev)
    state = GatherState(e, c, row_map, n_valid, perm if vocab_sorting else None, perm_padded, pos, tile_max,
                        int(vocab_start), float(softcap or 0.0), mean_logits)
    if n == 0:
        return lse_local, correct, state
    ws_bytes = lib.cce_fwd_workspace_bytes(n, d, v)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    ev = _ev_begin("fwd")
    _lib.check(lib.cce_fwd_gather(_p(e), _p(c), _p(perm_padded), _p(row_map), _p(n_valid), _p(pos), 0, n, d, v,
                                  float(softcap or 0.0), _p(ws), ws_bytes, _p(lse_local), _p(correct),
                                  _p(tile_max), _stream(dev)), "cce_fwd_gather")
    _ev_end("fwd", ev)
    return lse_local, correct, state


@dataclass
class StreamState:
    """What the bounded-memory training forward hands to the streamed backward: the caller's E and C
    (rows read through the compaction map / gathered per vocabulary group, never copied whole),
    O(N + V) maps and the per-row tile maxima [ceil(n/128)][ceil(v/256)][128]."""

    e: torch.Tensor
    c: torch.Tensor
    row_map: torch.Tensor
    n_valid: torch.Tensor
    perm: torch.Tensor | None
    perm_padded: torch.Tensor | None
    inv_perm: torch.Tensor | None
    pos: torch.Tensor
    tile_max: torch.Tensor
    vocab_start: int
    softcap: float
    mean_logits: torch.Tensor | None = None
    e_c: torch.Tensor | None = None  # compacted rows, when the batch is expected to ignore some

    def nbytes(self) -> int:
        own = [self.row_map, self.n_valid, self.pos, self.tile_max, self.perm, self.perm_padded, self.inv_perm,
               self.e_c]
        return sum(t.numel() * t.element_size() for t in own if t is not None)


# Whether the last batch of a shape ignored rows: {(n, d): [pinned n_valid copy, event, n_valid]}.
_IGNORED_HINT: dict = {}


def compact_copy_wanted(n: int, d: int, n_valid: torch.Tensor) -> bool:
    """The bounded forward reads E in place when no row is ignored, and through the compaction
    map otherwise.  Row gathers (cp.async) make the forward's E loads request-bound (Llama-3-8B
    with 25% padding: 30 vs 9 ms), so when rows are ignored the compacted rows are copied once
    (N_valid x D, the size of E) and read with plain TMA boxes.  Whether they are is known only on
    the device: the previous call of the same shape decides (its n_valid, read from a pinned copy
    once its event has completed -- never a host synchronisation); unknown counts as ignored.  A
    wrong guess only costs time: without the copy the kernels gather through the map."""
    key = (n, d)
    hint = _IGNORED_HINT.get(key)
    wanted = True
    if hint is not None:
        if hint[1] is not None and not _capturing() and hint[1].query():
            hint[2] = int(hint[0][0])
            hint[1] = None
        if hint[2] is not None:
            wanted = hint[2] < n
    if not _capturing() and (hint is None or hint[1] is None):
        pinned = hint[0] if hint is not None else torch.empty(1, dtype=torch.int32).pin_memory()
        pinned.copy_(n_valid, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        _IGNORED_HINT.pop(key, None)
        while len(_IGNORED_HINT) >= KEPT_HINT_MAX:  # shapes that vary every step: drop the oldest
            _IGNORED_HINT.pop(next(iter(_IGNORED_HINT)))
        _IGNORED_HINT[key] = [pinned, ev, hint[2] if hint is not None else None]
    return wanted


FWD_GROUP_MB = 52  # sorted classifier rows of one vocabulary group in the bounded forward (two buffers)
FWD_FOLD_GROUPS = 8  # groups whose (max, sum-exp) partials are folded by one combine launch


def fwd_group_tiles(d: int, mt: int, n: int = 0, sms: int = 0) -> int:
    """Vocab tiles per group of the bounded forward: the group's sorted rows within
    CCE_FWD_GROUP_MB (default 52 MB: 46 tiles at D = 2304, which keeps the forward's peak, 150 MiB,
    under the backward's 157 MiB), sized so each launch's tiles fill whole waves of the persistent
    grid.  Each group launch sweeps (token-tile pairs) x (group tiles) logit tiles over sms/2 CTA
    pairs and ends when its last wave does; every launch also costs its fill and drain
    (CCE_FWD_LAUNCH_WAVES, 1.5 waves: `scripts/fwd_split_probe.py` measured ~26 us per launch).
    At Gemma-2B: 46 tiles x 32 token-tile pairs = 19.9 waves of 74 pairs, 22 launches; 0.2-0.3 ms
    per forward faster than 37-tile groups (27 launches) and ~0.4 ms faster than the unfitted
    42-tile groups of the 48 MB budget (`scripts/ab_r2/r2_fgroup2.sh`, `r2_fgroup3.sh`).  The
    estimate (waves plus launches) is minimised over sizes down to 3/4 of the budget; batches the
    kernel rasters in bands (many token tiles) keep the budget's size."""
    budget = int(os.environ.get("CCE_FWD_GROUP_MB", FWD_GROUP_MB)) << 20
    cap = max(1, min(mt, budget // (BLOCK_VOCAB * d * 2)))
    if n <= 0 or sms <= 0 or os.environ.get("CCE_FWD_GROUP_FIT", "1") == "0":
        return cap
    return _fitted_group_tiles(d, mt, n, sms, cap, os.environ.get("CCE_PAIR", "1") != "0",
                               float(os.environ.get("CCE_FWD_LAUNCH_WAVES", 1.5)))


@functools.lru_cache(maxsize=256)
def _fitted_group_tiles(d: int, mt: int, n: int, sms: int, cap: int, pair_env: bool, launch_cost: float) -> int:
    pairs = pair_env and sms >= 2
    units = -(-(-(-n // BLOCK_TOKENS)) // (2 if pairs else 1))  # token tiles (pairs) per launch
    grid = sms // 2 if pairs else sms
    if units > max(1, (40 << 20) // (BLOCK_TOKENS * d * 2 * (2 if pairs else 1))) and units >= grid:
        return cap  # banded raster (cce_kernels.cu lse_raster): not whole-wave launches
    # launch_cost (waves): launch gap, pipeline fill and drain of one group launch
    # (scripts/fwd_split_probe.py: 27 launches instead of one cost ~0.67 ms at Gemma-2B, ~1.7 waves
    # of ~15 us each)

    def cost(g):
        full, rest = divmod(mt, g)
        waves = full * -(-(units * g) // grid) + (-(-(units * rest) // grid) if rest else 0)
        return waves + launch_cost * (full + (1 if rest else 0))

    return min(range(cap, max(1, (3 * cap) // 4) - 1, -1), key=cost)  # ties: the larger group


_SMS: dict = {}


def _sm_count(dev: torch.device) -> int:
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _SMS:
        _SMS[key] = torch.cuda.get_device_properties(key).multi_processor_count
    return _SMS[key]


_SIDE: dict = {}


def _side_stream(dev: torch.device) -> torch.cuda.Stream:
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    st = _SIDE.get(key)
    if st is None:
        st = _SIDE[key] = torch.cuda.Stream(dev)
    return st


def forward_stream(e, c, targets, ignore_index: int, vocab_start: int = 0, softcap: float = 0.0,
                   vocab_sorting: bool = True, perm: torch.Tensor | None = None):
    """Bounded-memory forward of the training path: (lse_local, correct, StreamState).

    indexed_matmul + lse_forward (kernels.py:204-319) over the backward's tiles (compacted rows,
    the reference's vocabulary order) with the per-row tile maxima the decision needs, run over
    vocabulary groups: each group's classifier rows are gathered into one of two <= 52 MB buffers (on
    a side stream, while the previous group is swept) and swept with plain TMA tiles; the groups'
    (max, sum-exp) partials are folded by log-add-exp (kernels.py:121-137).  E is read in place
    when no row is ignored and as a compacted copy otherwise (compact_copy_wanted).  Transients:
    the group buffers, the tile maxima, O(N + V) maps (and the compacted rows of a padded batch)."""
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    row_map, n_valid, perm, perm_padded, pos, mean_logits, inv_perm = prepare_order(
        e, c, targets, ignore_index, vocab_start, vocab_sorting, perm, with_inverse=True)
    sorted_ = vocab_sorting or perm is not None
    nt = max(1, -(-n // BLOCK_TOKENS))
    mt = -(-v // BLOCK_VOCAB)
    tile_max = torch.empty(nt * mt * BLOCK_TOKENS, dtype=torch.float32, device=dev)
    e_c = gather_rows(e, row_map, n) if n and compact_copy_wanted(n, d, n_valid) else None
    state = StreamState(e, c, row_map, n_valid, perm if sorted_ else None, perm_padded if sorted_ else None,
                        inv_perm if sorted_ else None, pos, tile_max, int(vocab_start), float(softcap or 0.0),
                        mean_logits, e_c)
    e_rows, e_gather = (e_c, 0) if e_c is not None else (e, 1)
    if n == 0:
        z = torch.zeros(0, dtype=torch.float32, device=dev)
        return z, z.clone(), state
    gt = fwd_group_tiles(d, mt, n, _sm_count(dev))
    groups = [(m0 * BLOCK_VOCAB, min(v, (m0 + gt) * BLOCK_VOCAB)) for m0 in range(0, mt, gt)]
    # the groups' (max, sum-exp) partials side by side after a running one (slot 0), folded into it
    # every FWD_FOLD_GROUPS groups and finished by one combine; the target logit lands in exactly
    # one group, so all groups write one zeroed array
    splits = [lib.cce_fwd_splits(n, d, v1 - v0) for v0, v1 in groups]
    fold = int(os.environ.get("CCE_FWD_FOLD", FWD_FOLD_GROUPS))
    slots = 1 + max(sum(splits[i:i + fold]) for i in range(0, len(groups), fold))
    parts = torch.empty(slots, n, 2, dtype=torch.float32, device=dev)
    parts[0, :, 0] = -float("inf")
    parts[0, :, 1] = 0.0
    correct = torch.zeros(n, dtype=torch.float32, device=dev)
    lse_local = torch.empty(n, dtype=torch.float32, device=dev)
    # two group buffers.  Default: group g + 1's rows are gathered on a side stream while group g
    # is swept, each launch waiting for its gather's event (CCE_FWD_OVERLAP=0: gathers in line).
    # CCE_FWD_CHAIN=1: the group launches form one chain of programmatic dependent launches
    # (cce_fwd_group_sync) -- launch g sweeps group g while its gather warp fills the other buffer
    # with group g + 1 -- synchronised by device flags, so a launch's CTAs start as the previous
    # launch's CTAs exit.  Bit-identical; its forward is 0.2-0.3 ms faster at Gemma-2B, but under
    # the power cap the backward after it runs ~0.15 ms slower (lower clocks), so the step gains
    # ~0.1 ms (`scripts/ab_r2/r2_chain2.sh`): opt-in.
    chain = sorted_ and len(groups) > 1 and os.environ.get("CCE_FWD_CHAIN", "0") == "1" and not _capturing()
    overlap = sorted_ and len(groups) > 1 and os.environ.get("CCE_FWD_OVERLAP", "1") != "0" and not _capturing() \
        and not chain
    rows_g = min(v, gt * BLOCK_VOCAB)
    bufs = [torch.empty(rows_g, d, dtype=torch.bfloat16, device=dev) for _ in range(2 if overlap or chain else 1)] \
        if sorted_ else []
    stream = _stream(dev)
    if chain:
        ev = _ev_begin("fwd")
        forward_chain(lib, e_rows, e_gather, c, perm, row_map, n_valid, pos, n, d, v, softcap, groups, splits,
                      fold, parts, correct, tile_max, lse_local, bufs, stream)
        _ev_end("fwd", ev)
        del parts, bufs
        return lse_local, correct, state
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev) if overlap else None
    gathered = [None, None]  # event: the buffer's gather is done
    released = [None, None]  # event: the sweep reading the buffer is done

    def gather(g):
        v0, v1 = groups[g]
        b = g % len(bufs)
        if side is None:
            _lib.check(lib.cce_gather_rows(_p(c), _p(perm[v0:v1]), v1 - v0, d, _p(bufs[b]), stream),
                       "cce_gather_rows")
            return
        if released[b] is not None:
            side.wait_event(released[b])
        with torch.cuda.stream(side):
            _lib.check(lib.cce_gather_rows(_p(c), _p(perm[v0:v1]), v1 - v0, d, _p(bufs[b]),
                                           ctypes.c_void_p(side.cuda_stream)), "cce_gather_rows")
            gathered[b] = torch.cuda.Event()
            gathered[b].record(side)

    ev = _ev_begin("fwd")
    if side is not None:
        side.wait_stream(main)  # the order (perm) and the caller's C are ready
    off = 1
    if sorted_:
        gather(0)
    for g, ((v0, v1), sp) in enumerate(zip(groups, splits)):
        if sorted_:
            b = g % len(bufs)
            if side is not None:
                main.wait_event(gathered[b])
                if g + 1 < len(groups):
                    gather(g + 1)
            c_g = bufs[b][: v1 - v0]
        else:
            c_g = c[v0:v1]
        ws = parts[off:off + sp]
        evk = _ev_begin("fwd_kernel")  # the logit-tile launches alone (bench roofline)
        _lib.check(lib.cce_fwd_group_ex(_p(e_rows), e_gather, _p(c_g), _p(row_map), _p(n_valid), _p(pos), v0, n, d,
                                        v1 - v0, v, float(softcap or 0.0), _p(ws), sp * n * 8, _p(None),
                                        _p(correct), _p(tile_max), 3, stream), "cce_fwd_group_ex")
        _ev_end("fwd_kernel", evk)
        if sorted_:
            if side is not None:
                released[b] = torch.cuda.Event()
                released[b].record(main)
            elif g + 1 < len(groups):
                gather(g + 1)
        off += sp
        if (g + 1) % fold == 0 and g + 1 < len(groups):
            _lib.check(lib.cce_combine_parts(_p(parts), off, n, _p(None), stream), "cce_combine_parts")
            off = 1
    _lib.check(lib.cce_combine_parts(_p(parts), off, n, _p(lse_local), stream), "cce_combine_parts")
    _ev_end("fwd", ev)
    # every side-stream gather is followed by a wait of the caller's stream on its event, and the
    # next call's gathers start after side.wait_stream(main): the buffers are the caller stream's
    # to free (no record_stream, which would hold them back from the allocator)
    del parts, bufs
    return lse_local, correct, state


def forward_chain(lib, e_rows, e_gather, c, perm, row_map, n_valid, pos, n, d, v, softcap, groups, splits, fold,
                  parts, correct, tile_max, lse_local, bufs, stream):
    """forward_stream's group launches as one chain (cce_fwd_group_sync): launch g waits for its
    rows (ready[g], set by launch g - 1's gather warps) instead of for launch g - 1 to finish, and
    gathers group g + 1 into the other buffer once launch g - 1 has exited (released[g - 1]).  A
    launch after a fold (cce_combine_parts, which reads the partial slots the next launch writes)
    waits for it as usual."""
    dev = e_rows.device
    ng = len(groups)
    flags = torch.zeros(4, ng, dtype=torch.int32, device=dev)  # ready, exited CTAs, released, gather shares
    ready, exits, released, shares = flags[0], flags[1], flags[2], flags[3]
    v0, v1 = groups[0]
    _lib.check(lib.cce_gather_rows(_p(c), _p(perm[v0:v1]), v1 - v0, d, _p(bufs[0]), stream), "cce_gather_rows")
    evk = _ev_begin("fwd_kernel")  # the chain's launches (and its folds) as one interval: events
    off = 1                        # between the launches would break the chain
    after_launch = False
    for g, ((v0, v1), sp) in enumerate(zip(groups, splits)):
        nxt = g + 1 < ng
        n0, n1 = groups[g + 1] if nxt else (0, 0)
        _lib.check(lib.cce_fwd_group_sync(
            _p(e_rows), e_gather, _p(bufs[g % 2][: v1 - v0]), _p(row_map), _p(n_valid), _p(pos), v0, n, d, v1 - v0, v,
            float(softcap or 0.0), _p(parts[off:off + sp]), sp * n * 8, _p(correct), _p(tile_max),
            _p(ready[g:]) if g else None, _p(exits[g:]), _p(released[g:]), int(after_launch), _p(c),
            _p(perm[n0:]) if nxt else None, n1 - n0, _p(bufs[(g + 1) % 2]) if nxt else None,
            _p(released[g - 1:]) if (nxt and g) else None, _p(shares[g + 1:]) if nxt else None,
            _p(ready[g + 1:]) if nxt else None, stream), "cce_fwd_group_sync")
        after_launch = True
        off += sp
        if (g + 1) % fold == 0 and g + 1 < ng:
            _lib.check(lib.cce_combine_parts(_p(parts), off, n, _p(None), stream), "cce_combine_parts")
            off = 1
            after_launch = False
    _ev_end("fwd_kernel", evk)
    _lib.check(lib.cce_combine_parts(_p(parts), off, n, _p(lse_local), stream), "cce_combine_parts")
    del flags


def backward_from_stream_state(state: StreamState, lse, upstream, *, eps: float = EPSILON_DEFAULT,
                               fp32_de: bool = False, de_done=None, label_split: bool = False,
                               correct=None, want_de: bool = True, want_dc: bool = True):
    """The streamed backward on a forward_stream state (the caller's E read in place, or its
    compacted copy when rows are ignored).  Batches of more than STREAM_CHUNK_TILES token tiles run
    as token chunks (backward_stream_chunked)."""
    n = state.e.shape[0]
    if -(-n // BLOCK_TOKENS) > stream_chunk_tiles():
        return backward_stream_chunked(state, lse, upstream, eps=eps, fp32_de=fp32_de, de_done=de_done,
                                       label_split=label_split, correct=correct, want_de=want_de, want_dc=want_dc)
    e_rows, e_gather = (state.e_c, False) if state.e_c is not None else (state.e, True)
    return backward_stream(e_rows, e_gather, state.c, state.perm_padded, state.inv_perm, state.row_map, state.n_valid,
                           state.pos, state.tile_max, lse, upstream, softcap=state.softcap, eps=eps, fp32_de=fp32_de,
                           de_done=de_done, label_split=label_split, correct=correct, want_de=want_de,
                           want_dc=want_dc, e_caller=state.e)


def backward_tiles(state: TileState, targets, lse, upstream, *, ignore_index: int,
                   eps: float = EPSILON_DEFAULT, fp32_de: bool = False,
                   de_done: torch.cuda.Event | None = None, label_split: bool = False,
                   correct: torch.Tensor | None = None, reuse_state: bool = False,
                   want_de: bool = True, want_dc: bool = True):
    """Backward of the filter-from-forward path (lse_backward, kernels.py:327-486).

    The skip decision of every tile comes from the forward's tile maxima (the same strict test
    as the in-kernel filter), so only kept tiles are recomputed.  If the kept tiles exceed the
    S-hat budget, the full filter pass (`backward`'s grouped path) runs instead, gated on a
    device flag.  Returns (dE, dC, counters[3]).  `de_done` (a CUDA event) is recorded on the
    current stream once dE is complete and before the dC pass runs.  Unless `reuse_state` (the
    state may see another backward, as the reference's backward closure allows), dC is written
    into the sorted classifier copy's storage and the state is spent.  want_de / want_dc False
    skip that pass (an input that needs no gradient) and return None in its place.
    """
    lib = _lib.load()
    e, c_t = state.e, state.c_t
    n, d = e.shape
    v = c_t.shape[0]
    dev = e.device
    stream = _stream(dev)
    lse = lse.to(torch.float32).contiguous()
    upstream = upstream.to(torch.float32).contiguous()
    de = torch.zeros(n, d, dtype=torch.float32 if fp32_de else torch.bfloat16, device=dev) if want_de else None
    # The sorted classifier copy is last read by the dE pass, so its storage becomes the dC output
    # (the library reads C through the permutation wherever C_t may already hold dC): no second
    # V x D matrix is ever live.  CCE_ALIAS_DC=0 allocates dC separately (A/B).
    if reuse_state and state.lab_cap:
        raise ValueError("reuse_state needs a forward without stored label tiles (store_labels=False)")
    alias = (want_dc and state.perm is not None and not reuse_state
             and os.environ.get("CCE_ALIAS_DC", "1") != "0")
    dc = (c_t if alias else torch.empty(v, d, dtype=torch.bfloat16, device=dev)) if want_dc else None
    if alias:
        state.c_t = None  # spent: its storage is now dC
    counters = torch.zeros(3, dtype=torch.int64, device=dev)
    if n == 0:
        return de, (dc.zero_() if dc is not None else None), counters
    if not eps:
        raise ValueError("backward_tiles needs filtering (eps > 0)")
    nt = -(-n // BLOCK_TOKENS)
    mt = -(-v // BLOCK_VOCAB)
    # S-hat slots (from the forward): label tiles stored there, the rest recomputed -- in one pass
    # if they fit; otherwise the library falls back (device flag, no host read) to token-tile
    # groups sized for the worst case
    if state.shat is None:
        state.rcap = shat_capacity(("recompute-", d, v, state.vocab_start, float(eps), state.softcap), nt, mt)
        state.shat = torch.empty(state.rcap * SHAT_TILE_BYTES, dtype=torch.uint8, device=dev)
    cap, lab_cap = state.rcap, state.lab_cap
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    stats = torch.zeros(2, dtype=torch.int32, device=dev)
    ws_bytes = lib.cce_bwd_kept_workspace_bytes(n, d, v, cap, lab_cap)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ev = _ev_begin("bwd")
    _lib.check(lib.cce_bwd_kept(_p(state.e_c), _p(c_t), _p(state.c if alias else None),
                                _p(state.perm_padded), _p(state.row_map),
                                _p(state.n_valid), _p(state.pos), 0, _p(lse), _p(upstream), _p(state.tile_max),
                                n, d, v, state.softcap, float(eps), int(bool(label_split)), _p(state.shat),
                                lab_cap, _p(state.lab_slot), _p(state.lab_list), _p(state.lab_count), cap,
                                _p(ws), ws_bytes, _p(de), int(fp32_de), 0, _p(dc), _p(counters), _p(overflow),
                                _p(stats), _p(None),
                                _event_handle(None if label_split else de_done), stream), "cce_bwd_kept")
    del ws
    if label_split:
        label_terms(e, state.c, state.perm_padded, state.row_map, state.n_valid, state.pos, upstream,
                    correct, state.softcap, de, dc)
        if de_done is not None:
            de_done.record()
    LAST_STATS["stats"] = stats  # [label tiles stored by the forward, tiles recomputed]
    if state.keys:
        _remember_count(state.keys[0], stats, 1, nt)
        if lab_cap:
            _remember_count(state.keys[1], stats, 0, nt)
    _ev_end("bwd", ev)
    LAST_COUNTERS["counters"] = counters
    LAST_OVERFLOW["flag"] = overflow
    return de, dc, counters


STREAM_RING_SLOTS = 512  # S-hat ring of the streamed backward (64 KiB slots: 32 MiB)


def stream_ring_slots(token_tiles: int = 0) -> int:
    """S-hat ring slots of one streamed pass: 512, or 8 per token tile (dE windows of half the
    ring then hold >= 4 items of every token tile), up to 4096 (256 MiB, 512 token tiles).
    Measured at Gemma-2-9B (256 token tiles): 84 ms per step with 2048 slots in one pass, against
    104 ms with four 64-tile chunks of 512 slots (scripts/ab_r2/r2_s57.sh); at NeMo (512 token
    tiles) one pass with 4096 slots takes 336 ms at a 1.70 GiB step peak, two 256-tile chunks
    323 ms at 2.78 GiB (scripts/ab_r2/r2_nemo.sh)."""
    env = os.environ.get("CCE_STREAM_RING")
    if env is not None:
        return max(128, int(env))
    return max(STREAM_RING_SLOTS, min(8 * STREAM_RING_SLOTS, 8 * token_tiles))


def stream_supported(d: int) -> bool:
    """The streamed backward's CTA-pair operand boxes need D % 64 == 0 (every LM head size)."""
    return d % 64 == 0


def backward_stream(e_rows, e_gather: bool, c, perm_padded, inv_perm, row_map, n_valid, pos, tile_max, lse,
                    upstream, *, softcap: float = 0.0, eps: float = EPSILON_DEFAULT, fp32_de: bool = False,
                    de_done: torch.cuda.Event | None = None, label_split: bool = False,
                    correct: torch.Tensor | None = None, want_de: bool = True, want_dc: bool = True,
                    e_caller: torch.Tensor | None = None):
    """Streamed backward of the training path (lse_backward, kernels.py:327-486): the decision from
    the forward's tile maxima, then the kept tiles recomputed in token-tile order (dE) and in
    vocabulary-tile order (dC), streamed through a fixed ring of S-hat slots.  Transients: the ring
    (32 MiB; 8 slots per token tile above 64 tiles), O(N + V) lists and maps, the split accumulators
    (N x D fp32 for dE) -- none grows with the kept
    count.  With a vocabulary order the sorted classifier lives in dC's own storage.
    `e_rows` is the caller's E (e_gather) or a compacted copy.  Returns (dE, dC, counters[3])."""
    lib = _lib.load()
    n, d = e_rows.shape
    v = c.shape[0]
    dev = e_rows.device
    lse = lse.to(torch.float32).contiguous()
    upstream = upstream.to(torch.float32).contiguous()
    de = torch.zeros(n, d, dtype=torch.float32 if fp32_de else torch.bfloat16, device=dev) if want_de else None
    dc = torch.empty(v, d, dtype=torch.bfloat16, device=dev) if want_dc else None
    counters = torch.zeros(3, dtype=torch.int64, device=dev)
    if n == 0:
        return de, (dc.zero_() if dc is not None else None), counters
    if not eps:
        raise ValueError("backward_stream needs filtering (eps > 0)")
    c_sorted = None
    if perm_padded is not None and os.environ.get("CCE_STREAM_GATHER", "0") == "0":
        # the sorted copy lives in dC's storage (dC then lands sorted and moves back in place);
        # CCE_STREAM_ALIAS=0 gives it its own buffer (A/B and diagnostics).  CCE_STREAM_GATHER=1:
        # no sorted copy, the pass gathers C rows through the order and scatters dC rows
        alias = dc is not None and os.environ.get("CCE_STREAM_ALIAS", "1") != "0"
        c_sorted = dc if alias else torch.empty(v, d, dtype=torch.bfloat16, device=dev)
    slots = stream_ring_slots(-(-n // BLOCK_TOKENS))
    ring = torch.empty(slots * SHAT_TILE_BYTES, dtype=torch.uint8, device=dev)
    ws_bytes = lib.cce_bwd_stream_workspace_bytes(n, d, v, slots)
    ws = (torch.zeros if os.environ.get("CCE_STREAM_ZERO_WS") else torch.empty)(ws_bytes, dtype=torch.uint8, device=dev)
    ev = _ev_begin("bwd")
    _lib.check(lib.cce_bwd_stream(_p(e_rows), int(bool(e_gather)), _p(c), _p(c_sorted), _p(perm_padded),
                                  _p(inv_perm), _p(row_map), _p(n_valid), _p(pos), _p(lse), _p(upstream),
                                  _p(tile_max), n, d, v, float(softcap or 0.0), float(eps), int(bool(label_split)),
                                  _p(ring), slots, _p(ws), ws_bytes, _p(de), int(fp32_de), _p(dc), _p(counters),
                                  _event_handle(None if label_split else de_done), _stream(dev)), "cce_bwd_stream")
    del ws, ring
    if label_split:
        label_terms(e_caller if e_caller is not None else e_rows, c, perm_padded, row_map, n_valid, pos, upstream, correct,
                    softcap, de, dc)
        if de_done is not None:
            de_done.record()
    _ev_end("bwd", ev)
    LAST_COUNTERS["counters"] = counters
    return de, dc, counters


STREAM_CHUNK_TILES = 512  # token tiles per streamed pass (65536 rows; ring sized by stream_ring_slots)


def stream_chunk_tiles() -> int:
    return max(1, int(os.environ.get("CCE_STREAM_CHUNK_TILES", STREAM_CHUNK_TILES)))


def backward_stream_chunked(state: StreamState, lse, upstream, *, eps: float = EPSILON_DEFAULT,
                            fp32_de: bool = False, de_done=None, label_split: bool = False, correct=None,
                            want_de: bool = True, want_dc: bool = True):
    """The streamed backward of a large batch as token chunks of STREAM_CHUNK_TILES tiles (65536 rows).

    The pass's dE segments are a token tile's items inside one window of ring / 2 stream items;
    with more token tiles than a quarter window they shrink below a few items, and every segment
    costs an fp32 read-modify-write of the tile's 128 x D partial sum.  The ring grows with the
    token tiles up to 4096 slots (stream_ring_slots); beyond that each chunk is its own
    pass over the same global decision inputs (tile maxima rows, lse, the vocabulary order): its
    tile decisions equal the whole batch's, dE rows are written once by their chunk, and dC adds
    over the chunks in bf16 (the fast path's group fallback does the same).  The sorted classifier
    copy is built once in its own buffer (dC accumulates in vocabulary order, so it cannot hold it)
    and E is read as a compacted copy.  Transients: O(V D) for the sorted copy and O(N D) for the
    compacted rows, independent of the kept tiles."""
    lib = _lib.load()
    e = state.e
    n, d = e.shape
    v = state.c.shape[0]
    dev = e.device
    stream = _stream(dev)
    lse = lse.to(torch.float32).contiguous()
    upstream = upstream.to(torch.float32).contiguous()
    if not eps:
        raise ValueError("backward_stream needs filtering (eps > 0)")
    de = torch.zeros(n, d, dtype=torch.float32 if fp32_de else torch.bfloat16, device=dev) if want_de else None
    dc = torch.empty(v, d, dtype=torch.bfloat16, device=dev) if want_dc else None
    counters = torch.zeros(3, dtype=torch.int64, device=dev)
    e_c = state.e_c if state.e_c is not None else gather_rows(e, state.row_map, n)
    c_sorted = gather_rows(state.c, state.perm, v) if state.perm_padded is not None and state.perm is not None else None
    chunk = stream_chunk_tiles() * BLOCK_TOKENS
    mt = -(-v // BLOCK_VOCAB)
    slots = stream_ring_slots(-(-min(n, chunk) // BLOCK_TOKENS))
    ring = torch.empty(slots * SHAT_TILE_BYTES, dtype=torch.uint8, device=dev)
    ws_bytes = lib.cce_bwd_stream_workspace_bytes(min(n, chunk), d, v, slots)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ev = _ev_begin("bwd")
    for k, r0 in enumerate(range(0, n, chunk)):
        r1 = min(n, r0 + chunk)
        nv = (state.n_valid - r0).clamp(0, r1 - r0).to(torch.int32)  # compacted rows of this chunk
        t0 = r0 // BLOCK_TOKENS
        tm = state.tile_max[t0 * mt * BLOCK_TOKENS:]
        last = r1 >= n
        flags = 3 if k > 0 else 0  # later chunks: the sorted copy is built, dC adds
        _lib.check(lib.cce_bwd_stream_ex(
            _p(e_c[r0:r1]), 0, _p(state.c), _p(c_sorted), _p(state.perm_padded if c_sorted is not None else None),
            _p(state.inv_perm), _p(state.row_map[r0:]), _p(nv), _p(state.pos), _p(lse), _p(upstream), _p(tm),
            r1 - r0, d, v, float(state.softcap or 0.0), float(eps), int(bool(label_split)), _p(ring), slots, _p(ws),
            ws_bytes, _p(de), int(fp32_de), _p(dc), _p(counters),
            _event_handle(de_done if (last and not label_split) else None), flags if dc is not None else (flags & 1),
            stream), "cce_bwd_stream_ex")
    del ws, ring, c_sorted
    if label_split:
        label_terms(e, state.c, state.perm_padded, state.row_map, state.n_valid, state.pos, upstream, correct,
                    state.softcap, de, dc)
        if de_done is not None:
            de_done.record()
    _ev_end("bwd", ev)
    LAST_COUNTERS["counters"] = counters
    return de, dc, counters


@dataclass
class GroupState:
    """What the grouped backward needs from forward_grouped: like TileState, but the sorted
    classifier is never materialised -- each vocabulary group's rows are gathered into a small
    buffer, once in the forward and once in the backward -- and the tile maxima are laid out
    group by group ([group][token tile][vocab tile of the group][128])."""
    e: torch.Tensor
    c: torch.Tensor
    e_c: torch.Tensor
    row_map: torch.Tensor
    n_valid: torch.Tensor
    perm: torch.Tensor | None
    perm_padded: torch.Tensor | None
    pos: torch.Tensor
    tile_max: torch.Tensor
    groups: list  # (first sorted row, end row) per group; starts are multiples of 256
    vocab_start: int
    softcap: float
    mean_logits: torch.Tensor | None = None
    slots: int = 0   # S-hat slots per group (grouped_plan)
    key: tuple = ()  # shape key of the learned kept count

    def nbytes(self) -> int:
        own = [self.e_c, self.row_map, self.n_valid, self.pos, self.tile_max, self.perm, self.perm_padded]
        return sum(t.numel() * t.element_size() for t in own if t is not None)


def _group_rows(c, perm, v0: int, v1: int) -> torch.Tensor:
    """The classifier rows of sorted positions [v0, v1): gathered, or a view without sorting."""
    return gather_rows(c, perm[v0:v1], v1 - v0) if perm is not None else c[v0:v1]


def forward_grouped(e, c, targets, ignore_index: int, vocab_start: int = 0, softcap: float = 0.0,
                    vocab_sorting: bool = True, perm: torch.Tensor | None = None,
                    eps: float = EPSILON_DEFAULT, label_split: bool = False):
    """Forward of the bounded-memory training path: (lse_local, correct, GroupState).

    The same sweep as forward_tiles (compacted rows, the reference's vocabulary order, per-row
    maxima of every 128 x 256 tile), run over vocabulary groups of the sorted order so that only
    one group's classifier rows are ever gathered (lowmem_group_vtiles budgets).  Each group is a
    vocabulary shard of its own: its (lse, correct) partials merge with the log-add-exp kernel of
    the vocab-parallel path (kernels.py:121-137).
    """
    lib = _lib.load()
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    stream = _stream(dev)
    row_map, n_valid = compact_rows(targets, ignore_index)
    e_c = gather_rows(e, row_map, n)
    mean_logits = None
    if vocab_sorting and perm is None:
        perm, mean_logits = vocab_order(e, c, targets, ignore_index, n_valid)
    vpad = -(-v // BLOCK_VOCAB) * BLOCK_VOCAB
    perm_padded = torch.empty(vpad, dtype=torch.int32, device=dev) if perm is not None else None
    inv_perm = torch.empty(v, dtype=torch.int32, device=dev) if perm is not None else None
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.cce_bwd_prep(_p(perm), v, _p(targets), int(ignore_index), int(vocab_start), n,
                                _p(perm_padded), _p(inv_perm), _p(pos), stream), "cce_bwd_prep")
    del inv_perm
    nt = -(-n // BLOCK_TOKENS)
    mt = -(-v // BLOCK_VOCAB)
    key = ("grouped", n, d, v, int(vocab_start), float(eps), float(softcap or 0.0), bool(label_split),
           perm is not None)
    bounds, slots = grouped_plan(n, d, v, key)
    groups = [(m0 * BLOCK_VOCAB, min(v, m1 * BLOCK_VOCAB)) for m0, m1 in bounds]
    tile_max = torch.empty(max(nt, 1) * mt * BLOCK_TOKENS, dtype=torch.float32, device=dev)
    state = GroupState(e, c, e_c, row_map, n_valid, perm, perm_padded, pos, tile_max, groups,
                       int(vocab_start), float(softcap or 0.0), mean_logits, slots, key)
    lse_parts = torch.empty(len(groups), n, dtype=torch.float32, device=dev)
    corr_parts = torch.empty(len(groups), n, dtype=torch.float32, device=dev)
    if n == 0:
        return lse_parts.sum(0), corr_parts.sum(0), state
    ws_bytes = max(lib.cce_fwd_workspace_bytes(n, d, v1 - v0) for v0, v1 in groups)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    ev = _ev_begin("fwd")
    c_g = None
    for g, (v0, v1) in enumerate(groups):
        c_g = None  # release the previous group's rows before gathering the next (one buffer live)
        c_g = _group_rows(c, perm, v0, v1)
        tm_g = tile_max[nt * (v0 // BLOCK_VOCAB) * BLOCK_TOKENS:]
        _lib.check(lib.cce_fwd_tiles(_p(e_c), _p(c_g), _p(row_map), _p(n_valid), _p(pos), v0, n, d, v1 - v0,
                                     float(softcap or 0.0), _p(ws), ws_bytes, _p(lse_parts[g]),
                                     _p(corr_parts[g]), _p(tm_g), _p(None), 0, _p(None), _p(None), _p(None),
                                     stream), "cce_fwd_tiles")
    # the groups are vocabulary shards of this call: log-add-exp of their partials; the target
    # logit sits in exactly one group (0 elsewhere)
    lse_local, loss = merge_shards(lse_parts, corr_parts, targets, ignore_index)
    correct = corr_parts.sum(0)
    del loss
    _ev_end("fwd", ev)
    return lse_local, correct, state


def backward_grouped(state: GroupState, targets, lse, upstream, *, ignore_index: int,
                     eps: float = EPSILON_DEFAULT, fp32_de: bool = False,
                     de_done: torch.cuda.Event | None = None, label_split: bool = False,
                     correct: torch.Tensor | None = None, want_de: bool = True, want_dc: bool = True):
    """Backward of the bounded-memory training path (lse_backward, kernels.py:327-486): per
    vocabulary group, the group's rows are gathered again, the skip decision is taken from the
    forward's tile maxima and only the kept tiles are recomputed (cce_bwd_kept with the group's
    S-hat slots sized for its worst case, so no overflow path exists); dE accumulates over the
    groups in fp32 in a fixed order, dC rows are written by their own group.
    Returns (dE, dC, counters[3])."""
    lib = _lib.load()
    e, c = state.e, state.c
    n, d = e.shape
    v = c.shape[0]
    dev = e.device
    stream = _stream(dev)
    lse = lse.to(torch.float32).contiguous()
    upstream = upstream.to(torch.float32).contiguous()
    de = torch.zeros(n, d, dtype=torch.float32, device=dev) if want_de else None
    dc = torch.empty(v, d, dtype=torch.bfloat16, device=dev) if want_dc else None
    counters = torch.zeros(3, dtype=torch.int64, device=dev)
    if n == 0:
        return ((de if fp32_de else de.to(torch.bfloat16)) if de is not None else None,
                dc.zero_() if dc is not None else None, counters)
    if not eps:
        raise ValueError("backward_grouped needs filtering (eps > 0)")
    nt = -(-n // BLOCK_TOKENS)
    gtiles = max(-(-(v1 - v0) // BLOCK_VOCAB) for v0, v1 in state.groups)
    # slots from grouped_plan: every tile of the group until a kept count is known, then the
    # learned density (a group that keeps more takes cce_bwd_kept's on-device overflow path)
    cap = max(gtiles, min(nt * gtiles, state.slots or nt * gtiles))
    shat = torch.empty(cap * SHAT_TILE_BYTES, dtype=torch.uint8, device=dev)
    ws_bytes = max(lib.cce_bwd_kept_workspace_bytes(n, d, v1 - v0, cap, 0) for v0, v1 in state.groups)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    overflow = torch.zeros(len(state.groups), dtype=torch.int32, device=dev)  # one flag per group
    vcounts = torch.zeros(-(-v // BLOCK_VOCAB), dtype=torch.int32, device=dev)  # kept per vocab tile
    split = bool(label_split)
    ev = _ev_begin("bwd")
    last = len(state.groups) - 1
    c_g = None
    for g, (v0, v1) in enumerate(state.groups):
        vg = v1 - v0
        c_g = None  # one group's rows live at a time
        c_g = _group_rows(c, state.perm, v0, v1)
        tm_g = state.tile_max[nt * (v0 // BLOCK_VOCAB) * BLOCK_TOKENS:]
        perm_g = state.perm_padded[v0:] if state.perm_padded is not None else None
        dc_g = None if dc is None else (dc if state.perm_padded is not None else dc[v0:v1])
        done = _event_handle(de_done if (g == last and not split) else None)
        _lib.check(lib.cce_bwd_kept(_p(state.e_c), _p(c_g), _p(None), _p(perm_g), _p(state.row_map),
                                    _p(state.n_valid), _p(state.pos), v0, _p(lse), _p(upstream), _p(tm_g),
                                    n, d, vg, state.softcap, float(eps), int(split), _p(shat), 0, _p(None),
                                    _p(None), _p(None), cap, _p(ws), ws_bytes, _p(de), 1, int(g > 0),
                                    _p(dc_g), _p(counters), _p(overflow[g:]), _p(None), _p(vcounts[v0 // BLOCK_VOCAB:]),
                                    done, stream), "cce_bwd_kept")
    del ws, shat
    if state.key:  # kept tiles per vocab tile: sizes the next call's groups
        _remember_vector(state.key + ("per-vtile",), vcounts)
    if split:
        label_terms(e, c, state.perm_padded, state.row_map, state.n_valid, state.pos, upstream, correct,
                    state.softcap, de, dc)
        if de_done is not None:
            de_done.record()
    _ev_end("bwd", ev)
    LAST_COUNTERS["counters"] = counters
    LAST_OVERFLOW["flag"] = overflow.max()  # 1 if any group took the fallback
    return (de if (fp32_de or de is None) else f32_to_bf16(de)), dc, counters


SHAT_TILE_BYTES = BLOCK_TOKENS * BLOCK_VOCAB * 2
LABEL_STORE_MIN_D = 1536      # hidden size from which the forward stores label tiles
FIRST_CALL_MB = 1024          # S-hat allocation before any kept count has been observed
KEPT_MARGIN = 1.15            # headroom over the last observed kept count
_KEPT_HINT: dict = {}         # shape key -> [pinned copy of a device count vector, CUDA event, last known value, index]
KEPT_HINT_MAX = 256           # shape keys remembered (least recently used dropped first)


def shat_budget_tiles() -> int:
    """Ceiling on S-hat slots (64 KiB each): CCE_SHAT_BUDGET_MB, else 10% of device memory."""
    env = os.environ.get("CCE_SHAT_BUDGET_MB")
    if env is not None:
        budget = int(env) << 20
    else:
        budget = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory // 10
    return max(1, budget // SHAT_TILE_BYTES)


def shat_capacity(key, nt: int, mt: int) -> int:
    """S-hat slots to allocate for this call.  A fixed CCE_SHAT_BUDGET_MB is used as is; otherwise
    the kept-tile count of the previous call with the same shape (read from a pinned copy only
    once its event has completed -- never a host synchronisation) plus a margin, or FIRST_CALL_MB
    on the first call.  Too small is safe: the grouped fallback runs on the device."""
    ceiling = shat_budget_tiles()
    if os.environ.get("CCE_SHAT_BUDGET_MB") is not None:
        cap = ceiling
    else:
        cap = min(ceiling, (FIRST_CALL_MB << 20) // SHAT_TILE_BYTES)
        hint = _KEPT_HINT.get(key)
        if hint is not None:
            _harvest(hint)
            if hint[2] is not None:
                cap = min(ceiling, max(int(_rescaled(hint, nt) * KEPT_MARGIN), mt))  # floor: one token tile's tiles
    return min(max(cap, mt), nt * mt)


def _capturing() -> bool:
    return torch.cuda.is_current_stream_capturing()


def _harvest(hint) -> None:
    if _capturing():  # no event queries inside a CUDA-graph capture: use what is already known
        return
    if hint[1] is not None and hint[1].query():
        hint[2] = int(hint[0][hint[3]]) if hint[3] is not None else hint[0].tolist()
        hint[1] = None
        if len(hint) > 5:
            hint[4] = hint[5]


LABEL_MARGIN = 1.1


def label_capacity(key, nt: int, mt: int) -> int:
    """Stored label-tile slots: the worst case (every valid row's label in its own vocab tile,
    ceil(n/128) * min(ceil(v/256), 128)) until a label count of this shape has been observed, then
    that count plus a margin.  Too small is safe: tiles without a slot are recomputed.  A fixed
    CCE_SHAT_BUDGET_MB pins it to the worst case as well (the overflow fallback's group size
    depends on it, and with it the bf16 summation order of dC across groups)."""
    worst = nt * min(mt, BLOCK_TOKENS)
    if os.environ.get("CCE_SHAT_BUDGET_MB") is not None:
        return worst
    hint = _KEPT_HINT.get(key)
    if hint is not None:
        _harvest(hint)
        if hint[2] is not None:
            return min(worst, int(_rescaled(hint, nt) * LABEL_MARGIN) + nt)
    return worst


def _rescaled(hint, nt: int) -> float:
    """The hint's count at `nt` token tiles (counts of the tile path grow with the token tiles)."""
    scale = hint[4] if len(hint) > 4 else None
    return hint[2] * nt / scale if scale else hint[2]


def _remember_count(key, counts: torch.Tensor, index: int, nt: int | None = None) -> None:
    """Queue an asynchronous copy of a device count (read by a later call once it has landed);
    `nt` records the token tiles it was observed at, so calls at another N can rescale it."""
    if _capturing():
        return
    hint = _KEPT_HINT.pop(key, None)
    if hint is None:
        # [pinned copy, event of the copy in flight, harvested value, index, token tiles of the
        #  harvested value, token tiles of the copy in flight]
        hint = [torch.zeros(counts.shape, dtype=counts.dtype).pin_memory(), None, None, index, nt, nt]
        while len(_KEPT_HINT) >= KEPT_HINT_MAX:  # shapes that vary every step: drop the oldest
            _KEPT_HINT.pop(next(iter(_KEPT_HINT)))
    _KEPT_HINT[key] = hint  # (re)inserted last: the dict's order is least recently used first
    _harvest(hint)
    if hint[1] is not None:
        return  # previous copy still in flight
    hint[0].copy_(counts, non_blocking=True)
    hint[1] = torch.cuda.Event()
    hint[1].record()
    if len(hint) > 5:
        hint[5] = nt


def _remember_vector(key, vec: torch.Tensor) -> None:
    """_remember_count for a whole device vector (read back as a list)."""
    _remember_count(key, vec, None)


def _remember_kept(key, counters: torch.Tensor, nt: int | None = None) -> None:
    """Queue an asynchronous copy of this call's kept-tile count (read by a later call once it
    has landed; the CPU usually runs ahead of the GPU, so the value may be a few calls old)."""
    _remember_count(key, counters, 0, nt)


REDUCTIONS = {"none": 0, "sum": 1, "mean": 2}


def reduce_loss(loss: torch.Tensor, targets: torch.Tensor, ignore_index: int, reduction: str) -> torch.Tensor:
    """Scalar sum / mean-over-valid of per-row losses (0 at ignored rows); device-side."""
    lib = _lib.load()
    out = torch.empty((), dtype=torch.float32, device=loss.device)
    _lib.check(lib.cce_reduce_loss(_p(loss), _p(targets), int(ignore_index), loss.shape[0],
                                   REDUCTIONS[reduction], _p(out), _stream(loss.device)), "cce_reduce_loss")
    return out


def upstream(grad: torch.Tensor, targets: torch.Tensor, ignore_index: int, reduction: str) -> torch.Tensor:
    """dLoss/dloss_i for each row (default_upstream, core.py:181-200), 0 at ignored rows."""
    lib = _lib.load()
    g = grad.to(torch.float32).contiguous()
    up = torch.empty(targets.shape[0], dtype=torch.float32, device=targets.device)
    _lib.check(lib.cce_upstream(_p(g), _p(targets), int(ignore_index), targets.shape[0],
                                REDUCTIONS[reduction], _p(up), _stream(targets.device)), "cce_upstream")
    return up


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
