"""`linear_cross_entropy`: the drop-in loss (north_star API) as a torch.autograd.Function.

Semantics follow the reference cce_loss (kernels.py:513-580) through the adapter of SURVEY §8(b):

  ignore_index   targets == ignore_index play the reference's IGNORE_INDEX = -1 (core.py:23)
  reduction      "mean" = "mean-over-valid" (core.py:194-197; an all-ignored batch gives 0 loss
                 and zero grads, never NaN), "sum", "none" (per-token, 0 at ignored rows)
  filter_eps     "auto" -> 2**-12 (EPSILON_DEFAULT, core.py:27); None / 0 -> filtering off
  softcap        z' = softcap * tanh(z / softcap) applied to every logit (absent from the
                 reference; restated in oracle/cce_oracle.py and pinned by finite differences)

Deviation (documented): for reduction="none" the reference raises on a nonzero upstream at an
ignored row (kernels.py:371-372); here the upstream is masked to 0 there instead.

Vocab-parallel: pass `process_group` and the classifier shard `c` holding global rows
[vocab_start, vocab_start + c.shape[0]).  E and targets are replicated; each rank returns the
full loss, dE is all-reduced, dC stays local (see vocab_parallel.py).
"""

from __future__ import annotations

import os

import torch

from . import ops
from .ops import EPSILON_DEFAULT


def _resolve_eps(filter_eps):
    if filter_eps is None or filter_eps is False:
        return 0.0
    if isinstance(filter_eps, str):
        if filter_eps != "auto":
            raise ValueError(f"filter_eps must be 'auto', a float in (0,1) or None, got {filter_eps!r}")
        return EPSILON_DEFAULT
    eps = float(filter_eps)
    if eps == 0.0:
        return 0.0
    if not (0.0 < eps < 1.0):
        raise ValueError(f"epsilon must be in (0, 1), got {eps}")  # core.py:151-152
    return eps


_GLOBAL_V: dict = {}


def _global_vocab(v_local: int, group) -> int:
    """Vocabulary size over all shards of `group` (one scalar all-reduce per group and shard size,
    then cached)."""
    import torch.distributed as dist

    key = (id(group), v_local)
    if key not in _GLOBAL_V:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        x = torch.tensor([v_local], dtype=torch.int64, device=dev)
        dist.all_reduce(x, group=group)
        _GLOBAL_V[key] = int(x.item())
    return _GLOBAL_V[key]


class _LinearCrossEntropy(torch.autograd.Function):
    @staticmethod
    def forward(ctx, e, c, targets, t_shard, ignore_index, softcap, reduction, eps, vocab_sorting, group,
                vocab_start, memory, exempt_label_tiles, training, v_total):
        # targets: the caller's labels (ignore mask, label-range check, upstream); t_shard: the same
        # labels in this shard's row coordinates (the kernels' targets; == targets unless the shard
        # is block-cyclic, see vocab_parallel.cyclic_rows)
        # Training with filtering: the forward sweeps the backward's tiles (compacted rows, sorted
        # vocabulary) and records per-row tile maxima, so the backward recomputes kept tiles only.
        # low_memory / no filtering / inference: plain forward, only O(N) state survives to the
        # backward, which then runs over vocabulary groups (ops.backward_lowmem).
        # `training` is decided by the caller (grad mode on and an input requires grad): inside
        # forward grad mode is always off, and needs_input_grad follows requires_grad even under
        # torch.no_grad(), so an eval call would otherwise pay for the training forward.
        ctx.state = None
        if eps > 0 and memory == "bounded" and training:
            # default: vocabulary-grouped forward into the per-row tile maxima, streamed backward
            lse_local, correct, ctx.state = ops.forward_stream(e, c, t_shard, ignore_index, vocab_start, softcap,
                                                               vocab_sorting)
        elif eps > 0 and memory == "fast" and training:
            lse_local, correct, ctx.state = ops.forward_tiles(e, c, t_shard, ignore_index, vocab_start,
                                                              softcap, vocab_sorting, eps=eps,
                                                              label_split=not exempt_label_tiles)
        elif eps > 0 and memory == "grouped" and training and os.environ.get("CCE_LOWMEM_RECOMPUTE", "0") == "0":
            # bounded memory: the same decision from the forward, over vocabulary groups
            lse_local, correct, ctx.state = ops.forward_grouped(e, c, t_shard, ignore_index, vocab_start,
                                                                softcap, vocab_sorting, eps=eps,
                                                                label_split=not exempt_label_tiles)
        else:
            lse_local, correct = ops.forward_local(e, c, t_shard, ignore_index, vocab_start, softcap)
        if group is None:
            lse, loss = ops.merge_shards(lse_local[None], correct[None], targets, ignore_index, v_total)
        else:
            from .vocab_parallel import gather_and_merge

            lse, loss = gather_and_merge(lse_local, correct, targets, ignore_index, group, v_total)
        ctx.save_for_backward(e, c, targets, t_shard, lse)
        ctx.cfg = (ignore_index, softcap, reduction, eps, vocab_sorting, group, vocab_start)
        # paper ordering: the label term is applied apart from the filtered tiles and needs the
        # forward's (softcapped) target logit of the rows whose label this shard owns (O(N): kept
        # for a second backward under retain_graph)
        ctx.split = not exempt_label_tiles and eps > 0
        ctx.correct = correct if ctx.split else None
        ctx.backwards = 0
        ctx.had_state = ctx.state is not None
        if reduction == "none":
            return loss
        return ops.reduce_loss(loss, targets, ignore_index, reduction)  # mean: 0 if nothing valid

    @staticmethod
    def backward(ctx, grad_out):
        e, c, targets, t_shard, lse = ctx.saved_tensors
        ignore_index, softcap, reduction, eps, vocab_sorting, group, vocab_start = ctx.cfg
        up = ops.upstream(grad_out, targets, ignore_index, reduction)  # default_upstream, core.py:181-200
        ctx.backwards += 1
        state, ctx.state = ctx.state, None
        if ctx.had_state and ctx.backwards > 1:
            raise RuntimeError("linear_cross_entropy: this forward's tile state was spent by the first backward "
                               "(a second backward under retain_graph=True needs low_memory=True or "
                               "filter_eps=None)")
        split, correct = ctx.split, ctx.correct
        # a pass whose input needs no gradient is skipped (e.g. a frozen classifier: no dC pass)
        want = dict(want_de=ctx.needs_input_grad[0], want_dc=ctx.needs_input_grad[1])
        if isinstance(state, ops.StreamState):
            done = ops.recorded_event() if group is not None else None
            de, dc, _ = ops.backward_from_stream_state(state, lse, up, eps=eps, fp32_de=group is not None,
                                                       de_done=done, label_split=split, correct=correct, **want)
            del state
            if group is not None and de is not None:
                from .vocab_parallel import all_reduce_de_overlapped

                de = all_reduce_de_overlapped(de, done, group)
        elif isinstance(state, ops.GroupState):
            done = ops.recorded_event() if group is not None else None
            de, dc, _ = ops.backward_grouped(state, t_shard, lse, up, ignore_index=ignore_index, eps=eps,
                                             fp32_de=group is not None, de_done=done, label_split=split,
                                             correct=correct, **want)
            del state
            if group is not None and de is not None:
                from .vocab_parallel import all_reduce_de_overlapped

                de = all_reduce_de_overlapped(de, done, group)
        elif state is not None:
            if group is None:
                de, dc, _ = ops.backward_tiles(state, t_shard, lse, up, ignore_index=ignore_index, eps=eps,
                                               label_split=split, correct=correct, **want)
            else:
                from .vocab_parallel import all_reduce_de_overlapped

                # dE is complete before the dC pass: its all-reduce runs on a side stream meanwhile
                done = ops.recorded_event()
                de, dc, _ = ops.backward_tiles(state, t_shard, lse, up, ignore_index=ignore_index, eps=eps,
                                               fp32_de=True, de_done=done, label_split=split, correct=correct,
                                               **want)
                if de is not None:
                    de = all_reduce_de_overlapped(de, done, group)
            del state
        else:  # low_memory=True or filtering off: vocabulary-grouped backward, bounded transients
            de, dc, _, _ = ops.backward_lowmem(e, c, t_shard, lse, up, ignore_index=ignore_index,
                                               vocab_start=vocab_start, softcap=softcap, eps=eps,
                                               vocab_sorting=vocab_sorting, fp32_de=group is not None,
                                               label_split=split, correct=correct)
            if group is not None:
                from .vocab_parallel import all_reduce_de

                de = all_reduce_de(de, group)
        return de, dc, None, None, None, None, None, None, None, None, None, None, None, None, None


def linear_cross_entropy(
    e: torch.Tensor,
    c: torch.Tensor,
    targets: torch.Tensor,
    ignore_index: int = -100,
    softcap: float | None = None,
    reduction: str = "mean",
    filter_eps: float | str | None = "auto",
    vocab_sorting: bool = True,
    process_group=None,
    vocab_start: int = 0,
    low_memory: bool = False,
    exempt_label_tiles: bool = True,
    memory: str | None = None,
    vocab_rows: torch.Tensor | None = None,
) -> torch.Tensor:
    """Cross-entropy of softmax(e @ c.T) against targets without materialising the logits.

    e: [..., D] CUDA embeddings; c: [V, D] classifier (nn.Linear weight layout); targets: [...]
    integer labels.  The kernels compute in bf16: fp32/fp16 operands are cast (gradients come
    back in the operands' dtype) and any D is accepted (zero-padded to a multiple of 8).  Returns a scalar for "mean"/"sum", else per-token losses of shape
    e.shape[:-1].

    memory selects the training path (filtering on):
      "bounded" (default)  the forward sweeps vocabulary groups of the sorted order (one group's
                 classifier rows gathered at a time) and keeps per-row tile maxima; the backward
                 streams the kept tiles through a fixed 32 MiB ring from recomputing CTAs to the dE /
                 dC CTAs of one persistent kernel (ops.backward_stream).  No transient grows with the
                 kept-tile count.  Needs D % 64 == 0; other shapes take "fast".
      "fast"     the forward keeps a sorted classifier copy and stores label tiles; the backward
                 keeps every kept tile's S-hat (memory grows with the kept count)
      "grouped"  (= low_memory=True) forward and backward over vocabulary groups with S-hat slots
                 sized from the learned kept density; with filter_eps=None, or
                 CCE_LOWMEM_RECOMPUTE=1, only O(N) state is kept and the backward recomputes every tile
    CCE_MEMORY overrides the default.

    vocab_rows (vocab-parallel, instead of vocab_start): the global vocabulary ids of `c`'s rows,
    for shards that are not one contiguous range -- e.g. vocab_parallel.cyclic_rows, which deals
    256-row blocks round-robin so that a frequency-ordered vocabulary (BPE ids) spreads its dense
    head over every rank.  The labels are mapped to shard coordinates on the device.

    exempt_label_tiles=True is the reference's filter (a tile holding a label is never skipped,
    kernels.py:447-455).  False is the paper's Alg. 3 ordering: tiles are filtered on the softmax
    alone and the -1 label term is applied exactly, apart from the tiles (PAPER.md:212-214,
    :330-335) -- label-only tiles then skip too.
    """
    if reduction not in ("mean", "sum", "none"):
        raise ValueError(f"unknown reduction {reduction!r}")
    lead = e.shape[:-1]
    e2 = e.reshape(-1, e.shape[-1])
    t2 = targets.reshape(-1)
    if t2.shape[0] != e2.shape[0]:
        raise ValueError(f"label count {t2.shape[0]} != token count {e2.shape[0]}")
    e2, c = ops.adapt_operands(e2, c)  # bf16, contiguous, hidden size padded to a multiple of 8
    ops.check_operands(e2, c, t2.to(torch.int64) if t2.dtype != torch.int64 else t2)
    t2 = t2.to(torch.int64).contiguous()
    v_total = c.shape[0] if process_group is None else _global_vocab(c.shape[0], process_group)
    # the reference's check_vocab (core.py:110-114): on the device, without a host read -- a label
    # outside [0, V) gives a NaN loss at its row and a sticky device flag, reported here by the
    # next call (ValueError) once its asynchronous copy has landed
    ops.raise_label_error(e2.device, v_total)
    if process_group is None and (os.environ.get("CCE_CHECK_LABELS") == "1" or torch.is_anomaly_enabled()):
        # debug mode: the same check on the host, raised by this call
        bad = (t2 != ignore_index) & ((t2 < 0) | (t2 >= c.shape[0]))
        if bool(bad.any()):
            raise ValueError(f"label out of range for vocab size {c.shape[0]}")
        for name, x in (("embeddings", e2), ("classifier", c)):  # core.py:47
            if not bool(torch.isfinite(x).all()):
                raise ValueError(f"{name} contains non-finite entries")
    t_shard = t2
    if vocab_rows is not None:
        if vocab_start:
            raise ValueError("pass vocab_rows or vocab_start, not both")
        if vocab_rows.shape != (c.shape[0],):
            raise ValueError(f"vocab_rows has shape {tuple(vocab_rows.shape)}, expected ({c.shape[0]},)")
        if 0 <= ignore_index <= c.shape[0]:
            raise ValueError("vocab_rows needs an ignore_index outside [0, shard rows]")
        t_shard = ops.shard_targets(t2, vocab_rows.to(e2.device), v_total, int(ignore_index))
    cap = float(softcap) if softcap else 0.0
    if cap < 0:
        raise ValueError("softcap must be positive")
    eps = _resolve_eps(filter_eps)
    training = torch.is_grad_enabled() and (e2.requires_grad or c.requires_grad)
    mode = "grouped" if low_memory else (memory or os.environ.get("CCE_MEMORY") or "bounded")
    if mode not in ("bounded", "fast", "grouped"):
        raise ValueError(f"memory must be 'bounded', 'fast' or 'grouped', got {mode!r}")
    if mode == "bounded" and not ops.stream_supported(e2.shape[1]):  # any N: large batches run in token chunks
        mode = "fast"  # the streamed backward's CTA-pair boxes need D % 64 == 0
    out = _LinearCrossEntropy.apply(e2, c, t2, t_shard, int(ignore_index), cap, reduction, eps,
                                    bool(vocab_sorting), process_group, int(vocab_start),
                                    mode, bool(exempt_label_tiles), training, int(v_total))
    if reduction == "none":
        return out.reshape(lead)
    return out
