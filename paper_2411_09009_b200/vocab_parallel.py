"""Vocab-parallel and token-parallel CCE over torch.distributed (NCCL on NVLink / NVSwitch).

Vocab-parallel (north_star (3); no reference counterpart): rank p holds classifier
rows [vocab_start_p, vocab_start_p + V_p); E and targets are replicated.

  forward   local fused kernel -> (lse_p[N], correct_p[N]); ONE all-gather of 2N floats per
            rank; local log-add-exp merge (kernels.py:121-137) -> global lse / loss on every rank
  backward  every rank filters with the GLOBAL lse (so skip decisions equal single-GPU
            semantics); the -1 label term lands only on the owner rank (pos = -1 elsewhere);
            dC_p stays local; the fp32 dE partials are all-reduced (SUM) before the bf16 cast

Token-parallel: independent token shards, no communication inside the loss (dC sync belongs to
the caller's DDP); see `token_parallel_loss`.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops


def shard_range(vocab: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous vocab shard [start, stop) of `rank`; sizes differ by at most one row."""
    base, rem = divmod(vocab, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


CYCLIC_BLOCK = 256  # rows per block of the block-cyclic layout: one vocabulary tile


def cyclic_rows(vocab: int, rank: int, world: int, block: int = CYCLIC_BLOCK) -> torch.Tensor:
    """Global vocabulary ids of `rank`'s rows in the block-cyclic layout: blocks
    of `block` consecutive ids are dealt round-robin, block b to rank b % world.  A vocabulary
    whose ids follow frequency (BPE merges) puts its dense head on every rank instead of rank 0;
    pass the result as linear_cross_entropy(vocab_rows=...) with c = C[rows]."""
    ids = torch.arange(vocab, dtype=torch.int64)
    return ids[(ids // block) % world == rank]


def gather_and_merge(lse_local, correct, targets, ignore_index, group, v_total: int = 0):
    world = dist.get_world_size(group)
    n = lse_local.shape[0]
    mine = torch.stack([lse_local, correct]).contiguous()          # [2, N]
    flat = torch.empty((world * 2, n), dtype=mine.dtype, device=mine.device)
    dist.all_gather_into_tensor(flat, mine, group=group)
    allp = flat.view(world, 2, n)
    return ops.merge_shards(allp[:, 0].contiguous(), allp[:, 1].contiguous(), targets, ignore_index, v_total)


def all_reduce_de(de_acc, group):
    """Sum the fp32 dE partials of all vocab shards, then cast to bf16."""
    dist.all_reduce(de_acc, op=dist.ReduceOp.SUM, group=group)
    return ops.f32_to_bf16(de_acc)


_SIDE_STREAMS: dict = {}


def all_reduce_de_overlapped(de_acc, de_done, group):
    """all_reduce_de on a side stream that starts at `de_done` (recorded by the backward before
    its dC pass), so the dE all-reduce overlaps dC; the caller's stream then waits for it."""
    main = torch.cuda.current_stream(de_acc.device)
    side = _SIDE_STREAMS.get(de_acc.device)
    if side is None:
        side = _SIDE_STREAMS[de_acc.device] = torch.cuda.Stream(de_acc.device)
    side.wait_event(de_done)
    with torch.cuda.stream(side):
        dist.all_reduce(de_acc, op=dist.ReduceOp.SUM, group=group)
    de_acc.record_stream(side)
    main.wait_stream(side)
    return ops.f32_to_bf16(de_acc)


def sharded_backward(e, c, targets, lse, upstream, *, ignore_index, vocab_start, softcap, eps,
                     vocab_sorting, group):
    de_acc, dc, _, _ = ops.backward(e, c, targets, lse, upstream, ignore_index=ignore_index,
                                    vocab_start=vocab_start, softcap=softcap, eps=eps,
                                    vocab_sorting=vocab_sorting, fp32_de=True)
    return all_reduce_de(de_acc, group), dc


def vocab_parallel_cross_entropy(e, c_shard, targets, *, vocab_start: int, group=None, **kw):
    """linear_cross_entropy with the classifier sharded by vocabulary across `group`."""
    from .linear_ce import linear_cross_entropy

    return linear_cross_entropy(e, c_shard, targets, process_group=group or dist.group.WORLD,
                                vocab_start=vocab_start, **kw)


def token_parallel_loss(e_shard, c, targets_shard, *, group=None, reduction="mean", **kw):
    """Token-sharded data parallelism: each rank computes its own shard with no communication
    inside the loss.  For a global mean over valid tokens, the per-rank sum is divided by the
    all-reduced valid count (one scalar all-reduce, outside the kernels)."""
    from .linear_ce import linear_cross_entropy

    if reduction != "mean":
        return linear_cross_entropy(e_shard, c, targets_shard, reduction=reduction, **kw)
    ignore_index = kw.get("ignore_index", -100)
    total = linear_cross_entropy(e_shard, c, targets_shard, reduction="sum", **kw)
    n_valid = (targets_shard != ignore_index).sum().to(torch.float32)
    if group is not False and dist.is_initialized():
        n_valid = n_valid.clone()
        dist.all_reduce(n_valid, group=group)
    return total / n_valid.clamp_min(1.0)
