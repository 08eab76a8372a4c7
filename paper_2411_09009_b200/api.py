"""The reference package's hot-path surface, on CUDA tensors, backed by libcce_b200.so.

Mirrors /root/reference/pkg/src/cce (core.py, kernels.py) name for name so code and tests written
against the reference port over mechanically:

  reference                                   here
  IGNORE_INDEX = -1 (core.py:23)              IGNORE_INDEX
  EPSILON_DEFAULT = 2**-12 (core.py:27)       EPSILON_DEFAULT
  BlockSpec (core.py:117-127)                 BlockSpec   (GPU tile fixed at n_b=128, m_b=256)
  CceOptions (core.py:130-156)                CceOptions  (thread_count accepted, ignored)
  LossOutput / Gradients (core.py:159-178)    LossOutput / Gradients (torch tensors)
  default_upstream (core.py:181-200)          default_upstream
  indexed_matmul (kernels.py:204-251)         indexed_matmul
  lse_forward (kernels.py:254-319)            lse_forward
  lse_backward (kernels.py:327-486)           lse_backward
  compute_vocab_order (kernels.py:145-160)    compute_vocab_order
  filter_ignored (kernels.py:494-510)         filter_ignored
  cce_loss (kernels.py:513-580)               cce_loss
  log_add_exp / block_skip_decision           log_add_exp / block_skip_decision

Inputs may be numpy arrays or tensors; E and C are rounded to bf16 on the device (the same RNE
rounding as round_to_bf16, core.py:208-226) because the tensor-core path is bf16 in / fp32
accumulate.  Errors are ValueError with the reference's messages.  Results are deterministic
(fixed reduction orders), so CceOptions.deterministic needs no special mode.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .ops import BackwardStats

IGNORE_INDEX = -1
EPSILON_DEFAULT = 2.0 ** -12


@dataclass(frozen=True)
class BlockSpec:
    """Tile sizes; the GPU kernels are built for 128 tokens x 256 vocab rows (d_b is free)."""

    n_b: int = ops.BLOCK_TOKENS
    m_b: int = ops.BLOCK_VOCAB
    d_b: int = 64

    def __post_init__(self):
        if min(self.n_b, self.m_b, self.d_b) < 1:
            raise ValueError(f"block sizes must be >= 1, got {self}")
        if (self.n_b, self.m_b) != (ops.BLOCK_TOKENS, ops.BLOCK_VOCAB):
            raise ValueError(
                f"the B200 kernels tile {ops.BLOCK_TOKENS} tokens x {ops.BLOCK_VOCAB} vocab rows; "
                f"got n_b={self.n_b}, m_b={self.m_b}")


@dataclass(frozen=True)
class CceOptions:
    epsilon: float = EPSILON_DEFAULT
    filtering: bool = True
    vocab_sorting: bool = True
    deterministic: bool = False
    reduction: str = "mean-over-valid"
    thread_count: int = 1

    def __post_init__(self):
        if not (0.0 < self.epsilon < 1.0):
            raise ValueError(f"epsilon must be in (0, 1), got {self.epsilon}")
        if self.reduction not in ("sum", "mean-over-valid", "none"):
            raise ValueError(f"unknown reduction {self.reduction!r}")
        if self.thread_count < 1:
            raise ValueError("thread_count must be >= 1")


@dataclass
class LossOutput:
    per_token_loss: torch.Tensor
    lse: torch.Tensor
    mean_logits: torch.Tensor | None = None


@dataclass
class Gradients:
    d_e: torch.Tensor
    d_c: torch.Tensor


@dataclass(frozen=True)
class VocabOrder:
    perm: torch.Tensor
    mean_logits: torch.Tensor


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("cce_b200 needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class EmbeddingMatrix:
    """Token embeddings [n_tokens, dim] (core.py:52-67): any array or tensor; checked on use."""
    data: object

    @property
    def n_tokens(self) -> int:
        return int(_shape(self.data)[0])

    @property
    def dim(self) -> int:
        return int(_shape(self.data)[1])


@dataclass(frozen=True)
class ClassifierMatrix:
    """Classifier rows [vocab, dim] (core.py:70-85)."""
    data: object

    @property
    def vocab(self) -> int:
        return int(_shape(self.data)[0])

    @property
    def dim(self) -> int:
        return int(_shape(self.data)[1])


@dataclass(frozen=True)
class TokenBatch:
    """Target labels, IGNORE_INDEX or a vocabulary row (core.py:88-114); validated on creation
    like the reference (1-D, >= -1)."""
    labels: object

    def __post_init__(self):
        t = torch.as_tensor(self.labels)
        if t.dim() != 1:
            raise ValueError(f"labels must be 1-D, got shape {tuple(t.shape)}")
        if t.numel() and int(t.min()) < IGNORE_INDEX:
            raise ValueError("labels must be -1 (ignore) or non-negative")

    @property
    def n_tokens(self) -> int:
        return int(_shape(self.labels)[0])

    @property
    def valid_mask(self) -> torch.Tensor:
        return torch.as_tensor(self.labels) != IGNORE_INDEX

    def check_vocab(self, vocab: int) -> None:
        t = torch.as_tensor(self.labels)
        if t.numel() and int(t.max()) >= vocab:
            raise ValueError(f"label {int(t.max())} out of range for vocab size {vocab}")


@dataclass(frozen=True)
class BlockSchedule:
    """The (token block, vocab block) pairs a pass visits, each once (kernels.py:48-63).  On the
    GPU the visit order is the persistent kernels' static unit schedule (a11); `order` keeps the
    reference's vocabulary: "row-major" = one fixed sweep (what the B200 kernels do: results are
    bit-reproducible), "work-stealing" = dynamic hand-out."""
    pairs: tuple
    order: str = "row-major"

    @classmethod
    def for_grid(cls, n_tiles: int, m_tiles: int, order: str = "row-major") -> "BlockSchedule":
        return cls(tuple((n, m) for n in range(n_tiles) for m in range(m_tiles)), order)


def round_to_bf16(x):
    """bf16 round-to-nearest-even, returned as float32 (core.py:208-226): scalars give a float,
    tensors a tensor, anything else a numpy array.  NaN stays NaN, +-inf stay infinite."""
    t = torch.as_tensor(x, dtype=torch.float32)
    r = t.to(torch.bfloat16).to(torch.float32)
    if isinstance(x, torch.Tensor):
        return r
    if r.dim() == 0:
        return float(r)
    return r.numpy()


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else tuple(torch.as_tensor(x).shape)


def _unwrap(x):
    if isinstance(x, (EmbeddingMatrix, ClassifierMatrix)):
        return x.data
    if isinstance(x, TokenBatch):
        return x.labels
    return x


def _matrix(x, name: str, min_rows: int) -> torch.Tensor:
    t = torch.as_tensor(_unwrap(x))
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if t.shape[0] < min_rows:
        raise ValueError(f"{name} needs at least {min_rows} rows, got {t.shape[0]}")
    if t.shape[1] < 1:
        raise ValueError(f"{name} needs at least one feature column")
    t = t.to(_device())
    if not bool(torch.isfinite(t).all()):
        raise ValueError(f"{name} contains non-finite entries")
    return t.to(torch.bfloat16).contiguous()


def _labels(x, vocab: int | None = None) -> torch.Tensor:
    t = torch.as_tensor(_unwrap(x)).to(torch.int64)
    if t.dim() != 1:
        raise ValueError(f"labels must be 1-D, got shape {tuple(t.shape)}")
    if t.numel() and int(t.min()) < IGNORE_INDEX:
        raise ValueError("labels must be -1 (ignore) or non-negative")
    if vocab is not None and t.numel() and int(t.max()) >= vocab:
        raise ValueError(f"label {int(t.max())} out of range for vocab size {vocab}")
    return t.to(_device()).contiguous()


def _pair(e, c, x=None):
    """(E, C, X) on the device in the kernels' layout; a hidden size that is not a multiple of 8 is
    zero-padded (logits unchanged) and _trim cuts the gradients back to the caller's D."""
    E = _matrix(e, "embeddings", 0)
    C = _matrix(c, "classifier", 1)
    if E.shape[1] != C.shape[1]:
        raise ValueError(f"feature dims differ: embeddings {E.shape[1]} vs classifier {C.shape[1]}")
    E, C = ops.adapt_operands(E, C)
    X = None
    if x is not None:
        X = _labels(x, C.shape[0])
        if X.shape[0] != E.shape[0]:
            raise ValueError(f"label count {X.shape[0]} != token count {E.shape[0]}")
    return E, C, X


def _hidden(e) -> int:
    return int(_shape(_unwrap(e))[1])


def _trim(g: torch.Tensor, d: int) -> torch.Tensor:
    return g if g.shape[1] == d else g[:, :d].contiguous()


def default_upstream(x, reduction: str, dtype=torch.float32) -> torch.Tensor:
    """core.py:181-200: 'sum' = 1 per valid token, 'mean-over-valid' = 1/#valid, 'none' raises."""
    labels = torch.as_tensor(_unwrap(x))
    if reduction == "none":
        raise ValueError('reduction "none" requires an explicit upstream vector')
    valid = labels != IGNORE_INDEX
    up = torch.zeros(labels.shape[0], dtype=dtype, device=labels.device)
    if reduction == "sum":
        up[valid] = 1.0
    elif reduction == "mean-over-valid":
        nv = int(valid.sum())
        if nv:
            up[valid] = 1.0 / nv
    else:
        raise ValueError(f"unknown reduction {reduction!r}")
    return up


def log_add_exp(a, b):
    """kernels.py:121-137 (elementwise, -inf identity)."""
    a = torch.as_tensor(a, dtype=torch.float64)
    b = torch.as_tensor(b, dtype=torch.float64)
    return torch.logaddexp(a, b)


def block_skip_decision(s_block, epsilon: float) -> bool:
    """kernels.py:140-142: every entry strictly below epsilon."""
    return bool((torch.as_tensor(s_block) < epsilon).all())


def compute_vocab_order(mean_logits, m_b: int = ops.BLOCK_VOCAB) -> VocabOrder:
    """Stable descending sort of the mean logits (kernels.py:145-160)."""
    mean = torch.as_tensor(mean_logits)
    if mean.dim() != 1:
        raise ValueError(f"mean logits must be 1-D, got shape {tuple(mean.shape)}")
    if m_b < 1:
        raise ValueError("m_b must be >= 1")
    perm = torch.sort(mean, descending=True, stable=True).indices
    return VocabOrder(perm=perm, mean_logits=mean)


def filter_ignored(e, x):
    """kernels.py:494-510: (compact_e, compact_x, index_map); wrapped inputs
    (EmbeddingMatrix / TokenBatch) come back wrapped, like the reference's."""
    E = torch.as_tensor(_unwrap(e))
    X = torch.as_tensor(_unwrap(x))
    if E.shape[0] != X.shape[0]:
        raise ValueError(f"label count {X.shape[0]} != token count {E.shape[0]}")
    valid = X != IGNORE_INDEX
    if bool(valid.all()):
        ce, cx, idx = E, X, torch.arange(X.shape[0], device=X.device)
    else:
        idx = torch.nonzero(valid).squeeze(1)
        ce, cx = E[idx], X[idx]
    if isinstance(e, EmbeddingMatrix):
        ce = EmbeddingMatrix(ce)
    if isinstance(x, TokenBatch):
        cx = TokenBatch(cx)
    return ce, cx, idx


def indexed_matmul(e, c, x, blocks: BlockSpec | None = None, options: CceOptions | None = None):
    """out[i] = C[x_i] . E[i], 0 at ignored rows (kernels.py:204-251)."""
    E, C, X = _pair(e, c, x)
    return ops.indexed_dot(E, C, X, IGNORE_INDEX)


def lse_forward(e, c, blocks: BlockSpec | None = None, options: CceOptions | None = None):
    """(lse over every vocabulary row for every token, mean_logits or None) (kernels.py:254-319)."""
    blocks = blocks or BlockSpec()
    options = options or CceOptions()
    E, C, _ = _pair(e, c)
    n = E.shape[0]
    no_labels = torch.full((n,), IGNORE_INDEX, dtype=torch.int64, device=E.device)
    lse, _ = ops.forward_local(E, C, no_labels, IGNORE_INDEX)
    mean = None
    if options.vocab_sorting:
        _, mean = ops.vocab_order(E, C, no_labels, IGNORE_INDEX - 1, n)
    return lse, mean


def lse_backward(e, c, x, lse, upstream, blocks: BlockSpec | None = None,
                 options: CceOptions | None = None, order: VocabOrder | None = None,
                 stats: BackwardStats | None = None) -> Gradients:
    """Filtered backward (kernels.py:327-486).  Like the reference, every row stays in place
    (ignored rows carry zero upstream; their token blocks count as zero-upstream skips when the
    whole block is ignored), so `stats` follows the reference's tile grid.  `order` (if given) is
    the vocab order; otherwise the natural order is used, like the reference.  The GPU tile is
    128 x 256 (BlockSpec.m_b other than 256 is rejected by BlockSpec itself)."""
    blocks = blocks or BlockSpec()
    options = options or CceOptions()
    E, C, X = _pair(e, c, x)
    n = E.shape[0]
    lse_t = torch.as_tensor(lse).to(E.device, torch.float32)
    if tuple(lse_t.shape) != (n,):
        raise ValueError(f"lse must have shape ({n},), got {tuple(lse_t.shape)}")
    up = torch.as_tensor(upstream).to(E.device, torch.float32)
    if tuple(up.shape) != (n,):
        raise ValueError(f"upstream must have shape ({n},), got {tuple(up.shape)}")
    if bool((up[X == IGNORE_INDEX] != 0).any()):
        raise ValueError("upstream must be 0 at ignored positions")
    perm = None
    if order is not None:
        perm = torch.as_tensor(order.perm).to(E.device, torch.int32)
        if perm.shape[0] != C.shape[0]:
            raise ValueError(f"vocab order has {perm.shape[0]} entries, expected {C.shape[0]}")
    de, dc, counters, _ = ops.backward(E, C, X, lse_t, up, ignore_index=IGNORE_INDEX,
                                       eps=options.epsilon if options.filtering else None,
                                       vocab_sorting=perm is not None, perm=perm, fp32_de=True,
                                       compact=False)
    if stats is not None:
        s = ops.stats_from_counters(counters, n, C.shape[0])
        stats.total_tiles, stats.skipped_epsilon, stats.skipped_zero_upstream = (
            s.total_tiles, s.skipped_epsilon, s.skipped_zero_upstream)
    d = _hidden(e)
    return Gradients(d_e=_trim(de, d), d_c=_trim(dc.float(), d))


def cce_loss(e, c, x, blocks: BlockSpec | None = None, options: CceOptions | None = None):
    """(LossOutput, backward) exactly like kernels.py:513-580: loss / lse 0 at ignored rows,
    mean_logits over valid rows when sorting, backward(upstream=None) from options.reduction."""
    blocks = blocks or BlockSpec()
    options = options or CceOptions()
    E, C, X = _pair(e, c, x)
    n, d = E.shape[0], _hidden(e)
    valid = X != IGNORE_INDEX
    mean = perm = state = None
    if options.filtering:
        # forward over the backward's tiles (compacted rows, vocab order fixed by the mean logits
        # of the valid rows), recording per-row tile maxima: the backward then recomputes only
        # the tiles it keeps
        # the backward closure may run more than once (kernels.py:549-580): no stored label tiles
        # (they become S-hat in place) and no dC in the sorted copy's storage (reuse_state)
        lse_l, corr, state = ops.forward_tiles(E, C, X, IGNORE_INDEX, vocab_sorting=options.vocab_sorting,
                                               eps=options.epsilon, store_labels=False)
        mean = state.mean_logits
    else:
        lse_l, corr = ops.forward_local(E, C, X, IGNORE_INDEX)
        if options.vocab_sorting:
            perm, mean = ops.vocab_order(E, C, X, IGNORE_INDEX, int(valid.sum()))
    lse, loss = ops.merge_shards(lse_l[None], corr[None], X, IGNORE_INDEX)
    out = LossOutput(per_token_loss=loss, lse=lse, mean_logits=mean)

    def backward(upstream=None, stats: BackwardStats | None = None) -> Gradients:
        if upstream is None:
            up = default_upstream(X, options.reduction)
        else:
            up = torch.as_tensor(upstream).to(E.device, torch.float32)
            if tuple(up.shape) != (n,):
                raise ValueError(f"upstream must have shape ({n},), got {tuple(up.shape)}")
            if bool((up[~valid] != 0).any()):
                raise ValueError("upstream must be 0 at ignored positions")
        if state is not None:
            de, dc, counters = ops.backward_tiles(state, X, lse, up.contiguous(), ignore_index=IGNORE_INDEX,
                                                  eps=options.epsilon, fp32_de=True, reuse_state=True)
        else:
            de, dc, counters, _ = ops.backward(
                E, C, X, lse, up.contiguous(), ignore_index=IGNORE_INDEX, eps=None,
                vocab_sorting=options.vocab_sorting, perm=perm, fp32_de=True)
        if stats is not None:
            s = ops.stats_from_counters(counters, int(valid.sum()), C.shape[0])
            stats.total_tiles, stats.skipped_epsilon, stats.skipped_zero_upstream = (
                s.total_tiles, s.skipped_epsilon, s.skipped_zero_upstream)
        return Gradients(d_e=_trim(de, d), d_c=_trim(dc.float(), d))

    return out, backward


__all__ = [
    "BackwardStats", "BlockSchedule", "BlockSpec", "CceOptions", "ClassifierMatrix", "EPSILON_DEFAULT",
    "EmbeddingMatrix", "Gradients", "IGNORE_INDEX", "LossOutput", "TokenBatch", "VocabOrder",
    "block_skip_decision", "cce_loss", "compute_vocab_order", "default_upstream", "filter_ignored",
    "indexed_matmul", "log_add_exp", "lse_backward", "lse_forward", "round_to_bf16",
]
