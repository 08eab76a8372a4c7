"""Transient-memory regression bound of the training default (memory="bounded").

The reference pins its loss-path transients (instrument.py:3-10: peak allocation minus inputs and
outputs) with a recorded formula, 4 * (8 (N + V) + 8 threads (n_b m_b + d_b (n_b + m_b)))
(/root/reference/pkg/tests/test_instrument.py:93-111).  The B200 path's transients are, per
ops.forward_stream / ops.backward_stream and stream_layout (csrc/cce_kernels.cu):

  forward   per-row tile maxima  ceil(N/128) * ceil(V/256) * 512 B
            two vocabulary groups of sorted classifier rows (at most CCE_FWD_GROUP_MB, 52 MiB, each: the
            next group is gathered on a side stream while one is swept)
            O(N + V) maps and partials; a batch with ignored rows adds their compacted copy
  backward  the S-hat ring (512 slots x 64 KiB = 32 MiB; 8 slots per token tile above 64 tiles)
            split-owner accumulators: ceil(N/128) * ceil(D/256) * 128 KiB (fp32 dE partial sums
            across stream windows) + 4 * ceil(D/256) * 256 KiB (vocab tiles over several segments),
            or, if larger, the unpermutation's saved break rows (V/64 * 5/4 + V/96 + 1024 rows of D)
            the tile maxima, O(N + V) maps and O(ceil(N/128) * ceil(V/256)) lists

No term depends on how many tiles the filter keeps: the test runs each head at two logit scales
whose kept-tile counts differ several-fold and requires the same peak.
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu

MIB = 1 << 20


def _budget(n, d, v):
    nt, mt, ndc = -(-n // 128), -(-v // 256), -(-d // 256)
    tile_max = nt * mt * 128 * 4
    lists = nt * mt * 72 + (n + v) * 64  # keep flags, item lists, segments, windows; O(N + V) maps
    # two group buffers (gather overlapped with the sweep) and the (max, sum-exp) partials of up to
    # 8 groups x 8 vocabulary splits between folds
    fwd = tile_max + 2 * 52 * MIB + 64 * n * 8 + lists + 2 * MIB
    acc = nt * ndc * 128 * 256 * 4 + 4 * ndc * 2 * 128 * 256 * 4
    # the unpermutation's saved break rows reuse the accumulators' storage after the pass: one row
    # per break (anchors 1 in 64 with headroom, cuts every 96 positions); larger at small N, large D
    perm_cap = v // 64 * 5 // 4 + v // 96 + 1024
    acc = max(acc, perm_cap * d * 2)
    ring = max(512, min(4096, 8 * nt)) * 64 * 1024  # ops.stream_ring_slots
    step = ring + acc + tile_max + lists + 4 * MIB
    return fwd, step


def _step(n, d, v, sigma, seed=0, pad=0.0):
    from paper_2411_09009_b200 import linear_cross_entropy, ops

    g = torch.Generator(device="cuda").manual_seed(seed)
    e = torch.randn(n, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
    c = (torch.randn(v, d, device="cuda", generator=g) * sigma / math.sqrt(d)).bfloat16().requires_grad_(True)
    t = torch.randint(0, v, (n,), device="cuda", generator=g)
    if pad:
        t[torch.rand(n, device="cuda", generator=g) < pad] = -100
    linear_cross_entropy(e, c, t).backward()  # warm-up (tensor maps, allocator)
    e.grad = c.grad = None
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    loss = linear_cross_entropy(e, c, t)
    torch.cuda.synchronize()
    fwd_peak = torch.cuda.max_memory_allocated() - base
    loss.backward()
    torch.cuda.synchronize()
    grads = e.grad.numel() * e.grad.element_size() + c.grad.numel() * c.grad.element_size()
    step_peak = torch.cuda.max_memory_allocated() - base - grads
    kept = int(ops.LAST_COUNTERS["counters"][0])
    return fwd_peak, step_peak, kept


@pytest.mark.parametrize("n,d,v", [(8192, 2304, 256000), (4096, 768, 50257), (2048, 4096, 128256)])
def test_training_transients_bounded_and_independent_of_kept_tiles(cuda_device, n, d, v):
    fwd_budget, step_budget = _budget(n, d, v)
    f1, s1, k1 = _step(n, d, v, sigma=0.25)  # label tiles only
    f3, s3, k3 = _step(n, d, v, sigma=4.0)   # most tiles kept
    print(f"N={n} D={d} V={v}: kept {k1} / {k3} tiles, forward peak {f1 / MIB:.1f} / {f3 / MIB:.1f} MiB "
          f"(budget {fwd_budget / MIB:.1f}), step peak {s1 / MIB:.1f} / {s3 / MIB:.1f} MiB "
          f"(budget {step_budget / MIB:.1f})")
    assert k3 > 1.5 * k1  # the two logit scales keep very different tile counts ...
    for f, s in ((f1, s1), (f3, s3)):
        assert f <= fwd_budget and s <= step_budget
    assert abs(s3 - s1) <= 2 * MIB and abs(f3 - f1) <= 2 * MIB  # ... and the same transients


def test_padded_batch_copies_only_the_compacted_rows(cuda_device):
    """An unpadded batch reads E in place; a 25%-padded one (after a call of the same shape has
    shown that rows are ignored) adds exactly the compacted copy of E (N x D bf16, read with plain
    TMA boxes: the row-gather forward is request-bound) and nothing else."""
    from paper_2411_09009_b200 import ops

    n, d, v = 4096, 2304, 128256
    ops._IGNORED_HINT.clear()
    _, s0, _ = _step(n, d, v, sigma=1.0)
    _, s1, _ = _step(n, d, v, sigma=1.0, pad=0.25)
    ecopy = n * d * 2
    assert s0 + ecopy - 2 * MIB <= s1 <= s0 + ecopy + 2 * MIB, (s0, s1)
