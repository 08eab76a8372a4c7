"""Host-side behaviour of the reference-mirroring API (no GPU): option validation, reductions,
vocabulary order, helpers - the same cases the reference's test_core.py / test_kernels.py pin."""

import math

import numpy as np
import pytest
import torch

from paper_2411_09009_b200 import api


def test_constants_match_reference():  # core.py:23, :27
    assert api.IGNORE_INDEX == -1
    assert api.EPSILON_DEFAULT == 2.0 ** -12


@pytest.mark.parametrize("kw", [dict(epsilon=0.0), dict(epsilon=1.0), dict(reduction="avg"),
                                dict(thread_count=0)])
def test_options_validation(kw):  # core.py:150-156
    with pytest.raises(ValueError):
        api.CceOptions(**kw)


def test_blockspec_validation():
    assert api.BlockSpec() == api.BlockSpec(128, 256, 64)
    with pytest.raises(ValueError):
        api.BlockSpec(n_b=0)
    with pytest.raises(ValueError, match="tile"):
        api.BlockSpec(n_b=128, m_b=128)


def test_default_upstream_reductions():  # core.py:181-200
    x = torch.tensor([3, -1, 0, 2])
    assert torch.allclose(api.default_upstream(x, "sum"), torch.tensor([1.0, 0, 1, 1]))
    assert torch.allclose(api.default_upstream(x, "mean-over-valid"), torch.tensor([1 / 3, 0, 1 / 3, 1 / 3]))
    assert torch.all(api.default_upstream(torch.tensor([-1, -1]), "mean-over-valid") == 0)
    with pytest.raises(ValueError):
        api.default_upstream(x, "none")


def test_vocab_order_descending_stable():  # test_kernels.py:206-225
    order = api.compute_vocab_order(torch.tensor([0.5, 2.0, 0.5, 2.0, -1.0]))
    assert order.perm.tolist() == [1, 3, 0, 2, 4]
    with pytest.raises(ValueError):
        api.compute_vocab_order(torch.zeros(2, 2))


def test_log_add_exp_and_skip_decision():  # test_kernels.py:87-99, kernels.py:140-142
    assert float(api.log_add_exp(1.0, 2.0)) == pytest.approx(2.3132616875182228, rel=1e-14)
    assert float(api.log_add_exp(-math.inf, -2.5)) == -2.5
    eps = 2.0 ** -12
    assert api.block_skip_decision(torch.full((2, 2), eps / 2), eps)
    assert not api.block_skip_decision(torch.full((2, 2), eps), eps)


def test_filter_ignored_compaction():  # kernels.py:494-510
    e = torch.arange(12.0).reshape(4, 3)
    x = torch.tensor([5, -1, 2, -1])
    ce, cx, idx = api.filter_ignored(e, x)
    assert idx.tolist() == [0, 2] and cx.tolist() == [5, 2] and torch.equal(ce, e[[0, 2]])
    ce, cx, idx = api.filter_ignored(e, torch.tensor([1, 1, 1, 1]))
    assert ce is e and idx.tolist() == [0, 1, 2, 3]


def test_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        api.cce_loss(np.zeros((2, 8), np.float32), np.zeros((3, 8), np.float32), np.array([0, 1]))


def test_reference_wrapper_types():  # core.py:52-114
    import numpy as np

    e = api.EmbeddingMatrix(np.zeros((5, 8), np.float32))
    c = api.ClassifierMatrix(np.zeros((7, 8), np.float32))
    x = api.TokenBatch(np.array([0, -1, 3, 6, -1]))
    assert (e.n_tokens, e.dim, c.vocab, c.dim, x.n_tokens) == (5, 8, 7, 8, 5)
    assert x.valid_mask.tolist() == [True, False, True, True, False]
    x.check_vocab(7)
    with pytest.raises(ValueError, match="out of range"):
        x.check_vocab(6)
    with pytest.raises(ValueError):
        api.TokenBatch(np.array([0, -2]))
    with pytest.raises(ValueError):
        api.TokenBatch(np.zeros((2, 2), np.int64))
    ce, cx, idx = api.filter_ignored(e, x)  # kernels.py:494-510, wrapped in, wrapped out
    assert isinstance(ce, api.EmbeddingMatrix) and isinstance(cx, api.TokenBatch)
    assert idx.tolist() == [0, 2, 3] and ce.n_tokens == 3
    assert api.default_upstream(x, "sum").tolist() == [1.0, 0.0, 1.0, 1.0, 0.0]


def test_block_schedule_covers_grid_once():  # test_kernels.py:228-232
    sched = api.BlockSchedule.for_grid(3, 5)
    assert len(sched.pairs) == 15 and len(set(sched.pairs)) == 15
    assert sched.order == "row-major"


def test_round_to_bf16_known_values():  # test_core.py:76-99 (round-to-nearest-even)
    import numpy as np

    assert api.round_to_bf16(1.0) == 1.0
    assert api.round_to_bf16(1.0 + 2.0 ** -8) == 1.0            # tie -> even
    assert api.round_to_bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6  # tie -> even (up)
    assert api.round_to_bf16(1.0 + 2.0 ** -7) == 1.0 + 2.0 ** -7  # exact
    r = api.round_to_bf16(np.array([np.nan, np.inf, -np.inf, 3.14159], np.float32))
    assert np.isnan(r[0]) and r[1] == np.inf and r[2] == -np.inf and r[3] == np.float32(3.140625)


def test_capacity_hint_cache_is_bounded(monkeypatch):
    """Shapes that change every step cannot grow the pinned capacity-hint cache without bound."""
    import torch

    from paper_2411_09009_b200 import ops

    monkeypatch.setattr(ops, "_KEPT_HINT", {})
    monkeypatch.setattr(ops, "KEPT_HINT_MAX", 8)
    monkeypatch.setattr(ops, "_capturing", lambda: False)
    monkeypatch.setattr(torch.Tensor, "pin_memory", lambda self: self)  # no CUDA here
    monkeypatch.setattr(torch.cuda, "Event", lambda: type("E", (), {"record": lambda s: None,
                                                                     "query": lambda s: True})())
    for i in range(50):
        ops._remember_count(("shape", i), torch.tensor([i, 2 * i]), 1)
    assert len(ops._KEPT_HINT) == 8
    assert ("shape", 49) in ops._KEPT_HINT and ("shape", 0) not in ops._KEPT_HINT


def test_forward_groups_fill_whole_waves(monkeypatch):
    """ops.fwd_group_tiles: the bounded forward's vocabulary groups stay within the byte budget
    and trade whole waves of the CTA-pair grid against launch count.  Gemma-2B on 148 SMs: the
    default 52 MB budget gives 46 tiles (19.9 waves, 22 launches); a 48 MB budget with cheap
    launches takes 37 tiles (32 token-tile pairs x 37 = exactly 16 waves of 74 pairs) over its
    budget's 42 (18.2 waves)."""
    from paper_2411_09009_b200 import ops

    for k in ("CCE_FWD_GROUP_MB", "CCE_FWD_GROUP_FIT", "CCE_FWD_LAUNCH_WAVES", "CCE_PAIR"):
        monkeypatch.delenv(k, raising=False)
    mt = 1000
    assert ops.fwd_group_tiles(2304, mt) == 46
    assert ops.fwd_group_tiles(2304, mt, 8192, 148) == 46
    monkeypatch.setenv("CCE_FWD_GROUP_MB", "48")
    monkeypatch.setenv("CCE_FWD_LAUNCH_WAVES", "0.4")
    assert ops.fwd_group_tiles(2304, mt) == 42
    g = ops.fwd_group_tiles(2304, mt, 8192, 148)
    assert g == 37 and (32 * g) % 74 == 0
    monkeypatch.delenv("CCE_FWD_GROUP_MB")
    monkeypatch.delenv("CCE_FWD_LAUNCH_WAVES")
    for n, d, v in [(4096, 768, 50257), (16384, 4096, 128256), (300, 64, 1000), (1, 64, 256),
                    (32768, 3584, 256000), (65536, 5120, 131072)]:
        m = -(-v // 256)
        cap = ops.fwd_group_tiles(d, m)
        g = ops.fwd_group_tiles(d, m, n, 148)
        assert 1 <= g <= cap and g * 256 * d * 2 <= max(52 << 20, 256 * d * 2)
    monkeypatch.setenv("CCE_FWD_GROUP_FIT", "0")
    assert ops.fwd_group_tiles(2304, mt, 8192, 148) == 46
