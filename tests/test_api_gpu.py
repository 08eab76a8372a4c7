"""The reference's own kernel tests (pkg/tests/test_kernels.py) replayed against the mirrored API
on the GPU, plus the reference-run fixtures through cce_loss."""

import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden_cases
from oracle import cce_oracle as O

pytestmark = pytest.mark.gpu


def _api():
    from paper_2411_09009_b200 import api

    return api


def _make(d, n, v, seed, sigma=1.0):
    rng = np.random.default_rng(seed)
    e = O.round_to_bf16(rng.standard_normal((n, d)).astype(np.float32))
    c = O.round_to_bf16((rng.standard_normal((v, d)) * sigma / math.sqrt(d)).astype(np.float32))
    x = rng.integers(0, v, n)
    return e, c, x


@pytest.mark.parametrize("name", golden_cases())
def test_cce_loss_reference_fixture(cuda_device, name):
    api = _api()
    g = np.load(GOLDEN / f"{name}.npz")
    opts = api.CceOptions(filtering=bool(g["filtering"]), vocab_sorting=bool(g["sorting"]))
    out, back = api.cce_loss(g["e"], g["c"], g["x"], options=opts)
    valid = g["x"] != -1
    tol = 1e-3 * max(1.0, float(np.abs(g["loss"]).max()))
    assert np.max(np.abs(out.per_token_loss.cpu().numpy() - g["loss"])) < tol
    assert np.max(np.abs(out.lse.cpu().numpy()[valid] - g["lse"][valid])) < tol
    if bool(g["sorting"]) and valid.any():
        assert O.rel_err(out.mean_logits.cpu().numpy(), g["mean_logits"]) < 1e-4
    if not valid.any():
        return
    stats = api.BackwardStats()
    if bool(g["sorting"]):
        # filtered parity needs the GPU's own order in the reference run
        perm = torch.sort(out.mean_logits, descending=True, stable=True).indices.cpu().numpy()
        ce, cl, idx = O.filter_ignored(g["e"], g["x"])
        rde_c, rdc = O.lse_backward_blocked(ce, g["c"], cl, g["lse"][idx], g["upstream"][idx],
                                            perm=perm, eps=O.EPSILON_DEFAULT if bool(g["filtering"]) else None)
        rde = np.zeros_like(g["e"])
        rde[idx] = rde_c
    else:
        rde, rdc = g["d_e"], g["d_c"]
    gr = back(stats=stats)
    assert O.rel_err(gr.d_e.cpu().numpy(), rde) < 1e-2
    assert O.rel_err(gr.d_c.cpu().numpy(), rdc) < 1e-2
    assert stats.total_tiles == int(g["stats"][0])


def test_zero_upstream_gives_zero_grads(cuda_device):  # test_kernels.py:240-246
    api = _api()
    e, c, x = _make(16, 300, 700, 1)
    out, back = api.cce_loss(e, c, x)
    stats = api.BackwardStats()
    g = back(np.zeros(300, np.float32), stats=stats)
    assert torch.all(g.d_e == 0) and torch.all(g.d_c == 0)
    assert stats.skipped_zero_upstream == stats.total_tiles


def test_vocab_one_zero_loss(cuda_device):  # test_kernels.py:139-143, :249-255
    api = _api()
    e, c, x = _make(16, 40, 1, 2)
    out, back = api.cce_loss(e, c, np.zeros(40, np.int64))
    assert torch.allclose(out.per_token_loss, torch.zeros_like(out.per_token_loss), atol=1e-6)
    g = back()
    assert float(g.d_e.abs().max()) < 1e-6 and float(g.d_c.abs().max()) < 1e-6


def test_upstream_at_ignored_rejected(cuda_device):  # kernels.py:553-558
    api = _api()
    e, c, x = _make(16, 10, 50, 3)
    x[2] = -1
    _, back = api.cce_loss(e, c, x)
    up = np.ones(10, np.float32)
    with pytest.raises(ValueError, match="ignored"):
        back(up)


def test_errors_match_reference(cuda_device):  # core.py:98-114, kernels.py:168-170
    api = _api()
    e, c, x = _make(16, 10, 50, 4)
    with pytest.raises(ValueError, match="out of range"):
        api.cce_loss(e, c, np.full(10, 50))
    with pytest.raises(ValueError, match="feature dims"):
        api.cce_loss(e, c[:, :8], x)
    with pytest.raises(ValueError, match="label count"):
        api.cce_loss(e, c, x[:5])
    with pytest.raises(ValueError, match="non-negative"):
        api.cce_loss(e, c, np.full(10, -2))


def test_sorting_and_order_invariance(cuda_device):  # test_kernels.py:496-517
    api = _api()
    e, c, x = _make(64, 500, 3000, 5, sigma=2.0)
    out_s, back_s = api.cce_loss(e, c, x, options=api.CceOptions(filtering=False, vocab_sorting=True))
    out_n, back_n = api.cce_loss(e, c, x, options=api.CceOptions(filtering=False, vocab_sorting=False))
    assert torch.allclose(out_s.per_token_loss, out_n.per_token_loss, atol=1e-5)
    gs, gn = back_s(), back_n()
    assert O.rel_err(gs.d_e.cpu().numpy(), gn.d_e.cpu().numpy()) < 1e-2
    assert O.rel_err(gs.d_c.cpu().numpy(), gn.d_c.cpu().numpy()) < 1e-2


def test_deterministic_bitwise(cuda_device):  # test_kernels.py:520-531
    api = _api()
    e, c, x = _make(64, 700, 5000, 6)
    x[::3] = -1
    outs = [api.cce_loss(e, c, x) for _ in range(2)]
    grads = [b() for _, b in outs]
    assert torch.equal(outs[0][0].per_token_loss, outs[1][0].per_token_loss)
    assert torch.equal(grads[0].d_e, grads[1].d_e) and torch.equal(grads[0].d_c, grads[1].d_c)


def test_lse_forward_and_indexed_matmul(cuda_device):  # test_kernels.py:26-39, :146-152
    api = _api()
    e, c, x = _make(32, 200, 900, 7)
    lse, mean = api.lse_forward(e, c)
    nl, nlse, _ = O.naive_forward(e, c, x)
    assert np.max(np.abs(lse.cpu().numpy() - nlse)) < 1e-3
    assert O.rel_err(mean.cpu().numpy(), c.astype(np.float64) @ e.astype(np.float64).mean(0)) < 1e-4
    ones = api.indexed_matmul(np.ones((5, 8), np.float32), np.ones((3, 8), np.float32), np.array([0, 1, 2, 0, -1]))
    assert ones.tolist() == [8, 8, 8, 8, 0]


@pytest.mark.parametrize("margin,kernel_tol", [(20.0, 5e-6), (10.0, 1e-5)])
def test_cce_loss_margin_closed_form_d4(cuda_device, margin, kernel_tol):  # test_kernels.py:354-371
    """The reference's own case at its own hidden size d=4 (zero-padded to 8 for the TMA rows)."""
    api = _api()
    v, d = 64, 4
    c = np.zeros((v, d), np.float32)
    c[13] = margin / d
    out, back = api.cce_loss(np.ones((1, d), np.float32), c, np.array([13]))
    expected = math.log(1.0 + (v - 1) * math.exp(-margin))
    assert float(out.per_token_loss[0]) == pytest.approx(expected, abs=kernel_tol)
    g = back()
    assert tuple(g.d_e.shape) == (1, d) and tuple(g.d_c.shape) == (v, d)


@pytest.mark.parametrize("d", [1, 4, 12, 30])
@pytest.mark.parametrize("filtering", [False, True])
def test_cce_loss_hidden_size_not_multiple_of_8(cuda_device, d, filtering):
    api = _api()
    e, c, x = _make(d, 300, 1100, 40 + d, sigma=3.0)
    x[::7] = -1
    opts = api.CceOptions(filtering=filtering)
    out, back = api.cce_loss(e, c, x, options=opts)
    nl, nlse, _ = O.naive_forward(e, c, x)
    valid = x != -1
    assert np.max(np.abs(out.per_token_loss.cpu().numpy()[valid] - nl[valid])) < 1e-3 * max(1.0, np.abs(nl).max())
    g = back()
    assert tuple(g.d_e.shape) == (300, d) and tuple(g.d_c.shape) == (1100, d)
    fde, fdc = O.naive_backward(e, c, x, O.default_upstream(x, "mean-over-valid"))
    tol = 2e-2 if filtering else 1e-2
    assert O.rel_err(g.d_e.float().cpu().numpy(), fde) < tol
    assert O.rel_err(g.d_c.float().cpu().numpy(), fdc) < tol


def test_backward_closure_callable_twice(cuda_device, monkeypatch):  # kernels.py:549-580
    """The reference's backward closure can be called again (e.g. with another upstream); the
    second call must equal a fresh run, whatever the first call did with its buffers.  A fixed
    S-hat budget keeps both runs on the same (whole-batch) path: a learned capacity from another
    test's data of this shape could send one of them through the overflow groups, which sum dC
    in a different order."""
    monkeypatch.setenv("CCE_SHAT_BUDGET_MB", "64")
    api = _api()
    e, c, x = _make(64, 700, 5000, 12, sigma=2.0)
    x[::5] = -1
    up2 = np.where(x == -1, 0.0, np.linspace(0.1, 1.0, 700)).astype(np.float32)
    out, back = api.cce_loss(e, c, x)
    g1 = back()
    g2 = back(up2)
    _, back_fresh = api.cce_loss(e, c, x)
    f2 = back_fresh(up2)
    assert torch.equal(g2.d_e, f2.d_e) and torch.equal(g2.d_c, f2.d_c)
    g1b = back()
    assert torch.equal(g1.d_e, g1b.d_e) and torch.equal(g1.d_c, g1b.d_c)


def test_cce_loss_accepts_reference_wrapper_types(cuda_device):  # core.py:52-114, kernels.py:513
    api = _api()
    e, c, x = _make(32, 300, 2000, 14)
    x[::4] = -1
    out_w, back_w = api.cce_loss(api.EmbeddingMatrix(e), api.ClassifierMatrix(c), api.TokenBatch(x))
    out_p, back_p = api.cce_loss(e, c, x)
    assert torch.equal(out_w.per_token_loss, out_p.per_token_loss)
    gw, gp = back_w(), back_p()
    assert torch.equal(gw.d_e, gp.d_e) and torch.equal(gw.d_c, gp.d_c)
    lse, mean = api.lse_forward(api.EmbeddingMatrix(e), api.ClassifierMatrix(c))
    assert torch.equal(lse, api.lse_forward(e, c)[0])
