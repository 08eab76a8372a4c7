"""Pin the CPU oracle (oracle/cce_oracle.py) before trusting it.

(a) the reference's own known-answer tests, ported value for value;
(b) the golden fixtures produced by running the reference itself (tests/golden/make_golden.py);
(c) finite differences for the softcap extension, which the reference lacks.
No GPU needed.
"""

import math
import struct

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases
from oracle import cce_oracle as O


# ---------------------------------------------------------------- (a) known answers
def test_log_add_exp_known_values():  # test_kernels.py:87-99
    assert O.log_add_exp(5.0, -np.inf) == 5.0
    assert O.log_add_exp(-np.inf, -2.5) == -2.5
    assert O.log_add_exp(-np.inf, -np.inf) == -np.inf
    assert O.log_add_exp(0.0, 0.0) == pytest.approx(math.log(2), abs=1e-12)
    assert O.log_add_exp(1.0, 2.0) == pytest.approx(2.3132616875182228, rel=1e-14)


def test_log_add_exp_elementwise_and_associative():  # test_kernels.py:102-124
    a = np.array([0.0, -np.inf, 3.0], np.float32)
    b = np.array([0.0, 1.0, -np.inf], np.float32)
    out = O.log_add_exp(a, b)
    assert out.dtype == np.float32
    assert out[0] == pytest.approx(math.log(2), rel=1e-6) and out[1] == 1.0 and out[2] == 3.0
    v = np.array([-3.0, 0.5, 2.0, -10.0])
    left = O.log_add_exp(O.log_add_exp(v[0], v[1]), v[2])
    right = O.log_add_exp(v[0], O.log_add_exp(v[1], v[2]))
    assert left == pytest.approx(right, rel=1e-12)


def test_logsumexp_known_values():  # test_oracle.py:19-45
    assert O.logsumexp_stable([0, 0, 0, 0]) == pytest.approx(math.log(4), abs=1e-15)
    assert O.logsumexp_stable([1, 2, 3]) == pytest.approx(3.4076059644443806, rel=1e-15)
    assert O.logsumexp_stable([-np.inf, -np.inf]) == -np.inf
    with pytest.raises(ValueError):
        O.logsumexp_stable([])


def _bf16_struct(x: float) -> float:  # independent rounding, tests/helpers.py:18-30
    (bits,) = struct.unpack("<I", struct.pack("<f", x))
    if (bits & 0x7F800000) == 0x7F800000:
        return x
    bits = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    return struct.unpack("<f", struct.pack("<I", bits & 0xFFFFFFFF))[0]


@pytest.mark.parametrize("value,expected", [
    (1.0, 1.0), (2.0 ** -12, 2.0 ** -12), (1.0 + 2.0 ** -9, 1.0), (0.0, 0.0), (-1.0, -1.0),
    (float("inf"), float("inf")), (float("-inf"), float("-inf")),
])
def test_bf16_known_values(value, expected):  # test_core.py:76-89
    assert O.round_to_bf16(value) == expected


def test_bf16_matches_independent_rounding():  # test_core.py:96-99
    assert math.isnan(O.round_to_bf16(float("nan")))
    for value in [3.14159, -0.1, 1e-30, 65504.0, 1.0 + 2.0 ** -8, 1.0 + 2.0 ** -7]:
        assert O.round_to_bf16(value) == _bf16_struct(value)


def test_block_skip_is_strict():  # kernels.py:140-142
    eps = 2.0 ** -12
    assert O.block_skip_decision(np.full((2, 2), eps / 2), eps)
    assert not O.block_skip_decision(np.full((2, 2), eps), eps)


def test_default_upstream():  # core.py:181-200
    x = np.array([3, -1, 0, 2])
    assert np.allclose(O.default_upstream(x, "sum"), [1, 0, 1, 1])
    assert np.allclose(O.default_upstream(x, "mean-over-valid"), [1 / 3, 0, 1 / 3, 1 / 3])
    assert np.all(O.default_upstream(np.array([-1, -1]), "mean-over-valid") == 0)
    with pytest.raises(ValueError):
        O.default_upstream(x, "none")


def test_vocab_order_stable_ties():  # test_kernels.py:206-225
    mean = np.array([0.5, 2.0, 0.5, 2.0, -1.0])
    assert O.compute_vocab_order(mean).tolist() == [1, 3, 0, 2, 4]


def test_uniform_classifier_loss_is_log_v():  # test_kernels.py:132-136, :343-351
    rng = np.random.default_rng(2)
    e = rng.standard_normal((24, 4)).astype(np.float32)
    c = np.zeros((16, 4), np.float32)
    x = rng.integers(0, 16, 24)
    loss, lse, _ = O.naive_forward(e, c, x)
    assert np.allclose(loss, math.log(16)) and np.allclose(lse, math.log(16))
    l2, _, _, de, dc, _ = O.cce_loss(e, c, x)
    up = O.default_upstream(x, "mean-over-valid")
    fde, fdc = O.naive_backward(e, c, x, up)
    assert np.allclose(l2, math.log(16), atol=1e-6)
    assert O.rel_err(dc, fdc) < 1e-5 and O.rel_err(de, fde) < 1e-5


@pytest.mark.parametrize("margin,tol", [(20.0, 5e-6), (10.0, 1e-5)])
def test_margin_closed_form(margin, tol):  # test_kernels.py:354-371
    v, d = 64, 4
    e = np.ones((1, d), np.float32)
    c = np.zeros((v, d), np.float32)
    c[13] = margin / d
    x = np.array([13])
    expected = math.log(1.0 + (v - 1) * math.exp(-margin))
    loss, _, _ = O.naive_forward(e, c, x)
    assert loss[0] == pytest.approx(expected, rel=1e-6)
    l2 = O.cce_loss(e, c, x)[0]
    assert l2[0] == pytest.approx(expected, abs=tol)


def test_vocab_one_and_all_ignored():  # test_kernels.py:139-143, :249-255, :408-415
    rng = np.random.default_rng(0)
    e = rng.standard_normal((7, 3)).astype(np.float32)
    c = rng.standard_normal((1, 3)).astype(np.float32)
    x = np.zeros(7, np.int64)
    loss, _, _, de, dc, _ = O.cce_loss(e, c, x)
    assert np.allclose(loss, 0, atol=1e-6) and np.allclose(de, 0) and np.allclose(dc, 0)
    c5 = rng.standard_normal((5, 3)).astype(np.float32)
    xi = np.full(7, -1)
    loss, lse, _, de, dc, _ = O.cce_loss(e, c5, xi)
    assert np.all(loss == 0) and np.all(lse == 0) and np.all(de == 0) and np.all(dc == 0)


def test_indexed_matmul_known_answers():  # test_kernels.py:26-39
    e = np.ones((5, 7), np.float32)
    c = np.ones((3, 7), np.float32)
    assert np.allclose(O.indexed_matmul(e, c, np.array([0, 1, 2, 0, -1])), [7, 7, 7, 7, 0])
    assert np.allclose(O.indexed_matmul(np.zeros((2, 7)), c, np.array([0, 1])), 0)


def test_zero_upstream_skips_everything():  # test_kernels.py:240-246
    rng = np.random.default_rng(1)
    e = rng.standard_normal((200, 8)).astype(np.float32)
    c = rng.standard_normal((600, 8)).astype(np.float32)
    x = rng.integers(0, 600, 200)
    lse = O.lse_forward_blocked(e, c)
    de, dc, st = O.lse_backward_blocked(e, c, x, lse, np.zeros(200, np.float32), return_stats=True)
    assert np.all(de == 0) and np.all(dc == 0)
    assert st["skipped_zero_upstream"] == st["total_tiles"]


# ---------------------------------------------------------------- (b) reference-run fixtures
@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference_fixture(name):
    g = np.load(GOLDEN / f"{name}.npz")
    e, c, x = g["e"], g["c"], g["x"]
    filt, srt = bool(g["filtering"]), bool(g["sorting"])
    loss, lse, mean, de, dc, st = O.cce_loss(
        e, c, x, eps=O.EPSILON_DEFAULT if filt else None, vocab_sorting=srt,
        perm=g["perm"] if srt else None)
    valid = x != -1
    tol = 1e-5 * max(1.0, float(np.abs(g["loss"]).max()))
    assert np.max(np.abs(loss - g["loss"])) < tol
    assert np.max(np.abs(lse[valid] - g["lse"][valid])) < tol
    if srt and valid.any():
        assert O.rel_err(mean, g["mean_logits"]) < 1e-5
        assert np.array_equal(O.compute_vocab_order(g["mean_logits"]), g["perm"])
    assert O.rel_err(de, g["d_e"]) < 1e-4
    assert O.rel_err(dc, g["d_c"]) < 1e-4
    ref_stats = g["stats"].tolist()
    if valid.any():
        assert [st["total_tiles"], st["skipped_epsilon"], st["skipped_zero_upstream"]] == ref_stats
    # exact oracle vs the reference's naive f64 oracle
    nl, nlse, _ = O.naive_forward(e, c, x)
    assert np.allclose(nl, g["naive_loss"], rtol=1e-12, atol=1e-12)
    assert np.allclose(nlse, g["naive_lse"], rtol=1e-12, atol=1e-12)
    nde, ndc = O.naive_backward(e, c, x, g["upstream"])
    assert np.allclose(nde, g["naive_d_e"], rtol=1e-10, atol=1e-14)
    assert np.allclose(ndc, g["naive_d_c"], rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- (c) softcap restatement
@pytest.mark.parametrize("cap", [3.0, 30.0])
def test_softcap_gradients_match_finite_differences(cap):
    rng = np.random.default_rng(7)
    n, d, v = 5, 4, 9
    e = rng.standard_normal((n, d))
    c = rng.standard_normal((v, d)) * 2.0
    x = rng.integers(0, v, n)
    x[2] = -1
    up = O.default_upstream(x, "mean-over-valid", np.float64)
    de, dc = O.naive_backward(e, c, x, up, softcap=cap)
    entries = [(j, k) for j in range(v) for k in range(d)]
    fde, fdc = O.finite_difference_gradients(e, c, x, up, classifier_entries=entries, softcap=cap)
    assert O.rel_err(de, fde) < 1e-7
    assert O.rel_err(dc.reshape(-1), fdc) < 1e-7
    assert np.all(de[2] == 0)


def test_softcap_blocked_matches_naive():
    rng = np.random.default_rng(3)
    e = rng.standard_normal((150, 16)).astype(np.float32)
    c = (rng.standard_normal((700, 16)) * 1.5).astype(np.float32)
    x = rng.integers(0, 700, 150)
    loss, lse, _, de, dc, _ = O.cce_loss(e, c, x, softcap=5.0, eps=None, vocab_sorting=False)
    nl, nlse, _ = O.naive_forward(e, c, x, softcap=5.0)
    nde, ndc = O.naive_backward(e, c, x, O.default_upstream(x, "mean-over-valid"), softcap=5.0)
    assert np.max(np.abs(loss - nl)) < 1e-4
    assert O.rel_err(de, nde) < 1e-4 and O.rel_err(dc, ndc) < 1e-4


def test_paper_ordering_restatement():
    """exempt_labels=False (Alg. 3: filter on S, then the label term): without filtering
    it is the unfiltered gradient; when every label tile is kept anyway it equals the reference's
    label-tile exemption; otherwise it skips at least as many tiles."""
    rng = np.random.default_rng(5)
    n, d, v = 300, 32, 10000  # mean S = 1e-4 < eps: only label tiles survive the reference rule
    e = O.round_to_bf16(rng.standard_normal((n, d)).astype(np.float32))
    c = O.round_to_bf16((rng.standard_normal((v, d)) * 0.1 / np.sqrt(d)).astype(np.float32))
    x = rng.integers(0, v, n)
    x[::7] = -1
    _, lse, _ = O.naive_forward(e, c, x)
    up = O.default_upstream(x, "mean-over-valid")
    a = O.lse_backward_blocked(e, c, x, lse.astype(np.float32), up, eps=None, exempt_labels=False,
                               dtype=np.float64)
    b = O.naive_backward(e, c, x, up)
    assert O.rel_err(a[0], b[0]) < 1e-6 and O.rel_err(a[1], b[1]) < 1e-6  # lse passed as f32
    ex = O.lse_backward_blocked(e, c, x, lse.astype(np.float32), up, return_stats=True)
    sp = O.lse_backward_blocked(e, c, x, lse.astype(np.float32), up, exempt_labels=False,
                                return_stats=True)
    assert sp[2]["skipped_epsilon"] > ex[2]["skipped_epsilon"]  # label-only tiles now skip
    # sharp logits: every label tile holds a big S, so both orderings keep the same tiles
    c2 = O.round_to_bf16((rng.standard_normal((v, d)) * 3.0 / np.sqrt(d)).astype(np.float32))
    _, lse2, _ = O.naive_forward(e, c2, x)
    ex2 = O.lse_backward_blocked(e, c2, x, lse2.astype(np.float32), up, return_stats=True)
    sp2 = O.lse_backward_blocked(e, c2, x, lse2.astype(np.float32), up, exempt_labels=False,
                                 return_stats=True)
    if ex2[2] == sp2[2]:
        assert O.rel_err(ex2[0], sp2[0]) < 1e-6 and O.rel_err(ex2[1], sp2[1]) < 1e-6
