"""Generate golden fixtures by running the REFERENCE implementation (build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every input is bf16-representable (rounded with the reference's own round_to_bf16, core.py:208-226)
so the GPU kernels see exactly the values the reference saw.  The reference runs with the GPU's
tile geometry BlockSpec(n_b=128, m_b=256, d_b=64), so ε-filter decisions are comparable tile by
tile.  Outputs are the reference's cce_loss (kernels.py:513-580) forward + backward with the
default "mean-over-valid" upstream, its naive f64 oracle (oracle.py:57-131), and, for the sorted
cases, the vocabulary order it computed (compute_vocab_order, kernels.py:145-160).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

import cce  # the reference package (PYTHONPATH=/root/reference/pkg/src)

OUT = Path(__file__).resolve().parent

CASES = [
    # name, n, d, v, sigma, ignore_frac, filtering, sorting, concentration(gen_synthetic)
    ("ragged_sorted", 200, 64, 700, 1.0, 0.0, True, True, None),
    ("ignored_unsorted", 300, 128, 1000, 3.0, 0.3, True, False, None),
    ("nofilter_sorted", 160, 64, 513, 2.0, 0.1, False, True, None),
    ("concentrated", 256, 32, 2048, None, 0.0, True, True, 2.0),
    ("vocab1", 40, 16, 1, 1.0, 0.0, True, False, None),
    ("sharp_filtered", 384, 64, 3000, None, 0.0, True, False, 1.0),
    ("wide_vocab", 256, 32, 8192, 0.12, 0.05, True, False, None),
]


def make_inputs(name, n, d, v, sigma, ignore_frac, conc, seed):
    rng = np.random.default_rng(seed)
    if conc is not None:
        e, c, x = cce.gen_synthetic(d, n, v, seed, concentration=conc)
        E, C, X = e.data, c.data, x.labels.copy()
    else:
        E = rng.standard_normal((n, d), dtype=np.float32)
        C = (rng.standard_normal((v, d)) * (sigma / np.sqrt(d))).astype(np.float32)
        X = rng.integers(0, v if name != "wide_vocab" else 600, size=n).astype(np.int64)
    if ignore_frac:
        X[rng.random(n) < ignore_frac] = -1
    return cce.round_to_bf16(E), cce.round_to_bf16(C), X


def main():
    for i, (name, n, d, v, sigma, ign, filt, srt, conc) in enumerate(CASES):
        E, C, X = make_inputs(name, n, d, v, sigma, ign, conc, seed=100 + i)
        e, c, x = cce.EmbeddingMatrix(E), cce.ClassifierMatrix(C), cce.TokenBatch(X)
        blocks = cce.BlockSpec(n_b=128, m_b=256, d_b=64)
        opts = cce.CceOptions(filtering=filt, vocab_sorting=srt)
        out, backward = cce.cce_loss(e, c, x, blocks, opts)
        grads = backward()
        perm = (cce.compute_vocab_order(out.mean_logits, blocks.m_b).perm
                if srt else np.arange(v, dtype=np.int64))
        nf, _ = cce.naive_forward(e, c, x, cce.CceOptions(vocab_sorting=True))
        up = cce.default_upstream(x, "mean-over-valid")
        ng = cce.naive_backward(e, c, x, up)
        # backward statistics with the same geometry (lse_backward on the compacted rows)
        ce, cx, idx = cce.filter_ignored(e, x)
        stats = cce.BackwardStats()
        if ce.n_tokens:
            lse_c, _ = cce.lse_forward(ce, c, blocks, cce.CceOptions(vocab_sorting=False))
            order = cce.VocabOrder(perm=perm, mean_logits=out.mean_logits) if srt else None
            cce.lse_backward(ce, c, cx, lse_c, up[idx], blocks, opts, order=order, stats=stats)
        np.savez_compressed(
            OUT / f"{name}.npz",
            e=E, c=C, x=X, filtering=filt, sorting=srt,
            loss=out.per_token_loss, lse=out.lse,
            mean_logits=(out.mean_logits if out.mean_logits is not None else np.zeros(0, np.float32)),
            perm=perm, d_e=grads.d_e, d_c=grads.d_c,
            naive_loss=nf.per_token_loss, naive_lse=nf.lse, naive_d_e=ng.d_e, naive_d_c=ng.d_c,
            upstream=up,
            stats=np.array([stats.total_tiles, stats.skipped_epsilon, stats.skipped_zero_upstream]),
        )
        print(f"{name}: n={n} d={d} v={v} stats={stats}", file=sys.stderr)


if __name__ == "__main__":
    main()
