"""World-size-2 gloo test of the vocab-parallel / token-parallel plumbing (CPU, no GPU).

The per-shard CUDA compute (ops.forward_local / merge_shards / backward / f32_to_bf16) is replaced
by exact float64 numpy test doubles so that only the collective logic is under test: the 2N-float
all-gather + log-add-exp merge in the forward, the global-LSE backward with the -1 label term on
the owner rank only, the dE all-reduce, and the token-parallel valid-count all-reduce.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cce_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _install_doubles(ops):
    def forward_local(e, c, t, ignore_index, vocab_start=0, softcap=0.0):
        z = e.double().numpy() @ c.double().numpy().T
        m = z.max(axis=1)
        lse = m + np.log(np.exp(z - m[:, None]).sum(axis=1))
        tt = t.numpy()
        loc = tt - vocab_start
        own = (tt != ignore_index) & (loc >= 0) & (loc < c.shape[0])
        corr = np.where(own, z[np.arange(len(tt)), np.clip(loc, 0, c.shape[0] - 1)], 0.0)
        return torch.from_numpy(lse), torch.from_numpy(corr)

    def merge_shards(lse_parts, correct_parts, t, ignore_index, v_total=0):
        lse = torch.logsumexp(lse_parts, dim=0)
        valid = t != ignore_index
        loss = torch.where(valid, lse - correct_parts.sum(0), torch.zeros_like(lse))
        return torch.where(valid, lse, torch.zeros_like(lse)), loss

    def backward(e, c, t, lse, up, *, ignore_index, vocab_start=0, softcap=0.0, eps=None,
                 vocab_sorting=True, perm=None, fp32_de=False):
        E, C = e.double().numpy(), c.double().numpy()
        s = np.exp(E @ C.T - lse.double().numpy()[:, None])
        tt = t.numpy()
        loc = tt - vocab_start
        own = (tt != ignore_index) & (loc >= 0) & (loc < C.shape[0])
        rows = np.nonzero(own)[0]
        s[rows, loc[rows]] -= 1.0
        s *= up.double().numpy()[:, None]
        return torch.from_numpy(s @ C), torch.from_numpy(s.T @ E), None, None

    ops.forward_local = forward_local
    ops.merge_shards = merge_shards
    ops.backward = backward
    ops.f32_to_bf16 = lambda x: x


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_09009_b200 import ops, vocab_parallel as vp

        _install_doubles(ops)
        rng = np.random.default_rng(0)
        n, d, v = 37, 8, 23
        e = torch.from_numpy(rng.standard_normal((n, d)))
        c = torch.from_numpy(rng.standard_normal((v, d)))
        t = torch.from_numpy(rng.integers(0, v, n))
        t[::5] = -100
        v0, v1 = vp.shard_range(v, rank, world)
        lse_l, corr = ops.forward_local(e, c[v0:v1], t, -100, v0)
        lse, loss = vp.gather_and_merge(lse_l, corr, t, -100, dist.group.WORLD)
        xo = np.where(t.numpy() == -100, -1, t.numpy())
        nl, nlse, _ = O.naive_forward(e.numpy(), c.numpy(), xo)
        valid = xo != -1
        up = torch.from_numpy(O.default_upstream(xo, "mean-over-valid", np.float64))
        de, dc = vp.sharded_backward(e, c[v0:v1], t, lse, up, ignore_index=-100, vocab_start=v0,
                                     softcap=0.0, eps=None, vocab_sorting=False, group=dist.group.WORLD)
        rde, rdc = O.naive_backward(e.numpy(), c.numpy(), xo, up.numpy())
        # token-parallel: global mean = all-reduced sum / all-reduced valid count
        n_valid = torch.tensor(float(valid[rank::world].sum()))
        dist.all_reduce(n_valid)
        q.put((rank, float(np.max(np.abs(loss.numpy() - nl))),
               float(np.max(np.abs(lse.numpy()[valid] - nlse[valid]))),
               O.rel_err(de.numpy(), rde), O.rel_err(dc.numpy(), rdc[v0:v1]),
               float(n_valid.item()) == float(valid.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_vocab_parallel_matches_single_shard(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, loss_err, lse_err, de_err, dc_err, count_ok in results:
        assert loss_err < 1e-10 and lse_err < 1e-10, (rank, loss_err, lse_err)
        assert de_err < 1e-10 and dc_err < 1e-10, (rank, de_err, dc_err)
        assert count_ok


def test_shard_range_partitions_vocab():
    from paper_2411_09009_b200.vocab_parallel import shard_range

    for v in (1, 7, 256000, 128256):
        for w in (1, 2, 3, 8):
            spans = [shard_range(v, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == v
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_cyclic_rows_partition_and_shard_targets():
    """Block-cyclic layout: the ranks' row sets partition the vocabulary; shard_targets maps an
    owned label to its shard row, any other label past the shard, and keeps ignore_index."""
    import torch

    from paper_2411_09009_b200 import ops
    from paper_2411_09009_b200.vocab_parallel import cyclic_rows

    v, world = 5001, 3
    rows = [cyclic_rows(v, r, world, block=256) for r in range(world)]
    allr = torch.cat(rows).sort().values
    assert torch.equal(allr, torch.arange(v))
    t = torch.tensor([0, 255, 256, 767, 768, 5000, -100])
    for r in range(world):
        loc = ops.shard_targets(t, rows[r], v, -100)
        for g, l in zip(t.tolist(), loc.tolist()):
            if g == -100:
                assert l == -100
            elif (g // 256) % world == r:
                assert rows[r][l] == g
            else:
                assert l == rows[r].shape[0]
