"""The copy-free training path: kernels read E through the compaction map and C through the
vocabulary order with cp.async row gathers (no compacted E, no sorted classifier).  Its forward
must be bit-identical to the forward over the materialised copies."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _head(n, d, v, seed, sigma=1.0, ign=0.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    e = torch.randn(n, d, device="cuda", generator=g).bfloat16()
    c = (torch.randn(v, d, device="cuda", generator=g) * sigma / math.sqrt(d)).bfloat16()
    t = torch.randint(0, v, (n,), device="cuda", generator=g)
    if ign:
        t[torch.rand(n, device="cuda", generator=g) < ign] = -100
    return e, c, t


@pytest.mark.parametrize("n,d,v,ign,cap,sort", [
    (300, 64, 1000, 0.0, 0.0, True),
    (1000, 200, 5003, 0.3, 0.0, True),     # hidden size not a multiple of 64: zero-filled tail
    (777, 128, 20000, 0.1, 30.0, True),
    (512, 256, 3000, 0.0, 0.0, False),
    (4096, 768, 50257, 0.25, 0.0, True),
    (2048, 2304, 65536, 0.0, 0.0, True),
])
def test_forward_gather_bit_identical_to_copies(cuda_device, n, d, v, ign, cap, sort):
    from paper_2411_09009_b200 import ops

    e, c, t = _head(n, d, v, n + d, ign=ign)
    l1, c1, s1 = ops.forward_tiles(e, c, t, -100, 0, cap, vocab_sorting=sort, store_labels=False)
    l2, c2, s2 = ops.forward_gather(e, c, t, -100, 0, cap, vocab_sorting=sort)
    torch.cuda.synchronize()
    valid = t != -100
    assert torch.equal(l1[valid], l2[valid]) and torch.equal(c1[valid], c2[valid])
    # tile maxima of the valid rows (rows past the compacted count hold no data)
    nv = int(s1.n_valid)
    tm1 = s1.tile_max.view(-1, s1.tile_max.numel() // max(1, -(-n // 128)) // 128, 128)
    tm2 = s2.tile_max.view_as(tm1)
    rows = torch.arange(tm1.shape[0] * 128, device=tm1.device).view(-1, 1, 128) < nv
    assert torch.equal(torch.where(rows, tm1, 0.0), torch.where(rows, tm2, 0.0))
    if sort:
        assert torch.equal(s1.perm, s2.perm)


def _stream_run(e, c, t, softcap=0.0, eps=2.0 ** -12, label_split=False):
    from paper_2411_09009_b200 import ops

    lse_l, corr, st = ops.forward_tiles(e, c, t, -100, 0, softcap, store_labels=False)
    lse, _ = ops.merge_shards(lse_l[None], corr[None], t, -100)
    up = ops.upstream(torch.ones((), device=e.device), t, -100, "mean")
    inv = torch.empty_like(st.perm)
    inv[st.perm.long()] = torch.arange(st.perm.shape[0], dtype=torch.int32, device=e.device)
    de, dc, cnt = ops.backward_stream(st.e_c, False, c, st.perm_padded, inv, st.row_map, st.n_valid, st.pos,
                                      st.tile_max, lse, up, softcap=softcap, eps=eps, label_split=label_split,
                                      correct=corr, e_caller=e)
    ref_de, ref_dc, ref_cnt = ops.backward_tiles(st, t, lse, up, ignore_index=-100, eps=eps,
                                                  label_split=label_split, correct=corr, reuse_state=True)
    torch.cuda.synchronize()
    return de, dc, cnt, ref_de, ref_dc, ref_cnt


def _rel(a, b):
    return float((a.float() - b.float()).abs().max()) / max(1e-30, float(b.float().abs().max()))


@pytest.mark.parametrize("n,d,v,ign,cap,sigma", [
    (300, 64, 1000, 0.0, 0.0, 1.0),
    (1000, 192, 5003, 0.3, 0.0, 2.0),
    (777, 128, 20000, 0.1, 30.0, 3.0),
    (4096, 768, 50257, 0.25, 0.0, 1.0),
])
def test_stream_backward_matches_stored_shat_backward(cuda_device, n, d, v, ign, cap, sigma):
    """Same decision, same S-hat tiles: the streamed backward equals the stored-S-hat backward up to
    the fp32 summation order of split owners (and bf16 rounding of the outputs)."""
    e, c, t = _head(n, d, v, 7 * n + d, sigma=sigma, ign=ign)
    de, dc, cnt, rde, rdc, rcnt = _stream_run(e, c, t, softcap=cap)
    assert torch.equal(cnt, rcnt), (cnt.tolist(), rcnt.tolist())
    # one bf16 ulp of the largest entry is 2**-8 = 3.9e-3 of the max-norm
    assert _rel(de, rde) < 8e-3 and _rel(dc, rdc) < 8e-3, (_rel(de, rde), _rel(dc, rdc))


@pytest.mark.parametrize("env", [
    {"CCE_STREAM_RING": "128", "CCE_STREAM_SEG_VOC": "1", "CCE_STREAM_WINDOW": "7", "CCE_STREAM_NACC": "1"},
    {"CCE_STREAM_RING": "128", "CCE_STREAM_SEG_VOC": "3", "CCE_STREAM_NACC": "2", "CCE_STREAM_P": "8",
     "CCE_STREAM_QC": "8"},
    {"CCE_STREAM_WINDOW": "500", "CCE_STREAM_P": "100", "CCE_STREAM_QC": "20"},
    {"CCE_STREAM_P": "10", "CCE_STREAM_QC": "100"},
])
def test_stream_backward_schedule_invariance(cuda_device, monkeypatch, env):
    """Small rings (many laps per slot), one-item dC segments (every vocab tile a long split chain),
    tiny dE windows, one accumulator region and lopsided role splits all give the same gradients."""
    e, c, t = _head(1500, 256, 30000, 11, sigma=2.5, ign=0.1)
    base = _stream_run(e, c, t)
    for k, val in env.items():
        monkeypatch.setenv(k, val)
    de, dc, cnt = _stream_run(e, c, t)[:3]
    assert torch.equal(cnt, base[2])
    assert _rel(de, base[0]) < 8e-3 and _rel(dc, base[1]) < 8e-3, (_rel(de, base[0]), _rel(dc, base[1]))


def test_stream_backward_bit_reproducible(cuda_device):
    e, c, t = _head(2048, 512, 40000, 5, sigma=2.0, ign=0.05)
    a = _stream_run(e, c, t)
    b = _stream_run(e, c, t)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])


def test_stream_backward_paper_ordering(cuda_device):
    e, c, t = _head(900, 128, 7000, 9, sigma=2.0, ign=0.1)
    de, dc, cnt, rde, rdc, rcnt = _stream_run(e, c, t, label_split=True)
    assert torch.equal(cnt, rcnt)
    assert _rel(de, rde) < 8e-3 and _rel(dc, rdc) < 8e-3


@pytest.mark.parametrize("n,d,v,ign,cap,sigma", [
    (300, 64, 1000, 0.0, 0.0, 1.0),
    (1000, 192, 5003, 0.3, 0.0, 2.0),
    (777, 128, 20000, 0.1, 30.0, 3.0),
    (4096, 768, 50257, 0.25, 0.0, 1.0),
])
def test_stream_gather_mode_bit_identical(cuda_device, monkeypatch, n, d, v, ign, cap, sigma):
    """CCE_STREAM_GATHER=1: no sorted classifier copy -- the recompute CTAs gather C rows through the
    order with cp.async, the dE CTAs with TMA gather4, and dC rows are scattered to vocabulary order
    by the dC epilogue (no in-place unpermute).  Same operands, same order: bit-identical."""
    e, c, t = _head(n, d, v, 3 * n + d, sigma=sigma, ign=ign)
    base = _stream_run(e, c, t, softcap=cap)[:3]
    monkeypatch.setenv("CCE_STREAM_GATHER", "1")
    got = _stream_run(e, c, t, softcap=cap)[:3]
    for a, b in zip(got, base):
        assert torch.equal(a, b)


@pytest.mark.parametrize("v,d,kind", [(1000, 64, "random"), (5003, 192, "random"), (256000, 2304, "random"),
                                      (3000, 128, "identity"), (3000, 128, "shift"), (4096, 256, "swaps"),
                                      (2000, 520, "random"), (20000, 256, "freecycle")])
def test_unpermute_rows_in_place(cuda_device, v, d, kind):
    """The in-place unpermutation of dC (cycle segments cut at anchors, chain tables, batched row
    moves per column block) equals an out-of-place index copy, for random permutations (one giant
    cycle plus small ones), the identity, one long shift, many 2-cycles (rotated) and a 500-long
    cycle without anchors (cut from its smallest position)."""
    from paper_2411_09009_b200 import _lib, ops

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(v + d)
    if kind == "random":
        perm = torch.randperm(v, device="cuda", generator=g)
    elif kind == "identity":
        perm = torch.arange(v, device="cuda")
    elif kind == "shift":
        perm = (torch.arange(v, device="cuda") + 1) % v
    elif kind == "swaps":
        perm = torch.arange(v, device="cuda").view(-1, 2).flip(1).reshape(-1)
    else:  # one 500-long cycle through positions that are not anchors (cut every 96 from its minimum)
        idx = [p for p in range(v) if ((p * 2654435761) & 0xFFFFFFFF) >> 26 != 0][:500]
        perm = torch.arange(v, device="cuda")
        src = torch.tensor(idx, device="cuda")
        perm[src] = torch.roll(src, 1)
    perm = perm.to(torch.int32)
    inv = torch.empty_like(perm)
    inv[perm.long()] = torch.arange(v, dtype=torch.int32, device="cuda")
    x = torch.randn(v, d, device="cuda", generator=g).bfloat16()
    want = torch.empty_like(x)
    want[perm.long()] = x
    ws_bytes = lib.cce_bwd_stream_workspace_bytes(1, d, v, 512)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    _lib.check(lib.cce_unpermute_rows(ops._p(x), ops._p(perm), ops._p(inv), v, d, ops._p(ws), ws_bytes,
                                      ops._stream(x.device)), "cce_unpermute_rows")
    torch.cuda.synchronize()
    assert torch.equal(x, want)


@pytest.mark.parametrize("n,d,v,ign,cap,sort,fp32", [(1000, 128, 5003, 0.2, 0.0, True, False),
                                                     (1500, 256, 30000, 0.0, 30.0, True, False),
                                                     (700, 192, 4000, 0.1, 0.0, False, False),
                                                     (900, 128, 6000, 0.1, 0.0, True, True)])
def test_stream_token_chunks_match_whole_batch(cuda_device, monkeypatch, n, d, v, ign, cap, sort, fp32):
    """Large batches run the streamed backward as token chunks over a shared sorted copy (dC added
    over the chunks in bf16): the same tile decisions as the whole-batch pass, gradients within
    the bf16 rounding of the chunk sums."""
    from paper_2411_09009_b200 import ops

    e, c, t = _head(n, d, v, 5 * n + d, sigma=2.0, ign=ign)

    def run():
        lse_l, corr, st = ops.forward_stream(e, c, t, -100, 0, cap, vocab_sorting=sort)
        lse, _ = ops.merge_shards(lse_l[None], corr[None], t, -100)
        up = ops.upstream(torch.ones((), device=e.device), t, -100, "mean")
        out = ops.backward_from_stream_state(st, lse, up, fp32_de=fp32)  # fp32: the vocab-parallel dE
        torch.cuda.synchronize()
        return out

    de0, dc0, cnt0 = run()
    monkeypatch.setenv("CCE_STREAM_CHUNK_TILES", "2")
    de1, dc1, cnt1 = run()
    assert torch.equal(cnt0, cnt1), (cnt0.tolist(), cnt1.tolist())
    assert _rel(de1, de0) < 8e-3 and _rel(dc1, dc0) < 1e-2, (_rel(de1, de0), _rel(dc1, dc0))
    assert torch.all(de1[t == -100] == 0)


def test_bounded_default_beyond_2048_token_tiles(cuda_device):
    """linear_cross_entropy's bounded default at N = 270000 (2110 token tiles, more than one
    streamed pass can hold): token chunks of 256 tiles, against memory="fast" on the same batch."""
    from paper_2411_09009_b200 import linear_cross_entropy

    n, d, v = 270000, 64, 2000
    e0, c0, t = _head(n, d, v, 17, sigma=2.0, ign=0.05)
    out = {}
    for mode in ("bounded", "fast"):
        e = e0.clone().requires_grad_(True)
        c = c0.clone().requires_grad_(True)
        loss = linear_cross_entropy(e, c, t, memory=mode)
        loss.backward()
        torch.cuda.synchronize()
        out[mode] = (loss.item(), e.grad, c.grad)
    lb, lf = out["bounded"][0], out["fast"][0]
    assert abs(lb - lf) <= 1e-4 * abs(lf), (lb, lf)
    assert _rel(out["bounded"][1], out["fast"][1]) < 1e-2
    assert _rel(out["bounded"][2], out["fast"][2]) < 1e-2


def test_bounded_default_across_changing_batches(cuda_device):
    """A training loop whose batches change shape and padding from step to step (the learned
    compaction choice and ring sizing follow the batch): every step equals memory="fast"."""
    from paper_2411_09009_b200 import linear_cross_entropy

    d, v = 256, 30000
    for step, (n, ign) in enumerate([(3000, 0.0), (3000, 0.3), (5000, 0.3), (5000, 0.0), (700, 0.5), (3000, 0.0)]):
        e0, c0, t = _head(n, d, v, 100 + step, sigma=2.0, ign=ign)
        out = {}
        for mode in ("bounded", "fast"):
            e = e0.clone().requires_grad_(True)
            c = c0.clone().requires_grad_(True)
            loss = linear_cross_entropy(e, c, t, memory=mode)
            loss.backward()
            torch.cuda.synchronize()
            out[mode] = (loss.item(), e.grad, c.grad)
        assert abs(out["bounded"][0] - out["fast"][0]) <= 1e-4 * abs(out["fast"][0]), step
        assert _rel(out["bounded"][1], out["fast"][1]) < 1e-2, step
        assert _rel(out["bounded"][2], out["fast"][2]) < 1e-2, step
        assert torch.all(out["bounded"][1][t == -100] == 0), step


@pytest.mark.parametrize("n,d,v,ign,cap,group_mb", [(4096, 768, 50257, 0.0, 0.0, 4), (1000, 256, 30000, 0.2, 30.0, 1),
                                                      (8192, 2304, 256000, 0.0, 0.0, 52)])
def test_forward_chain_bit_identical(cuda_device, monkeypatch, n, d, v, ign, cap, group_mb):
    """The bounded forward's group launches as one flag-synchronised chain (CCE_FWD_CHAIN=1: each
    launch gathers the next group in a warp of its own and no launch waits for the previous one to
    finish) give the same lse, target logits and tile maxima, bit for bit, as the per-group stream
    waits -- over many groups (small CCE_FWD_GROUP_MB), folds, ignored rows and softcap."""
    from paper_2411_09009_b200 import ops

    monkeypatch.setenv("CCE_FWD_GROUP_MB", str(group_mb))
    e, c, t = _head(n, d, v, n + d + 7, ign=ign)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("CCE_FWD_CHAIN", mode)
        for _ in range(2):  # the second call runs on the learned compaction hint
            lse_l, corr, st = ops.forward_stream(e, c, t, -100, 0, cap)
        torch.cuda.synchronize()
        out[mode] = (lse_l, corr, st.tile_max)
    valid = t != -100
    nv = int(valid.sum())
    tm0, tm1 = out["0"][2], out["1"][2]
    mt = -(-v // 256)
    rows = (torch.arange(tm0.numel() // (mt * 128) * 128, device=e.device).view(-1, 1, 128) < nv)
    assert torch.equal(out["0"][0][valid], out["1"][0][valid]) and torch.equal(out["0"][1][valid], out["1"][1][valid])
    assert torch.equal(torch.where(rows, tm0.view(-1, mt, 128), 0.0), torch.where(rows, tm1.view(-1, mt, 128), 0.0))
