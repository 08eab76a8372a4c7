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
    assert torch.equal(s1.tile_max, s2.tile_max)
    if sort:
        assert torch.equal(s1.perm, s2.perm)
