"""Developer probe: compare the tile path and the low-memory path against torch fp32 on one case."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2411_09009_b200 import linear_cross_entropy, ops

def rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))

def run(n, d, v, sigma, ign, cap, seed=77, eps="auto"):
    g = torch.Generator().manual_seed(seed)
    e0 = torch.randn(n, d, generator=g).bfloat16().cuda()
    c0 = (torch.randn(v, d, generator=g) * sigma / math.sqrt(d)).bfloat16().cuda()
    t = torch.randint(0, v, (n,), generator=g).cuda()
    if ign:
        t[(torch.rand(n, generator=g) < ign).cuda()] = -100
    e2 = e0.float().requires_grad_(True); c2 = c0.float().requires_grad_(True)
    z = e2 @ c2.T
    if cap: z = cap * torch.tanh(z / cap)
    torch.nn.functional.cross_entropy(z, t, ignore_index=-100).backward()
    res = {}
    for low in (False, True):
        e = e0.clone().requires_grad_(True); c = c0.clone().requires_grad_(True)
        loss = linear_cross_entropy(e, c, t, softcap=cap or None, low_memory=low, filter_eps=eps)
        loss.backward()
        cnt = ops.LAST_COUNTERS["counters"].tolist()
        bad = (e.grad.float() - e2.grad).abs().max(dim=1).values
        rows = torch.nonzero(bad > 0.05 * e2.grad.abs().max()).flatten().tolist()
        print(f"n={n} d={d} v={v} ign={ign} cap={cap} low={low}: dE {rel(e.grad.float(), e2.grad):.2e} "
              f"dC {rel(c.grad.float(), c2.grad):.2e} cnt {cnt} bad rows {len(rows)} {rows[:10]} "
              f"ignored-bad {[(r, int(t[r])) for r in rows[:5]]}")
        res[low] = (e.grad.float(), c.grad.float())
    print("  tiles vs low:", rel(res[False][0], res[True][0]), rel(res[False][1], res[True][1]))

run(1000, 256, 20000, 0.4, 0.2, 0.0)
run(1000, 256, 20000, 0.4, 0.0, 0.0)
run(1000, 256, 20000, 0.4, 0.2, 0.0, eps=None)
run(640, 128, 3001, 2.0, 0.2, 0.0)
run(1024, 256, 20000, 0.4, 0.2, 0.0)
