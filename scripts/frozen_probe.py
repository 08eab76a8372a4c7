"""Step time with a frozen classifier / frozen hidden states (the backward skips that pass) at the
Gemma-2-2B head.  Usage: python scripts/frozen_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math, torch
from paper_2411_09009_b200 import linear_cross_entropy
N, D, V = 8192, 2304, 256000
g = torch.Generator(device="cuda").manual_seed(0)
e0 = torch.randn(N, D, device="cuda", generator=g).bfloat16()
c0 = (torch.randn(V, D, device="cuda", generator=g) / math.sqrt(D)).bfloat16()
t = torch.randint(0, V, (N,), device="cuda", generator=g)
for rep in range(2):
    for frozen in (None, "c", "e"):
        e = e0.clone().requires_grad_(frozen != "e")
        c = c0.clone().requires_grad_(frozen != "c")
        def step():
            e.grad = c.grad = None
            linear_cross_entropy(e, c, t).backward()
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            step()
        b.record(); torch.cuda.synchronize()
        print(f"frozen={frozen} {a.elapsed_time(b) / 20:.3f} ms/step")
