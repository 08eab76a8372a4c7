"""Eager step vs the same step captured in a CUDA graph (same box, same inputs): the difference
is what launch gaps and host work cost.  Also checks the graph replay's gradients."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_09009_b200 import linear_cross_entropy

N, D, V = 8192, 2304, 256000
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(N, D, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(V, D, device=dev, generator=g) / math.sqrt(D)).bfloat16().requires_grad_(True)
t = torch.randint(0, V, (N,), device=dev, generator=g)


def step():
    e.grad = None
    c.grad = None
    loss = linear_cross_entropy(e, c, t)
    loss.backward()
    return loss


def timed(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


eager = timed(step)
ref = (step().item(), e.grad.clone(), c.grad.clone())
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
try:
    e.grad = None
    c.grad = None
    with torch.cuda.graph(graph):
        loss = linear_cross_entropy(e, c, t)
        loss.backward()
    replay = timed(graph.replay)
    graph.replay()
    torch.cuda.synchronize()
    same = torch.equal(e.grad, ref[1]) and torch.equal(c.grad, ref[2]) and loss.item() == ref[0]
    print(f"eager {eager:.3f} ms/step, graph replay {replay:.3f} ms/step, identical results: {same}")
except Exception as exc:
    print(f"eager {eager:.3f} ms/step; capture failed: {type(exc).__name__}: {exc}")
