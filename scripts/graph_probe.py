"""Eager vs CUDA-graph replay of the default training step (linear_cross_entropy fwd+bwd) at a
BASELINE head: per-step device time over REPS steps, and the replayed step's loss and gradients
against the eager step on the same inputs (bitwise).  Usage: python scripts/graph_probe.py [config]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_09009_b200 import linear_cross_entropy  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
reps = int(os.environ.get("REPS", 20))
n, d, v, cap, pad, sigma = bench.CONFIGS[cfg]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(n, d, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(v, d, device=dev, generator=g) * sigma / math.sqrt(d)).bfloat16().requires_grad_(True)
t = torch.randint(0, v, (n,), device=dev, generator=g)


def step():
    e.grad = c.grad = None
    loss = linear_cross_entropy(e, c, t, softcap=cap or None)
    loss.backward()
    return loss


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(side)
timed(step)  # settle
ref_loss = step().detach().clone()
ref_de, ref_dc = e.grad.clone(), c.grad.clone()
graph = torch.cuda.CUDAGraph()
e.grad = c.grad = None
with torch.cuda.graph(graph):
    g_loss = linear_cross_entropy(e, c, t, softcap=cap or None)
    g_loss.backward()
g_de, g_dc = e.grad, c.grad
graph.replay()
torch.cuda.synchronize()
same = torch.equal(g_loss, ref_loss) and torch.equal(g_de, ref_de) and torch.equal(g_dc, ref_dc)
rounds = []
for _ in range(3):  # interleaved: clocks drift under the power cap
    rounds.append((timed(step), timed(graph.replay)))
print(f"{cfg}: " + "  ".join(f"eager {a:.3f} / graph {b:.3f} ms" for a, b in rounds) +
      f"  bitwise-equal {same}")
