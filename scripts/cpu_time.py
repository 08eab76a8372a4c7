"""Host-side enqueue time of one training step (no synchronisation inside the timed loop) vs the
device time: if the CPU needs longer than the GPU, kernels wait on launches."""
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


def fwd():
    e.grad = c.grad = None
    return linear_cross_entropy(e, c, t)


for _ in range(4):
    fwd().backward()
torch.cuda.synchronize()
K = 10
tf = tb = 0.0
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
t0 = time.perf_counter()
for _ in range(K):
    s = time.perf_counter()
    loss = fwd()
    m = time.perf_counter()
    loss.backward()
    tf += m - s
    tb += time.perf_counter() - m
t1 = time.perf_counter()
b.record()
torch.cuda.synchronize()
print(f"host enqueue per step: {(t1 - t0) / K * 1e3:.2f} ms (forward {tf / K * 1e3:.2f}, backward {tb / K * 1e3:.2f}); "
      f"device per step {a.elapsed_time(b) / K:.2f} ms")
