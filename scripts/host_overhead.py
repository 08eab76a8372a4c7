"""Host time to enqueue one training step (Python + ctypes + allocator, no device sync) vs the
device time of the step.  If the host time is larger, the GPU starves.
Usage: python scripts/host_overhead.py [config]"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2411_09009_b200 import linear_cross_entropy

cfg = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
n, d, v, cap, pad, sigma = bench.CONFIGS[cfg]
g = torch.Generator(device="cuda").manual_seed(0)
e = torch.randn(n, d, device="cuda", generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(v, d, device="cuda", generator=g) * sigma / math.sqrt(d)).bfloat16().requires_grad_(True)
t = torch.randint(0, v, (n,), device="cuda", generator=g)


def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t, softcap=cap or None).backward()


for _ in range(10):
    step()
torch.cuda.synchronize()
K = int(os.environ.get("HOST_K", "5"))  # few steps: a deep queue would block the host on the device
h0 = time.perf_counter()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(K):
    step()
h1 = time.perf_counter()
b.record()
torch.cuda.synchronize()
print(f"{cfg}: host enqueue {1e3 * (h1 - h0) / K:.3f} ms/step, device {a.elapsed_time(b) / K:.3f} ms/step")
