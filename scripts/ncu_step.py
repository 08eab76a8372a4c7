"""One steady-state training step for ncu: warm-up steps (capacities learned, caches hot) run
unprofiled, then one step between cudaProfilerStart / Stop.  Run under
`ncu --profile-from-start off -k regex:... -c K` to capture that step's kernels.
Usage: python scripts/ncu_step.py [config] [warm steps]"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2411_09009_b200 import linear_cross_entropy

cfg = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n, d, v, cap, pad, sigma = bench.CONFIGS[cfg]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(n, d, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(v, d, device=dev, generator=g) * sigma / math.sqrt(d)).bfloat16().requires_grad_(True)
t = torch.randint(0, v, (n,), device=dev, generator=g)
low = os.environ.get("NCU_LOW", "0") == "1"


def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t, softcap=cap or None, low_memory=low).backward()


for _ in range(warm):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
