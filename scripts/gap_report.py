"""Where the device idles between kernels in a default training step (torch.profiler trace):
gaps summed by the kernel that follows them."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2411_09009_b200 import linear_cross_entropy

N, D, V = 8192, 2304, 256000
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(N, D, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(V, D, device=dev, generator=g) / math.sqrt(D)).bfloat16().requires_grad_(True)
t = torch.randint(0, V, (N,), device=dev, generator=g)


def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t).backward()


for _ in range(4):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
evs = sorted([x for x in prof.events() if x.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda x: x.time_range.start)
agg = {}
prev = None
for x in evs:
    if prev is not None:
        gap = x.time_range.start - prev
        name = x.name.split("(")[0].replace("void ", "")[:60]
        a = agg.setdefault(name, [0.0, 0, 0.0])
        a[0] += gap / 3
        a[1] += 1
        a[2] = max(a[2], gap)
    prev = max(prev or 0, x.time_range.end)
print(f"{len(evs) / 3:.0f} device ops per step")
for name, (tot, cnt, mx) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {tot:8.1f} us/step  n/step={cnt / 3:5.1f}  max {mx:7.1f} us  before {name}")
