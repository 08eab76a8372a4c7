"""Kernel timeline of a few bench steps (torch.profiler / CUPTI): per-kernel device time and the
idle gaps between consecutive kernels, to find host-side stalls."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2411_09009_b200 import linear_cross_entropy

cfg = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
import bench
n, d, v, cap, pad, sigma = bench.CONFIGS[cfg]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(n, d, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(v, d, device=dev, generator=g) * sigma / math.sqrt(d)).bfloat16().requires_grad_(True)
t = torch.randint(0, v, (n,), device=dev, generator=g)

def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t, softcap=cap or None,
                         low_memory=os.environ.get("TRACE_LOW", "0") == "1").backward()

for _ in range(int(os.environ.get("TRACE_WARM", "3"))):  # e.g. 40: settle the power state first
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
prev_end = None
rows = []
for ev in evs:
    s, en = ev.time_range.start, ev.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0
    rows.append((s, en - s, gap, ev.name[:70]))
    prev_end = en if prev_end is None else max(prev_end, en)
tot_gap = sum(r[2] for r in rows if r[2] > 0)
span = rows[-1][0] + rows[-1][1] - rows[0][0]
print(f"span {span/1e3:.2f} ms for 2 steps, kernel-busy {sum(r[1] for r in rows)/1e3:.2f} ms, gaps {tot_gap/1e3:.2f} ms")
full = os.environ.get("TRACE_ALL") == "1"
for s, dur, gap, name in rows:
    if full or dur > 50 or gap > 50:
        print(f"  gap {gap:8.1f} us  dur {dur:9.1f} us  {name}")
# CPU-side ops that took long (syncs)
cpu = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU], key=lambda e: -e.cpu_time_total)[:15]
for e_ in cpu:
    print(f"  cpu {e_.cpu_time_total/1e3:8.2f} ms  {e_.name[:80]}")
